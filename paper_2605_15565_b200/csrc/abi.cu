// C-ABI plumbing: status strings, thread-local error detail, parameter defaults.
#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace rl {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

rl_status fail(rl_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return s;
}

rl_status check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RL_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return RL_OK;
}

static DevInfo g_dev[kMaxDevices];
static std::atomic<int> g_dev_ready[kMaxDevices];

const DevInfo& dev_info() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (g_dev_ready[dev].load(std::memory_order_acquire) != 1) {
    DevInfo d{dev, 148, 0, 0};
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (g_dev_ready[dev].load(std::memory_order_relaxed) != 1) {
      g_dev[dev] = d;
      g_dev_ready[dev].store(1, std::memory_order_release);
    }
  }
  return g_dev[dev];
}

rl_status require_sm100() {
  const DevInfo& d = dev_info();
  if (d.cc_major != 10 || d.cc_minor != 0)
    return fail(RL_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a (B200) only",
                d.ordinal, d.cc_major, d.cc_minor);
  return RL_OK;
}

int& dev_slot(int* table) { return table[dev_info().ordinal]; }

static std::atomic<int> g_opt[OPT_COUNT];
int dev_option(int key) { return (key >= 0 && key < OPT_COUNT) ? g_opt[key].load(std::memory_order_relaxed) : 0; }

}  // namespace rl

extern "C" int32_t rl_dev_set_option(int32_t key, int32_t value) {
  if (key < 0 || key >= rl::OPT_COUNT) return -1;
  const int old = rl::g_opt[key].exchange(value);
  return old;
}

extern "C" const char* rl_status_string(rl_status s) {
  switch (s) {
    case RL_OK: return "ok";
    case RL_ERR_INVALID_ARGUMENT: return "invalid-argument";
    case RL_ERR_ALIGNMENT: return "alignment";
    case RL_ERR_UNSUPPORTED: return "unsupported";
    case RL_ERR_WORKSPACE: return "workspace";
    case RL_ERR_CUDA: return "cuda-error";
    case RL_ERR_NCCL: return "nccl-error";
  }
  return "unknown-status";
}

extern "C" const char* rl_last_error(void) { return rl::g_last_error; }

extern "C" int32_t rl_abi_version(void) { return RL_POLICY_ABI_VERSION; }

extern "C" void rl_loss_params_default(rl_loss_params* p) {
  if (!p) return;
  p->clip_eps_low = 0.2f;
  p->clip_eps_high = 0.2f;
  p->inv_temperature = 1.0f;
  p->log_ratio_clamp = 20.0f;
  p->grad_scale = 1.0f;
  p->agg = RL_AGG_TOKEN_MEAN;
  p->trainer_version = 0;
  p->max_staleness = -1;
  p->global_num_seqs = 0;
  p->flags = 0;
  p->global_active_tokens = 0.0;
  p->active_tokens_dev = nullptr;
  p->kl_coef = 0.f;
  p->ref_logp = nullptr;
  p->prox_logp = nullptr;
}
