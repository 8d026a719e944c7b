// (3) Token log-probs — c3 of DESIGN.md §3 (north_star: "a log-softmax over the
// vocabulary followed by a gather").  Read-only single streaming pass: each CTA owns one
// row at a time; 128-bit loads, U vectors in flight per thread, per-thread online
// (max, sum-exp2) and a block reduction.  HBM-bound: V*elem + 12 B per token.
#include <algorithm>

#include "rowstats.cuh"

namespace rl {

constexpr int kLpThreads = 256;
constexpr int kLpUnroll = 4;

template <typename T>
__global__ void __launch_bounds__(kLpThreads) token_logprob_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t V, int64_t ld,
    const int32_t* __restrict__ targets, float inv_t, float* __restrict__ logp_out,
    float* __restrict__ lse_out, double* __restrict__ bad_count) {
  __shared__ float red[64];
  const float k = inv_t * RL_LOG2E;
  const uint64_t pol = policy_evict_first();
  const int64_t row_bytes = ld * elem_bytes<T>();
  unsigned bad = 0;
  for (int64_t row = blockIdx.x; row < n_tokens; row += gridDim.x) {
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    const int32_t y = targets[row];
    MS st = row_stats_thread<T, kLpThreads, kLpUnroll>(rp, V, k, pol);
    st = block_reduce_ms<kLpThreads>(st, red);
    if (threadIdx.x == 0) {
      const float c2 = st.m + fast_log2(st.s);  // log2-domain log-sum-exp
      float lp;
      if (y >= 0 && (int64_t)y < V) lp = VecTraits<T>::load1(rp, y) * inv_t - c2 * RL_LN2;
      else if (y < 0) lp = 0.f;
      else { lp = __int_as_float(0x7fc00000); ++bad; }
      logp_out[row] = lp;
      if (lse_out) lse_out[row] = c2 * RL_LN2;
    }
  }
  if (threadIdx.x == 0 && bad && bad_count) atomicAdd(bad_count, (double)bad);
}

int logprob_grid(int64_t n_tokens) {
  static int max_ctas = 0;
  if (!max_ctas) {
    int dev = 0, sms = 148, occ = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, token_logprob_kernel<bf16_t>, kLpThreads, 0);
    max_ctas = sms * std::max(occ, 1);
  }
  return (int)std::min<int64_t>(n_tokens, max_ctas);
}

}  // namespace rl

extern "C" rl_status rl_token_logprob(const void* logits, int32_t dtype, int64_t n_tokens,
                                      int64_t vocab, int64_t ld, const int32_t* targets,
                                      float inv_temperature, float* logp_out, float* lse_out,
                                      double* bad_target_count, rl_stream stream) {
  using namespace rl;
  if (n_tokens < 0 || vocab < 1 || ld < vocab)
    return fail(RL_ERR_INVALID_ARGUMENT, "n_tokens < 0, vocab < 1 or ld < vocab");
  if (dtype != RL_F32 && dtype != RL_BF16) return fail(RL_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (!(inv_temperature > 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be > 0");
  if (n_tokens == 0) return RL_OK;
  if (!logits || !targets || !logp_out) return fail(RL_ERR_INVALID_ARGUMENT, "NULL logits/targets/logp_out");
  const int64_t eb = dtype == RL_BF16 ? 2 : 4;
  if (((uintptr_t)logits & 15) || (ld * eb) % 16)
    return fail(RL_ERR_ALIGNMENT, "logits must be 16-B aligned with ld*elem %% 16 == 0");
  const int grid = logprob_grid(n_tokens);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RL_BF16)
    token_logprob_kernel<bf16_t><<<grid, kLpThreads, 0, s>>>(logits, n_tokens, vocab, ld, targets,
                                                             inv_temperature, logp_out, lse_out,
                                                             bad_target_count);
  else
    token_logprob_kernel<float><<<grid, kLpThreads, 0, s>>>(logits, n_tokens, vocab, ld, targets,
                                                            inv_temperature, logp_out, lse_out,
                                                            bad_target_count);
  return check_launch("token_logprob_kernel");
}
