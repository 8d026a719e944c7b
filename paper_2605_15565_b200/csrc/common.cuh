// Shared device helpers for the sm_100a kernels of the policy-loss path.
// (CUDA side only; the CPU oracle in oracle/ shares nothing with this file.)
#pragma once
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rl_policy.h"

#define RL_LOG2E 1.4426950408889634f
#define RL_LN2 0.6931471805599453f

namespace rl {

// ---------------------------------------------------------------- host-side error plumbing
void set_error(const char* fmt, ...);
rl_status fail(rl_status s, const char* fmt, ...);
rl_status check_launch(const char* what);

// ---------------------------------------------------------------- per-device host state
// Everything the launchers derive from the device (SM count, compute capability) is cached per
// device ordinal, so one process may drive several GPUs; entry points first call
// require_sm100() (RL_ERR_UNSUPPORTED on anything but a compute-capability 10.0 device).
constexpr int kMaxDevices = 64;
struct DevInfo {
  int ordinal;
  int sms;
  int cc_major, cc_minor;
};
const DevInfo& dev_info();  // current device
rl_status require_sm100();
// per-device cache slot for a launcher-derived integer (0 = not computed yet)
int& dev_slot(int* table);

// Development options (include/rl_policy_dev.h): alternative kernels kept for A/B tests.
// Set explicitly through rl_dev_set_option; the library never reads the environment.
enum DevOpt {
  OPT_LOSS_KERNEL = 0,  // 0 = single-visit cluster kernel (default), 1 = exact two-pass kernel
  OPT_VP_PATH = 1,      // fused vocab-parallel loss: 0 = in-kernel peer exchange when enabled, 1 = NCCL path
  OPT_LM_SPLITS = 2,    // LM-head vocabulary split override (0 = cost model)
  OPT_VP_KERNEL = 3,    // peer-exchange vocab-parallel kernel: 0 = default (see vocab_parallel.cu), 1 = L2 ring, 2 = register cache when it fits
  OPT_VC_GROUPS = 4,    // vp_cache_kernel collector groups override (0 = min(8, 32 / P))
  OPT_VC_ROWS = 5,      // vp_cache_kernel rows parked in shared memory: 0 = default, else that number + 1
  OPT_VC_PUB = 6,       // vp_cache_kernel record send, value + 1: 0 collector strong, 1 last warp weak (default), 2 collector weak
  OPT_LM_PAIR = 7,      // LM-head kernels: 0 = pairs for the gradient kernel only, 1 = single CTAs, 2 = pairs for both
  OPT_LM_GEMM = 8,      // LM-head backward GEMMs: 0 / 1 = cuBLAS (default), 2 = lm_gemm_kernel (tcgen05)
  OPT_VR_DELAY = 9,     // vp_ring_kernel rows between a slice's two reads (0 = L2-window rule; sets G = 1)
  OPT_VC_TMEM = 10,     // vp_cache_kernel parked rows in tensor memory: 0 = default (on for narrow shards on > 1 rank), 1 = off, 2 = on
  OPT_COUNT = 11
};
int dev_option(int key);

// ---------------------------------------------------------------- debug checks
// python -m paper_2605_15565_b200.build --variant checks (-DRL_DEBUG_CHECKS): bounds / index
// assertions at the kernels' global stores and ring accesses (the stand-in for compute-sanitizer,
// which this GPU pool refuses); compiled out of the product library.
#ifdef RL_DEBUG_CHECKS
#define RL_DCHECK(c)                                                                                    \
  do {                                                                                                  \
    if (!(c)) {                                                                                         \
      printf("RL_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, blockIdx.x, \
             threadIdx.x);                                                                              \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define RL_DCHECK(c) \
  do {               \
  } while (0)
#endif

// ---------------------------------------------------------------- element access
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// pack two floats to bf16x2 with round-to-nearest-even (cvt.rn.bf16x2.f32: hi operand first)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fast_log2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 128-bit streaming global load, no L1 allocation
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 128-bit load with an L2 cache-policy hint (evict_last keeps the line for a re-read)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_hint_v4(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// 128-bit read-only load through L1 (consecutive per-thread vectors share cache lines)
__device__ __forceinline__ uint4 ld_hint_v4_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 128-bit streaming store (evict-first in L2: dlogits are not re-read by this kernel)
__device__ __forceinline__ void st_stream_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// predicated form (no branch around it in unrolled loops)
__device__ __forceinline__ void st_stream_v4_if(void* p, uint4 v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\n\t}" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"((uint32_t)pred)
               : "memory");
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- (max, sum) in log2 domain
// A partial softmax state over a set of columns: m = max t, s = sum 2^(t - m), t = x*k.
struct MS {
  float m;
  float s;
};

__device__ __forceinline__ MS ms_combine(MS a, MS b) {
  float m = fmaxf(a.m, b.m);
  if (m == -INFINITY) return MS{-INFINITY, 0.f};
  float sa = (a.m == -INFINITY) ? 0.f : a.s * fast_exp2(a.m - m);
  float sb = (b.m == -INFINITY) ? 0.f : b.s * fast_exp2(b.m - m);
  return MS{m, sa + sb};
}

__device__ __forceinline__ MS warp_reduce_ms(MS v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MS w;
    w.m = __shfl_xor_sync(0xffffffffu, v.m, o);
    w.s = __shfl_xor_sync(0xffffffffu, v.s, o);
    v = ms_combine(v, w);
  }
  return v;
}

// Row validity (c2 rule), shared by the bookkeeping and loss kernels.
struct RowMeta {
  int32_t y;
  int32_t seq;
  bool in_range;   // 0 <= y < V
  bool bad;        // y >= V
  bool neg_stale;  // staleness < 0
  bool stale_drop; // staleness > max_staleness >= 0
  bool valid;
};

__device__ __forceinline__ RowMeta row_meta(int64_t row, int64_t vocab, const int32_t* targets,
                                            const uint8_t* loss_mask, const int32_t* token_seq,
                                            const int32_t* seq_version, int32_t trainer_version,
                                            int32_t max_staleness) {
  RowMeta m;
  m.y = targets[row];
  m.seq = token_seq ? token_seq[row] : 0;
  m.in_range = (m.y >= 0) && ((int64_t)m.y < vocab);
  m.bad = (int64_t)m.y >= vocab;
  int32_t stale = seq_version ? (trainer_version - seq_version[m.seq]) : 0;
  m.neg_stale = stale < 0;
  m.stale_drop = (!m.neg_stale) && max_staleness >= 0 && stale > max_staleness;
  bool mask = loss_mask ? (loss_mask[row] != 0) : true;
  m.valid = mask && m.in_range && !m.neg_stale && !m.stale_drop;
  m.stale_drop = m.stale_drop && mask && m.in_range;
  return m;
}

}  // namespace rl
