// (3) Token log-probs — c3 of DESIGN.md §3 (north_star: "a log-softmax over the
// vocabulary followed by a gather").  Read-only single streaming pass: each CTA owns one
// row at a time; 128-bit loads, U vectors in flight per thread, per-thread online
// (max, sum-exp2) and a block reduction.  HBM-bound: V*elem + 12 B per token.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cluster_common.cuh"
#include "rowstats.cuh"

namespace rl {

// Warp-per-row kernel (default): each warp streams whole rows (U 16-B loads in flight per lane,
// no block barriers) and sums e_v = 2^(x_v k - R) with the TARGET logit as reference, R = x_y k
// (as the fused SV loss kernel, reading R1): one MUFU.EX2 per element, no max.  Since
// x_y <= max, S >= 1; lse = (R + log2 S) ln2 and logp = -ln2 log2 S.  A row with S >= 2^115 or a
// non-finite S (inf / NaN logits), or without an in-range target when lse is requested, is
// recomputed by the same warp with the max-referenced online pass (rare: a second read).
constexpr int kLwThreads = 256;
constexpr float kLwRedo = 0x1p115f;

template <typename T, int U>
__global__ void __launch_bounds__(kLwThreads) logprob_warp_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t V, int64_t ld,
    const int32_t* __restrict__ targets, float inv_t, float* __restrict__ logp_out,
    float* __restrict__ lse_out, double* __restrict__ bad_count) {
  constexpr int EPV = VecTraits<T>::EPV;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float k = inv_t * RL_LOG2E;
  const uint64_t pol = policy_evict_first();
  const int64_t row_bytes = ld * elem_bytes<T>();
  const int64_t nvec = V / EPV;
  unsigned bad = 0;
  for (int64_t row = gw; row < n_tokens; row += nw) {
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    const uint4* vrow = reinterpret_cast<const uint4*>(rp);
    const int32_t y = targets[row];
    const bool in_range = y >= 0 && (int64_t)y < V;
    float lp = 0.f, lse2 = 0.f;
    bool slow = !in_range;
    if (in_range) {
      const float R = VecTraits<T>::load1(rp, y) * k;
      const uint64_t k2 = f2pack(k, k), r2 = f2pack(-R, -R);
      uint64_t acc = f2pack(0.f, 0.f);
      int64_t i = lane;
      for (; i + (int64_t)(U - 1) * 32 < nvec; i += (int64_t)U * 32) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_hint_v4(vrow + i + u * 32, pol);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = ClVec<T>::exp_sum(v[u], k2, r2, acc);
      }
      for (; i < nvec; i += 32) acc = ClVec<T>::exp_sum(ld_hint_v4(vrow + i, pol), k2, r2, acc);
      float s0, s1;
      f2unpack(acc, s0, s1);
      float S = s0 + s1;
      for (int64_t c = nvec * EPV + lane; c < V; c += 32) S += fast_exp2(fmaf(VecTraits<T>::load1(rp, c), k, -R));
      S = warp_sum(S);
      if (S < kLwRedo) {
        const float l2 = fast_log2(S);
        lse2 = R + l2;
        lp = -l2 * RL_LN2;
      } else {
        slow = true;
      }
    }
    if (slow && (in_range || lse_out)) {  // max-referenced online pass (second read of the row)
      MS st = row_stats_thread<T, 32, 4>(rp, V, k, pol, lane);
      st = warp_reduce_ms(st);
      lse2 = st.m + fast_log2(st.s);
      if (in_range) lp = VecTraits<T>::load1(rp, y) * inv_t - lse2 * RL_LN2;
    }
    if (!in_range) {
      if (y < 0) lp = 0.f;
      else {
        lp = __int_as_float(0x7fc00000);
        ++bad;
      }
    }
    if (lane == 0) {
      logp_out[row] = lp;
      if (lse_out) lse_out[row] = lse2 * RL_LN2;
    }
  }
  if (lane == 0 && bad && bad_count) atomicAdd(bad_count, (double)bad);
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
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cudaStream_t s = (cudaStream_t)stream;
  {
    static int ctas_tab[kMaxDevices] = {};
    int& ctas = dev_slot(ctas_tab);
    if (!ctas) {
      int occ = 8;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, logprob_warp_kernel<bf16_t, 4>, kLwThreads, 0);
      ctas = dev_info().sms * std::max(occ, 1);
    }
    const int grid = (int)std::min<int64_t>((n_tokens + kLwThreads / 32 - 1) / (kLwThreads / 32), ctas);
    if (dtype == RL_BF16)
      logprob_warp_kernel<bf16_t, 4><<<grid, kLwThreads, 0, s>>>(logits, n_tokens, vocab, ld, targets,
                                                                inv_temperature, logp_out, lse_out,
                                                                bad_target_count);
    else
      logprob_warp_kernel<float, 4><<<grid, kLwThreads, 0, s>>>(logits, n_tokens, vocab, ld, targets,
                                                               inv_temperature, logp_out, lse_out,
                                                               bad_target_count);
    return check_launch("logprob_warp_kernel");
  }
}
