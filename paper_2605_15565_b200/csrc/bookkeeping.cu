// (2) Sequence / version bookkeeping — c2 of DESIGN.md §3.
// token -> sequence map from cu_seqlens, staleness = trainer_version - seq_version
// (PAPER.md:160 model-version tags; "max staleness 8"; SPEC.md:142
// 20 - 11 = 9 > 8 -> discarded), valid-token mask and per-sequence active counts.
// Integer work, bit-exact.  ~9 B/token: grid-stride over tokens, each thread owning a
// contiguous run of tokens so per-sequence counts flush with few atomics.
#include "common.cuh"

namespace rl {

constexpr int kBkThreads = 256;
constexpr int kBkRun = 16;  // tokens per thread run

__global__ void bk_seq_kernel(const int32_t* __restrict__ seq_version, int32_t n_seq,
                              int32_t trainer_version, int32_t* __restrict__ seq_active_out,
                              int32_t* __restrict__ seq_staleness_out,
                              rl_batch_counts* __restrict__ counts) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seq; i += gridDim.x * blockDim.x) {
    seq_active_out[i] = 0;
    const int32_t st = seq_version ? trainer_version - seq_version[i] : 0;
    if (seq_staleness_out) seq_staleness_out[i] = st;
    if (counts) {
      if (st < 0) atomicAdd(&counts->neg_staleness, 1.0);
      else atomicAdd(&counts->stale_hist[st < RL_STALE_HIST_BINS ? st : RL_STALE_HIST_BINS - 1], 1.0);
    }
  }
}

__device__ __forceinline__ int find_seq(const int32_t* cu, int32_t n_seq, int64_t t) {
  // largest i with cu[i] <= t  (cu[0] = 0 <= t < cu[n_seq])
  int lo = 0, hi = n_seq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)cu[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kBkThreads) bk_token_kernel(
    const int32_t* __restrict__ cu_seqlens, int32_t n_seq, int64_t n_tokens,
    const uint8_t* __restrict__ loss_mask, const int32_t* __restrict__ targets, int64_t vocab,
    const int32_t* __restrict__ seq_version, int32_t trainer_version, int32_t max_staleness,
    const float* __restrict__ seq_adv, int32_t* __restrict__ token_seq_out,
    int32_t* __restrict__ seq_active_out, float* __restrict__ adv_token_out,
    uint8_t* __restrict__ valid_out, rl_batch_counts* __restrict__ counts) {
  unsigned long long c_active = 0, c_stale = 0, c_bad = 0;
  const int64_t nruns = (n_tokens + kBkRun - 1) / kBkRun;
  for (int64_t run = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; run < nruns;
       run += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t0 = run * kBkRun;
    const int64_t t1 = min(n_tokens, t0 + kBkRun);
    int seq = find_seq(cu_seqlens, n_seq, t0);
    int64_t seq_end = cu_seqlens[seq + 1];
    int32_t stale = seq_version ? trainer_version - seq_version[seq] : 0;
    int cnt = 0;
    for (int64_t t = t0; t < t1; ++t) {
      while (t >= seq_end) {  // next non-empty sequence
        if (cnt) atomicAdd(&seq_active_out[seq], cnt);
        cnt = 0;
        ++seq;
        seq_end = cu_seqlens[seq + 1];
        stale = seq_version ? trainer_version - seq_version[seq] : 0;
      }
      token_seq_out[t] = seq;
      const int32_t y = targets[t];
      const bool in_range = y >= 0 && (int64_t)y < vocab;
      const bool m = loss_mask ? loss_mask[t] != 0 : true;
      const bool usable = stale >= 0 && (max_staleness < 0 || stale <= max_staleness);
      const bool valid = m && in_range && usable;
      c_bad += (int64_t)y >= vocab;
      c_stale += (m && in_range && stale >= 0 && !usable);
      c_active += valid;
      cnt += valid;
      if (valid_out) valid_out[t] = valid;
      if (adv_token_out) adv_token_out[t] = seq_adv[seq];
    }
    if (cnt) atomicAdd(&seq_active_out[seq], cnt);
  }
  if (counts) {
    // integer-valued partial sums: exact and order-independent in fp64
    for (int o = 16; o > 0; o >>= 1) {
      c_active += __shfl_xor_sync(0xffffffffu, c_active, o);
      c_stale += __shfl_xor_sync(0xffffffffu, c_stale, o);
      c_bad += __shfl_xor_sync(0xffffffffu, c_bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
      if (c_active) atomicAdd(&counts->active_tokens, (double)c_active);
      if (c_stale) atomicAdd(&counts->stale_masked, (double)c_stale);
      if (c_bad) atomicAdd(&counts->bad_targets, (double)c_bad);
    }
  }
}

}  // namespace rl

extern "C" rl_status rl_seq_bookkeeping(const int32_t* cu_seqlens, int32_t n_seq, int64_t n_tokens,
                                        const uint8_t* loss_mask, const int32_t* targets,
                                        int64_t vocab, const int32_t* seq_version,
                                        int32_t trainer_version, int32_t max_staleness,
                                        const float* seq_adv, int32_t* token_seq_out,
                                        int32_t* seq_active_out, int32_t* seq_staleness_out,
                                        float* adv_token_out, uint8_t* valid_out,
                                        rl_batch_counts* counts_out, rl_stream stream) {
  using namespace rl;
  if (n_seq < 0 || n_tokens < 0 || vocab < 1)
    return fail(RL_ERR_INVALID_ARGUMENT, "n_seq/n_tokens < 0 or vocab < 1");
  if (n_tokens > 0 && n_seq == 0) return fail(RL_ERR_INVALID_ARGUMENT, "tokens without sequences");
  if (!cu_seqlens || (n_tokens > 0 && (!targets || !token_seq_out)) || (n_seq > 0 && !seq_active_out))
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL required pointer");
  if (adv_token_out && !seq_adv) return fail(RL_ERR_INVALID_ARGUMENT, "adv_token_out needs seq_adv");
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cudaStream_t s = (cudaStream_t)stream;
  if (counts_out && cudaMemsetAsync(counts_out, 0, sizeof(rl_batch_counts), s) != cudaSuccess)
    return check_launch("memset counts");
  if (n_seq > 0) {
    const int blocks = (int)std::min<int64_t>(148 * 4, (n_seq + 255) / 256);
    bk_seq_kernel<<<blocks, 256, 0, s>>>(seq_version, n_seq, trainer_version, seq_active_out,
                                         seq_staleness_out, counts_out);
    rl_status st = check_launch("bk_seq_kernel");
    if (st != RL_OK) return st;
  }
  if (n_tokens == 0) return RL_OK;
  const int64_t nruns = (n_tokens + kBkRun - 1) / kBkRun;
  const int blocks = (int)std::min<int64_t>(148 * 8, (nruns + kBkThreads - 1) / kBkThreads);
  bk_token_kernel<<<blocks, kBkThreads, 0, s>>>(cu_seqlens, n_seq, n_tokens, loss_mask, targets,
                                                vocab, seq_version, trainer_version, max_staleness,
                                                seq_adv, token_seq_out, seq_active_out,
                                                adv_token_out, valid_out, counts_out);
  return check_launch("bk_token_kernel");
}
