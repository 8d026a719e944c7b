// (5) Vocab-parallel log-prob (+ fused loss/grad on the local shard) — c8 of DESIGN.md §3
// (north_star: "by vocabulary (vocab-parallel log-softmax), with an NCCL all-reduce of
// per-token max, sum-exp and target logit over NVLink"; BASELINE.json configs[3]).
//
// Phase 1 (vp_stats_kernel): per row, (m_r, s_r) in the log2 domain over the local columns
//   and the target logit z_y if this rank owns column y -> 16 B per row.
// Phase 2: one ncclAllGather of those 16-B records over NVLink/NVSwitch.
// Phase 3 (vp_finish_kernel): M = max m_r, S = sum s_r 2^(m_r - M), lse, logp — identical
//   on every rank; with the loss, the token epilogue (stats counted on comm rank 0 only) and
//   the local dlogits shard s_t*(softmax - onehot) written in a second pass over the shard.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cluster_common.cuh"
#include "loss_common.cuh"
#include "rowstats.cuh"
#include "sm100.cuh"

namespace rl {

ncclComm_t comm_nccl(rl_comm* c);
int32_t comm_rank(const rl_comm* c);
int32_t comm_size(const rl_comm* c);
bool comm_peer_exchange(rl_comm* c, int64_t n_tokens, void** peers, int64_t* max_tokens, uint32_t* epoch);
rl_status launch_stats_reduce(const double* partials, int n_ctas, rl_loss_stats* stats,
                              bool accumulate, cudaStream_t s);

constexpr int kVpThreads = 256;
constexpr int kVpUnroll = 4;

template <typename T>
__global__ void __launch_bounds__(kVpThreads) vp_stats_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t Vr, int64_t offset, int64_t ld,
    const int32_t* __restrict__ targets, float inv_t, float4* __restrict__ rec) {
  __shared__ float red[64];
  const float k = inv_t * RL_LOG2E;
  const uint64_t keep = policy_evict_last();  // the finish pass re-reads the shard
  const int64_t row_bytes = ld * elem_bytes<T>();
  for (int64_t row = blockIdx.x; row < n_tokens; row += gridDim.x) {
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    MS st = row_stats_thread<T, kVpThreads, kVpUnroll>(rp, Vr, k, keep);
    st = block_reduce_ms<kVpThreads>(st, red);
    if (threadIdx.x == 0) {
      const int64_t yl = (int64_t)targets[row] - offset;
      const bool owned = targets[row] >= 0 && yl >= 0 && yl < Vr;
      const float zy = owned ? VecTraits<T>::load1(rp, yl) * inv_t : 0.f;
      rec[row] = make_float4(st.m, st.s, zy, owned ? 1.f : 0.f);
    }
  }
}

__device__ __forceinline__ float vp_combine(const float4* __restrict__ all, int64_t n_tokens,
                                            int P, int64_t row, float* zy_out) {
  float M = -INFINITY;
  for (int r = 0; r < P; ++r) M = fmaxf(M, all[(int64_t)r * n_tokens + row].x);
  float S = 0.f, zy = 0.f;
  for (int r = 0; r < P; ++r) {
    const float4 e = all[(int64_t)r * n_tokens + row];
    if (e.x != -INFINITY) S += e.y * fast_exp2(e.x - M);
    zy += e.z;
  }
  *zy_out = zy;
  return M + fast_log2(S);  // c2: log2-domain log-sum-exp
}

// logprob only: one thread per row
__global__ void vp_logp_kernel(const float4* __restrict__ all, int64_t n_tokens, int P,
                               int64_t vocab_total, const int32_t* __restrict__ targets,
                               float* __restrict__ logp_out, float* __restrict__ lse_out) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n_tokens;
       row += (int64_t)gridDim.x * blockDim.x) {
    float zy;
    const float c2 = vp_combine(all, n_tokens, P, row, &zy);
    const int32_t y = targets[row];
    float lp = 0.f;
    if (y >= 0 && (int64_t)y < vocab_total) lp = zy - c2 * RL_LN2;
    else if ((int64_t)y >= vocab_total) lp = __int_as_float(0x7fc00000);
    logp_out[row] = lp;
    if (lse_out) lse_out[row] = c2 * RL_LN2;
  }
}

template <typename T>
__global__ void __launch_bounds__(kVpThreads) vp_finish_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t Vr, int64_t offset,
    int64_t vocab_total, int64_t ld, const float4* __restrict__ all, int P,
    const int32_t* __restrict__ targets, const float* __restrict__ old_logp,
    const uint8_t* __restrict__ loss_mask, const int32_t* __restrict__ token_seq,
    const float* __restrict__ seq_adv, const int32_t* __restrict__ seq_version,
    const int32_t* __restrict__ seq_active, Knobs kn, int count_stats, void* dlogits,
    float* __restrict__ logp_out, float* __restrict__ lse_out, double* __restrict__ partials) {
  constexpr int EPV = VecTraits<T>::EPV;
  __shared__ float s_row[2];
  const float k = kn.inv_t * RL_LOG2E;
  const uint64_t drop = policy_evict_first();
  const int64_t row_bytes = ld * elem_bytes<T>();
  const double inv_tm = token_mean_inv(kn);
  Acc acc;
  acc.zero();
  for (int64_t row = blockIdx.x; row < n_tokens; row += gridDim.x) {
    if (threadIdx.x == 0) {
      const RowMeta mt = row_meta(row, vocab_total, targets, loss_mask, token_seq, seq_version,
                                  kn.trainer_version, kn.max_staleness);
      float zy;
      const float c2 = vp_combine(all, n_tokens, P, row, &zy);
      const float lp = logp_from(mt, zy, c2);
      if (logp_out) logp_out[row] = lp;
      if (lse_out) lse_out[row] = c2 * RL_LN2;
      const float A = mt.valid ? seq_adv[mt.seq] : 0.f;
      const float old = mt.valid ? old_logp[row] : 0.f;
      Acc tmp;
      tmp.zero();
      float prox_, ref_;
      token_extra(kn, row, old, prox_, ref_);
      const float s = token_epilogue(mt, lp, old, A, seq_active, inv_tm, kn, tmp, nullptr, prox_, ref_);
      if (count_stats)
        for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
      s_row[0] = s;
      s_row[1] = c2;
    }
    __syncthreads();
    const float s = s_row[0], c2 = s_row[1];
    __syncthreads();
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    char* dp = reinterpret_cast<char*>(dlogits) + row * row_bytes;
    const uint4* vrow = reinterpret_cast<const uint4*>(rp);
    uint4* vout = reinterpret_cast<uint4*>(dp);
    const int64_t nvec = Vr / EPV;
    const int64_t yl = (int64_t)targets[row] - offset;
    if (s == 0.f) {
      for (int64_t i = threadIdx.x; i < nvec; i += kVpThreads) st_stream_v4(vout + i, make_uint4(0, 0, 0, 0));
      for (int64_t c = nvec * EPV + threadIdx.x; c < Vr; c += kVpThreads) VecTraits<T>::store1(dp, c, 0.f);
      continue;
    }
    for (int64_t i = threadIdx.x; i < nvec; i += kVpThreads) {
      float f[EPV];
      VecTraits<T>::unpack(ld_hint_v4(vrow + i, drop), f);
#pragma unroll
      for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
      const int64_t c0 = i * EPV;
      onehot_sub(f, yl - c0, s);  // static indices: f stays in registers
      st_stream_v4(vout + i, VecTraits<T>::pack(f));
    }
    for (int64_t c = nvec * EPV + threadIdx.x; c < Vr; c += kVpThreads) {
      float v = s * fast_exp2(fmaf(VecTraits<T>::load1(rp, c), k, -c2));
      if (c == yl) v -= s;
      VecTraits<T>::store1(dp, c, v);
    }
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = acc.v[i];
}


// Warp-per-row forms of the two NCCL-path passes (default; the CTA-per-row kernels above are
// kept for RL_VP_KERNEL=block): a warp streams one row slice with 4 x 16-B loads in flight per
// lane and no block barriers (the layout of logprob_warp_kernel, 7 TB/s read).
constexpr int kVwThreads = 256;
constexpr int kVwWarps = kVwThreads / 32;

template <typename T>
__global__ void __launch_bounds__(kVwThreads) vp_stats_warp_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t Vr, int64_t offset, int64_t ld,
    const int32_t* __restrict__ targets, float inv_t, float4* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float k = inv_t * RL_LOG2E;
  const uint64_t pol = policy_evict_first();
  const int64_t row_bytes = ld * elem_bytes<T>();
  for (int64_t row = gw; row < n_tokens; row += nw) {
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    MS st = row_stats_thread<T, 32, 4>(rp, Vr, k, pol, lane);
    st = warp_reduce_ms(st);
    if (lane == 0) {
      const int32_t y = targets[row];
      const int64_t yl = (int64_t)y - offset;
      const bool owned = y >= 0 && yl >= 0 && yl < Vr;
      const float zy = owned ? VecTraits<T>::load1(rp, yl) * inv_t : 0.f;
      rec[row] = make_float4(st.m, st.s, zy, owned ? 1.f : 0.f);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kVwThreads, 4) vp_finish_warp_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t Vr, int64_t offset,
    int64_t vocab_total, int64_t ld, const float4* __restrict__ all, int P,
    const int32_t* __restrict__ targets, const float* __restrict__ old_logp,
    const uint8_t* __restrict__ loss_mask, const int32_t* __restrict__ token_seq,
    const float* __restrict__ seq_adv, const int32_t* __restrict__ seq_version,
    const int32_t* __restrict__ seq_active, Knobs kn, int count_stats, void* dlogits,
    float* __restrict__ logp_out, float* __restrict__ lse_out, double* __restrict__ partials) {
  constexpr int EPV = VecTraits<T>::EPV;
  __shared__ double wacc[kVwWarps][RL_LOSS_STATS_N];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float k = kn.inv_t * RL_LOG2E;
  const uint64_t pol = policy_evict_first();
  const int64_t row_bytes = ld * elem_bytes<T>();
  const int64_t nvec = Vr / EPV;
  const double inv_tm = token_mean_inv(kn);
  if (lane == 0)  // the warp's statistics live in shared memory (no fp64 registers in the loop)
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) wacc[warp][i] = 0.0;
  for (int64_t row = gw; row < n_tokens; row += nw) {
    float s = 0.f, c2 = 0.f;
    int64_t yl = -1;
    if (lane == 0) {
      const RowMeta mt = row_meta(row, vocab_total, targets, loss_mask, token_seq, seq_version,
                                  kn.trainer_version, kn.max_staleness);
      float zy;
      c2 = vp_combine(all, n_tokens, P, row, &zy);
      const float lp = logp_from(mt, zy, c2);
      if (logp_out) logp_out[row] = lp;
      if (lse_out) lse_out[row] = c2 * RL_LN2;
      const float A = mt.valid ? seq_adv[mt.seq] : 0.f;
      const float old = mt.valid ? old_logp[row] : 0.f;
      Acc tmp;
      tmp.zero();
      float prox_, ref_;
      token_extra(kn, row, old, prox_, ref_);
      s = token_epilogue(mt, lp, old, A, seq_active, inv_tm, kn, tmp, nullptr, prox_, ref_);
      if (count_stats)
        for (int i = 0; i < RL_LOSS_STATS_N; ++i) wacc[warp][i] += tmp.v[i];
      yl = (int64_t)mt.y - offset;
      if (!(mt.in_range && yl >= 0 && yl < Vr)) yl = -1;
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    c2 = __shfl_sync(0xffffffffu, c2, 0);
    yl = __shfl_sync(0xffffffffu, yl, 0);
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    char* dp = reinterpret_cast<char*>(dlogits) + row * row_bytes;
    const uint4* vrow = reinterpret_cast<const uint4*>(rp);
    uint4* vout = reinterpret_cast<uint4*>(dp);
    if (s == 0.f) {
      for (int64_t i = lane; i < nvec; i += 32) st_stream_v4(vout + i, make_uint4(0, 0, 0, 0));
      for (int64_t c = nvec * EPV + lane; c < Vr; c += 32) VecTraits<T>::store1(dp, c, 0.f);
      continue;
    }
    int64_t i = lane;
    for (; i + 3 * 32 < nvec; i += 4 * 32) {  // 4 vectors in flight per lane
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld_hint_v4(vrow + i + u * 32, pol);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[EPV];
        VecTraits<T>::unpack(v[u], f);
#pragma unroll
        for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
        const int64_t c0 = (i + u * 32) * EPV;
        onehot_sub(f, yl - c0, s);  // static indices: f stays in registers
        st_stream_v4(vout + i + u * 32, VecTraits<T>::pack(f));
      }
    }
    for (; i < nvec; i += 32) {
      float f[EPV];
      VecTraits<T>::unpack(ld_hint_v4(vrow + i, pol), f);
#pragma unroll
      for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
      const int64_t c0 = i * EPV;
      onehot_sub(f, yl - c0, s);  // static indices: f stays in registers
      st_stream_v4(vout + i, VecTraits<T>::pack(f));
    }
    for (int64_t c = nvec * EPV + lane; c < Vr; c += 32) {
      float v = s * fast_exp2(fmaf(VecTraits<T>::load1(rp, c), k, -c2));
      if (c == yl) v -= s;
      VecTraits<T>::store1(dp, c, v);
    }
  }
  // per-CTA partials: the warps' accumulators summed in warp order (deterministic)
  __syncthreads();
  if (threadIdx.x < RL_LOSS_STATS_N) {
    double t = 0.0;
    for (int w = 0; w < kVwWarps; ++w) t += wacc[w][threadIdx.x];
    partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + threadIdx.x] = t;
  }
}

// Finish pass, TMA-streamed (default): one CTA per SM walks rows blockIdx.x + k * gridDim.x.
// Warp 15 streams the row slices through a ring of 30 KB shared-memory slots (TMA bulk
// copies — the copy size that reads at full rate); warp 16 combines the
// ranks' records, runs the loss epilogue and publishes (s, c2, target column) one row ahead;
// warps 0..14 turn each landed chunk into dlogits (one MUFU.EX2 per element) with 128-bit
// streaming stores.
constexpr int kVtCons = 480, kVtThreads = 544, kVtVpt = 4;  // 15 consumer warps + producer + service
constexpr int kVtSlot = kVtVpt * kVtCons * 16;  // 30 KB
constexpr int kVtScale = 8;                     // rows of scales published ahead

template <typename T>
__global__ void __launch_bounds__(kVtThreads, 1) vp_finish_tma_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t Vr, int64_t offset,
    int64_t vocab_total, int64_t ld, const float4* __restrict__ all, int P,
    const int32_t* __restrict__ targets, const float* __restrict__ old_logp,
    const uint8_t* __restrict__ loss_mask, const int32_t* __restrict__ token_seq,
    const float* __restrict__ seq_adv, const int32_t* __restrict__ seq_version,
    const int32_t* __restrict__ seq_active, Knobs kn, int count_stats, void* dlogits,
    float* __restrict__ logp_out, float* __restrict__ lse_out, double* __restrict__ partials,
    int nslots) {
  constexpr int EPV = VecTraits<T>::EPV;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nslots;
  uint64_t* scbar = empty + nslots;          // [kVtScale] service warp published row k's scale
  uint64_t* donebar = scbar + kVtScale;      // [kVtScale] consumers finished row k (15 arrivals)
  float4* sc = reinterpret_cast<float4*>(smem + 8 * (2 * nslots + 2 * kVtScale) + 64);  // [kVtScale]
  unsigned char* ring = smem + ((8 * (2 * nslots + 2 * kVtScale) + 64 + 16 * kVtScale + 127) & ~127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nvec = Vr / EPV;
  const int64_t row_bytes = ld * elem_bytes<T>();
  const int64_t slice_bytes = nvec * 16;
  const int nch = (int)((slice_bytes + kVtSlot - 1) / kVtSlot);
  const int64_t nk = blockIdx.x < n_tokens ? (n_tokens - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const float k = kn.inv_t * RL_LOG2E;
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], 15);
    }
    for (int i = 0; i < kVtScale; ++i) {
      sm100::mbar_init(&scbar[i], 1);
      sm100::mbar_init(&donebar[i], 15);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t full_s = sm100::smem_u32(full), empty_s = sm100::smem_u32(empty);
  const uint32_t ring_s = sm100::smem_u32(ring);
  if (warp >= 15) {
    if (warp == 15 && lane == 0 && nch > 0) {  // ---- TMA producer (its own warp)
      RingPos rp{0, 0};
      for (int64_t kk = 0; kk < nk; ++kk) {
        const char* src = reinterpret_cast<const char*>(logits) + ((int64_t)blockIdx.x + kk * gridDim.x) * row_bytes;
        for (int c = 0; c < nch; ++c) {
          sm100::mbar_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1);
          const uint32_t bytes = (uint32_t)min((int64_t)kVtSlot, slice_bytes - (int64_t)c * kVtSlot);
          sm100::mbar_arrive_expect_tx(&full[rp.slot], bytes);
          sm100::bulk_g2s_nohint(ring + (size_t)rp.slot * kVtSlot, src + (size_t)c * kVtSlot, bytes, &full[rp.slot]);
          rp.advance(1, nslots);
        }
      }
    } else if (warp == 16 && lane == 0) {  // ---- service warp: combine + loss epilogue, rows ahead
      const double inv_tm = token_mean_inv(kn);
      Acc acc;
      acc.zero();
      for (int64_t kk = 0; kk < nk; ++kk) {
        const int64_t row = (int64_t)blockIdx.x + kk * gridDim.x;
        const RowMeta mt = row_meta(row, vocab_total, targets, loss_mask, token_seq, seq_version,
                                    kn.trainer_version, kn.max_staleness);
        float zy;
        const float c2 = vp_combine(all, n_tokens, P, row, &zy);
        const float lp = logp_from(mt, zy, c2);
        if (logp_out) logp_out[row] = lp;
        if (lse_out) lse_out[row] = c2 * RL_LN2;
        const float A = mt.valid ? seq_adv[mt.seq] : 0.f;
        const float old = mt.valid ? old_logp[row] : 0.f;
        Acc tmp;
        tmp.zero();
        float prox_, ref_;
        token_extra(kn, row, old, prox_, ref_);
        const float st = token_epilogue(mt, lp, old, A, seq_active, inv_tm, kn, tmp, nullptr, prox_, ref_);
        if (count_stats)
          for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
        const int64_t yl = (int64_t)mt.y - offset;
        const int ycol = (mt.in_range && yl >= 0 && yl < Vr) ? (int)yl : -1;
        const int q = (int)(kk % kVtScale);
        if (kk >= kVtScale) sm100::mbar_wait_polite(&donebar[q], (uint32_t)(((kk - kVtScale) / kVtScale) & 1), false);
        sc[q] = make_float4(st, c2, 0.f, __int_as_float(ycol));
        sm100::mbar_arrive(&scbar[q]);
      }
      for (int i = 0; i < RL_LOSS_STATS_N; ++i) partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = acc.v[i];
    }
    return;
  }
  // ---- consumers
  uint32_t slot = 0, rph = 0;
  const uint32_t my_off = (uint32_t)tid * 16u;
  for (int64_t kk = 0; kk < nk; ++kk) {
    const int64_t row = (int64_t)blockIdx.x + kk * gridDim.x;
    const int q = (int)(kk % kVtScale);
    sm100::mbar_wait(&scbar[q], (uint32_t)((kk / kVtScale) & 1));
    const float4 r = sc[q];
    const float s = r.x, c2 = r.y;
    const int64_t yl = __float_as_int(r.w);
    char* dp = reinterpret_cast<char*>(dlogits) + row * row_bytes;
    uint4* vout = reinterpret_cast<uint4*>(dp);
    for (int c = 0; c < nch; ++c) {
      sm100::mbar_wait_a(full_s + slot * 8, rph);
#pragma unroll
      for (int u = 0; u < kVtVpt; ++u) {
        const int64_t i = ((int64_t)c * kVtVpt + u) * kVtCons + tid;  // vector index in the slice
        if (i < nvec) {
          uint4 o = make_uint4(0, 0, 0, 0);
          if (s != 0.f) {
            float f[EPV];
            VecTraits<T>::unpack(sm100::lds128_a(ring_s + slot * (uint32_t)kVtSlot + u * (kVtCons * 16) + my_off), f);
#pragma unroll
            for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
            const int64_t c0 = i * EPV;
            onehot_sub(f, yl - c0, s);  // static indices: f stays in registers
            o = VecTraits<T>::pack(f);
          }
          st_stream_v4(vout + i, o);
        }
      }
      sm100::mbar_arrive_lane0(empty_s + slot * 8, lane);
      if (++slot == (uint32_t)nslots) {
        slot = 0;
        rph ^= 1u;
      }
    }
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    for (int64_t cc = nvec * EPV + tid; cc < Vr; cc += kVtCons) {  // scalar tail columns
      float v = (s == 0.f) ? 0.f : s * fast_exp2(fmaf(VecTraits<T>::load1(rp, cc), k, -c2));
      if (s != 0.f && cc == yl) v -= s;
      VecTraits<T>::store1(dp, cc, v);
    }
    sm100::mbar_arrive_lane0(sm100::smem_u32(&donebar[q]), lane);
  }
}

// ---------------------------------------------------------------------------------------
// Fused vocab-parallel loss with in-kernel peer exchange (rl_comm_enable_peer_exchange).
// One CTA per SM; each CTA walks its rows (row = blockIdx.x + k * gridDim.x, the same on every
// rank).  A 4-deep ring of row slices in shared memory (TMA bulk loads): the statistics of row
// k+1 are computed and published to every rank (NVLink stores of a 16-B record + a flag carrying
// the call's epoch) BEFORE the kernel waits for the peers' records of row k, so the exchange
// latency hides behind the next row's pass; then row k is combined (M, S, lse, logp, loss
// epilogue) and its dlogits slice written from shared memory.  Logits read once, dlogits once.
constexpr int kVfThreads = 512;
constexpr int kVfBufs = 4;

struct VfArgs {
  const void* logits;
  void* dlogits;
  int64_t n, Vr, off, Vtot, ld, max_tokens;
  const int32_t* targets;
  const float* old_logp;
  const uint8_t* mask;
  const int32_t* token_seq;
  const float* seq_adv;
  const int32_t* seq_version;
  const int32_t* seq_active;
  float* logp_out;
  float* lse_out;
  double* partials;
  Knobs kn;
  int32_t count_stats, P, me;
  int32_t nb;  // vp_fused_kernel: shared-memory row buffers (2..4)
  int32_t pf;  // vp_fused2_kernel: L2 prefetch distance in row groups (0 = off)
  int32_t trace;  // vp_fused2_kernel: record g_trace_vp2
  uint32_t epoch;
  float4* rec[8];     // rank q's record array  [P][max_tokens]
  uint32_t* flag[8];  // rank q's flag array    [P][max_tokens]
};

template <typename T>
__global__ void __launch_bounds__(kVfThreads, 1) vp_fused_kernel(const VfArgs a) {
  constexpr int EPV = VecTraits<T>::EPV;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  float* red = reinterpret_cast<float*>(smem + 64);                 // 64 floats
  float4* rsc = reinterpret_cast<float4*>(smem + 64 + 256);         // per buffer (st, c2, dy, ycol)
  unsigned char* bufs = smem + 1024;
  const int64_t nvec = a.Vr / EPV;                                  // whole 16-B vectors per slice
  const int64_t slice_bytes = (a.Vr * elem_bytes<T>() + 15) / 16 * 16;
  const int64_t row_bytes = a.ld * elem_bytes<T>();
  const int tid = threadIdx.x;
  const float k = a.kn.inv_t * RL_LOG2E;
  const int64_t nk = blockIdx.x < a.n ? (a.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const double inv_tm = token_mean_inv(a.kn);
  Acc acc;
  acc.zero();
  if (tid == 0) {
    for (int i = 0; i < kVfBufs; ++i) sm100::mbar_init(&full[i], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  auto row_of = [&](int64_t kk) { return (int64_t)blockIdx.x + kk * gridDim.x; };
  const int nb = a.nb;
  auto issue = [&](int64_t kk) {
    if (tid == 0 && kk < nk) {
      const int b = (int)(kk % nb);
      sm100::mbar_arrive_expect_tx(&full[b], (uint32_t)slice_bytes);
      sm100::bulk_g2s_nohint(bufs + (size_t)b * slice_bytes,
                             reinterpret_cast<const char*>(a.logits) + row_of(kk) * row_bytes, (uint32_t)slice_bytes,
                             &full[b]);
    }
  };
  // statistics of row kk (buffer kk % 4) -> record published to every rank
  auto stats_publish = [&](int64_t kk) {
    const int b = (int)(kk % nb);
    sm100::mbar_wait(&full[b], (uint32_t)((kk / nb) & 1));
    const unsigned char* rowp = bufs + (size_t)b * slice_bytes;
    const uint4* vrow = reinterpret_cast<const uint4*>(rowp);
    MS st{-INFINITY, 0.f};
    int64_t i = tid;
    for (; i + kVfThreads < nvec; i += 2 * kVfThreads) {  // two shared-memory vectors per step
      float f[2 * EPV];
      VecTraits<T>::unpack(vrow[i], f);
      VecTraits<T>::unpack(vrow[i + kVfThreads], f + EPV);
      ms_update<2 * EPV>(st, f, k);
    }
    for (; i < nvec; i += kVfThreads) {
      float f[EPV];
      VecTraits<T>::unpack(vrow[i], f);
      ms_update<EPV>(st, f, k);
    }
    st = block_reduce_ms<kVfThreads>(st, red);
    if (tid == 0) {
      const int64_t row = row_of(kk);
      const int32_t y = a.targets[row];
      const int64_t yl = (int64_t)y - a.off;
      // columns past the whole vectors (Vr % EPV) live in the same smem row
      MS tail{-INFINITY, 0.f};
      for (int64_t c = nvec * EPV; c < a.Vr; ++c) {
        float f[1] = {VecTraits<T>::load1(rowp, c)};
        ms_update<1>(tail, f, k);
      }
      st = ms_combine(st, tail);
      const bool owned = y >= 0 && yl >= 0 && yl < a.Vr;
      const float zy = owned ? VecTraits<T>::load1(rowp, yl) * a.kn.inv_t : 0.f;
      const float4 rec = make_float4(st.m, st.s, zy, owned ? 1.f : 0.f);
      for (int q = 0; q < a.P; ++q) a.rec[q][(int64_t)a.me * a.max_tokens + row] = rec;
      __threadfence_system();
      for (int q = 0; q < a.P; ++q)
        *reinterpret_cast<volatile uint32_t*>(&a.flag[q][(int64_t)a.me * a.max_tokens + row]) = a.epoch;
    }
  };
  for (int q = 0; q < nb - 1; ++q) issue(q);
  if (nk > 0) stats_publish(0);
  for (int64_t kk = 0; kk < nk; ++kk) {
    issue(kk + nb - 1);                   // buffer (kk+nb-1)%nb == (kk-1)%nb, freed at the end of kk-1
    if (kk + 1 < nk) stats_publish(kk + 1);
    const int b = (int)(kk % nb);
    const int64_t row = row_of(kk);
    if (tid == 0) {  // wait for every rank's record of this row, then combine + loss epilogue
      for (int q = 0; q < a.P; ++q) {
        const volatile uint32_t* f = &a.flag[a.me][(int64_t)q * a.max_tokens + row];
        while (*f != a.epoch) {
        }
      }
      __threadfence_system();
      float M = -INFINITY;
      for (int q = 0; q < a.P; ++q) M = fmaxf(M, a.rec[a.me][(int64_t)q * a.max_tokens + row].x);
      float S = 0.f, zy = 0.f;
      for (int q = 0; q < a.P; ++q) {
        const float4 e = a.rec[a.me][(int64_t)q * a.max_tokens + row];
        if (e.x != -INFINITY) S += e.y * fast_exp2(e.x - M);
        zy += e.z;
      }
      const float c2 = M + fast_log2(S);
      const RowMeta mt = row_meta(row, a.Vtot, a.targets, a.mask, a.token_seq, a.seq_version,
                                  a.kn.trainer_version, a.kn.max_staleness);
      const float lp = logp_from(mt, zy, c2);
      if (a.logp_out) a.logp_out[row] = lp;
      if (a.lse_out) a.lse_out[row] = c2 * RL_LN2;
      const float A = mt.valid ? a.seq_adv[mt.seq] : 0.f;
      const float old = mt.valid ? a.old_logp[row] : 0.f;
      Acc tmp;
      tmp.zero();
      float prox_, ref_;
      token_extra(a.kn, row, old, prox_, ref_);
      const float s = token_epilogue(mt, lp, old, A, a.seq_active, inv_tm, a.kn, tmp, nullptr, prox_, ref_);
      if (a.count_stats)
        for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
      const int64_t yl = (int64_t)mt.y - a.off;
      const int ycol = (mt.in_range && yl >= 0 && yl < a.Vr) ? (int)yl : -1;
      rsc[b] = make_float4(s, c2, s * (fast_exp2(zy * RL_LOG2E - c2) - 1.f), __int_as_float(ycol));
    }
    __syncthreads();
    const float4 sc = rsc[b];
    const float s = sc.x, c2 = sc.y, dy = sc.z;
    const int ycol = __float_as_int(sc.w);
    const unsigned char* rowp = bufs + (size_t)b * slice_bytes;
    char* dp = reinterpret_cast<char*>(a.dlogits) + row * row_bytes;
    const uint4* vin = reinterpret_cast<const uint4*>(rowp);
    uint4* vout = reinterpret_cast<uint4*>(dp);
    for (int64_t i = tid; i < nvec; i += kVfThreads) {
      float f[EPV];
      if (s == 0.f) {
#pragma unroll
        for (int j = 0; j < EPV; ++j) f[j] = 0.f;
      } else {
        VecTraits<T>::unpack(vin[i], f);
#pragma unroll
        for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
        const int64_t c0 = i * EPV;
        onehot_set(f, ycol - c0, dy);
      }
      st_stream_v4(vout + i, VecTraits<T>::pack(f));
    }
    for (int64_t c = nvec * EPV + tid; c < a.Vr; c += kVfThreads) {
      float v = (s == 0.f) ? 0.f : s * fast_exp2(fmaf(VecTraits<T>::load1(rowp, c), k, -c2));
      if (s != 0.f && c == ycol) v = dy;
      VecTraits<T>::store1(dp, c, v);
    }
    __syncthreads();  // buffer b free for the load of row kk + nb
  }
  if (tid == 0)
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = acc.v[i];
}

// ---------------------------------------------------------------------------------------
// Fused vocab-parallel loss v2 (default with peer exchange): 2 HBM units per row slice.
// Rows blockIdx.x + k * gridDim.x are processed in groups of G = 16 / WPR, one row per team of WPR
// consumer warps (two groups of every CTA fit in L2: G * slice <= ~300 KB).  Each team runs, per
// group g: pass 1 of its row of group g — streamed from HBM (evict_last, 8 vectors in flight per
// thread) into the row's (max, sum 2^(t - max), target logit) record — then pass 2 of its row of
// group g-1, re-read from L2 (evict_first) into dlogits.  Service warp 16 lane 0 (it stores no
// dlogits, so its system fence covers only its own few stores) publishes a group's records to
// every rank's buffer with ONE fence, waits for the peers' records of that group, combines them
// in rank order, runs the loss epilogue and publishes the row scales — while the teams stream
// the next group.
// development phase trace (RL_TRACE): per CTA, team 0 thread 0's cycles in pass 1, waiting for
// the row scales, and pass 2, plus the service lane's cycles waiting for the peers' records
__device__ unsigned long long g_trace_vp2[256][4];
constexpr int kV2Warps = 16;
constexpr int kV2U1 = 10;  // pass-1 vectors in flight per thread
constexpr int kV2U2 = 4;   // pass-2 (L2 re-read) vectors in flight per thread (10 spills: slower)
constexpr int kV2Cons = kV2Warps * 32;

template <typename T, int WPR>
__global__ void __launch_bounds__(kV2Cons + 32, 1) vp_fused2_kernel(const VfArgs a) {
  constexpr int EPV = VecTraits<T>::EPV;
  constexpr int G = kV2Warps / WPR;  // rows per group = teams
  constexpr int NT = WPR * 32;       // threads per team
  __shared__ float4 grp_rec[2][G];   // [group parity][team] this rank's records
  __shared__ float4 grp_sc[2][G];    // (s, c2, -, target column or -1)
  __shared__ float red_m[2][kV2Warps], red_s[2][kV2Warps];
  __shared__ __align__(8) uint64_t stats_bar[2], scale_bar[2], done_bar[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nk = blockIdx.x < a.n ? (a.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t ng = (nk + G - 1) / G;
  const int64_t row_bytes = a.ld * elem_bytes<T>();
  const int64_t nvec = a.Vr / EPV;
  const float k = a.kn.inv_t * RL_LOG2E;
  auto row_of = [&](int64_t kk) { return (int64_t)blockIdx.x + kk * gridDim.x; };
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&stats_bar[i], G);
      sm100::mbar_init(&scale_bar[i], 1);
      sm100::mbar_init(&done_bar[i], kV2Warps);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (warp == kV2Warps) {
    if (lane != 0) return;
    // ------------------------------------------------------------------ service lane
    const double inv_tm = token_mean_inv(a.kn);
    Acc acc;
    acc.zero();
    for (int64_t g = 0; g < ng; ++g) {
      const int b = (int)(g & 1);
      const int64_t k0 = g * G, k1 = min(nk, k0 + G);
      sm100::mbar_wait_polite(&stats_bar[b], (uint32_t)((g >> 1) & 1), false);
      for (int64_t kk = k0; kk < k1; ++kk) {  // records -> every rank (this rank's slot [me][row])
        const float4 r = grp_rec[b][kk - k0];
        const int64_t row = row_of(kk);
        for (int q = 0; q < a.P; ++q) a.rec[q][(int64_t)a.me * a.max_tokens + row] = r;
      }
      __threadfence_system();
      for (int64_t kk = k0; kk < k1; ++kk)
        for (int q = 0; q < a.P; ++q)
          *reinterpret_cast<volatile uint32_t*>(&a.flag[q][(int64_t)a.me * a.max_tokens + row_of(kk)]) = a.epoch;
      // the scale slot of group g-2 must be free: its pass 2 is done
      if (g >= 2) sm100::mbar_wait_polite(&done_bar[b], (uint32_t)(((g - 2) >> 1) & 1), false);
      const long long tw0 = clock64();
      for (int64_t kk = k0; kk < k1; ++kk) {
        const int64_t row = row_of(kk);
        for (int q = 0; q < a.P; ++q) {
          const volatile uint32_t* f = &a.flag[a.me][(int64_t)q * a.max_tokens + row];
          while (*f != a.epoch) __nanosleep(20);
        }
      }
      if (a.trace && blockIdx.x < 256) g_trace_vp2[blockIdx.x][3] += (unsigned long long)(clock64() - tw0);
      __threadfence_system();
      for (int64_t kk = k0; kk < k1; ++kk) {
        const int64_t row = row_of(kk);
        float M = -INFINITY;
        for (int q = 0; q < a.P; ++q) M = fmaxf(M, a.rec[a.me][(int64_t)q * a.max_tokens + row].x);
        float S = 0.f, zy = 0.f;
        for (int q = 0; q < a.P; ++q) {
          const float4 e = a.rec[a.me][(int64_t)q * a.max_tokens + row];
          if (e.x != -INFINITY) S += e.y * fast_exp2(e.x - M);
          zy += e.z;
        }
        const float c2 = M + fast_log2(S);
        const RowMeta mt = row_meta(row, a.Vtot, a.targets, a.mask, a.token_seq, a.seq_version,
                                    a.kn.trainer_version, a.kn.max_staleness);
        const float lp = logp_from(mt, zy, c2);
        if (a.logp_out) a.logp_out[row] = lp;
        if (a.lse_out) a.lse_out[row] = c2 * RL_LN2;
        const float A = mt.valid ? a.seq_adv[mt.seq] : 0.f;
        const float old = mt.valid ? a.old_logp[row] : 0.f;
        float prox_, ref_;
        token_extra(a.kn, row, old, prox_, ref_);
        Acc tmp;
        tmp.zero();
        const float st = token_epilogue(mt, lp, old, A, a.seq_active, inv_tm, a.kn, tmp, nullptr, prox_, ref_);
        if (a.count_stats)
          for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
        const int64_t yl = (int64_t)mt.y - a.off;
        const int ycol = (mt.in_range && yl >= 0 && yl < a.Vr) ? (int)yl : -1;
        grp_sc[b][kk - k0] = make_float4(st, c2, st * (fast_exp2(zy * RL_LOG2E - c2) - 1.f), __int_as_float(ycol));
      }
      sm100::mbar_arrive(&scale_bar[b]);
    }
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = acc.v[i];
    return;
  }
  // -------------------------------------------------------------------- row teams
  const int team = warp / WPR, t = tid % NT;
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  const int pf = a.pf;  // L2 prefetch distance in groups (0 = off)
  const uint32_t slice16 = (uint32_t)((a.Vr * elem_bytes<T>() + 15) / 16 * 16);
  if (t == 0)
    for (int64_t gg = 0; gg < ((int64_t)pf < ng ? (int64_t)pf : ng); ++gg)
      if (gg * G + team < nk)
        sm100::bulk_prefetch_l2(reinterpret_cast<const char*>(a.logits) + row_of(gg * G + team) * row_bytes, slice16);
  for (int64_t g = 0; g <= ng; ++g) {
    const bool tr = a.trace && tid == 0 && blockIdx.x < 256;
    long long tc = tr ? clock64() : 0;
    if (g < ng) {  // ---- pass 1 of group g: this team's row record
      const int b = (int)(g & 1);
      const int64_t kk = g * G + team;
      if (pf > 0 && t == 0 && kk + pf * G < nk)  // pull the team's row of group g + pf into L2
        sm100::bulk_prefetch_l2(reinterpret_cast<const char*>(a.logits) + row_of(kk + pf * G) * row_bytes, slice16);
      MS st{-INFINITY, 0.f};
      const char* rp = nullptr;
      if (kk < nk) {
        rp = reinterpret_cast<const char*>(a.logits) + row_of(kk) * row_bytes;
        // every load of a round in flight, predicated (no serial tail: a thread owns ~nvec / NT
        // vectors, e.g. 18.5 at P = 4, which two rounds of kV2U1 cover)
        const uint4* vrow = reinterpret_cast<const uint4*>(rp);
        for (int64_t i0 = t; i0 < nvec; i0 += (int64_t)kV2U1 * NT) {
          uint4 v[kV2U1];
#pragma unroll
          for (int u = 0; u < kV2U1; ++u)
            v[u] = (i0 + u * NT < nvec) ? ld_hint_v4(vrow + i0 + u * NT, keep) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int u = 0; u < kV2U1; ++u) {
            float f[EPV];
            VecTraits<T>::unpack(v[u], f);
            if (i0 + u * NT >= nvec) {
#pragma unroll
              for (int j = 0; j < EPV; ++j) f[j] = -INFINITY;
            }
            ms_update<EPV>(st, f, k);
          }
        }
        for (int64_t c = nvec * EPV + t; c < a.Vr; c += NT) {
          float f[1] = {VecTraits<T>::load1(rp, c)};
          ms_update<1>(st, f, k);
        }
      }
      st = warp_reduce_ms(st);
      if (WPR > 1) {
        if (lane == 0) {
          red_m[b][warp] = st.m;
          red_s[b][warp] = st.s;
        }
        sm100::named_bar_sync(1 + team, NT);
      }
      if (t == 0) {
        if (kk < nk) {
          MS r = st;
          for (int w = 1; w < WPR; ++w) r = ms_combine(r, MS{red_m[b][warp + w], red_s[b][warp + w]});
          const int32_t y = a.targets[row_of(kk)];
          const int64_t yl = (int64_t)y - a.off;
          const bool owned = y >= 0 && yl >= 0 && yl < a.Vr;
          const float zy = owned ? VecTraits<T>::load1(rp, yl) * a.kn.inv_t : 0.f;
          grp_rec[b][team] = make_float4(r.m, r.s, zy, owned ? 1.f : 0.f);
        }
        sm100::mbar_arrive(&stats_bar[b]);
      }
    }
    if (g >= 1) {  // ---- pass 2 of group g-1: this team's row, from L2
      const int64_t gp = g - 1;
      const int b = (int)(gp & 1);
      const int64_t kk = gp * G + team;
      if (tr) {
        const long long t1 = clock64();
        g_trace_vp2[blockIdx.x][0] += (unsigned long long)(t1 - tc);
        tc = t1;
      }
      sm100::mbar_wait(&scale_bar[b], (uint32_t)((gp >> 1) & 1));
      if (tr) {
        const long long t1 = clock64();
        g_trace_vp2[blockIdx.x][1] += (unsigned long long)(t1 - tc);
        tc = t1;
      }
      if (kk < nk) {
        const int64_t row = row_of(kk);
        const float4 sc = grp_sc[b][team];
        const float s = sc.x, c2 = sc.y, dy = sc.z;
        const int64_t yl = __float_as_int(sc.w);
        const char* rp = reinterpret_cast<const char*>(a.logits) + row * row_bytes;
        char* dp = reinterpret_cast<char*>(a.dlogits) + row * row_bytes;
        const uint4* vrow = reinterpret_cast<const uint4*>(rp);
        uint4* vout = reinterpret_cast<uint4*>(dp);
        if (s == 0.f) {
          for (int64_t i = t; i < nvec; i += NT) st_stream_v4(vout + i, make_uint4(0, 0, 0, 0));
        } else {
          constexpr int U = kV2U2;
          for (int64_t i0 = t; i0 < nvec; i0 += U * NT) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (i0 + u * NT < nvec) v[u] = ld_hint_v4(vrow + i0 + u * NT, drop);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int64_t i = i0 + u * NT;
              if (i < nvec) {
                float f[EPV];
                VecTraits<T>::unpack(v[u], f);
#pragma unroll
                for (int j = 0; j < EPV; ++j) f[j] = s * fast_exp2(fmaf(f[j], k, -c2));
                onehot_set(f, yl - i * EPV, dy);
                st_stream_v4(vout + i, VecTraits<T>::pack(f));
              }
            }
          }
        }
        for (int64_t c = nvec * EPV + t; c < a.Vr; c += NT) {
          float v = (s == 0.f) ? 0.f : s * fast_exp2(fmaf(VecTraits<T>::load1(rp, c), k, -c2));
          if (s != 0.f && c == yl) v = dy;
          VecTraits<T>::store1(dp, c, v);
        }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&done_bar[b]);
      if (tr) g_trace_vp2[blockIdx.x][2] += (unsigned long long)(clock64() - tc);
    }
  }
}

template <typename T>
static void launch_vp_fused2(const VfArgs& v0, int64_t slice_bytes, int grid, cudaStream_t s) {
  // rows per group G = 16 / WPR: the largest power of two with G * slice <= 300 KB
  // (RL_VP2_WPR=1|2|4|8|16 forces the team size: tests run every instantiation at small shapes)
  // (RL_VP2_PF = L2 prefetch distance in groups, default 1; the groups resident in L2 are then
  //  pass 2's, pass 1's and the prefetched ones: budget 200 KB per group, 300 KB without prefetch)
  static int forced = -1, pf = -1;
  if (forced < 0) forced = getenv("RL_VP2_WPR") ? atoi(getenv("RL_VP2_WPR")) : 0;
  if (pf < 0) pf = getenv("RL_VP2_PF") ? std::max(0, atoi(getenv("RL_VP2_PF"))) : 1;
  VfArgs v = v0;
  v.pf = pf;
  static int trace = -1;
  if (trace < 0) trace = getenv("RL_TRACE") ? 1 : 0;
  v.trace = trace;
  const int64_t budget = getenv("RL_VP2_BUDGET_KB") ? (int64_t)atoi(getenv("RL_VP2_BUDGET_KB")) << 10
                                                     : (pf > 0 ? 200 << 10 : 300 << 10);
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16) slice_bytes = budget / (16 / forced);
  if (slice_bytes * 16 <= budget) vp_fused2_kernel<T, 1><<<grid, kV2Cons + 32, 0, s>>>(v);
  else if (slice_bytes * 8 <= budget) vp_fused2_kernel<T, 2><<<grid, kV2Cons + 32, 0, s>>>(v);
  else if (slice_bytes * 4 <= budget) vp_fused2_kernel<T, 4><<<grid, kV2Cons + 32, 0, s>>>(v);
  else if (slice_bytes * 2 <= budget) vp_fused2_kernel<T, 8><<<grid, kV2Cons + 32, 0, s>>>(v);
  else vp_fused2_kernel<T, 16><<<grid, kV2Cons + 32, 0, s>>>(v);
}

static int vp_grid(int64_t n) {
  static int ctas = 0;
  if (!ctas) {
    int dev = 0, sms = 148, occ = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vp_stats_kernel<bf16_t>, kVpThreads, 0);
    ctas = std::min(sms * std::max(occ, 1), kMaxStatCtas);
  }
  return (int)std::min<int64_t>(n, ctas);
}

}  // namespace rl

extern "C" size_t rl_vocab_parallel_workspace_size(int64_t n_tokens, int32_t nranks) {
  if (n_tokens < 0 || nranks < 1) return 0;
  const size_t rec = (size_t)n_tokens * 16;
  return rl::kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double) + rec * (1 + (size_t)nranks);
}

extern "C" rl_status rl_vocab_parallel_logprob(
    const void* logits_shard, int32_t dtype, int64_t n_tokens, int64_t vocab_shard,
    int64_t vocab_offset, int64_t vocab_total, int64_t ld, const int32_t* targets,
    float inv_temperature, rl_comm* comm, float* logp_out, float* lse_out, const float* old_logp,
    const uint8_t* loss_mask, const int32_t* token_seq, const float* seq_adv,
    const int32_t* seq_version, const int32_t* seq_active, const rl_loss_params* p,
    void* dlogits_shard, rl_loss_stats* stats, void* workspace, size_t workspace_bytes,
    rl_stream stream) {
  using namespace rl;
  if (!comm) return fail(RL_ERR_INVALID_ARGUMENT, "NULL comm");
  if (n_tokens < 0 || vocab_shard < 0 || vocab_offset < 0 || vocab_total < 1 ||
      vocab_offset + vocab_shard > vocab_total || ld < vocab_shard || ld < 1)
    return fail(RL_ERR_INVALID_ARGUMENT, "bad sizes (n_tokens/vocab_shard/offset/total/ld)");
  if (dtype != RL_F32 && dtype != RL_BF16) return fail(RL_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (!(inv_temperature > 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be > 0");
  const int P = comm_size(comm);
  if (!workspace || workspace_bytes < rl_vocab_parallel_workspace_size(n_tokens, P))
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes",
                rl_vocab_parallel_workspace_size(n_tokens, P));
  const bool with_loss = old_logp != nullptr;
  if (n_tokens > 0 && (!targets || !logp_out || (vocab_shard > 0 && !logits_shard)))
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL logits_shard/targets/logp_out");
  if (with_loss) {
    if (!p || !token_seq || !seq_adv || !stats || (vocab_shard > 0 && !dlogits_shard))
      return fail(RL_ERR_INVALID_ARGUMENT, "fused loss needs p, token_seq, seq_adv, stats, dlogits_shard");
    if (p->agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN && !seq_active)
      return fail(RL_ERR_INVALID_ARGUMENT, "SEQ_MEAN_TOKEN_MEAN needs seq_active");
    if (p->kl_coef != 0.f && !p->ref_logp) return fail(RL_ERR_INVALID_ARGUMENT, "kl_coef != 0 needs ref_logp");
    if (p->flags & RL_F_ENTROPY)
      return fail(RL_ERR_UNSUPPORTED, "RL_F_ENTROPY is not available on the vocab-parallel path");
  }
  const int64_t eb = dtype == RL_BF16 ? 2 : 4;
  if (((uintptr_t)logits_shard & 15) || ((uintptr_t)dlogits_shard & 15) || (ld * eb) % 16)
    return fail(RL_ERR_ALIGNMENT, "shards must be 16-B aligned with ld*elem %% 16 == 0");
  cudaStream_t s = (cudaStream_t)stream;
  double* partials = (double*)workspace;
  float4* send = reinterpret_cast<float4*>((char*)workspace + kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double));
  float4* recv = send + n_tokens;
  if (n_tokens == 0) {
    if (with_loss && !(p->flags & RL_F_STATS_ACCUMULATE)) cudaMemsetAsync(stats, 0, sizeof(rl_loss_stats), s);
    return check_launch("vp empty");
  }
  void* peers[8];
  int64_t max_tok = 0;
  uint32_t epoch = 0;
  const int64_t slice_bytes = (vocab_shard * eb + 15) / 16 * 16;
  const int nbuf = (int)std::min<int64_t>(kVfBufs, (232448 - 1024) / std::max<int64_t>(slice_bytes, 16));
  const size_t vf_smem = 1024 + (size_t)nbuf * slice_bytes;
  static int fused_v1 = -1;  // RL_VP_FUSED=smem: the first in-kernel exchange kernel (row slices in smem)
  if (fused_v1 < 0) fused_v1 = (getenv("RL_VP_FUSED") && strcmp(getenv("RL_VP_FUSED"), "smem") == 0) ? 1 : 0;
  if (with_loss && (!fused_v1 || nbuf >= 2) && comm_peer_exchange(comm, n_tokens, peers, &max_tok, &epoch)) {
    VfArgs v;
    v.logits = logits_shard;
    v.dlogits = dlogits_shard;
    v.n = n_tokens;
    v.Vr = vocab_shard;
    v.off = vocab_offset;
    v.Vtot = vocab_total;
    v.ld = ld;
    v.max_tokens = max_tok;
    v.targets = targets;
    v.old_logp = old_logp;
    v.mask = loss_mask;
    v.token_seq = token_seq;
    v.seq_adv = seq_adv;
    v.seq_version = seq_version;
    v.seq_active = seq_active;
    v.logp_out = logp_out;
    v.lse_out = lse_out;
    v.partials = partials;
    v.kn = make_knobs(p);
    v.count_stats = comm_rank(comm) == 0;
    v.P = P;
    v.me = comm_rank(comm);
    v.epoch = epoch;
    v.nb = nbuf;
    for (int q = 0; q < 8; ++q) {
      v.rec[q] = q < P ? reinterpret_cast<float4*>(peers[q]) : nullptr;
      v.flag[q] = q < P ? reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(peers[q]) + (size_t)P * max_tok * 16)
                        : nullptr;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int vgrid = (int)std::min<int64_t>(n_tokens, std::min(sms, kMaxStatCtas));
    if (!fused_v1) {
      if (dtype == RL_BF16) launch_vp_fused2<bf16_t>(v, slice_bytes, vgrid, s);
      else launch_vp_fused2<float>(v, slice_bytes, vgrid, s);
    } else if (dtype == RL_BF16) {
      cudaFuncSetAttribute(vp_fused_kernel<bf16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vf_smem);
      vp_fused_kernel<bf16_t><<<vgrid, kVfThreads, vf_smem, s>>>(v);
    } else {
      cudaFuncSetAttribute(vp_fused_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vf_smem);
      vp_fused_kernel<float><<<vgrid, kVfThreads, vf_smem, s>>>(v);
    }
    rl_status st0 = check_launch("vp_fused_kernel");
    if (st0 != RL_OK) return st0;
    return launch_stats_reduce(partials, vgrid, stats, (p->flags & RL_F_STATS_ACCUMULATE) != 0, s);
  }
  static int block_kernels = -1;  // RL_VP_KERNEL=block: the CTA-per-row passes
  if (block_kernels < 0)
    block_kernels = (getenv("RL_VP_KERNEL") && strcmp(getenv("RL_VP_KERNEL"), "block") == 0) ? 1 : 0;
  int grid = vp_grid(n_tokens);
  if (!block_kernels) {
    static int wctas = 0;
    if (!wctas) {
      int dev = 0, sms = 148, occ = 4;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vp_finish_warp_kernel<bf16_t>, kVwThreads, 0);
      wctas = std::min(sms * std::max(occ, 1), kMaxStatCtas);
    }
    grid = (int)std::min<int64_t>((n_tokens + kVwWarps - 1) / kVwWarps, wctas);
    if (dtype == RL_BF16)
      vp_stats_warp_kernel<bf16_t><<<grid, kVwThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                               vocab_offset, ld, targets, inv_temperature, send);
    else
      vp_stats_warp_kernel<float><<<grid, kVwThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                              vocab_offset, ld, targets, inv_temperature, send);
  } else if (dtype == RL_BF16)
    vp_stats_kernel<bf16_t><<<grid, kVpThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                        vocab_offset, ld, targets, inv_temperature, send);
  else
    vp_stats_kernel<float><<<grid, kVpThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                       vocab_offset, ld, targets, inv_temperature, send);
  rl_status st = check_launch("vp_stats_kernel");
  if (st != RL_OK) return st;
  ncclResult_t r = ncclAllGather(send, recv, (size_t)n_tokens * 4, ncclFloat, comm_nccl(comm), s);
  if (r != ncclSuccess) return fail(RL_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  if (!with_loss) {
    const int blocks = (int)std::min<int64_t>(148 * 4, (n_tokens + 255) / 256);
    vp_logp_kernel<<<blocks, 256, 0, s>>>(recv, n_tokens, P, vocab_total, targets, logp_out, lse_out);
    return check_launch("vp_logp_kernel");
  }
  const Knobs kn = make_knobs(p);
  const int count = comm_rank(comm) == 0;
  static int finish_warp = -1;  // RL_VP_FINISH=warp: the warp-per-row finish pass
  if (finish_warp < 0)
    finish_warp = (getenv("RL_VP_FINISH") && strcmp(getenv("RL_VP_FINISH"), "warp") == 0) ? 1 : 0;
  if (!block_kernels && !finish_warp) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tgrid = (int)std::min<int64_t>(n_tokens, std::min(sms, kMaxStatCtas));
    const int nslots = 7;
    const size_t smem = ((8 * (2 * nslots + 2 * kVtScale) + 64 + 16 * kVtScale + 127) & ~(size_t)127) +
                        (size_t)nslots * kVtSlot;
    auto kern = dtype == RL_BF16 ? vp_finish_tma_kernel<bf16_t> : vp_finish_tma_kernel<float>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<tgrid, kVtThreads, smem, s>>>(logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv,
                                         P, targets, old_logp, loss_mask, token_seq, seq_adv, seq_version,
                                         seq_active, kn, count, dlogits_shard, logp_out, lse_out, partials, nslots);
    grid = tgrid;
  } else if (!block_kernels) {
    if (dtype == RL_BF16)
      vp_finish_warp_kernel<bf16_t><<<grid, kVwThreads, 0, s>>>(
          logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv, P, targets,
          old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active, kn, count, dlogits_shard,
          logp_out, lse_out, partials);
    else
      vp_finish_warp_kernel<float><<<grid, kVwThreads, 0, s>>>(
          logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv, P, targets,
          old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active, kn, count, dlogits_shard,
          logp_out, lse_out, partials);
  } else if (dtype == RL_BF16)
    vp_finish_kernel<bf16_t><<<grid, kVpThreads, 0, s>>>(
        logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv, P, targets,
        old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active, kn, count, dlogits_shard,
        logp_out, lse_out, partials);
  else
    vp_finish_kernel<float><<<grid, kVpThreads, 0, s>>>(
        logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv, P, targets,
        old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active, kn, count, dlogits_shard,
        logp_out, lse_out, partials);
  st = check_launch("vp_finish_kernel");
  if (st != RL_OK) return st;
  return launch_stats_reduce(partials, grid, stats, (p->flags & RL_F_STATS_ACCUMULATE) != 0, s);
}

// development only (not part of include/rl_policy.h): copy / clear the vp_fused2 phase trace
extern "C" int rl_debug_trace_vp2(unsigned long long* host, size_t bytes, int clear) {
  const size_t n = sizeof(rl::g_trace_vp2) < bytes ? sizeof(rl::g_trace_vp2) : bytes;
  if (host && cudaMemcpyFromSymbol(host, rl::g_trace_vp2, n) != cudaSuccess) return 1;
  if (clear) {
    static unsigned long long zero[256 * 4] = {};
    if (cudaMemcpyToSymbol(rl::g_trace_vp2, zero, sizeof(zero)) != cudaSuccess) return 1;
  }
  return 0;
}

