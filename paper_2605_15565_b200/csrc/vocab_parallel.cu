// (5) Vocab-parallel log-prob (+ fused loss/grad on the local shard) — c8 of DESIGN.md §3
// (north_star: "by vocabulary (vocab-parallel log-softmax), with an NCCL all-reduce of
// per-token max, sum-exp and target logit over NVLink"; BASELINE.json configs[3]).
//
// Two exchange paths for the per-row statistics of the P column shards:
//  * NCCL (always available; logprob-only calls always take it):
//      vp_stats_warp_kernel — per row, (m_r, s_r) in the log2 domain over the local columns and
//        the target logit z_y if this rank owns column y -> one 16-B record per row;
//      one ncclAllGather of the records over NVLink / NVSwitch;
//      vp_finish_tma_kernel — M = max m_r, S = sum s_r 2^(m_r - M), lse, logp (identical on every
//        rank), the token epilogue (statistics counted on comm rank 0 only) and the local dlogits
//        slice s_t (softmax - onehot) from a second read of the shard: 3 HBM units per slice.
//  * in-kernel peer exchange (rl_comm_enable_peer_exchange; the default for the fused loss):
//      vp_ring_kernel — one kernel, the records travel over NVLink inside it, the shard is read
//        from HBM once, re-read from L2 once and dlogits written once: 2 HBM units per slice.
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


// NCCL path, pass 1: a warp streams one row slice with 4 x 16-B loads in flight per lane and no
// block barriers (the layout of logprob_warp_kernel).
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
      sm100::mbar_init(&empty[i], 15 * sm100::kRelPerWarp);
    }
    for (int i = 0; i < kVtScale; ++i) {
      sm100::mbar_init(&scbar[i], 1);
      sm100::mbar_init(&donebar[i], 15 * sm100::kRelPerWarp);
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
  const uint32_t rt_zero = (uint32_t)nslots >> 31;  // 0 at run time (sm100::mbar_release_after)
  uint32_t dep = 0;                                  // bits of what this thread read from the ring
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
          dep ^= o.x;
          st_stream_v4(vout + i, o);
        }
      }
      sm100::mbar_release_after(empty_s + slot * 8, dep, rt_zero);
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
    sm100::mbar_release_after(sm100::smem_u32(&donebar[q]), dep, rt_zero);
  }
}


// ---------------------------------------------------------------------------------------
// Fused vocab-parallel loss with the in-kernel peer exchange: vp_ring_kernel.
//
// One CTA per SM walks its rows row(k) = blockIdx.x + k * gridDim.x (the same rows on every
// rank).  The shard's row slices stream through ONE ring of 30 KB shared-memory slots, filled by
// TMA bulk copies from a producer lane in the order
//     for j = 0 .. nk + D - 1:   pass 1 of row j (if j < nk),  pass 2 of row j - D (if j >= D)
// so pass 1 reads a slice from HBM (L2 evict_last) and pass 2 re-reads it D rows later from L2
// (evict_first) — 2 HBM units per slice; D is sized so the grid's D-row window stays L2-resident.
//   consumers (warps 0..14): pass 1 -> per-thread online (max, sum 2^(t - max)) over packed bf16
//     chunk maxima, warp-reduced into the row's stats slot; the thread holding the target column
//     also records z_y.  Pass 2 -> dlogits = s (2^(t - c2) - [v == y]) with 128-bit streaming
//     stores (the target column rewritten with dy = s (p_y - 1) by the thread that stored it).
//   producer (warp 15 lane 0): the TMA bulk copies.
//   service (warp 16): in groups of G rows — (A) reduce the group's 15 warp partials per row into
//     c2_r = m + log2 s and publish (c2_r, z_y) to every rank as two 8-byte "LL" words that carry
//     the call's epoch in their high half (single-copy atomic NVLink stores: no fence, no flag);
//     (B) LG groups later, poll the P records of each row of group g - LG (lane r*P + q reads rank
//     q's record of row r), combine them in rank order (M = max c2_q, S = sum 2^(c2_q - M), the
//     same float operations on every rank), run the token epilogue and publish the row scales.
// Exchange slots are double-buffered by the epoch's parity: a rank can only start call e + 2
// after every peer finished call e (finishing e + 1 needs every peer's e + 1 records), so a slot
// is never rewritten while a peer may still read it.  A peer that never publishes (a dead rank)
// ends the kernel with __trap() after kVrTimeoutNs, which surfaces as RL_ERR_CUDA.
constexpr int kVrCons = 480, kVrThreads = 576;  // 15 consumer warps + producer + 2 service warps
constexpr int kVrStat = 32;                                 // row stats slots
constexpr int kVrScale = 32;                                // row scale slots
constexpr long long kVrTimeoutNs = 30LL * 1000 * 1000 * 1000;

struct VrArgs {
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
  int32_t G, LG, D, nslots;
  int32_t pub_mode;  // vp_cache_kernel: 0 collector sends (strong), 1 last consumer warp (weak), 2 collector (weak)
  uint32_t epoch;
  unsigned long long* xr[8];  // rank q's slots of this call's parity: [src P][max_tokens] x 2 words
};

struct VrShared {
  uint64_t stats_full[kVrStat], stats_free[kVrStat];
  uint64_t scale_full[kVrScale], scale_free[kVrScale];
  float2 red[kVrStat][15];  // per consumer warp (m, s) of the row
  float zyv[kVrStat];       // target logit * inv_t of the row (0 when not owned)
  float4 sc[kVrScale];      // (s, c2, dy, target column or -1)
  double acc[32][RL_LOSS_STATS_N];
};

__device__ __forceinline__ void st_ll2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// weak (posted) form: no ordering with the thread's later accesses is requested, so the store does
// not hold up the issuing thread; each 8-byte word stays single-copy atomic
__device__ __forceinline__ void st_ll2_weak(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_ll2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// dlogits of one 16-B vector: s * 2^(x k - c2), packed fp32x2 math, RNE to the logits' type
template <typename T>
struct VrGrad;
template <>
struct VrGrad<bf16_t> {
  __device__ static __forceinline__ uint4 run(const uint4& v, uint64_t k2, uint64_t nc2, uint64_t s2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float a, b;
      f2unpack(ffma2(f2pack(bf16_lo(w[i]), bf16_hi(w[i])), k2, nc2), a, b);
      o[i] = f2_to_bf2(fmul2(f2pack(fast_exp2(a), fast_exp2(b)), s2));
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
};
template <>
struct VrGrad<float> {
  __device__ static __forceinline__ uint4 run(const uint4& v, uint64_t k2, uint64_t nc2, uint64_t s2) {
    float a, b, c, d;
    f2unpack(ffma2(f2pack(__uint_as_float(v.x), __uint_as_float(v.y)), k2, nc2), a, b);
    f2unpack(ffma2(f2pack(__uint_as_float(v.z), __uint_as_float(v.w)), k2, nc2), c, d);
    float e, f, g, h;
    f2unpack(fmul2(f2pack(fast_exp2(a), fast_exp2(b)), s2), e, f);
    f2unpack(fmul2(f2pack(fast_exp2(c), fast_exp2(d)), s2), g, h);
    return make_uint4(__float_as_uint(e), __float_as_uint(f), __float_as_uint(g), __float_as_uint(h));
  }
};

// VPT: 16-B vectors per consumer thread per ring slot (4: 30 KB slots, 5: 37.5 KB), chosen on the host
// so the slot count covers the row slice with the least idle tail (P = 4 / 8 widths: 5; 2 chunks of
// 2,400 vectors for 4,748, where 4 left the third chunk 47 % full)
template <typename T, int VPT>
__global__ void __launch_bounds__(kVrThreads, 1) vp_ring_kernel(const VrArgs a) {
  constexpr int kVrVpt = VPT;
  constexpr int kVrChunkVec = VPT * kVrCons;   // 16-B vectors per slot
  constexpr int kVrSlot = kVrChunkVec * 16;    // slot bytes
  constexpr int EPV = VecTraits<T>::EPV;
  extern __shared__ __align__(128) unsigned char smem[];
  VrShared& sh = *reinterpret_cast<VrShared*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + sizeof(VrShared));
  uint64_t* empty = full + a.nslots;
  unsigned char* ring = smem + ((sizeof(VrShared) + 16 * (size_t)a.nslots + 127) & ~(size_t)127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nk = blockIdx.x < a.n ? (a.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t row_bytes = a.ld * elem_bytes<T>();
  const int64_t nvec = a.Vr / EPV;
  const int nch = (int)((nvec + kVrChunkVec - 1) / kVrChunkVec);
  const int D = a.D;
  const float k = a.kn.inv_t * RL_LOG2E;
  auto row_of = [&](int64_t kk) { return (int64_t)blockIdx.x + kk * gridDim.x; };
  if (tid == 0) {
    for (int i = 0; i < a.nslots; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], 15 * sm100::kRelPerWarp);
    }
    for (int i = 0; i < kVrStat; ++i) {
      sm100::mbar_init(&sh.stats_full[i], 15);
      sm100::mbar_init(&sh.stats_free[i], 1);
      sh.zyv[i] = 0.f;
    }
    for (int i = 0; i < kVrScale; ++i) {
      sm100::mbar_init(&sh.scale_full[i], 1);
      sm100::mbar_init(&sh.scale_free[i], 15);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t full_s = sm100::smem_u32(full), empty_s = sm100::smem_u32(empty);
  const uint32_t ring_s = sm100::smem_u32(ring);

  if (warp == 15) {  // ------------------------------------------------------------ producer
    if (lane == 0 && nch > 0) {
      const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
      RingPos rp{0, 0};
      for (int64_t j = 0; j < nk + D; ++j) {
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const int64_t kk = pass == 0 ? j : j - D;
          if (pass == 0 ? (j >= nk) : (j < D)) continue;
          const char* src = reinterpret_cast<const char*>(a.logits) + row_of(kk) * row_bytes;
          for (int c = 0; c < nch; ++c) {
            sm100::mbar_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1);
            const uint32_t bytes = (uint32_t)min((int64_t)kVrChunkVec, nvec - (int64_t)c * kVrChunkVec) * 16u;
            sm100::mbar_arrive_expect_tx(&full[rp.slot], bytes);
            sm100::bulk_g2s(ring + (size_t)rp.slot * kVrSlot, src + (size_t)c * kVrSlot, bytes, &full[rp.slot],
                            pass == 0 ? keep : drop);
            rp.advance(1, a.nslots);
          }
        }
      }
    }
    return;
  }

  if (warp >= 16) {  // ------------------------------------------------ service: warp 16 (A), warp 17 (B)
    // (A) and (B) run in their own warps, so a row's scale never waits behind the next row's
    // publication (at D = 1, P = 2, the serial order exposed the service latency every row)
    const bool pubw = warp == 16;
    const int G = a.G, P = a.P;
    const int rl_ = lane / P, ql = lane % P;  // this lane: row rl_ of a group, rank ql
    const bool lane_on = rl_ < G;
    const double inv_tm = token_mean_inv(a.kn);
    Acc acc;
    acc.zero();
    float my_c2 = -INFINITY, my_zy = 0.f;
    const unsigned long long ep = (unsigned long long)a.epoch << 32;
    const int64_t ngr = (nk + G - 1) / G;
    // this lane's row of the next B group, level-1 metadata (loaded one group ahead)
    int32_t ny = 0, nseq = 0;
    uint8_t nmask = 1;
    float nold = 0.f, nprox = 0.f, nref = 0.f;
    auto load_l1 = [&](int64_t gb) {
      const int64_t kk = gb * G + rl_;
      if (lane_on && ql == 0 && kk < nk) {
        const int64_t row = row_of(kk);
        ny = a.targets[row];
        nseq = a.token_seq ? a.token_seq[row] : 0;
        nmask = a.mask ? a.mask[row] : 1;
        nold = a.old_logp[row];
        token_extra(a.kn, row, nold, nprox, nref);
      }
    };
    load_l1(0);
    for (int64_t g = 0; g < ngr; ++g) {
      if (pubw) {  // ---- (A) publish the records of group g
        for (int r = 0; r < G; ++r) {
          const int64_t kk = g * G + r;
          if (kk >= nk) break;
          const int ss = (int)(kk % kVrStat);
          sm100::mbar_wait(&sh.stats_full[ss], (uint32_t)((kk / kVrStat) & 1));
          MS st = lane < 15 ? MS{sh.red[ss][lane].x, sh.red[ss][lane].y} : MS{-INFINITY, 0.f};
          st = warp_reduce_ms(st);
          const float zy = sh.zyv[ss];
          __syncwarp();
          if (lane == 0) {
            sh.zyv[ss] = 0.f;
            sm100::mbar_arrive(&sh.stats_free[ss]);
          }
          if (rl_ == r) {
            my_c2 = st.s > 0.f ? st.m + fast_log2(st.s) : -INFINITY;
            my_zy = zy;
          }
        }
        const int64_t kk = g * G + rl_;
        if (lane_on && kk < nk)
          st_ll2(a.xr[ql] + ((int64_t)a.me * a.max_tokens + row_of(kk)) * 2, ep | __float_as_uint(my_c2),
                 ep | __float_as_uint(my_zy));
      }
      if (!pubw) {  // ---- (B) combine group g, run the epilogue, publish the scales
        const int64_t gb = g;
        const int64_t kk = gb * G + rl_;
        const bool has = lane_on && kk < nk;
        const int64_t row = has ? row_of(kk) : 0;
        // this group's metadata (level 1 was loaded one group ago; level 2 issued before polling)
        const int32_t y = ny, seq = nseq;
        const uint8_t mk = nmask;
        const float old = nold, prox = nprox, ref = nref;
        const bool lead = has && ql == 0;
        int32_t ver = 0, act = 0;
        float A = 0.f;
        const bool pre = lead && mk != 0 && y >= 0 && (int64_t)y < a.Vtot;
        if (lead && a.seq_version) ver = a.seq_version[seq];
        if (pre) {
          A = a.seq_adv[seq];
          if (a.seq_active) act = a.seq_active[seq];
        }
        float c2q = -INFINITY, zyq = 0.f;
        if (has) {
          const unsigned long long* slot = a.xr[a.me] + ((int64_t)ql * a.max_tokens + row) * 2;
          unsigned long long w0, w1;
          const unsigned long long t0 = globaltimer();
          for (int it = 0;; ++it) {
            ld_ll2(slot, w0, w1);
            if ((w0 >> 32) == a.epoch && (w1 >> 32) == a.epoch) break;
            if ((it & 1023) == 1023 && globaltimer() - t0 > (unsigned long long)kVrTimeoutNs) {
              printf("rl_vocab_parallel_logprob: rank %d waited > %lld s for rank %d's record of row %lld "
                     "(epoch %u); a peer is not running the matching call\n",
                     a.me, kVrTimeoutNs / 1000000000LL, ql, (long long)row, a.epoch);
              __trap();
            }
          }
          c2q = __uint_as_float((uint32_t)w0);
          zyq = __uint_as_float((uint32_t)w1);
        }
        load_l1(gb + 1);
        const int base = (lane / P) * P;
        float M = -INFINITY;
        for (int q = 0; q < P; ++q) M = fmaxf(M, __shfl_sync(0xffffffffu, c2q, (base + q) & 31));
        float S = 0.f, zy = 0.f;
        for (int q = 0; q < P; ++q) {
          const float cq = __shfl_sync(0xffffffffu, c2q, (base + q) & 31);
          const float zq = __shfl_sync(0xffffffffu, zyq, (base + q) & 31);
          if (cq != -INFINITY) S += fast_exp2(cq - M);
          zy += zq;
        }
        if (lead) {
          const float c2 = M + fast_log2(S);
          RowMeta mt;
          mt.y = y;
          mt.seq = a.token_seq ? seq : 0;
          mt.in_range = y >= 0 && (int64_t)y < a.Vtot;
          mt.bad = (int64_t)y >= a.Vtot;
          const int32_t stale = a.seq_version ? a.kn.trainer_version - ver : 0;
          mt.neg_stale = stale < 0;
          mt.stale_drop = !mt.neg_stale && a.kn.max_staleness >= 0 && stale > a.kn.max_staleness;
          const bool m_on = mk != 0;
          mt.valid = m_on && mt.in_range && !mt.neg_stale && !mt.stale_drop;
          mt.stale_drop = mt.stale_drop && m_on && mt.in_range;
          const float lp = logp_from(mt, zy, c2);
          if (a.logp_out) a.logp_out[row] = lp;
          if (a.lse_out) a.lse_out[row] = c2 * RL_LN2;
          Acc tmp;
          tmp.zero();
          const int32_t Li = (mt.valid && a.kn.agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN) ? act : 0;
          const float st = token_epilogue_li(mt, lp, mt.valid ? old : 0.f, mt.valid ? A : 0.f, Li, inv_tm, a.kn,
                                             tmp, nullptr, prox, ref);
          if (a.count_stats)
            for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
          const int64_t yl = (int64_t)y - a.off;
          const int ycol = (mt.in_range && yl >= 0 && yl < a.Vr) ? (int)yl : -1;
          const float dy = st * (fast_exp2(zy * RL_LOG2E - c2) - 1.f);
          const int sl = (int)(kk % kVrScale);
          if (kk >= kVrScale) sm100::mbar_wait_polite(&sh.scale_free[sl], (uint32_t)(((kk / kVrScale) - 1) & 1), false);
          sh.sc[sl] = make_float4(st, c2, dy, __int_as_float(ycol));
          sm100::mbar_arrive(&sh.scale_full[sl]);
        }
      }
    }
    if (pubw) return;
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) sh.acc[lane][i] = acc.v[i];
    __syncwarp();
    if (lane < RL_LOSS_STATS_N) {  // lane-ordered (deterministic) sum of the row leaders' statistics
      double t = 0.0;
      for (int l = 0; l < 32; ++l) t += sh.acc[l][lane];
      a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + lane] = t;
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumers
  using V = ClVec<T>;
  uint32_t slot = 0, rph = 0;
  const uint32_t rt_zero = (uint32_t)a.nslots >> 31;  // 0 at run time (sm100::mbar_release_after)
  const uint32_t my_off = (uint32_t)tid * 16u;
  const uint64_t k2 = f2pack(k, k);
  const int64_t tail0 = nvec * EPV;
  int32_t y_next = nk > 0 ? a.targets[row_of(0)] : 0;
  for (int64_t j = 0; j < nk + D; ++j) {
    if (j < nk) {  // ---- pass 1 of row j
      const int64_t row = row_of(j);
      const int32_t y = y_next;
      if (j + 1 < nk) y_next = a.targets[row_of(j + 1)];
      const int64_t yl = (int64_t)y - a.off;  // target column in this shard (any value)
      const int64_t yv = (y >= 0 && yl >= 0 && yl < tail0) ? yl / EPV : -1;
      float m = -INFINITY, zy = 0.f;
      bool own = false;
      uint64_t acc2 = f2pack(0.f, 0.f);
      for (int c = 0; c < nch; ++c) {
        sm100::mbar_wait_a(full_s + slot * 8, rph);
        const uint32_t sb = ring_s + slot * (uint32_t)kVrSlot;
        uint4 v[kVrVpt];
        typename V::MaxT mx = V::max_init();
#pragma unroll
        for (int u = 0; u < kVrVpt; ++u) {
          const int64_t i = (int64_t)c * kVrChunkVec + u * kVrCons + tid;
          v[u] = i < nvec ? sm100::lds128_a(sb + u * (kVrCons * 16) + my_off) : V::neg_inf_vec();
          V::max_acc(v[u], mx);
        }
        if (yv >= 0 && yv / kVrChunkVec == c && yv % kVrCons == tid) {  // this thread holds z_y
          const uint32_t off = (uint32_t)((yl - (int64_t)c * kVrChunkVec * EPV) * elem_bytes<T>());
          uint32_t w;
          if (EPV == 8) {
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(w) : "r"(sb + off));
            zy = __uint_as_float(w << 16);
          } else {
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(sb + off));
            zy = __uint_as_float(w);
          }
          own = true;
        }
        sm100::mbar_release_after(empty_s + slot * 8, v[0].x ^ v[kVrVpt - 1].w, rt_zero);
        if (++slot == (uint32_t)a.nslots) {
          slot = 0;
          rph ^= 1u;
        }
        const float nm = fmaxf(m, V::max_to_float(mx) * k);
        if (nm != -INFINITY) {
          if (nm > m) {
            const float sc = fast_exp2(m - nm);  // 0 while m = -inf
            acc2 = fmul2(acc2, f2pack(sc, sc));
            m = nm;
          }
          const uint64_t mn2 = f2pack(-nm, -nm);
#pragma unroll
          for (int u = 0; u < kVrVpt; ++u) acc2 = V::exp_sum(v[u], k2, mn2, acc2);
        }
      }
      float lo, hi;
      f2unpack(acc2, lo, hi);
      MS st{m, lo + hi};
      const char* rp = reinterpret_cast<const char*>(a.logits) + row * row_bytes;
      for (int64_t cc = tail0 + tid; cc < a.Vr; cc += kVrCons) {  // scalar tail columns
        float f[1] = {VecTraits<T>::load1(rp, cc)};
        ms_update<1>(st, f, k);
        if (cc == yl && y >= 0) {
          zy = f[0];
          own = true;
        }
      }
      st = warp_reduce_ms(st);
      const int ss = (int)(j % kVrStat);
      if (j >= kVrStat) sm100::mbar_wait(&sh.stats_free[ss], (uint32_t)(((j / kVrStat) - 1) & 1));
      if (own) sh.zyv[ss] = zy * a.kn.inv_t;
      __syncwarp();
      if (lane == 0) {
        sh.red[ss][warp] = make_float2(st.m, st.s);
        sm100::mbar_arrive(&sh.stats_full[ss]);
      }
    }
    if (j >= D) {  // ---- pass 2 of row j - D
      const int64_t kk = j - D;
      const int64_t row = row_of(kk);
      RL_DCHECK(row < a.n);
      const int sl = (int)(kk % kVrScale);
      sm100::mbar_wait(&sh.scale_full[sl], (uint32_t)((kk / kVrScale) & 1));
      const float4 r = sh.sc[sl];
      const float s = r.x, c2 = r.y, dy = r.z;
      const int ycol = __float_as_int(r.w);
      const uint64_t s2 = f2pack(s, s), nc2 = f2pack(-c2, -c2);
      char* dp = reinterpret_cast<char*>(a.dlogits) + row * row_bytes;
      uint4* vout = reinterpret_cast<uint4*>(dp);
      for (int c = 0; c < nch; ++c) {
        sm100::mbar_wait_a(full_s + slot * 8, rph);
        const uint32_t sb = ring_s + slot * (uint32_t)kVrSlot;
        uint4 v[kVrVpt];
#pragma unroll
        for (int u = 0; u < kVrVpt; ++u) v[u] = sm100::lds128_a(sb + u * (kVrCons * 16) + my_off);
        sm100::mbar_release_after(empty_s + slot * 8, v[0].x ^ v[kVrVpt - 1].w, rt_zero);
        if (++slot == (uint32_t)a.nslots) {
          slot = 0;
          rph ^= 1u;
        }
#pragma unroll
        for (int u = 0; u < kVrVpt; ++u) {
          const int64_t i = (int64_t)c * kVrChunkVec + u * kVrCons + tid;
          const uint4 o = s != 0.f ? VrGrad<T>::run(v[u], k2, nc2, s2) : make_uint4(0, 0, 0, 0);
          st_stream_v4_if(vout + i, o, i < nvec);
        }
      }
      const char* rp = reinterpret_cast<const char*>(a.logits) + row * row_bytes;
      for (int64_t cc = tail0 + tid; cc < a.Vr; cc += kVrCons) {
        float v = (s == 0.f) ? 0.f : s * fast_exp2(fmaf(VecTraits<T>::load1(rp, cc), k, -c2));
        if (s != 0.f && cc == ycol) v = dy;
        VecTraits<T>::store1(dp, cc, v);
      }
      // the target column: rewritten by the thread that stored its vector (same-thread order)
      RL_DCHECK(ycol < a.Vr);
      if (s != 0.f && ycol >= 0 && ycol < tail0 && (ycol / EPV) % kVrCons == tid) VecTraits<T>::store1(dp, ycol, dy);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&sh.scale_free[sl]);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Fused vocab-parallel loss, register-cache form: vp_cache_kernel<NV, R> (the default for bf16
// shards of <= 4928 16-B vectors, i.e. the P >= 4 shard widths of V = 151936).
//
// One HBM read and one exp2 per element: a CTA walks its rows; each consumer thread holds NV
// vectors (vector t + 448 i) of a row slice in registers, converted in place into
//     e'_v = 2^(x_v k - m_w)          m_w = the max of x k over the thread's WARP (no CTA barrier)
// and keeps them (bf16) for R rows while the row statistics travel: warp partials
// (m_w, S_w = sum e') -> the LAST consumer warp to post its record (a shared-memory counter) combines
// the 14 warps into c2_r = lse2 of the shard and sends (c2_r, z_y) to every rank (LL words, as vp_ring_kernel) -> the collector warp polls the P
// records of the row, combines them in rank order (identical on every rank), runs the token
// epilogue and publishes (s_t, c2, dy, target column).  R + RS - 1 rows after a row was loaded its
// gradient is written from the cache (RS older rows parked in shared memory across GPUs):
// dlogits_v = e'_v q_w,  q_w = s_t 2^(m_w - c2)  (q split into bf16 hi + lo, HMUL2 + HFMA2: one
// rounding in the product, reading R2), target column dy = s_t (p_y - 1).  So the exchange latency
// hides behind R + RS - 1 rows of streaming.  Ring slots are released per thread after the data
// read from them is in registers (sm100::mbar_release_after).
//   warps 0..13   consumers (thread t holds vectors t + 448 i, i < NV)
//   warp 14       lane 0: TMA producer (ring of 28 KB slots) — alone in its warp, so a copy is
//                 issued the moment a slot frees (sharing the warp with polling lanes starved it)
//   warp 15       collector: G = min(8, 32 / P) groups of P lanes, group g owning rows g, g + G, ...
//                 (lane q polls rank q's record, lane 0 of the group runs the epilogue), so G rows
//                 are combined concurrently
// 16 warps = 4 per SM sub-partition, so each thread may use 128 registers (the NV = 11 cache is 88).
constexpr int kVcWarps = 14, kVcCons = kVcWarps * 32;
constexpr int kVcThreads = kVcCons + 64;
constexpr int kVcColl = 0;  // first collector lane
constexpr int kVcStat = 32, kVcScale = 32;

#ifdef RL_VC_TRACE
// development build only (python -m paper_2605_15565_b200.build --variant trace): per-CTA cycle
// counters — 0 consumer wait for the row scale, 1 consumer wait for ring data, 2 collector wait for
// the row's own record, 3 collector poll for the peers' records, 4 collector chain per row, 5 rows,
// 6 consumer thread 0's cycles in the kernel, 7 the CTA's SM id (last call), 8 collector: peers'
// records in -> row scale posted
__device__ unsigned long long g_vc_trace[256][12];
#define RL_VC_T0(v) const long long v = clock64()
#define RL_VC_ADD(i, v) do { if (blockIdx.x < 256) atomicAdd(&g_vc_trace[blockIdx.x][i], (unsigned long long)(clock64() - (v))); } while (0)
#else
#define RL_VC_T0(v)
#define RL_VC_ADD(i, v)
#endif

struct VcShared {
  uint32_t cnt[kVcStat];    // consumer warps that posted the row's record
  uint64_t pub_full[kVcStat];  // the row's shard record (c2, z_y) is in pub[]
  float2 pub[kVcStat];
  uint64_t scale_full[kVcScale], scale_free[kVcScale];
  float2 red[kVcStat][kVcWarps];
  float zyv[kVcStat];
  float4 sc[kVcScale];  // (s, c2, dy, target column or -1)
  double acc[8][RL_LOSS_STATS_N];  // collector groups' statistics
  uint32_t tmem_base;              // PK: the parked rows' tensor-memory allocation
};

// parked rows in tensor memory (PK): thread (warp w, lane l) owns TMEM lane 32 (w % 4) + l; the four
// warps sharing a sub-partition take disjoint column ranges.  Plain 32-bit stores / loads
// (tcgen05.st / ld .32x32b.x4: one 16-B vector per thread), no tensor-core work.
__device__ __forceinline__ void tm_st4(uint32_t taddr, uint4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// the caller issues tcgen05.wait::ld before using the registers
__device__ __forceinline__ uint4 tm_ld4(uint32_t taddr) {
  uint4 v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(taddr)
               : "memory");
  return v;
}

// warp max in one instruction (redux.sync .f32, sm_100a)
__device__ __forceinline__ float warp_max_redux(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// CV: 16-B vectors per consumer thread per ring slot; PK: the RS parked rows live in tensor memory
// (1) instead of shared memory (0), which leaves all of shared memory to the copy ring
template <int NV, int R, int RS, int CV = 4, int PK = 0>
__global__ void __launch_bounds__(kVcThreads, 1) vp_cache_kernel(const VrArgs a) {
  static_assert(!PK || (RS > 0 && ((kVcWarps + 3) / 4) * RS * NV * 4 <= 512), "parked rows exceed 512 TMEM columns");
  constexpr int CHV = CV * kVcCons;  // vectors per ring slot
  constexpr int SLOT = CHV * 16;     // ring slot bytes (28 KB at CV = 4)
  using V = ClVec<bf16_t>;
  extern __shared__ __align__(128) unsigned char smem[];
  VcShared& sh = *reinterpret_cast<VcShared*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + sizeof(VcShared));
  uint64_t* empty = full + a.nslots;
  unsigned char* ring = smem + ((sizeof(VcShared) + 16 * (size_t)a.nslots + 127) & ~(size_t)127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nk = blockIdx.x < a.n ? (a.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t row_bytes = a.ld * 2;
  const int nvec = (int)(a.Vr / 8);
  const int nch = (nvec + CHV - 1) / CHV;
  const float k = a.kn.inv_t * RL_LOG2E;
  auto row_of = [&](int64_t kk) { return (int64_t)blockIdx.x + kk * gridDim.x; };
  if (tid == 0) {
    for (int i = 0; i < a.nslots; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], kVcWarps * sm100::kRelPerWarp);
    }
    for (int i = 0; i < kVcStat; ++i) {
      sh.cnt[i] = 0;
      sh.zyv[i] = 0.f;
      sm100::mbar_init(&sh.pub_full[i], 1);
    }
    for (int i = 0; i < kVcScale; ++i) {
      sm100::mbar_init(&sh.scale_full[i], 1);
      sm100::mbar_init(&sh.scale_free[i], kVcWarps);
    }
    sm100::fence_mbar_init();
  }
  if constexpr (PK) {
    if (threadIdx.x < 32) {  // warp 0 allocates 512 columns (one CTA per SM)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sm100::smem_u32(&sh.tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if constexpr (PK) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t full_s = sm100::smem_u32(full), empty_s = sm100::smem_u32(empty);
  const uint32_t ring_s = sm100::smem_u32(ring);
  // RS older rows of e' parked in shared memory after the ring (thread t's vector i of slot s at
  // ((s NV + i) 448 + t) 16: conflict-free, only the owning thread touches it)
  const uint32_t rowc_s = ring_s + (uint32_t)a.nslots * (uint32_t)SLOT;
  const uint32_t tmem = PK ? sh.tmem_base : 0u;

  if (warp == kVcWarps) {
    if (lane == 0) {  // -------------------------------------------------------- TMA producer
      RingPos rp{0, 0};
      for (int64_t kk = 0; kk < nk; ++kk) {
        const char* src = reinterpret_cast<const char*>(a.logits) + row_of(kk) * row_bytes;
        for (int c = 0; c < nch; ++c) {
          sm100::mbar_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1);
          const uint32_t bytes = (uint32_t)min(CHV, nvec - c * CHV) * 16u;
          sm100::mbar_arrive_expect_tx(&full[rp.slot], bytes);
          sm100::bulk_g2s_nohint(ring + (size_t)rp.slot * SLOT, src + (size_t)c * SLOT, bytes, &full[rp.slot]);
          rp.advance(1, a.nslots);
        }
      }
    }
    return;
  }
  if (warp == kVcWarps + 1) {
    {  // ----------------------------------------------------------------------- collector
      // lanes 8..31 form G = min(8, 24 / P) groups of P lanes; group g owns rows g, g + G, ... (its
      // own serial poll -> combine -> epilogue chain), lane q of a group polls rank q's record
      const int cl = lane - kVcColl;
      const int G = a.G > 0 ? min(a.G, 32 / a.P) : min(8, 32 / a.P);
      const int grp = cl / a.P, q = cl - grp * a.P;
      const int lead = kVcColl + grp * a.P;
      const unsigned gmask = (a.P == 32 ? 0xffffffffu : ((1u << a.P) - 1u)) << lead;
      if (grp < G) {
    const double inv_tm = token_mean_inv(a.kn);
    Acc acc;
    acc.zero();
    // metadata pipeline (lane 0 of the group), so no global-load latency sits between the peers'
    // records and the row's scale: while row kk is combined, the sequence-indexed (level-2) loads
    // of row kk + G and the row-indexed (level-1) loads of row kk + 2G are in flight
    struct Meta {
      int32_t y = 0, seq = 0, ver = 0, act = 0;
      uint8_t mk = 1;
      float old = 0.f, prox = 0.f, ref = 0.f, A = 0.f;
    };
    auto load_l1 = [&](Meta& m, int64_t kk) {
      if (q == 0 && kk < nk) {
        const int64_t row = row_of(kk);
        m.y = a.targets[row];
        m.seq = a.token_seq ? a.token_seq[row] : 0;
        m.mk = a.mask ? a.mask[row] : 1;
        m.old = a.old_logp[row];
        token_extra(a.kn, row, m.old, m.prox, m.ref);
      }
    };
    auto load_l2 = [&](Meta& m, int64_t kk) {
      if (q == 0 && kk < nk) {
        if (a.seq_version) m.ver = a.seq_version[m.seq];
        if (m.mk != 0 && m.y >= 0 && (int64_t)m.y < a.Vtot) {
          m.A = a.seq_adv[m.seq];
          if (a.seq_active) m.act = a.seq_active[m.seq];
        }
      }
    };
    Meta mnext, mnext2;
    load_l1(mnext, grp);
    load_l2(mnext, grp);
    load_l1(mnext2, grp + G);
    for (int64_t kk = grp; kk < nk; kk += G) {
      const int64_t row = row_of(kk);
      const Meta cur = mnext;
      mnext = mnext2;
      load_l2(mnext, kk + G);
      mnext2 = Meta{};
      load_l1(mnext2, kk + 2 * G);
      const int32_t y = cur.y, seq = cur.seq, ver = cur.ver, act = cur.act;
      const uint8_t mk = cur.mk;
      const float old = cur.old, prox = cur.prox, ref = cur.ref, A = cur.A;
      RL_VC_T0(tc0);
      {  // publish this rank's record of the row: lane q of the group sends it to rank q
        const int ss = (int)(kk % kVcStat);
        sm100::mbar_wait(&sh.pub_full[ss], (uint32_t)((kk / kVcStat) & 1));
        if (grp == 0 && q == 0) RL_VC_ADD(2, tc0);
        const float2 pr = sh.pub[ss];
        const unsigned long long ep = (unsigned long long)a.epoch << 32;
        unsigned long long* dst = a.xr[q] + ((int64_t)a.me * a.max_tokens + row) * 2;
        if (a.pub_mode == 0) st_ll2(dst, ep | __float_as_uint(pr.x), ep | __float_as_uint(pr.y));
        else if (a.pub_mode == 2) st_ll2_weak(dst, ep | __float_as_uint(pr.x), ep | __float_as_uint(pr.y));
      }
      float c2q = -INFINITY, zyq = 0.f;
      RL_VC_T0(tc1);
      {
        RL_DCHECK(q < a.P && row < a.max_tokens);
        const unsigned long long* slot = a.xr[a.me] + ((int64_t)q * a.max_tokens + row) * 2;
        unsigned long long w0, w1;
        const unsigned long long t0 = globaltimer();
        for (int it = 0;; ++it) {
          ld_ll2(slot, w0, w1);
          if ((w0 >> 32) == a.epoch && (w1 >> 32) == a.epoch) break;
          __nanosleep(32);  // the warp's other groups poll their own rows
          if ((it & 1023) == 1023 && globaltimer() - t0 > (unsigned long long)kVrTimeoutNs) {
            printf("rl_vocab_parallel_logprob: rank %d waited > %lld s for rank %d's record of row %lld "
                   "(epoch %u); a peer is not running the matching call\n",
                   a.me, kVrTimeoutNs / 1000000000LL, q, (long long)row, a.epoch);
            __trap();
          }
        }
        c2q = __uint_as_float((uint32_t)w0);
        zyq = __uint_as_float((uint32_t)w1);
      }
      if (grp == 0 && q == 0) RL_VC_ADD(3, tc1);
      RL_VC_T0(tc2);
      float M = -INFINITY;
      for (int j = 0; j < a.P; ++j) M = fmaxf(M, __shfl_sync(gmask, c2q, lead + j));
      float S = 0.f, zy = 0.f;
      for (int j = 0; j < a.P; ++j) {
        const float cq = __shfl_sync(gmask, c2q, lead + j);
        const float zq = __shfl_sync(gmask, zyq, lead + j);
        if (cq != -INFINITY) S += fast_exp2(cq - M);
        zy += zq;
      }
      if (q == 0) {
        const float c2 = M + fast_log2(S);
        RowMeta mt;
        mt.y = y;
        mt.seq = a.token_seq ? seq : 0;
        mt.in_range = y >= 0 && (int64_t)y < a.Vtot;
        mt.bad = (int64_t)y >= a.Vtot;
        const int32_t stale = a.seq_version ? a.kn.trainer_version - ver : 0;
        mt.neg_stale = stale < 0;
        mt.stale_drop = !mt.neg_stale && a.kn.max_staleness >= 0 && stale > a.kn.max_staleness;
        const bool m_on = mk != 0;
        mt.valid = m_on && mt.in_range && !mt.neg_stale && !mt.stale_drop;
        mt.stale_drop = mt.stale_drop && m_on && mt.in_range;
        const float lp = logp_from(mt, zy, c2);
        if (a.logp_out) a.logp_out[row] = lp;
        if (a.lse_out) a.lse_out[row] = c2 * RL_LN2;
        Acc tmp;
        tmp.zero();
        const int32_t Li = (mt.valid && a.kn.agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN) ? act : 0;
        const float st = token_epilogue_li(mt, lp, mt.valid ? old : 0.f, mt.valid ? A : 0.f, Li, inv_tm, a.kn,
                                           tmp, nullptr, prox, ref);
        if (a.count_stats)
          for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
        const int64_t yl = (int64_t)y - a.off;
        const int ycol = (mt.in_range && yl >= 0 && yl < a.Vr) ? (int)yl : -1;
        const float dy = st * (fast_exp2(zy * RL_LOG2E - c2) - 1.f);
        const int sl = (int)(kk % kVcScale);
        if (kk >= kVcScale) sm100::mbar_wait_polite(&sh.scale_free[sl], (uint32_t)(((kk / kVcScale) - 1) & 1), false);
        sh.sc[sl] = make_float4(st, c2, dy, __int_as_float(ycol));
        sm100::mbar_arrive(&sh.scale_full[sl]);
        if (grp == 0) {
          RL_VC_ADD(4, tc0);
          RL_VC_ADD(8, tc2);
#ifdef RL_VC_TRACE
          if (blockIdx.x < 256) atomicAdd(&g_vc_trace[blockIdx.x][5], 1ull);
#endif
        }
      }
    }
      if (q == 0)
        for (int i = 0; i < RL_LOSS_STATS_N; ++i) sh.acc[grp][i] = acc.v[i];
      }
      __syncwarp(0xffffffffu << kVcColl);
      if (cl < RL_LOSS_STATS_N) {  // group-ordered (deterministic) sum of the groups' statistics
        double tsum = 0.0;
        for (int g = 0; g < G; ++g) tsum += sh.acc[g][cl];
        a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + cl] = tsum;
      }
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumers
  RL_VC_T0(tk0);
  uint4 cache[R][NV];
  const uint32_t my_off = (uint32_t)tid * 16u;
  const uint64_t k2 = f2pack(k, k);
  uint32_t slot = 0, rph = 0;
  const uint32_t rt_zero = (uint32_t)a.nslots >> 31;  // 0 at run time (sm100::mbar_release_after)
  uint32_t dep = 0;                                    // bits of the ring vectors this thread read
  int32_t y_next = nk > 0 ? a.targets[row_of(0)] : 0;
  // load row kk into cache[r] (raw bf16), then convert in place to e' (bf16) and post the warp record
  auto load_row = [&](auto rc, int64_t kk) {
    constexpr int r = decltype(rc)::value;
    const int32_t y = y_next;
    if (kk + 1 < nk) y_next = a.targets[row_of(kk + 1)];
    const int64_t yl = (int64_t)y - a.off;
    const int yv = (y >= 0 && yl >= 0 && yl < a.Vr) ? (int)(yl >> 3) : -1;  // target's vector
    typename V::MaxT mx = V::max_init();
    // a chunk's slot is released after the NEXT chunk's loads were issued (its own loads have
    // returned by then, so the data-dependent release does not stall); the row's last slot after
    // the chunk loop
    uint32_t pend = 0;  // empty-barrier address of the slot awaiting release (0: none)
#pragma unroll
    for (int c = 0; c < (NV + CV - 1) / CV; ++c) {
      if (c < nch) {
        RL_DCHECK(slot < (uint32_t)a.nslots && row_of(kk) < a.n);
        RL_VC_T0(tf0);
        sm100::mbar_wait_a(full_s + slot * 8, rph);
        if (tid == 0) RL_VC_ADD(1, tf0);
        const uint32_t sb = ring_s + slot * (uint32_t)SLOT;
        const uint32_t dprev = dep;
#pragma unroll
        for (int u = 0; u < CV; ++u) {
          const int i = CV * c + u;
          if (i < NV) {
            const bool ok = i * kVcCons + tid < nvec;
            cache[r][i] = ok ? sm100::lds128_a(sb + u * (kVcCons * 16) + my_off) : V::neg_inf_vec();
            V::max_acc(cache[r][i], mx);
            dep ^= cache[r][i].x;
          }
        }
        if (pend) sm100::mbar_release_after(pend, dprev, rt_zero);
        pend = empty_s + slot * 8;
        if (++slot == (uint32_t)a.nslots) {
          slot = 0;
          rph ^= 1u;
        }
      } else {
#pragma unroll
        for (int u = 0; u < CV; ++u)
          if (CV * c + u < NV) cache[r][CV * c + u] = V::neg_inf_vec();
      }
    }
    // z_y from the raw vector that holds it (its owner thread; compile-time vector index)
    float zy = 0.f;
    bool own = false;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (yv == i * kVcCons + tid) {
        const uint4 v = cache[r][i];
        const int e = (int)(yl & 7);
        const uint32_t wd = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
        zy = (e & 1) ? bf16_hi(wd) : bf16_lo(wd);
        own = true;
      }
    }
    const float m = warp_max_redux(V::max_to_float(mx)) * k;  // also the row's red[].x (grad reads it)
    float s = 0.f;
    if (m != -INFINITY) {
      const uint64_t mn2 = f2pack(-m, -m);
      uint64_t acc2 = f2pack(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < NV; ++i) acc2 = V::exp_sv(cache[r][i], k2, mn2, acc2, cache[r][i]);
      float lo, hi;
      f2unpack(acc2, lo, hi);
      s = lo + hi;
    }
    // the row's last slot: released once the row's max / exp pass consumed its data (no wait)
    if (pend) sm100::mbar_release_after(pend, dep, rt_zero);
    s = warp_sum(s);
    // slot ss is reused 32 rows later: the consumer warps stay within a few rows of each other
    // (a ring slot is refilled only once all 14 warps released it)
    const int ss = (int)(kk % kVcStat);
    if (own) sh.zyv[ss] = zy * a.kn.inv_t;
    __syncwarp();
    if (lane == 0) {
      sh.red[ss][warp] = make_float2(m, s);
      if (sm100::atom_add_acqrel(sm100::smem_u32(&sh.cnt[ss]), 1u) == kVcWarps - 1) {  // last warp: publish
        float M = -INFINITY;
        for (int w = 0; w < kVcWarps; ++w) M = fmaxf(M, sh.red[ss][w].x);
        float S = 0.f;
        for (int w = 0; w < kVcWarps; ++w) {
          const float2 rw = sh.red[ss][w];
          if (rw.x != -INFINITY) S += rw.y * fast_exp2(rw.x - M);
        }
        const float zr = sh.zyv[ss];
        sh.zyv[ss] = 0.f;
        atomicExch(&sh.cnt[ss], 0u);
        const float c2r = S > 0.f ? M + fast_log2(S) : -INFINITY;
        if (a.pub_mode == 1) {  // this warp sends the record itself, weak (posted) stores
          const unsigned long long ep = (unsigned long long)a.epoch << 32;
          const int64_t row = row_of(kk);
          for (int q = 0; q < a.P; ++q)
            st_ll2_weak(a.xr[q] + ((int64_t)a.me * a.max_tokens + row) * 2, ep | __float_as_uint(c2r),
                        ep | __float_as_uint(zr));
        }
        // hand the record to the collector, which sends it (pub_mode 0 / 2: remote NVLink stores
        // stay off the consumers' path; a consumer warp stalled on them holds every ring slot)
        sh.pub[ss] = make_float2(c2r, zr);
        sm100::mbar_arrive(&sh.pub_full[ss]);
      }
    }
  };
  // dlogits of row kk from its e' vectors (getv(i): the cached vector i of this thread)
  auto grad_vecs = [&](int64_t kk, auto&& getv) {
    const int64_t row = row_of(kk);
    const int sl = (int)(kk % kVcScale);
    RL_VC_T0(tw0);
    sm100::mbar_wait(&sh.scale_full[sl], (uint32_t)((kk / kVcScale) & 1));
    if (tid == 0) RL_VC_ADD(0, tw0);
    const float4 sc = sh.sc[sl];
    const float st = sc.x, c2 = sc.y, dy = sc.z;
    const int ycol = __float_as_int(sc.w);
    const float mw = sh.red[kk % kVcStat][warp].x;  // this warp's exponent reference of the row
    const float q = st == 0.f ? 0.f : st * fast_exp2(mw - c2);
    const uint32_t qb2 = pack_bf16x2(q, q);
    const float qh = __uint_as_float(qb2 << 16);
    const uint32_t ql2 = pack_bf16x2(q - qh, q - qh);
    uint4* out = reinterpret_cast<uint4*>(reinterpret_cast<char*>(a.dlogits) + row * row_bytes) + tid;
    RL_DCHECK(row < a.n && ycol < a.Vr);
    if constexpr (PK) {
      // parked in tensor memory: four loads in flight per wait (one tcgen05.wait::ld per 4 vectors)
#pragma unroll
      for (int i0 = 0; i0 < NV; i0 += 4) {
        uint4 t[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < NV) t[u] = getv(i0 + u);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < NV)
            st_stream_v4_if(out + (i0 + u) * kVcCons, V::grad_sv(t[u], qb2, ql2, q), (i0 + u) * kVcCons + tid < nvec);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        st_stream_v4_if(out + i * kVcCons, V::grad_sv(getv(i), qb2, ql2, q), i * kVcCons + tid < nvec);
    }
    if (st != 0.f && ycol >= 0 && ((ycol >> 3) % kVcCons) == tid)  // same thread, after its vector store
      VecTraits<bf16_t>::store1(reinterpret_cast<char*>(a.dlogits) + row * row_bytes, ycol, dy);
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&sh.scale_free[sl]);
  };
  if constexpr (RS == 0) {
    // window R - 1 rows: row p is loaded into cache[p % R], row p - R + 1 written from cache[(p + 1) % R]
    for (int64_t p0 = 0; p0 < nk + R - 1; p0 += R) {
      static_for<0, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        const int64_t p = p0 + r;
        if (p < nk) load_row(rc, p);
        const int64_t g = p - (R - 1);
        constexpr int rg = (r + 1) % R;
        if (g >= 0 && g < nk) grad_vecs(g, [&](int i) { return cache[rg][i]; });
      });
    }
  } else {
    // window R + RS - 1 rows: before row p is loaded into cache[p % R], the row held there (p - R)
    // moves to shared-memory slot (p - R) % RS, whose row (p - R - RS) is written out first
    for (int64_t p0 = 0; p0 < nk + R + RS; p0 += R) {
      static_for<0, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        const int64_t p = p0 + r;
        const int64_t g = p - R - RS;
        if constexpr (PK) {
          // TMEM lane 32 (warp % 4) + lane, columns ((warp / 4) RS + slot) 4 NV + 4 i
          const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * RS * NV * 4);
          if (g >= 0 && g < nk) {
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            const uint32_t tb = tl + (uint32_t)((g % RS) * NV * 4);
            grad_vecs(g, [&](int i) { return tm_ld4(tb + (uint32_t)(4 * i)); });
          }
          const int64_t mv = p - R;
          if (mv >= 0 && mv < nk) {
            const uint32_t tb = tl + (uint32_t)((mv % RS) * NV * 4);
#pragma unroll
            for (int i = 0; i < NV; ++i) tm_st4(tb + (uint32_t)(4 * i), cache[r][i]);
          }
        } else {
          if (g >= 0 && g < nk) {
            const uint32_t base = rowc_s + (uint32_t)((g % RS) * NV * kVcCons) * 16u + my_off;
            RL_DCHECK(base + (uint32_t)((NV - 1) * kVcCons * 16) < rowc_s + (uint32_t)(RS * NV * kVcCons * 16));
            grad_vecs(g, [&](int i) { return sm100::lds128_a(base + (uint32_t)(i * kVcCons * 16)); });
          }
          const int64_t mv = p - R;
          if (mv >= 0 && mv < nk) {
            const uint32_t base = rowc_s + (uint32_t)((mv % RS) * NV * kVcCons) * 16u + my_off;
#pragma unroll
            for (int i = 0; i < NV; ++i) sm100::sts128(base + (uint32_t)(i * kVcCons * 16), cache[r][i]);
          }
        }
        if (p < nk) load_row(rc, p);
      });
    }
  }
  if constexpr (PK) {  // every consumer warp is done with its parked rows -> warp 0 frees the columns
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(kVcCons) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#ifdef RL_VC_TRACE
  if (tid == 0 && blockIdx.x < 256) {  // 6: consumer thread 0's cycles in the kernel, 7: SM id
    RL_VC_ADD(6, tk0);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_vc_trace[blockIdx.x][7] = smid;
  }
#endif
}


// L2 window of the ring kernel: D rows per CTA between a slice's two reads; G rows per service
// group, published LG groups before they are combined.  D >= (LG + 1) G - 1 is required (the
// service combines group g - LG only after the consumers finished pass 1 of group g).  A CTA keeps
// D + 1 row slices in L2 between their two reads (rows j - D .. j), so the grid's window
// grid (D + 1) slice is kept <= kVrWindow: at P = 2 (152 KB slices) D = 1 — with D = 3 the 90 MB
// window missed L2 on 97 % of the re-reads (ncu: 18.6 GB of DRAM reads for 10.0 GB algorithmic).
constexpr int64_t kVrWindow = 48ll << 20;
static void vr_geometry(int P, int64_t slice_bytes, int grid, int* G, int* LG, int* D) {
  *LG = 1;
  const int64_t rows = kVrWindow / std::max<int64_t>(1, (int64_t)grid * slice_bytes);  // max D + 1
  int g = std::min(4, 32 / std::max(P, 1));
  while (g > 1 && (int64_t)(2 * g + 2) > rows) g /= 2;
  *G = g;
  *D = g > 1 ? 2 * g + 1 : (int)std::max<int64_t>(1, std::min<int64_t>(3, rows - 1));
  const int dopt = dev_option(OPT_VR_DELAY);  // development override of D (G = 1)
  if (dopt > 0) {
    *G = 1;
    *D = dopt;
  }
}

static int vp_warp_grid(int64_t n_tokens) {
  static int ctas_tab[kMaxDevices] = {};
  int& ctas = dev_slot(ctas_tab);
  if (!ctas) {
    int occ = 4;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vp_stats_warp_kernel<bf16_t>, kVwThreads, 0);
    ctas = std::min(dev_info().sms * std::max(occ, 1), kMaxStatCtas);
  }
  return (int)std::min<int64_t>((n_tokens + kVwWarps - 1) / kVwWarps, ctas);
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
  if (rl_status e = require_sm100(); e != RL_OK) return e;
  cudaStream_t s = (cudaStream_t)stream;
  double* partials = (double*)workspace;
  float4* send = reinterpret_cast<float4*>((char*)workspace + kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double));
  float4* recv = send + n_tokens;
  if (n_tokens == 0) {
    if (with_loss && !(p->flags & RL_F_STATS_ACCUMULATE)) cudaMemsetAsync(stats, 0, sizeof(rl_loss_stats), s);
    return check_launch("vp empty");
  }
  const bool accumulate = with_loss && (p->flags & RL_F_STATS_ACCUMULATE) != 0;
  void* peers[8];
  int64_t max_tok = 0;
  uint32_t epoch = 0;
  if (with_loss && dev_option(OPT_VP_PATH) != 1 && comm_peer_exchange(comm, n_tokens, peers, &max_tok, &epoch)) {
    VrArgs v;
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
    const size_t par = (size_t)(epoch & 1) * P * max_tok * 2;  // u64 words
    for (int q = 0; q < 8; ++q) v.xr[q] = q < P ? reinterpret_cast<unsigned long long*>(peers[q]) + par : nullptr;
    const int grid = (int)std::min<int64_t>(n_tokens, std::min(dev_info().sms, kMaxStatCtas));
    // bf16 shards of <= 4800 whole vectors: the register-cache kernel (one read, one exp2 per
    // element); anything else: the L2 re-read ring kernel (same exchange protocol)
    const int64_t nv = vocab_shard / 8;
    // Across GPUs the register cache's exchange window (R + RS - 1 rows) does not absorb the ranks'
    // lockstep jitter, the L2 ring's (~14 us) does: 4 x B200, P = 4 width: ring 1.84 ms, cache 2.12;
    // P = 8 width: ring 1.09, cache 1.37 (rows parked in tensor memory).  One rank: cache 1.64 / 0.95,
    // ring 1.83 / 1.10.  So the cache on one rank, the ring on more.
    const int vk = dev_option(OPT_VP_KERNEL);  // 0 default, 1 ring, 2 cache whenever it fits
    const bool cache_fits = dtype == RL_BF16 && vocab_shard % 8 == 0 && nv >= 1 && nv <= 11 * kVcCons;
    const bool use_cache = cache_fits && (vk == 2 || (vk == 0 && P == 1));
    if (use_cache) {
      // rows parked in shared memory (RS): the exchange window is R + RS - 1 rows
      const bool wide = nv > 6 * kVcCons;
      const int rs_opt = dev_option(OPT_VC_ROWS);  // 0 = default, else RS + 1
      // default: parked rows across GPUs widen the exchange window (P = 8 width on 4 GPUs: RS = 0 /
      // 1 / 2 -> 1.59 / 1.55 / 1.47 ms; the wide shards have room for one); none on one rank, where
      // the records are back within a row and parking costs 11 % at the P = 8 width (0.95 vs 1.06 ms)
      // parked rows in tensor memory (RL_DEV_VC_TMEM: 0 default, 1 off, 2 on): RS = 2 wide / 4 narrow
      // rows, all of shared memory left to the ring.  Default on more than one rank at the narrow
      // (P >= 8) widths: P = 8 width on 4 GPUs 1.37 ms against 1.47 with two rows in shared memory
      // (and 1.54 for the ring); the wide shards lose (2.14 vs 2.12 ms across GPUs, 1.87 vs 1.64 on one)
      const int tm_opt = dev_option(OPT_VC_TMEM);
      const bool pk = tm_opt == 2 || (tm_opt == 0 && P > 1 && !wide);
      const int RS = pk ? (wide ? 2 : 4)
                        : rs_opt > 0 ? std::min(rs_opt - 1, 2) : (P > 1 ? (wide ? 1 : 2) : 0);
      // two parked wide rows in shared memory leave 62 KB of ring: 14 KB slots (CV = 2)
      const int slot_b = (!pk && wide && RS == 2 ? 2 : 4) * kVcCons * 16;
      const int NVc = wide ? 11 : 6;
      const size_t head = (sizeof(VcShared) + 127) & ~(size_t)127;
      const size_t rowc = pk ? 0 : (size_t)RS * NVc * kVcCons * 16;
      v.nslots = (int)((kSmemMax - head - rowc - 256) / (slot_b + 16));
      const size_t smem = ((sizeof(VcShared) + 16 * (size_t)v.nslots + 127) & ~(size_t)127) +
                          (size_t)v.nslots * slot_b + rowc;
      auto kern = pk ? (wide ? vp_cache_kernel<11, 2, 2, 4, 1> : vp_cache_kernel<6, 3, 4, 4, 1>)
                : wide ? (RS == 2 ? vp_cache_kernel<11, 2, 2, 2> : RS == 1 ? vp_cache_kernel<11, 2, 1> : vp_cache_kernel<11, 2, 0>)
                       : (RS == 2 ? vp_cache_kernel<6, 3, 2> : RS == 1 ? vp_cache_kernel<6, 3, 1>
                                                                      : vp_cache_kernel<6, 3, 0>);
      v.G = std::min(8, std::max(0, dev_option(OPT_VC_GROUPS)));
      // record send (measured, tools/vptrace.py / vpbench.py): across GPUs the last consumer warp's
      // weak stores (2.31 vs 2.42 ms at P = 4 on 4 GPUs); one rank: the collector's (weak) store
      v.pub_mode = dev_option(OPT_VC_PUB) > 0 ? std::min(2, dev_option(OPT_VC_PUB) - 1) : (P > 1 ? 1 : 2);
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute(vp_cache_kernel)");
      kern<<<grid, kVcThreads, smem, s>>>(v);
      rl_status stc = check_launch("vp_cache_kernel");
      if (stc != RL_OK) return stc;
      return launch_stats_reduce(partials, grid, stats, accumulate, s);
    }
    const int64_t slice_bytes = (vocab_shard / (16 / eb)) * 16;
    vr_geometry(P, std::max<int64_t>(slice_bytes, 16), grid, &v.G, &v.LG, &v.D);
    // vectors per thread per slot: the fewest idle tail lanes (ties: the smaller slot, more of them)
    const int64_t nvec_r = vocab_shard / (16 / eb);
    auto waste = [&](int vpt) {
      const int64_t cv = (int64_t)vpt * kVrCons;
      return ((nvec_r + cv - 1) / cv) * cv - nvec_r;
    };
    const int vpt = waste(5) < waste(4) ? 5 : 4;
    const int slot_b = vpt * kVrCons * 16;
    const size_t head = (sizeof(VrShared) + 127) & ~(size_t)127;
    v.nslots = (int)((kSmemMax - head - 256) / (slot_b + 16));
    const size_t smem = ((sizeof(VrShared) + 16 * (size_t)v.nslots + 127) & ~(size_t)127) + (size_t)v.nslots * slot_b;
    auto kern = dtype == RL_BF16 ? (vpt == 5 ? vp_ring_kernel<bf16_t, 5> : vp_ring_kernel<bf16_t, 4>)
                                 : (vpt == 5 ? vp_ring_kernel<float, 5> : vp_ring_kernel<float, 4>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute(vp_ring_kernel)");
    kern<<<grid, kVrThreads, smem, s>>>(v);
    rl_status st0 = check_launch("vp_ring_kernel");
    if (st0 != RL_OK) return st0;
    return launch_stats_reduce(partials, grid, stats, accumulate, s);
  }
  int grid = vp_warp_grid(n_tokens);
  if (dtype == RL_BF16)
    vp_stats_warp_kernel<bf16_t><<<grid, kVwThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                             vocab_offset, ld, targets, inv_temperature, send);
  else
    vp_stats_warp_kernel<float><<<grid, kVwThreads, 0, s>>>(logits_shard, n_tokens, vocab_shard,
                                                            vocab_offset, ld, targets, inv_temperature, send);
  rl_status st = check_launch("vp_stats_warp_kernel");
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
  const int tgrid = (int)std::min<int64_t>(n_tokens, std::min(dev_info().sms, kMaxStatCtas));
  const int nslots = 7;
  const size_t smem = ((8 * (2 * nslots + 2 * kVtScale) + 64 + 16 * kVtScale + 127) & ~(size_t)127) +
                      (size_t)nslots * kVtSlot;
  auto kern = dtype == RL_BF16 ? vp_finish_tma_kernel<bf16_t> : vp_finish_tma_kernel<float>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(vp_finish_tma_kernel)");
  kern<<<tgrid, kVtThreads, smem, s>>>(logits_shard, n_tokens, vocab_shard, vocab_offset, vocab_total, ld, recv, P,
                                       targets, old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active,
                                       kn, count, dlogits_shard, logp_out, lse_out, partials, nslots);
  st = check_launch("vp_finish_tma_kernel");
  if (st != RL_OK) return st;
  return launch_stats_reduce(partials, tgrid, stats, accumulate, s);
}

#ifdef RL_VC_TRACE
// development build only: copy (and optionally clear) the vp_cache_kernel cycle counters
extern "C" int rl_debug_vc_trace(unsigned long long* host, size_t bytes, int clear) {
  const size_t n = sizeof(rl::g_vc_trace) < bytes ? sizeof(rl::g_vc_trace) : bytes;
  if (host && cudaMemcpyFromSymbol(host, rl::g_vc_trace, n) != cudaSuccess) return 1;
  if (clear) {
    static unsigned long long zero[256 * 12] = {};
    if (cudaMemcpyToSymbol(rl::g_vc_trace, zero, sizeof(zero)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif
