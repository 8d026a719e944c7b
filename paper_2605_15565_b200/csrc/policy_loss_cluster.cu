// Row-resident cluster kernel "R" of the fused policy loss — the hot kernel.
//
// North_star: "a single streaming pass over bf16 logits with online max and sum-exp, using
// vectorised 128-bit coalesced loads staged through TMA or shared memory ... the gather,
// ratio, clip, mask and gradient write fused into that same pass, so logits are read once
// and dlogits written once."
//
// A row of V = 151936 bf16 logits is 297 KB, more than one SM's shared memory, so each row is
// split over a thread-block CLUSTER of CL CTAs (CL = 2 at V = 151936: 148 KB per CTA).  Per CTA:
//   producer warp : cp.async.bulk (TMA bulk copy) of 7.5 KB chunks of this CTA's column slice
//                   into a ring of shared-memory slots (mbarrier full/empty pipeline), running
//                   ahead into the next rows as slots free up.
//   consumer warps (15), per row i, software-pipelined so the cross-CTA exchange of row i
//   overlaps the arrival / max pass of row i+1:
//     pass B(i)  e' = 2^(x k - m_c + 15) from the ring, sum e' (the only MUFU.EX2 per element);
//                e' is kept as fp16 in REGISTERS (20 x 16 B per thread) and the ring slot is
//                released immediately -> the ring refills with the next rows during the rest.
//     send(i)    (m_c, s_c, z_y) record -> peer CTA(s): st.shared::cluster + remote mbarrier arrive
//     pass A(i+1) max over row i+1's slice as its chunks land (packed bf16 max)
//     recv(i)    combine in rank order -> lse, logp, ratio, clip, s_t (c3-c7; identical in every
//                CTA of the cluster, rank 0 records the statistics)
//     pass C(i)  dlogits = s_t 2^(m_c - 15 - lse2) e'  (target column: s_t (p_y - 1)), bf16 RNE,
//                128-bit streaming stores straight from the register cache.
// HBM traffic: logits read once (TMA), dlogits written once.  dlogits may alias logits: a CTA
// writes only its own slice of row i, after that slice is fully resident.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "cluster_common.cuh"

namespace rl {

// Development trace (RL_TRACE=1 selects the traced instantiation): per CTA, the first 64 rows'
// phase boundaries in globaltimer ns.  Read with rl_debug_trace (tools/trace_cluster.py).
constexpr int kTraceRows = 64, kTraceEv = 8, kTraceCtas = 256;
__device__ unsigned long long g_trace[kTraceCtas][kTraceRows][kTraceEv];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RL_TRACE_EV(row_it, ev)                                                           \
  do {                                                                                   \
    if (TRACE && blockIdx.x < kTraceCtas && (row_it) < kTraceRows)                       \
      g_trace[blockIdx.x][(row_it)][(ev)] = gtimer();                                    \
  } while (0)

struct __align__(16) ClShared {
  float4 xch[2][8];             // [row parity][cluster rank]: (m_c log2 units, s_c, z_y, owned)
  float red_max[2][kNcw];       // [pass-A call parity][warp] block reduction
  float red_sum[2][kNcw];       // [row parity][warp] pass-B partial sums (2^15-scaled)
  float mrow[2];                // [row parity] slice max m_c (log2 units)
  float4 row_sc[2];             // [row parity] (s_t, lse2, d_y, target column as int bits or -1)
  float rref[2][8];             // [row parity][group] reference max R_g of each chunk group (log2)
  uint64_t xbar[2];             // peer records landed (CL - 1 remote arrivals)
  uint64_t sumbar[2];           // consumers finished pass B (kNcw arrivals)
  uint64_t scalebar[2];         // epilogue published row_sc (1 arrival)
  // followed by full[nslots], empty[nslots] (uint64) then the ring (128-B aligned)
};

// NCH = compile-time upper bound of chunks per CTA slice (the register cache is uint4[NCH]).
//
// Warp roles: warps 0..14 consume (passes A/B/C); warp 15 is the service warp: lane 0 issues the
// TMA bulk copies, lane 1 runs the per-row epilogue (DSMEM exchange with the peer CTA(s),
// combine, ratio/clip/scale, statistics) off the consumers' critical path.
// cache operations: fp16 e' + fp32 multiply (default) or bf16 e' + packed bf16 multiply (BFC)
template <typename T, bool BFC>
struct CacheOps {
  __device__ static __forceinline__ uint64_t exp(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc, uint4& c) {
    return ClVec<T>::exp_cache(v, k2, mn2, acc, c);
  }
  __device__ static __forceinline__ uint4 grad(const uint4& c, uint64_t q2, uint32_t) { return ClVec<T>::grad(c, q2); }
};
template <>
struct CacheOps<bf16_t, true> {
  __device__ static __forceinline__ uint64_t exp(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc, uint4& c) {
    return ClVec<bf16_t>::exp_cache_bf(v, k2, mn2, acc, c);
  }
  __device__ static __forceinline__ uint4 grad(const uint4& c, uint64_t, uint32_t qb2) {
    return ClVec<bf16_t>::grad_bf(c, qb2);
  }
};

template <typename T, int CL, int NCH, bool EXACT, int H, bool TRACE = false, bool BFC = false>
__global__ void __launch_bounds__(kClThreads, 1) loss_cluster_kernel(const ClArgs a) {
  static_assert(H >= 1 && H <= 8, "chunk groups per row");
  constexpr int EPV = ClVec<T>::EPV;
  using MaxT = typename ClVec<T>::MaxT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ClShared& sh = *reinterpret_cast<ClShared*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + sizeof(ClShared));
  uint64_t* empty = full + a.nslots;
  const size_t ring_off = (sizeof(ClShared) + 2 * sizeof(uint64_t) * a.nslots + 127) & ~(size_t)127;
  uint4* ring = reinterpret_cast<uint4*>(smem_raw + ring_off);
  const int nslots = a.nslots;
  const uint32_t full_s = sm100::smem_u32(full), empty_s = sm100::smem_u32(empty);
  const uint32_t ring_s = sm100::smem_u32(ring);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = sm100::cluster_ctarank();
  const int64_t cid = sm100::cluster_id_x();
  const int64_t ncl = sm100::nclusters_x();
  const int64_t v0 = (int64_t)crank * a.h_vec;
  const int64_t v1 = min(a.nvec, v0 + a.h_vec);
  const int my_nv = (int)max((int64_t)0, v1 - v0);
  const int nfull = my_nv / kChunkVec;             // full chunks
  const int last_nv = my_nv - nfull * kChunkVec;   // vectors of the partial last chunk
  const int nch = nfull + (last_nv > 0);           // <= NCH (checked at launch)
  const bool tail_owner = crank == CL - 1;
  const int n_tail = (int)(a.V - a.nvec * EPV);    // < EPV scalar columns after the vectors
  const int64_t row_bytes = a.ld * elem_bytes<T>();

  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], kNcw);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&sh.xbar[i], CL - 1);
      sm100::mbar_init(&sh.sumbar[i], kNcw);
      sm100::mbar_init(&sh.scalebar[i], 1);
    }
    sm100::fence_mbar_init();
  }
  sm100::cluster_sync();  // barriers initialised before any remote arrive / TMA

  if (warp == kNcw) {
    if (lane == 0 && nch > 0) {
      // ---------------------------------------------------------- TMA producer (lane 0)
      const uint64_t pol = policy_evict_first();
      RingPos rp{0, 0};
      // L2 lookahead: when the ring is full, the chunks that must wait for a free slot are
      // prefetched into L2 (up to pf_chunks ahead) so their later TMA loads are L2 hits.
      const int pf_chunks = a.prefetch_chunks;
      int64_t g = 0, g_pf = 0;
      for (int64_t row = cid; row < a.n_tokens; row += ncl) {
        const char* src = reinterpret_cast<const char*>(a.logits) + row * row_bytes + v0 * 16;
        for (int j = 0; j < nch; ++j, ++g) {
          if (pf_chunks > 0 && g >= g_pf && !sm100::mbar_try_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1)) {
            int64_t rr = row, jj = j;
            for (int q = 0; q < pf_chunks; ++q) {
              if (rr >= a.n_tokens) break;
              const uint32_t pb = (jj < nfull ? kChunkVec : last_nv) * 16u;
              sm100::bulk_prefetch_l2(reinterpret_cast<const char*>(a.logits) + rr * row_bytes + v0 * 16 +
                                          (size_t)jj * kChunkBytes, pb);
              if (++jj == nch) {
                jj = 0;
                rr += ncl;
              }
            }
            g_pf = g + pf_chunks;
          }
          sm100::mbar_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1);
          const uint32_t bytes = (j < nfull ? kChunkVec : last_nv) * 16u;
          sm100::mbar_arrive_expect_tx(&full[rp.slot], bytes);
          if (a.debug == 3)
            sm100::bulk_g2s(ring + (size_t)rp.slot * kChunkVec, src + (size_t)j * kChunkBytes, bytes,
                            &full[rp.slot], pol);
          else
            sm100::bulk_g2s_nohint(ring + (size_t)rp.slot * kChunkVec, src + (size_t)j * kChunkBytes, bytes,
                                   &full[rp.slot]);
          rp.advance(1, nslots);
        }
      }
    } else if (lane == 1) {
      // ---------------------------------------------------------- row epilogue (lane 1)
      const double inv_tm = token_mean_inv(a.kn);
      Acc acc;
      acc.zero();
      uint32_t it = 0;
      for (int64_t row = cid; row < a.n_tokens; row += ncl, ++it) {
        const int par = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        const char* rp = reinterpret_cast<const char*>(a.logits) + row * row_bytes;
        const RowMeta mt = row_meta(row, a.V, a.targets, a.mask, a.token_seq, a.seq_version,
                                    a.kn.trainer_version, a.kn.max_staleness);
        float A = 0.f, old = 0.f, zy = 0.f;
        bool owned = false;
        if (mt.valid) {
          A = a.seq_adv[mt.seq];
          old = a.old_logp[row];
        }
        if (mt.in_range) {
          const int64_t vy = mt.y / EPV;
          owned = (vy >= v0 && vy < v1) || (tail_owner && vy >= a.nvec);
          if (owned) zy = VecTraits<T>::load1(rp, mt.y) * a.kn.inv_t;
        }
        RL_TRACE_EV(it, 4);
        if (a.debug == 4) sm100::mbar_wait(&sh.sumbar[par], ph);
        else sm100::mbar_wait_polite(&sh.sumbar[par], ph, false);
        RL_TRACE_EV(it, 5);
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kNcw; ++w) s += sh.red_sum[par][w];
        s *= 1.f / 32768.f;  // undo the 2^15 cache shift (exact)
        const float m = sh.mrow[par];
        const float4 rec = make_float4(m, s, owned ? zy : 0.f, owned ? 1.f : 0.f);
        sh.xch[par][crank] = rec;
#pragma unroll
        for (int r = 0; r < CL; ++r)
          if (r != (int)crank) {
            sm100::st_remote_v4(&sh.xch[par][crank], r, rec.x, rec.y, rec.z, rec.w);
            sm100::mbar_arrive_remote(&sh.xbar[par], r);
          }
        if (CL > 1) {
          if (a.debug == 4) sm100::mbar_wait_cluster(&sh.xbar[par], ph);
          else sm100::mbar_wait_polite(&sh.xbar[par], ph, true);
        }
        RL_TRACE_EV(it, 6);
        // combine in rank order (bitwise identical in every CTA of the cluster)
        float M = -INFINITY;
#pragma unroll
        for (int r = 0; r < CL; ++r) M = fmaxf(M, sh.xch[par][r].x);
        float S = 0.f, z = 0.f;
#pragma unroll
        for (int r = 0; r < CL; ++r) {
          const float4 e = sh.xch[par][r];
          if (e.x != -INFINITY) S += e.y * fast_exp2(e.x - M);
          z += e.z;
        }
        const float c2 = M + fast_log2(S);
        const float lp = logp_from(mt, z, c2);
        uint8_t cl = 0;
        Acc tmp;
        tmp.zero();
        float prox_, ref_;
        token_extra(a.kn, row, old, prox_, ref_);
        const float st = token_epilogue(mt, lp, old, A, a.seq_active, inv_tm, a.kn, tmp, &cl, prox_, ref_);
        if (crank == 0) {
#pragma unroll
          for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
          if (a.logp_out) a.logp_out[row] = lp;
          if (a.clipped_out) a.clipped_out[row] = cl;
        }
        // q = s_t 2^(m_c - 15 - lse2): p_v = (q / s_t) e'_v.  An all -inf / empty slice has no
        // cache (pass B skipped) and q = 0.  Target column: d_y = s_t (p_y - 1).
        (void)m;
        const float dy = st * (fast_exp2(z * RL_LOG2E - c2) - 1.f);
        sh.row_sc[par] = make_float4(st, c2, dy, __int_as_float(owned ? mt.y : -1));
        sm100::mbar_arrive(&sh.scalebar[par]);
        RL_TRACE_EV(it, 7);
      }
#pragma unroll
      for (int i = 0; i < RL_LOSS_STATS_N; ++i)
        a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = crank == 0 ? acc.v[i] : 0.0;
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ consumer warps
    const float k = a.kn.inv_t * RL_LOG2E;
    const uint64_t k2 = f2pack(k, k);
    const uint32_t my_off = (uint32_t)tid * 16u;
    const bool last_mine = tid < last_nv;  // this thread's vector exists in the partial last chunk
    uint4 cache[NCH];  // this thread's fp16 e' values for the current row (registers)
    RingPos pos{0, 0};
    constexpr int GS = (NCH + H - 1) / H;  // chunks per group; each group has its own reference
    // chunk j of a row: present (uniform), partial (uniform: the ragged last chunk), mine (per thread)
#define RL_PRESENT(j) (EXACT ? true : ((j) < nch))
#define RL_PARTIAL(j) (EXACT ? ((j) == NCH - 1 && last_nv > 0) : ((j) == nfull))
#define RL_MINE(j) (!RL_PARTIAL(j) || last_mine)

    // pass A of chunk group g of `row` (ring position p of the row's first chunk): waits for the
    // group's chunks, returns their block-reduced log2-domain max R_g (the last group also covers
    // this thread's scalar tail column, returned in xt).
    uint32_t acall = 0;  // pass-A call counter (red_max double buffer)
    auto group_a = [&](int64_t row, RingPos p, int g, float& xt) -> float {
      MaxT mx = ClVec<T>::max_init();
      const int ab = (acall++) & 1;
      uint32_t slot = p.slot + g * GS, ph = p.phase;
      while (slot >= (uint32_t)nslots) {
        slot -= nslots;
        ph ^= 1u;
      }
#pragma unroll
      for (int j = g * GS; j < (g + 1) * GS && j < NCH; ++j) {
        if (RL_PRESENT(j)) {
          sm100::mbar_wait_a(full_s + slot * 8, ph);
          uint4 v = sm100::lds128_a(ring_s + slot * (uint32_t)kChunkBytes + my_off);
          if (!RL_MINE(j)) v = ClVec<T>::neg_inf_vec();  // stale bytes past the slice
          ClVec<T>::max_acc(v, mx);
          if (++slot == (uint32_t)nslots) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
      float m = ClVec<T>::max_to_float(mx);
      if (g == H - 1) {
        xt = -INFINITY;
        if (tail_owner && tid < n_tail) {
          xt = VecTraits<T>::load1(reinterpret_cast<const char*>(a.logits) + row * row_bytes, a.nvec * EPV + tid);
          m = fmaxf(m, xt);
        }
      }
      m = warp_max(m);
      if (lane == 0) sh.red_max[ab][warp] = m;
      sm100::named_bar_sync(1, kCons);
      m = sh.red_max[ab][0];
#pragma unroll
      for (int w = 1; w < kNcw; ++w) m = fmaxf(m, sh.red_max[ab][w]);
      return m * k;
    };
    // running (R_run, S_run) of a row: group sums fold into the largest reference seen so far
    float R_run = -INFINITY, S_run = 0.f;
    auto fold = [&](float Rg, uint64_t acc2) {
      float s0, s1;
      f2unpack(acc2, s0, s1);
      const float sg = s0 + s1;
      if (Rg == -INFINITY) return;
      if (Rg > R_run) {
        S_run = (R_run == -INFINITY ? 0.f : S_run * fast_exp2(R_run - Rg)) + sg;
        R_run = Rg;
      } else {
        S_run += sg * fast_exp2(Rg - R_run);
      }
    };
    auto send_sum = [&](uint32_t itn) {
      const float sum = warp_sum(S_run);
      if (lane == 0) {
        sh.red_sum[itn & 1][warp] = sum;
        if (warp == 0) sh.mrow[itn & 1] = R_run;
        sm100::mbar_arrive(&sh.sumbar[itn & 1]);
      }
    };

    int64_t row = cid;
    uint32_t it = 0;
    float xt = -INFINITY, xt_next = -INFINITY;
    float Rg0 = 0.f;  // group-0 reference of the next row, computed while the exchange runs
    if (row < a.n_tokens) {  // pass A + B of the first row, group by group
      R_run = -INFINITY;
      S_run = 0.f;
      uint32_t slot = pos.slot;
#pragma unroll
      for (int g = 0; g < H; ++g) {
        const float Rg = group_a(row, pos, g, xt);
        if (tid == 0) sh.rref[0][g] = Rg;
        const bool live = Rg != -INFINITY;
        const uint64_t mn2 = f2pack(kCacheShift - Rg, kCacheShift - Rg);
        uint64_t acc2 = f2pack(0.f, 0.f);
#pragma unroll
        for (int j = g * GS; j < (g + 1) * GS && j < NCH; ++j) {
          if (RL_PRESENT(j)) {
            if (live) {
              const uint4 v = sm100::lds128_a(ring_s + slot * (uint32_t)kChunkBytes + my_off);
              const uint64_t nacc = CacheOps<T, BFC>::exp(v, k2, mn2, acc2, cache[j]);
              acc2 = RL_MINE(j) ? nacc : acc2;
            }
            sm100::mbar_arrive_lane0(empty_s + slot * 8, lane);
            if (++slot == (uint32_t)nslots) slot = 0;
          }
        }
        if (g == H - 1 && tail_owner && tid < n_tail && live) {
          xt = fast_exp2(fmaf(xt, k, kCacheShift - Rg));
          acc2 = fadd2(acc2, f2pack(xt, 0.f));
        }
        fold(Rg, acc2);
      }
      pos.advance(nch, nslots);
      send_sum(0);
    }
    for (; row < a.n_tokens; row += ncl, ++it) {
      const int par = it & 1;
      char* dp = reinterpret_cast<char*>(a.dlogits) + row * row_bytes;
      // ---- pass A of the next row's first chunk group overlaps the exchange of this one
      const int64_t next = row + ncl;
      const bool has_next = next < a.n_tokens;
      if (tid == 0) RL_TRACE_EV(it, 0);
      if (has_next) Rg0 = group_a(next, pos, 0, xt_next);
      if (tid == 0) RL_TRACE_EV(it, 1);
      sm100::mbar_wait(&sh.scalebar[par], (it >> 1) & 1);
      if (tid == 0) RL_TRACE_EV(it, 2);
      const float4 sc = sh.row_sc[par];
      const float st = sc.x, c2 = sc.y, dy = sc.z;
      const int ycol = __float_as_int(sc.w);
      uint4* out = reinterpret_cast<uint4*>(dp) + v0 + tid;
      // ---- fused pass C(row) + pass A/B(next) group by group: the dlogits stores of this row
      // drain while the next row's groups are max-reduced (as they land) and exp2'd; each
      // register-cache entry is emptied (stored) and refilled in place.
      R_run = -INFINITY;
      S_run = 0.f;
      uint32_t slot = pos.slot;
      float q_last = 0.f;
#pragma unroll
      for (int g = 0; g < H; ++g) {
        float Rg = Rg0;
        if (has_next && g > 0) Rg = group_a(next, pos, g, xt_next);
        if (has_next && tid == 0) sh.rref[(it + 1) & 1][g] = Rg;
        const float Rc = sh.rref[par][g];  // this row's group reference
        const float q = (st == 0.f || Rc == -INFINITY) ? 0.f : st * fast_exp2(Rc - kCacheShift - c2);
        q_last = q;
        const uint64_t q2 = f2pack(q, q);
        const uint32_t qb2 = pack_bf16x2(q, q);
        const bool zero = q == 0.f;
        const bool live = has_next && Rg != -INFINITY;
        const uint64_t mn2 = f2pack(kCacheShift - Rg, kCacheShift - Rg);
        uint64_t acc2 = f2pack(0.f, 0.f);
#pragma unroll
        for (int j = g * GS; j < (g + 1) * GS && j < NCH; ++j) {
          if (RL_PRESENT(j)) {
            if (RL_MINE(j) && (!TRACE || a.debug != 1))
              st_stream_v4(out + j * kChunkVec, zero ? make_uint4(0, 0, 0, 0) : CacheOps<T, BFC>::grad(cache[j], q2, qb2));
            if (has_next) {
              if (live && (!TRACE || a.debug != 2)) {
                const uint4 v = sm100::lds128_a(ring_s + slot * (uint32_t)kChunkBytes + my_off);
                const uint64_t nacc = CacheOps<T, BFC>::exp(v, k2, mn2, acc2, cache[j]);
                acc2 = RL_MINE(j) ? nacc : acc2;
              }
              sm100::mbar_arrive_lane0(empty_s + slot * 8, lane);
              if (++slot == (uint32_t)nslots) slot = 0;
            }
          }
        }
        if (g == H - 1) {
          if (tail_owner && tid < n_tail) {  // this row's tail column (cached e' in xt)
            const float o = (q == 0.f) ? 0.f : xt * q;
            VecTraits<T>::store1(dp, a.nvec * EPV + tid, o);
          }
          if (has_next && tail_owner && tid < n_tail && live) {
            xt_next = fast_exp2(fmaf(xt_next, k, kCacheShift - Rg));
            acc2 = fadd2(acc2, f2pack(xt_next, 0.f));
          }
        }
        if (has_next) fold(Rg, acc2);
      }
      (void)q_last;
      // target column: rewritten by the thread that stored its vector (or tail column) above —
      // same-thread program order to the same address.
      if (st != 0.f && ycol >= 0) {
        const bool in_tail = ycol >= a.nvec * EPV;
        const int owner = in_tail ? (int)(ycol - a.nvec * EPV) : (int)((ycol / EPV - v0) % kChunkVec);
        if (tid == owner) VecTraits<T>::store1(dp, ycol, dy);
      }
      if (has_next) {
        pos.advance(nch, nslots);
        send_sum(it + 1);
      }
      if (tid == 0) RL_TRACE_EV(it, 3);
      xt = xt_next;
    }
#undef RL_PRESENT
#undef RL_PARTIAL
#undef RL_MINE
  }
  __syncwarp();
  sm100::cluster_sync();  // no CTA leaves while a peer may still arrive on / write its smem
}

template <typename T, int CL, int NCH, bool EXACT = false, int H = 1, bool TRACE = false,
          bool BFC = std::is_same<T, bf16_t>::value>
static rl_status launch_cl(const ClArgs& a0, int64_t n, cudaStream_t s, int* n_ctas) {
  ClArgs a = a0;
  auto kern = loss_cluster_kernel<T, CL, NCH, EXACT, H, TRACE, BFC>;
  const size_t head = (sizeof(ClShared) + 127) & ~(size_t)127;
  int nslots = (int)((kSmemMax - head - 256) / (kChunkBytes + 16));
  const int nch = (int)((a.h_vec + kChunkVec - 1) / kChunkVec);
  static int slots_cap = -1;  // RL_CLUSTER_SLOTS: cap on the ring depth (tuning knob)
  if (slots_cap < 0) slots_cap = getenv("RL_CLUSTER_SLOTS") ? atoi(getenv("RL_CLUSTER_SLOTS")) : 0;
  if (slots_cap > 0) nslots = std::min(nslots, std::max(slots_cap, nch));
  if (nch > nslots || nch > NCH || (EXACT && nch != NCH)) return RL_ERR_UNSUPPORTED;
  a.nslots = nslots;
  const size_t smem = ((sizeof(ClShared) + 2 * sizeof(uint64_t) * nslots + 127) & ~(size_t)127) +
                      (size_t)nslots * kChunkBytes;
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute(max dynamic smem)");
    attr_done = true;
  }
  static int max_clusters = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!max_clusters) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(sms / CL * CL);
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      max_clusters = sms / CL;
    }
  }
  const int64_t ncl = std::min<int64_t>(std::min<int64_t>(n, max_clusters), kMaxStatCtas / CL);
  cfg.gridDim = dim3((unsigned)(ncl * CL));
  *n_ctas = (int)(ncl * CL);
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return check_launch("loss_cluster_kernel");
  return check_launch("loss_cluster_kernel");
}

rl_status launch_loss_cluster(const void* logits, int32_t dtype, int64_t n, int64_t V, int64_t ld,
                              const int32_t* targets, const float* old_logp, const uint8_t* mask,
                              const int32_t* token_seq, const float* seq_adv,
                              const int32_t* seq_version, const int32_t* seq_active,
                              const Knobs& kn, void* dlogits, float* logp_out, uint8_t* clipped_out,
                              double* partials, int* n_ctas, cudaStream_t s) {
  // masked-row skipping and the entropy moment are not in this kernel: the two-pass kernel runs
  if (kn.flags & (RL_F_SKIP_MASKED_READS | RL_F_ENTROPY)) return RL_ERR_UNSUPPORTED;
  ClArgs a;
  a.logits = logits;
  a.dlogits = dlogits;
  a.n_tokens = n;
  a.V = V;
  a.ld = ld;
  const int epv = dtype == RL_BF16 ? 8 : 4;
  a.nvec = V / epv;
  a.targets = targets;
  a.old_logp = old_logp;
  a.mask = mask;
  a.token_seq = token_seq;
  a.seq_adv = seq_adv;
  a.seq_version = seq_version;
  a.seq_active = seq_active;
  a.logp_out = logp_out;
  a.clipped_out = clipped_out;
  a.partials = partials;
  a.kn = kn;
  a.nslots = 0;
  static int pfc = -1;
  if (pfc < 0) pfc = getenv("RL_L2_PREFETCH_CHUNKS") ? atoi(getenv("RL_L2_PREFETCH_CHUNKS")) : 0;
  a.prefetch_chunks = pfc;
  a.debug = getenv("RL_CLUSTER_DEBUG") ? atoi(getenv("RL_CLUSTER_DEBUG")) : 0;
  // Half rows per 2-CTA cluster by default (all 148 SMs).  RL_CLUSTER_CL=3 selects thirds of a
  // row per 3-CTA cluster (more ring slack, 56-register cache) — measured slower.
  static int cl_env = -1;
  if (cl_env < 0) {
    cl_env = 2;
    if (const char* e = getenv("RL_CLUSTER_CL")) cl_env = atoi(e) == 3 ? 3 : 2;
  }
  const bool bf = dtype == RL_BF16;
  auto nchunks = [&](int64_t h) { return (h + kChunkVec - 1) / kChunkVec; };
  const int64_t h2 = (a.nvec + 1) / 2, nch2 = nchunks(h2);
  const int64_t h3 = (a.nvec + 2) / 3, nch3 = nchunks(h3);
  if (cl_env == 3 && nch2 > 10 && nch3 <= 20) {
    a.h_vec = h3;
    if (bf && nch3 == 14) return launch_cl<bf16_t, 3, 14, true>(a, n, s, n_ctas);  // V = 151936
    if (bf && nch3 == 12) return launch_cl<bf16_t, 3, 12, true>(a, n, s, n_ctas);  // V = 128256
    return bf ? launch_cl<bf16_t, 3, 20>(a, n, s, n_ctas) : launch_cl<float, 3, 20>(a, n, s, n_ctas);
  }
  a.h_vec = h2;
  if (bf && nch2 == 20) {  // V = 151936: 4 chunk groups (RL_CLUSTER_GROUPS = 1, 2, 4, 5)
    static int groups = -1;
    if (groups < 0) groups = getenv("RL_CLUSTER_GROUPS") ? atoi(getenv("RL_CLUSTER_GROUPS")) : 1;
    if (getenv("RL_TRACE")) return launch_cl<bf16_t, 2, 20, true, 1, true, true>(a, n, s, n_ctas);
    static int f16c = -1;  // RL_CACHE=fp16: fp16 row cache + fp32 multiply in pass C (comparison)
    if (f16c < 0) f16c = (getenv("RL_CACHE") && strcmp(getenv("RL_CACHE"), "fp16") == 0) ? 1 : 0;
    if (groups == 1 && f16c) return launch_cl<bf16_t, 2, 20, true, 1, false, false>(a, n, s, n_ctas);
    if (groups == 1) return launch_cl<bf16_t, 2, 20, true, 1>(a, n, s, n_ctas);
    if (groups == 2) return launch_cl<bf16_t, 2, 20, true, 2>(a, n, s, n_ctas);
    if (groups == 5) return launch_cl<bf16_t, 2, 20, true, 5>(a, n, s, n_ctas);
    return launch_cl<bf16_t, 2, 20, true, 4>(a, n, s, n_ctas);
  }
  if (bf && nch2 == 17) return launch_cl<bf16_t, 2, 17, true>(a, n, s, n_ctas);  // V = 128256
  if (nch2 <= 2) return bf ? launch_cl<bf16_t, 2, 2>(a, n, s, n_ctas) : launch_cl<float, 2, 2>(a, n, s, n_ctas);
  if (nch2 <= 5) return bf ? launch_cl<bf16_t, 2, 5>(a, n, s, n_ctas) : launch_cl<float, 2, 5>(a, n, s, n_ctas);
  if (nch2 <= 10) return bf ? launch_cl<bf16_t, 2, 10>(a, n, s, n_ctas) : launch_cl<float, 2, 10>(a, n, s, n_ctas);
  if (nch2 <= 20) return bf ? launch_cl<bf16_t, 2, 20>(a, n, s, n_ctas) : launch_cl<float, 2, 20>(a, n, s, n_ctas);
  a.h_vec = (a.nvec + 3) / 4;
  return bf ? launch_cl<bf16_t, 4, 20>(a, n, s, n_ctas) : launch_cl<float, 4, 20>(a, n, s, n_ctas);
}

}  // namespace rl

// development only (not part of include/rl_policy.h): copy the phase trace to the host
extern "C" int rl_debug_trace(unsigned long long* host, size_t bytes) {
  const size_t n = sizeof(rl::g_trace) < bytes ? sizeof(rl::g_trace) : bytes;
  return cudaMemcpyFromSymbol(host, rl::g_trace, n) == cudaSuccess ? 0 : 1;
}
