// Single-visit cluster kernel "SV" of the fused policy loss — the hot kernel.
//
// North_star: "a single streaming pass over bf16 logits with online max and sum-exp ... the
// gather, ratio, clip, mask and gradient write fused into that same pass, so logits are read
// once and dlogits written once."
//
// Like kernel "R" (policy_loss_cluster.cu) a row of V = 151936 bf16 logits is split over a
// 2-CTA cluster and each thread keeps its e' values of the current row in a register cache.
// The difference is the exponent reference.  R takes the slice max first (pass A), which keeps
// every ring slot of a row occupied until pass B has re-read it — the ring then holds a whole
// row and only its remaining slots (9 of 29) overlap HBM latency.  SV uses the TARGET logit as
// the reference, known before the row is read (one 2-byte load per row by the service warp):
//     e'_v = 2^(x_v k - R + 15),  R = x_y k,  k = inv_T log2(e)
// so each chunk is exp2'd the moment it lands and its slot is released at once: all ring slots
// are read slack.  Since x_y <= max_v x_v, e'_y = 2^15 and the sum S' = sum_v e'_v >= 2^15
// never underflows; the largest term is 2^(15 + (max - x_y) k), bf16/fp32 range up to 2^127.
// Rows whose S' >= 2^115 (max - x_y > ~69 nats) or is not finite (NaN / inf logits) are
// flagged and redone by the exact two-pass kernel (policy_loss.cu, fixup launch); the fast
// kernel writes nothing for them.  Then (c3-c7):
//     lse2 = R - 15 + log2 S'    logp = ln(2^15 / S')    p_v = e'_v / S'
//     dlogits_v = (s_t / S') e'_v  (bf16 x bf16 HMUL2),  target column s_t (p_y - 1).
//
// Per CTA: warps 0..14 consume; warp 15 lane 0 issues the TMA bulk copies of this CTA's column
// slice into a ring of smem slots (mbarrier full/empty); lane 1 is the service lane.  A slot
// holds VPT x 7.5 KB (VPT 16-B vectors per consumer thread; default 4 -> 30 KB, 7 slots): the
// copy probe (tools/copy_probe.cu) reads 3.6-4.5 TB/s from 7.5 KB bulk copies but
// 7.5 TB/s from 15-30 KB ones, so the copy size, not the ring depth, bounds the read side.
// Consumer iteration p: wait ref(p) (reference and metadata of row p, published two rows ahead by
// the service lane), then one loop over the chunks: store dlogits chunk j of row p-1 from
// cache[j], refill cache[j] with row p's chunk j as it lands; then the row exchange, done by the
// consumers themselves to keep it short: warp sums -> named barrier -> CTA sum -> thread 0
// st.async's it to the peer (no release fence) -> every thread combines and computes the row's
// scale (token_ratio / token_scale, the statistics' own functions).  Thread 0 posts (S', logp) and
// the service lane writes logp, clip flag, redo flag and the statistics off the critical path.
#include <cuda_bf16.h>

#include "cluster_common.cuh"

namespace rl {

struct __align__(16) SvShared {
  float4 xch[2][8];    // [row parity][cluster rank]: (S'_c, -, -, -), written by the peers' st.async
  float red_sum[2][kNcw];
  float red_ent[2][kNcw];  // RL_F_ENTROPY: per-warp sum e' x
  // row p's metadata in slot p % 4: published two rows ahead and read by the consumers up to the
  // end of row p's exchange, so the slot of ref(p+2) must differ from row p's (a 2-deep ring let a
  // slow consumer warp read row p+2's values)
  float4 refa[4];      // row p: (15 - R_p, A, old_logp, (float) w)
  float4 refc[4];      // row p: (prox_logp, ref_logp, -, -)
  int4 refb[4];        // row p: (need | valid << 1, target column if in this CTA's slice else -1, -, -)
  float4 res[2];       // row p: (S', logp, sum e' x, -) from consumer thread 0 for the statistics lane
  uint64_t xbar[2];    // peer records landed (thread 0's expect_tx arrive + 16 B st.async per peer)
  uint64_t refbar[4];  // service lane published ref(p) (1 arrival)
  uint64_t resbar[2];  // consumer thread 0 posted res(p) (1 arrival)
};
enum : uint32_t { SV_NONE = 0, SV_ZERO = 1, SV_GRAD = 2 };  // how row p-1's dlogits are written
constexpr float kSvRedo = 0x1p115f;                         // S' bound of the fast path
static_assert(kCacheShift == 15.f, "p_y = 2^15 / S' below");

constexpr int kSvThreads = kClThreads;  // 15 consumer warps + 1 service warp (128 registers)

// XF: compile-time extensions — bit 0 the entropy moment (RL_F_ENTROPY), bit 1 the KL / proximal
// terms (kl_coef, prox_logp); the default instantiation (XF = 0) carries neither.
template <typename T, int CL, int NCH, bool EXACT, int VPT = 4, int XF = 0>
__global__ void __launch_bounds__(kSvThreads, 1) loss_sv_kernel(const ClArgs a) {
  constexpr int EPV = ClVec<T>::EPV;
  constexpr bool ENT = (XF & 1) != 0, EXT = (XF & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SvShared& sh = *reinterpret_cast<SvShared*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + sizeof(SvShared));
  uint64_t* empty = full + a.nslots;
  const size_t ring_off = (sizeof(SvShared) + 2 * sizeof(uint64_t) * a.nslots + 127) & ~(size_t)127;
  uint4* ring = reinterpret_cast<uint4*>(smem_raw + ring_off);
  const int nslots = a.nslots;
  const uint32_t rt_zero = (uint32_t)nslots >> 31;  // 0 at run time (sm100::mbar_release_after)
  uint32_t dep = 0;                                  // bits of the ring vectors this thread read
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
  const int nfull = my_nv / kChunkVec;
  const int last_nv = my_nv - nfull * kChunkVec;
  const int nch = nfull + (last_nv > 0);
  const bool tail_owner = crank == CL - 1;
  const int n_tail = (int)(a.V - a.nvec * EPV);
  const int64_t row_bytes = a.ld * elem_bytes<T>();
  const bool skip_masked = (a.kn.flags & RL_F_SKIP_MASKED_READS) != 0;
  const float k = a.kn.inv_t * RL_LOG2E;

  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], kNcw * sm100::kRelPerWarp);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&sh.xbar[i], 1);
      sm100::mbar_init(&sh.resbar[i], 1);
    }
    for (int i = 0; i < 4; ++i) sm100::mbar_init(&sh.refbar[i], 1);
    sm100::fence_mbar_init();
  }
  sm100::cluster_sync();

  if (warp == kNcw) {
    if (lane == 0 && nch > 0) {
      // ---------------------------------------------------------- TMA producer (lane 0)
      // a row is read iff it has an in-range target (and, under SKIP_MASKED_READS, is valid):
      // the same predicate the service lane publishes as need_p.
      auto need_of = [&](int64_t row) -> bool {
        const RowMeta mt = row_meta(row, a.V, a.targets, a.mask, a.token_seq, a.seq_version,
                                    a.kn.trainer_version, a.kn.max_staleness);
        return mt.in_range && !(skip_masked && !mt.valid);
      };
      RingPos rp{0, 0};
      bool need = cid < a.n_tokens && need_of(cid);
      uint32_t pp = 0;
      for (int64_t row = cid; row < a.n_tokens; row += ncl, ++pp) {
        const int64_t nx = row + ncl;
        const int32_t y_nx = nx < a.n_tokens ? a.targets[nx] : -1;  // load in flight during the row
        if (need) {
          const char* src = reinterpret_cast<const char*>(a.logits) + row * row_bytes + v0 * 16;
          for (int c = 0; c * VPT < nch; ++c) {  // one bulk copy of VPT x 7.5 KB per ring slot
            sm100::mbar_wait_a(empty_s + rp.slot * 8, rp.phase ^ 1);
            const uint32_t bytes = (uint32_t)min(VPT * kChunkVec, my_nv - c * VPT * kChunkVec) * 16u;
            sm100::mbar_arrive_expect_tx(&full[rp.slot], bytes);
            sm100::bulk_g2s_nohint(ring + (size_t)rp.slot * (VPT * kChunkVec), src + (size_t)c * VPT * kChunkBytes,
                                   bytes, &full[rp.slot]);
            rp.advance(1, nslots);
          }
        }
        need = nx < a.n_tokens && (skip_masked ? need_of(nx) : (y_nx >= 0 && (int64_t)y_nx < a.V));
      }
    } else if (lane == 1) {
      // ---------------------------------------------------------- service lane (lane 1)
      // Row metadata two rows ahead (ref), and — off the consumers' critical path — each row's
      // statistics, logp, clip flag and redo flag from the record consumer thread 0 posts.
      const double inv_tm = token_mean_inv(a.kn);
      Acc acc;
      acc.zero();
      struct Pre {
        RowMeta mt;
        float xk, A, old, prox, ref;
        double w;
        bool need, owned;
      };
      auto fetch = [&](int64_t row) {
        Pre r;
        r.mt = row_meta(row, a.V, a.targets, a.mask, a.token_seq, a.seq_version, a.kn.trainer_version,
                        a.kn.max_staleness);
        r.need = r.mt.in_range && !(skip_masked && !r.mt.valid);
        r.xk = 0.f;
        r.owned = false;
        if (r.need) {
          r.xk = VecTraits<T>::load1(reinterpret_cast<const char*>(a.logits) + row * row_bytes, r.mt.y) * k;
          const int64_t vy = r.mt.y / EPV;
          r.owned = (vy >= v0 && vy < v1) || (tail_owner && vy >= a.nvec);
        }
        r.A = r.mt.valid ? a.seq_adv[r.mt.seq] : 0.f;
        r.old = r.mt.valid ? a.old_logp[row] : 0.f;
        r.w = r.mt.valid ? token_weight(r.mt, a.seq_active, inv_tm, a.kn) : 0.0;
        r.prox = r.old;
        r.ref = 0.f;
        if (EXT) token_extra(a.kn, row, r.old, r.prox, r.ref);
        return r;
      };
      auto publish_ref = [&](uint32_t p, const Pre& r) {
        sh.refa[p & 3] = make_float4(kCacheShift - r.xk, r.A, r.old, (float)r.w);
        if (EXT) sh.refc[p & 3] = make_float4(r.prox, r.ref, 0.f, 0.f);
        sh.refb[p & 3] = make_int4((r.need ? 1 : 0) | (r.mt.valid ? 2 : 0), r.owned ? r.mt.y : -1, 0, 0);
        sm100::mbar_arrive(&sh.refbar[p & 3]);
      };
      if (cid < a.n_tokens) {
        Pre cur = fetch(cid), nxt;
        publish_ref(0, cur);
        if (cid + ncl < a.n_tokens) {
          nxt = fetch(cid + ncl);
          publish_ref(1, nxt);
        }
        uint32_t p = 0;
        for (int64_t row = cid; row < a.n_tokens; row += ncl, ++p) {
          sm100::mbar_wait_polite(&sh.resbar[p & 1], (p >> 1) & 1, false);
          const float4 rs = sh.res[p & 1];
          const float S = rs.x;
          const RowMeta& mt = cur.mt;
          const bool redo = cur.need && !(S < kSvRedo);
          if (crank == 0) {
            a.redo[row] = redo ? 1 : 0;
            if (!redo) {
              const float lp = cur.need ? rs.y : (mt.in_range ? 0.f : logp_from(mt, 0.f, 0.f));
              uint8_t cl = 0;
              if (EXT) token_epilogue(mt, lp, cur.old, cur.A, a.seq_active, inv_tm, a.kn, acc, &cl, cur.prox, cur.ref);
              else token_epilogue_basic(mt, lp, cur.old, cur.A, a.seq_active, inv_tm, a.kn, acc, &cl);
              if (ENT && (a.kn.flags & RL_F_ENTROPY) && cur.need && mt.valid)  // H = lse - sum p z
                acc.v[ST_ENT] += (double)((cur.xk + fast_log2(S) - kCacheShift) * RL_LN2 - rs.z * a.kn.inv_t / S);
              if (a.logp_out) a.logp_out[row] = lp;
              if (a.clipped_out) a.clipped_out[row] = cl;
            }
          }
          // ref(p+2) goes to slot (p+2) % 4: row p's slot stays intact for its late readers
          const int64_t n2 = row + 2 * ncl;
          cur = nxt;
          if (n2 < a.n_tokens) {
            nxt = fetch(n2);
            publish_ref(p + 2, nxt);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < RL_LOSS_STATS_N; ++i)
        a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = crank == 0 ? acc.v[i] : 0.0;
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ consumer warps
    const uint64_t k2 = f2pack(k, k);
    const uint32_t my_off = (uint32_t)tid * 16u;
    const bool last_mine = tid < last_nv;
    // EXACT shapes (V = 151936, 128256) have V % 8 == 0: no scalar tail columns
    const bool tail_mine = !EXACT && tail_owner && tid < n_tail;
    uint4 cache[NCH];  // bf16 e' of this thread's vectors of the current row
#pragma unroll
    for (int j = 0; j < NCH; ++j) cache[j] = make_uint4(0, 0, 0, 0);
    uint32_t slot = 0, rph = 0;
    float xt = 0.f;  // e' of this thread's scalar tail column (V % EPV != 0)
    // row p-1's gradient (set by the exchange at the end of iteration p-1)
    uint32_t mode = SV_NONE, qb2 = 0, ql2 = 0;  // q split into bf16 hi + lo (ClVec::grad_sv)
    float q = 0.f, dy = 0.f;
    int ycol = -1;
#define RL_PRESENT(j) (EXACT ? true : ((j) < nch))
#define RL_PARTIAL(j) (EXACT ? ((j) == NCH - 1 && last_nv > 0) : ((j) == nfull))
#define RL_MINE(j) (!RL_PARTIAL(j) || last_mine)
#define RL_CHUNK_END(j) ((j) % VPT == VPT - 1 || (EXACT ? (j) == NCH - 1 : (j) == nch - 1))
    int64_t row = cid;
    for (uint32_t p = 0;; ++p, row += ncl) {
      const bool has_row = row < a.n_tokens;
      if (!has_row && p == 0) break;
      const uint32_t b = p & 1;
      bool need = false;
      float mn = 0.f;
      const uint32_t q4 = p & 3;
      if (has_row) {
        sm100::mbar_wait(&sh.refbar[q4], (p >> 2) & 1);
        need = (sh.refb[q4].x & 1) != 0;
        mn = sh.refa[q4].x;
      }
      const uint64_t mn2 = f2pack(mn, mn);
      const bool stores = mode != SV_NONE;
      char* dp = reinterpret_cast<char*>(a.dlogits) + (row - ncl) * row_bytes;  // row p-1
      uint4* out = reinterpret_cast<uint4*>(dp) + v0 + tid;
      float x_tail = -INFINITY;
      if (need && tail_mine)
        x_tail = VecTraits<T>::load1(reinterpret_cast<const char*>(a.logits) + row * row_bytes, a.nvec * EPV + tid);
      uint64_t acc2 = f2pack(0.f, 0.f), accx = f2pack(0.f, 0.f);
      // one pass over the chunks: dlogits of row p-1 out of cache[j] (predicated store; a row
      // with s = 0 has q = 0 and a finite cache -> exact zeros), row p's chunk j into cache[j]
      auto chunk_loop = [&](auto need_c) {
        const bool NEED = decltype(need_c)::value == 2 ? need : decltype(need_c)::value == 1;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          if (RL_PRESENT(j)) {
            RL_DCHECK(!(stores && RL_MINE(j)) ||
                      (row - ncl >= 0 && row - ncl < a.n_tokens && v0 + tid + j * kChunkVec < a.nvec));
            st_stream_v4_if(out + j * kChunkVec, ClVec<T>::grad_sv(cache[j], qb2, ql2, q),
                            stores && RL_MINE(j));
            if (NEED) {
              RL_DCHECK(slot < (uint32_t)nslots && row < a.n_tokens);
              if (j % VPT == 0) sm100::mbar_wait_a(full_s + slot * 8, rph);
              const uint4 v = sm100::lds128_a(ring_s + slot * (uint32_t)(VPT * kChunkBytes) + (j % VPT) * kChunkBytes + my_off);
              dep ^= v.x;
              if (ENT) {
                uint64_t nx = accx;
                const uint64_t nacc = ClVec<T>::exp_sv_ent(v, k2, mn2, acc2, nx, cache[j]);
                acc2 = RL_MINE(j) ? nacc : acc2;
                accx = RL_MINE(j) ? nx : accx;
              } else if (EXACT && j < NCH - 1) {
                acc2 = ClVec<T>::exp_sv(v, k2, mn2, acc2, cache[j]);
              } else {
                const uint64_t nacc = ClVec<T>::exp_sv(v, k2, mn2, acc2, cache[j]);
                acc2 = RL_MINE(j) ? nacc : acc2;
              }
              // release the slot after the chunk's arithmetic consumed its data (no extra stall)
              if (RL_CHUNK_END(j)) sm100::mbar_release_after(empty_s + slot * 8, dep, rt_zero);
              if (RL_CHUNK_END(j) && ++slot == (uint32_t)nslots) {
                slot = 0;
                rph ^= 1u;
              }
            } else {
              cache[j] = make_uint4(0, 0, 0, 0);  // an unread row writes zeros next iteration
            }
          }
        }
      };
      chunk_loop(std::integral_constant<int, 2>{});  // runtime need (one loop body: no spills)
      if (tail_mine) {
        RL_DCHECK(!stores || (a.nvec * EPV + tid < a.V && row - ncl < a.n_tokens));
        if (stores) VecTraits<T>::store1(dp, a.nvec * EPV + tid, xt * q);
        xt = 0.f;
        if (need) {
          xt = fast_exp2(fmaf(x_tail, k, mn));
          acc2 = fadd2(acc2, f2pack(xt, 0.f));
          if (ENT) accx = fadd2(accx, f2pack(xt * x_tail, 0.f));
        }
      }
      // target column of row p-1: rewritten by the thread that stored its vector (or tail
      // column) above — same-thread program order to the same address.
      if (mode == SV_GRAD && ycol >= 0) {
        const bool in_tail = ycol >= a.nvec * EPV;
        const int owner = in_tail ? (int)(ycol - a.nvec * EPV) : (int)((ycol / EPV - v0) % kChunkVec);
        RL_DCHECK(tid != owner || (ycol < a.V && row - ncl >= 0 && row - ncl < a.n_tokens));
        if (tid == owner) VecTraits<T>::store1(dp, ycol, dy);
      }
      if (!has_row) break;
      // ---- exchange of row p: CTA sum (named barrier), cluster sum (st.async), row scale
      {
        float s0, s1;
        f2unpack(acc2, s0, s1);
        const float ws = warp_sum(s0 + s1);
        if (lane == 0) sh.red_sum[b][warp] = ws;
        if (ENT) {
          f2unpack(accx, s0, s1);
          const float wx = warp_sum(s0 + s1);
          if (lane == 0) sh.red_ent[b][warp] = wx;
        }
      }
      sm100::named_bar_sync(1, kCons);
      float Sc = 0.f, Tc = 0.f;
#pragma unroll
      for (int w = 0; w < kNcw; ++w) Sc += sh.red_sum[b][w];
      if (ENT && tid == 0)
        for (int w = 0; w < kNcw; ++w) Tc += sh.red_ent[b][w];
      if (CL > 1) {
        if (tid == 0) {
          sm100::mbar_arrive_expect_tx(&sh.xbar[b], 16u * (CL - 1));
#pragma unroll
          for (int r = 0; r < CL; ++r)
            if (r != (int)crank) sm100::st_async_v4(&sh.xch[b][crank], &sh.xbar[b], r, Sc, Tc, 0.f, 0.f);
        }
        // the peer's st.async completes THIS CTA's barrier (async proxy, like a TMA load): a
        // CTA-scope wait makes its bytes visible — no cluster-scope acquire (an L1 invalidate)
        sm100::mbar_wait_cluster(&sh.xbar[b], (p >> 1) & 1);
      }
      float S = 0.f, Tx = 0.f;  // rank order: bitwise identical in every CTA of the cluster
#pragma unroll
      for (int r = 0; r < CL; ++r) S += r == (int)crank ? Sc : sh.xch[b][r].x;
      if (ENT && tid == 0)
        for (int r = 0; r < CL; ++r) Tx += r == (int)crank ? Tc : sh.xch[b][r].y;
      const float4 ra = sh.refa[q4];
      const float4 rc = EXT ? sh.refc[q4] : make_float4(ra.z, 0.f, 0.f, 0.f);
      const int4 rb = sh.refb[q4];
      const bool valid = (rb.x & 2) != 0;
      const bool redo = need && !(S < kSvRedo);
      const float lp = need ? (kCacheShift - fast_log2(S)) * RL_LN2 : 0.f;  // ln(2^15 / S')
      float st = 0.f;
      if (valid && !redo) {
        if (EXT) st = token_scale(token_ratio(lp, ra.z, rc.x, rc.y, ra.y, a.kn), ra.w, ra.y, a.kn);
        else st = token_scale_basic(token_ratio_basic(lp, ra.z, ra.y, a.kn), ra.w, ra.y, a.kn);
      }
      mode = redo ? SV_NONE : (st == 0.f ? SV_ZERO : SV_GRAD);
      const float inv_s = 1.f / S;
      q = st == 0.f ? 0.f : st * inv_s;  // (an unread row has S' = 0)
      dy = st == 0.f ? 0.f : st * (32768.f * inv_s - 1.f);  // p_y = e'_y / S' = 2^15 / S'
      qb2 = pack_bf16x2(q, q);
      {
        const float qh = __uint_as_float(qb2 << 16);
        ql2 = pack_bf16x2(q - qh, q - qh);
      }
      ycol = rb.y;
      if (tid == 0) {
        sh.res[b] = make_float4(S, lp, Tx, 0.f);
        sm100::mbar_arrive(&sh.resbar[b]);
      }
    }
#undef RL_PRESENT
#undef RL_PARTIAL
#undef RL_MINE
#undef RL_CHUNK_END
  }
  __syncwarp();
  sm100::cluster_sync();  // no CTA leaves while a peer may still write its smem
}

template <typename T, int CL, int NCH, bool EXACT = false, int VPT = 4, int XF = 0>
static rl_status launch_sv(const ClArgs& a0, int64_t n, cudaStream_t s, int* n_ctas) {
  ClArgs a = a0;
  auto kern = loss_sv_kernel<T, CL, NCH, EXACT, VPT, XF>;
  const size_t head = (sizeof(SvShared) + 127) & ~(size_t)127;
  constexpr size_t slot_bytes = (size_t)VPT * kChunkBytes;
  const int nslots = (int)((kSmemMax - head - 256) / (slot_bytes + 16));
  const int nch = (int)((a.h_vec + kChunkVec - 1) / kChunkVec);
  if (nch > NCH || (EXACT && nch != NCH)) return RL_ERR_UNSUPPORTED;
  a.nslots = nslots;
  const size_t smem = ((sizeof(SvShared) + 2 * sizeof(uint64_t) * nslots + 127) & ~(size_t)127) +
                      (size_t)nslots * slot_bytes;
  // the >48 KB opt-in is per device and cheap: set it on every launch
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(max dynamic smem)");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kSvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_clusters_tab[kMaxDevices] = {};
  int& max_clusters = dev_slot(max_clusters_tab);
  if (!max_clusters) {
    const int sms = dev_info().sms;
    cfg.gridDim = dim3(sms / CL * CL);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = sms / CL;
    }
    max_clusters = mc;
  }
  const int64_t ncl = std::min<int64_t>(std::min<int64_t>(n, max_clusters), kMaxStatCtas / 2 / CL);
  cfg.gridDim = dim3((unsigned)(ncl * CL));
  *n_ctas = (int)(ncl * CL);
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return check_launch("loss_sv_kernel");
  return check_launch("loss_sv_kernel");
}

rl_status launch_loss_sv(const void* logits, int32_t dtype, int64_t n, int64_t V, int64_t ld,
                         const int32_t* targets, const float* old_logp, const uint8_t* mask,
                         const int32_t* token_seq, const float* seq_adv, const int32_t* seq_version,
                         const int32_t* seq_active, const Knobs& kn, void* dlogits, float* logp_out,
                         uint8_t* clipped_out, double* partials, uint8_t* redo, int* n_ctas,
                         cudaStream_t s) {
  ClArgs a;
  a.logits = logits;
  a.dlogits = dlogits;
  a.n_tokens = n;
  a.V = V;
  a.ld = ld;
  const bool bf = dtype == RL_BF16;
  a.nvec = V / (bf ? 8 : 4);
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
  a.redo = redo;
  a.kn = kn;
  a.nslots = 0;
  auto nchunks = [&](int64_t h) { return (h + kChunkVec - 1) / kChunkVec; };
  a.h_vec = (a.nvec + 1) / 2;
  const int64_t nch2 = nchunks(a.h_vec);
  // The EXACT instantiations (V = 151936, 128256: 20 / 17 chunks per CTA) carry no scalar tail
  // code, so they are taken only when V has no tail columns (V % 8 == 0); a vocabulary of the
  // same width with a tail (e.g. 151665 in a 151936-wide buffer) takes the general instantiation.
  const bool exact_ok = bf && V % 8 == 0;
  const int xf = ((kn.flags & RL_F_ENTROPY) ? 1 : 0) | ((kn.kl_coef != 0.f || kn.prox_logp) ? 2 : 0);
  if (xf) {  // NEXT-2 terms: compile-time variants of the hot shapes, the general one otherwise
#define RL_SV_XF(X)                                                                                      \
    if (xf == X && exact_ok) {                                                                           \
      if (nch2 == 20) return launch_sv<bf16_t, 2, 20, true, 4, X>(a, n, s, n_ctas);                      \
      if (nch2 == 17) return launch_sv<bf16_t, 2, 17, true, 4, X>(a, n, s, n_ctas);                      \
    }
    RL_SV_XF(1) RL_SV_XF(2) RL_SV_XF(3)
#undef RL_SV_XF
    if (nch2 <= 20)
      return bf ? launch_sv<bf16_t, 2, 20, false, 4, 3>(a, n, s, n_ctas)
                : launch_sv<float, 2, 20, false, 4, 3>(a, n, s, n_ctas);
    return RL_ERR_UNSUPPORTED;  // very wide rows: the two-pass kernel computes them
  }
  if (exact_ok && nch2 == 20) return launch_sv<bf16_t, 2, 20, true>(a, n, s, n_ctas);  // V = 151936
  if (exact_ok && nch2 == 17) return launch_sv<bf16_t, 2, 17, true>(a, n, s, n_ctas);  // V = 128256
  if (nch2 <= 2) return bf ? launch_sv<bf16_t, 2, 2>(a, n, s, n_ctas) : launch_sv<float, 2, 2>(a, n, s, n_ctas);
  if (nch2 <= 5) return bf ? launch_sv<bf16_t, 2, 5>(a, n, s, n_ctas) : launch_sv<float, 2, 5>(a, n, s, n_ctas);
  if (nch2 <= 10) return bf ? launch_sv<bf16_t, 2, 10>(a, n, s, n_ctas) : launch_sv<float, 2, 10>(a, n, s, n_ctas);
  if (nch2 <= 20) return bf ? launch_sv<bf16_t, 2, 20>(a, n, s, n_ctas) : launch_sv<float, 2, 20>(a, n, s, n_ctas);
  a.h_vec = (a.nvec + 3) / 4;
  return bf ? launch_sv<bf16_t, 4, 20>(a, n, s, n_ctas) : launch_sv<float, 4, 20>(a, n, s, n_ctas);
}

}  // namespace rl
