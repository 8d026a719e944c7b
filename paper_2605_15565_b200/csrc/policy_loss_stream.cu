// Streaming row-resident loss kernel "S": the variant that never waits on the
// cluster exchange.
//
// Like the cluster kernel, a 2-CTA cluster owns each row (half the columns per CTA) and logits
// arrive by TMA bulk copies into a shared-memory ring.  Differences:
//  * single visit per chunk: when chunk j lands, each consumer warp takes the warp max of its
//    values (redux.sync), raises its running reference R (rescaling its partial sum on the rare
//    raise), caches e' = 2^(x k - R + 15) as fp16 and releases the ring slot immediately;
//  * TWO row caches: even rows cache e' in registers (20 x 16 B per thread), odd rows in shared
//    memory (150 KB), so the exp pass of row i+1 runs while the cluster exchange of row i is in
//    flight and pass C of row i (stores) is fused with the exp pass of row i+2;
//  * warp 15 is a service warp running one non-blocking event loop: TMA issue for free ring slots
//    (lane 0) and the per-row epilogue (warp-parallel combine of the 15 warps' partial sums,
//    DSMEM exchange, ratio/clip/scale, statistics, scalar tail columns).
// HBM traffic: logits read once, dlogits written once.  dlogits may alias logits.
#include <cstdlib>
#include <cstring>
#include <algorithm>

#include "cluster_common.cuh"

namespace rl {

struct __align__(16) StShared {
  float4 xch[2][8];        // [row parity][cluster rank]: (m_c log2 units, s_c, z_y, owned)
  float red_sum[2][kNcw];  // [row parity][warp] sum of e' in the warp's frame (2^15-scaled)
  float red_R[2][kNcw];    // [row parity][warp] the warp's final reference max R_w (log2)
  float4 row_sc[2];        // [row parity] (s_t, lse2, d_y, target column as int bits or -1)
  uint64_t xbar[2];        // peer records landed (CL - 1 remote arrivals)
  uint64_t sumbar[2];      // consumers finished the row's exp pass (kNcw arrivals)
  uint64_t scalebar[2];    // epilogue published row_sc (1 arrival)
  // followed by full[nslots], empty[nslots] (uint64); then (128-B aligned) the shared-memory row
  // cache [NCH][kCons] x 16 B and the ring [nslots][kCons] x 16 B
};

__device__ __forceinline__ bool mbar_test_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test_cluster_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void sts128_a(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

constexpr int kStCL = 2;

template <typename T, int NCH, bool EXACT, bool DUAL>
__global__ void __launch_bounds__(kClThreads, 1) loss_stream_kernel(const ClArgs a) {
  static_assert(NCH <= 32, "chunk references live in one lane each");
  constexpr int CL = kStCL;
  constexpr int EPV = ClVec<T>::EPV;
  using MaxT = typename ClVec<T>::MaxT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StShared& sh = *reinterpret_cast<StShared*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + sizeof(StShared));
  uint64_t* empty = full + a.nslots;
  const size_t cache_off = (sizeof(StShared) + 2 * sizeof(uint64_t) * a.nslots + 127) & ~(size_t)127;
  const size_t ring_off = cache_off + (DUAL ? (size_t)NCH * kChunkBytes : 0);
  uint4* ring = reinterpret_cast<uint4*>(smem_raw + ring_off);
  const int nslots = a.nslots;
  const uint32_t full_s = sm100::smem_u32(full), empty_s = sm100::smem_u32(empty);
  const uint32_t ring_s = sm100::smem_u32(ring);
  const uint32_t scache_s = sm100::smem_u32(smem_raw + cache_off);

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
  const float k = a.kn.inv_t * RL_LOG2E;
  const int64_t nrows = cid < a.n_tokens ? (a.n_tokens - 1 - cid) / ncl + 1 : 0;  // rows cid + t ncl
  const int64_t total_chunks = nrows * nch;

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
    // ------------------------------------------------------------ service warp: event loop
    const uint64_t pol = policy_evict_first();
    const double inv_tm = token_mean_inv(a.kn);
    Acc acc;
    acc.zero();
    int64_t g_issue = 0, g_row = 0;  // next chunk to issue: row ordinal g_row, chunk g_j
    int g_j = 0;
    RingPos ip{0, 0};
    int64_t t = 0;  // row ordinal of the epilogue
    int stage = 0;  // 0: waiting for the consumers' sums, 1: waiting for the peer records
    // per-row epilogue state (lane 0 unless noted)
    RowMeta mt;
    float A = 0.f, old = 0.f, zy = 0.f, xt = -INFINITY;
    bool owned = false, loaded = false;
    while (t < nrows || g_issue < total_chunks) {
      // ---- TMA issue (lane 0): every free ring slot gets its next chunk
      if (lane == 0) {
        while (g_issue < total_chunks && mbar_test_a(empty_s + ip.slot * 8, ip.phase ^ 1)) {
          const char* src = reinterpret_cast<const char*>(a.logits) + (cid + g_row * ncl) * row_bytes + v0 * 16 +
                            (size_t)g_j * kChunkBytes;
          const uint32_t bytes = (g_j < nfull ? kChunkVec : last_nv) * 16u;
          sm100::mbar_arrive_expect_tx(&full[ip.slot], bytes);
          sm100::bulk_g2s(ring + (size_t)ip.slot * kChunkVec, src, bytes, &full[ip.slot], pol);
          ip.advance(1, nslots);
          ++g_issue;
          if (++g_j == nch) {
            g_j = 0;
            ++g_row;
          }
        }
      }
      g_issue = __shfl_sync(0xffffffffu, g_issue, 0);
      if (t >= nrows) continue;
      const int64_t row = cid + t * ncl;
      const int par = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      const char* rp = reinterpret_cast<const char*>(a.logits) + row * row_bytes;
      if (!loaded) {  // row scalars (and the tail columns, read before any write of the row)
        if (lane == 0) {
          mt = row_meta(row, a.V, a.targets, a.mask, a.token_seq, a.seq_version, a.kn.trainer_version,
                        a.kn.max_staleness);
          A = mt.valid ? a.seq_adv[mt.seq] : 0.f;
          old = mt.valid ? a.old_logp[row] : 0.f;
          owned = false;
          zy = 0.f;
          if (mt.in_range) {
            const int64_t vy = mt.y / EPV;
            owned = (vy >= v0 && vy < v1) || (tail_owner && vy >= a.nvec);
            if (owned) zy = VecTraits<T>::load1(rp, mt.y) * a.kn.inv_t;
          }
        }
        xt = -INFINITY;
        if (tail_owner && lane >= kNcw && lane < kNcw + n_tail)
          xt = VecTraits<T>::load1(rp, a.nvec * EPV + (lane - kNcw)) * k;
        loaded = true;
      }
      const bool tail_lane = tail_owner && lane >= kNcw && lane < kNcw + n_tail;
      if (stage == 0) {
        const bool ready = __shfl_sync(0xffffffffu, mbar_test_a(sm100::smem_u32(&sh.sumbar[par]), ph) ? 1 : 0, 0);
        if (!ready) continue;
        // slice (m_c, s_c): lanes 0..14 carry the consumer warps' (R_w, sum_w), lanes 15.. the tail
        float Rw = -INFINITY, Sw = 0.f;
        if (lane < kNcw) {
          Rw = sh.red_R[par][lane];
          Sw = sh.red_sum[par][lane];
        } else if (tail_lane) {
          Rw = xt;
          Sw = 32768.f;  // one element at its own reference, in the 2^15-scaled frame
        }
        float m;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(Rw));
        const float s = warp_sum((Rw != -INFINITY) ? Sw * fast_exp2(Rw - m - kCacheShift) : 0.f);
        if (lane == 0) {
          const float4 rec = make_float4(m, s, owned ? zy : 0.f, owned ? 1.f : 0.f);
          sh.xch[par][crank] = rec;
#pragma unroll
          for (int r = 0; r < CL; ++r)
            if (r != (int)crank) {
              sm100::st_remote_v4(&sh.xch[par][crank], r, rec.x, rec.y, rec.z, rec.w);
              sm100::mbar_arrive_remote(&sh.xbar[par], r);
            }
        }
        stage = 1;
      }
      if (stage == 1) {
        const bool ready =
            __shfl_sync(0xffffffffu, mbar_test_cluster_a(sm100::smem_u32(&sh.xbar[par]), ph) ? 1 : 0, 0);
        if (!ready) continue;
        float st = 0.f, c2 = 0.f, dy = 0.f;
        int ycol = -1;
        if (lane == 0) {
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
          c2 = M + fast_log2(S);
          const float lp = logp_from(mt, z, c2);
          uint8_t cl = 0;
          Acc tmp;
          tmp.zero();
          st = token_epilogue(mt, lp, old, A, a.seq_active, inv_tm, a.kn, tmp, &cl);
          if (crank == 0) {
#pragma unroll
            for (int i = 0; i < RL_LOSS_STATS_N; ++i) acc.v[i] += tmp.v[i];
            if (a.logp_out) a.logp_out[row] = lp;
            if (a.clipped_out) a.clipped_out[row] = cl;
          }
          dy = st * (fast_exp2(z * RL_LOG2E - c2) - 1.f);  // target column: s_t (p_y - 1)
          ycol = owned ? mt.y : -1;
          sh.row_sc[par] = make_float4(st, c2, dy, __int_as_float(ycol));
          sm100::mbar_arrive(&sh.scalebar[par]);
        }
        if (tail_owner && n_tail > 0) {  // the tail columns' gradient (their owner lanes)
          st = __shfl_sync(0xffffffffu, st, 0);
          c2 = __shfl_sync(0xffffffffu, c2, 0);
          dy = __shfl_sync(0xffffffffu, dy, 0);
          ycol = __shfl_sync(0xffffffffu, ycol, 0);
          if (tail_lane) {
            char* dp = reinterpret_cast<char*>(a.dlogits) + row * row_bytes;
            const int64_t col = a.nvec * EPV + (lane - kNcw);
            const float o = (st == 0.f) ? 0.f : (col == ycol ? dy : st * fast_exp2(xt - c2));
            VecTraits<T>::store1(dp, col, o);
          }
        }
        stage = 0;
        loaded = false;
        ++t;
      }
    }
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < RL_LOSS_STATS_N; ++i)
        a.partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = crank == 0 ? acc.v[i] : 0.0;
  } else {
    // ------------------------------------------------------------ consumer warps
    const uint64_t k2 = f2pack(k, k);
    const uint32_t my_off = (uint32_t)tid * 16u;
    const bool last_mine = tid < last_nv;  // this thread's vector exists in the partial last chunk
    uint4 cache[NCH];  // register row cache (even row ordinals); odd ones live in shared memory
    float rr[2];       // lane j of rr[b]: the warp's reference R used for chunk j of the row in cache b
    rr[0] = rr[1] = -INFINITY;
    RingPos pos{0, 0};
#define RL_PRESENT(j) (EXACT ? true : ((j) < nch))
#define RL_PARTIAL(j) (EXACT ? ((j) == NCH - 1 && last_nv > 0) : ((j) == nfull))
#define RL_MINE(j) (!RL_PARTIAL(j) || last_mine)

    // exp pass of one chunk (state: running reference R, packed partial sum acc2, mn2 = 15 - R)
    float R = -INFINITY;
    uint64_t acc2 = 0, mn2 = 0;
    // fetch: wait for the chunk, read this thread's vector, release the slot (ring order)
    auto fetch = [&](uint32_t& slot, uint32_t& ph) -> uint4 {
      sm100::mbar_wait_a(full_s + slot * 8, ph);
      const uint4 v = sm100::lds128_a(ring_s + slot * (uint32_t)kChunkBytes + my_off);
      sm100::mbar_arrive_lane0(empty_s + slot * 8, lane);  // data is in registers: slot free
      if (++slot == (uint32_t)nslots) {
        slot = 0;
        ph ^= 1u;
      }
      return v;
    };
    // compute: warp max -> running reference -> e' (fp16 cache word) and partial sum
    auto compute = [&](int j, const uint4& v, bool mine, uint4& cj, float& rrb) {
      MaxT mv = ClVec<T>::max_init();
      ClVec<T>::max_acc(v, mv);
      float wm = mine ? ClVec<T>::max_to_float(mv) : -INFINITY;
      asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(wm) : "f"(wm));
      const float Rn = fmaxf(R, wm * k);
      if (Rn > R) {  // warp-uniform, rare after the first chunks
        if (R != -INFINITY) {
          const float f = fast_exp2(R - Rn);
          acc2 = fmul2(acc2, f2pack(f, f));
        }
        R = Rn;
        mn2 = f2pack(kCacheShift - R, kCacheShift - R);
      }
      if (R != -INFINITY) {
        const uint64_t nacc = ClVec<T>::exp_cache(v, k2, mn2, acc2, cj);
        acc2 = mine ? nacc : acc2;
      } else {
        cj = make_uint4(0, 0, 0, 0);
      }
      rrb = (lane == j) ? R : rrb;
    };
    auto finish_row = [&](int64_t tr) {
      float s0, s1;
      f2unpack(acc2, s0, s1);
      const float sum = warp_sum(s0 + s1);
      if (lane == 0) {
        sh.red_sum[tr & 1][warp] = sum;
        sh.red_R[tr & 1][warp] = R;
        sm100::mbar_arrive(&sh.sumbar[tr & 1]);
      }
    };
    auto scache = [&](int j) { return scache_s + (uint32_t)j * (uint32_t)kChunkBytes + my_off; };
    // full exp pass of row ordinal tr into cache b (prologue); chunk j+1 is fetched before chunk
    // j is computed so its shared-memory latency overlaps the math
    auto exp_row = [&](int b, int64_t tr) {
      R = -INFINITY;
      acc2 = f2pack(0.f, 0.f);
      uint32_t slot = pos.slot, ph = pos.phase;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        if (RL_PRESENT(j)) {
          const uint4 vcur = fetch(slot, ph);
          if (b == 0) {
            compute(j, vcur, RL_MINE(j), cache[j], rr[0]);
          } else {
            uint4 cv;
            compute(j, vcur, RL_MINE(j), cv, rr[1]);
            sts128_a(scache(j), cv);
          }
        }
      pos.slot = slot;
      pos.phase = ph;
      finish_row(tr);
    };
    // pass C of row ordinal tr from cache b, fused with the exp pass of row tr + NB into cache b
    constexpr int NB = DUAL ? 2 : 1;
    auto fused = [&](int b, int64_t tr, bool has_e) {
      sm100::mbar_wait(&sh.scalebar[tr & 1], (tr >> 1) & 1);
      const float4 sc = sh.row_sc[tr & 1];
      const float st = sc.x, c2 = sc.y, dy = sc.z;
      const int ycol = __float_as_int(sc.w);
      char* dp = reinterpret_cast<char*>(a.dlogits) + (cid + tr * ncl) * row_bytes;
      uint4* out = reinterpret_cast<uint4*>(dp) + v0 + tid;
      R = -INFINITY;
      acc2 = f2pack(0.f, 0.f);
      uint32_t slot = pos.slot, ph = pos.phase;
      float Rq = __int_as_float(0x7fc00000);  // reference of the cached q (NaN: none yet)
      uint64_t q2 = 0;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        if (RL_PRESENT(j)) {
          uint4 vcur = make_uint4(0, 0, 0, 0);
          if (has_e) vcur = fetch(slot, ph);
          const float Rj = __shfl_sync(0xffffffffu, rr[b], j);
          if (Rj != Rq) {  // warp-uniform; the reference changes a few times per row
            Rq = Rj;
            const float q = (st == 0.f || Rj == -INFINITY) ? 0.f : st * fast_exp2(Rj - kCacheShift - c2);
            q2 = f2pack(q, q);
          }
          if (b == 0) {
            if (RL_MINE(j)) st_stream_v4(out + j * kChunkVec, ClVec<T>::grad(cache[j], q2));
            if (has_e) compute(j, vcur, RL_MINE(j), cache[j], rr[0]);
          } else {
            if (RL_MINE(j)) st_stream_v4(out + j * kChunkVec, ClVec<T>::grad(sm100::lds128_a(scache(j)), q2));
            if (has_e) {
              uint4 cv;
              compute(j, vcur, RL_MINE(j), cv, rr[1]);
              sts128_a(scache(j), cv);
            }
          }
        }
      }
      // target column: rewritten by the thread that stored its vector above — same-thread
      // program order to the same address (tail columns are the service warp's).
      if (st != 0.f && ycol >= 0 && ycol < a.nvec * EPV) {
        const int owner = (int)((ycol / EPV - v0) % kChunkVec);
        if (tid == owner) VecTraits<T>::store1(dp, ycol, dy);
      }
      if (has_e) {
        pos.slot = slot;
        pos.phase = ph;
        finish_row(tr + NB);
      }
    };

    if (DUAL) {
      if (nrows > 0) exp_row(0, 0);
      if (nrows > 1) exp_row(1, 1);
      for (int64_t tr = 0; tr < nrows; tr += 2) {
        fused(0, tr, tr + 2 < nrows);
        if (tr + 1 < nrows) fused(1, tr + 1, tr + 3 < nrows);
      }
    } else {
      if (nrows > 0) exp_row(0, 0);
      for (int64_t tr = 0; tr < nrows; ++tr) fused(0, tr, tr + 1 < nrows);
    }
#undef RL_PRESENT
#undef RL_PARTIAL
#undef RL_MINE
  }
  __syncwarp();
  sm100::cluster_sync();  // no CTA leaves while a peer may still arrive on / write its smem
}

template <typename T, int NCH, bool EXACT, bool DUAL = true>
static rl_status launch_st(const ClArgs& a0, int64_t n, cudaStream_t s, int* n_ctas) {
  ClArgs a = a0;
  auto kern = loss_stream_kernel<T, NCH, EXACT, DUAL>;
  const int nch = (int)((a.h_vec + kChunkVec - 1) / kChunkVec);
  if (nch > NCH || (EXACT && nch != NCH)) return RL_ERR_UNSUPPORTED;
  const size_t head = (sizeof(StShared) + 127) & ~(size_t)127;
  const size_t cache = DUAL ? (size_t)NCH * kChunkBytes : 0;
  int nslots = (int)((kSmemMax - head - cache - 256) / (kChunkBytes + 16));
  static int slots_cap = -1;  // RL_STREAM_SLOTS: cap on the ring depth (fewer loads in flight)
  if (slots_cap < 0) slots_cap = getenv("RL_STREAM_SLOTS") ? atoi(getenv("RL_STREAM_SLOTS")) : 0;
  if (slots_cap > 0) nslots = std::min(nslots, std::max(slots_cap, 4));
  if (nslots < 4) return RL_ERR_UNSUPPORTED;
  a.nslots = nslots;
  const size_t smem = ((sizeof(StShared) + 2 * sizeof(uint64_t) * nslots + 127) & ~(size_t)127) + cache +
                      (size_t)nslots * kChunkBytes;
  (void)0;
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
  attr[0].val.clusterDim.x = kStCL;
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
    cfg.gridDim = dim3(sms / kStCL * kStCL);
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
      cudaGetLastError();
      max_clusters = sms / kStCL;
    }
  }
  const int64_t ncl = std::min<int64_t>(std::min<int64_t>(n, max_clusters), kMaxStatCtas / kStCL);
  cfg.gridDim = dim3((unsigned)(ncl * kStCL));
  *n_ctas = (int)(ncl * kStCL);
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return check_launch("loss_stream_kernel");
  return check_launch("loss_stream_kernel");
}

rl_status launch_loss_stream(const void* logits, int32_t dtype, int64_t n, int64_t V, int64_t ld,
                             const int32_t* targets, const float* old_logp, const uint8_t* mask,
                             const int32_t* token_seq, const float* seq_adv, const int32_t* seq_version,
                             const int32_t* seq_active, const Knobs& kn, void* dlogits, float* logp_out,
                             uint8_t* clipped_out, double* partials, int* n_ctas, cudaStream_t s) {
  if (kn.flags & RL_F_SKIP_MASKED_READS) return RL_ERR_UNSUPPORTED;
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
  a.prefetch_chunks = 0;
  a.debug = 0;
  a.inflight_cap = 0;
  a.h_vec = (a.nvec + 1) / 2;
  const int64_t c = (a.h_vec + kChunkVec - 1) / kChunkVec;
  const bool bf = dtype == RL_BF16;
  static int dual = -1;  // RL_STREAM_CACHE=single: one register row cache (exchange exposed)
  if (dual < 0) dual = (getenv("RL_STREAM_CACHE") && strcmp(getenv("RL_STREAM_CACHE"), "single") == 0) ? 0 : 1;
  if (bf && c == 20)
    return dual ? launch_st<bf16_t, 20, true, true>(a, n, s, n_ctas) : launch_st<bf16_t, 20, true, false>(a, n, s, n_ctas);
  if (c <= 2) return bf ? launch_st<bf16_t, 2, false>(a, n, s, n_ctas) : launch_st<float, 2, false>(a, n, s, n_ctas);
  if (c <= 5) return bf ? launch_st<bf16_t, 5, false>(a, n, s, n_ctas) : launch_st<float, 5, false>(a, n, s, n_ctas);
  if (c <= 10) return bf ? launch_st<bf16_t, 10, false>(a, n, s, n_ctas) : launch_st<float, 10, false>(a, n, s, n_ctas);
  if (c <= 20) return bf ? launch_st<bf16_t, 20, false>(a, n, s, n_ctas) : launch_st<float, 20, false>(a, n, s, n_ctas);
  return RL_ERR_UNSUPPORTED;
}

}  // namespace rl
