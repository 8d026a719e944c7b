// (8) Fused LM-head log-prob — NEXT 4 of SURVEY.md §8(f), forward half ("Fused LM-head GEMM +
// loss (tcgen05, logits never materialised) ... it takes hidden states and W").
//
// logp_t = x_{t,y} - lse_t with x = (h W^T) * inv_T (c3 of SURVEY.md §8(c) on the LM head's
// output), computed without writing the [N, V] logits: the logits tile lives only in TMEM.
//
// Per CTA: one block of kBM = 128 token rows against one range of vocabulary tiles of kBN = 256 rows
// of W (grid = (vocabulary splits, token blocks), split fastest; the split count is an L2 decision,
// lm_splits below; with several splits a combine kernel merges the per-split row records).
//   warp 0 (one lane)  TMA producer: 2-D tensor copies (128-B swizzle) of the hidden block's and
//                      the W tile's K-slices (64 bf16 = 128 B) into a kStages-deep smem ring
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M = 128, N = 256, K = 16,
//                      bf16 x bf16 -> fp32 in TMEM; two accumulators (2 x 256 TMEM columns) so
//                      the MMAs of vocabulary tile j+1 run while tile j is reduced
//   warps 2..5         epilogue: tcgen05.ld 32 columns at a time (thread = token row = TMEM
//                      lane), online (max, sum 2^(t - max)) over the row, the target logit picked
//                      with compile-time indices; after the last tile lse and logp are written
// The hidden block is re-read from L2 once per vocabulary tile; W streams from HBM / L2.
#include <cublas_v2.h>
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace rl {

constexpr int kLmBM = 128, kLmBN = 256, kLmBK = 64, kLmStages = 4;
// PAIR mode (cta_group::2): a cluster of two CTAs = 256 token rows x one 256-row W tile per MMA
// (M = 256); each CTA stages its own 128 token rows and HALF of the W tile (128 rows), so the W
// bytes per SM halve and six 32 KB stages fit where four 48 KB ones did
constexpr int kLmPairStages = 6;
constexpr uint32_t kLmPairBBytes = (kLmBN / 2) * kLmBK * 2;
constexpr int kLmThreads = 192;
constexpr uint32_t kLmABytes = kLmBM * kLmBK * 2, kLmBBytes = kLmBN * kLmBK * 2;
constexpr uint32_t kLmStageBytes = kLmABytes + kLmBBytes;  // 48 KB
constexpr size_t kLmSmem = (size_t)kLmStages * kLmStageBytes + 1024;

struct LmArgs {
  const int32_t* targets;
  int64_t n, V;
  int32_t kblocks, vtiles, tiles_per_split;
  float inv_t;
  float* logp_out;
  float* lse_out;
  float4* partial;  // [splits][n] (max2, sum, raw target logit, -) when gridDim.x > 1
  // gradient mode (lmhead_grad_kernel): G = s_t (softmax(x_t) - onehot(y_t)) written as bf16
  const float* lse;     // [n] natural-log lse of the forward (rl_lmhead_logprob)
  const float* scale;   // [n] s_t (rl_policy_loss_from_logp)
  uint16_t* g_out;      // [n, ld_g] bf16 bits
  int64_t ld_g;
  int32_t n_splits;     // PAIR launches: the split count (the grid is 1-D)
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sm100::smem_u32(bar))
      : "memory");
}
// K-major operand, 128-B swizzle (8-row groups of 1024 B), descriptor version 1 (sm100)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sm100::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t f2pack_lm(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack_lm(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2_lm(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fmul2_lm(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// instruction descriptor, kind::f16: D fp32 (bit 4), A bf16 (bits 7-9 = 1), B bf16 (bits 10-12 = 1),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kLmIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLmBN >> 3) << 17) |
                              ((uint32_t)(kLmBM >> 4) << 24);
constexpr uint32_t kLmPairIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kLmBN >> 3) << 17) |
                                  ((uint32_t)((2 * kLmBM) >> 4) << 24);

// PAIR-mode primitives: the MMA of the CTA pair (issued by the leader), its commit multicast to
// both CTAs' barrier at the same offset, and the TMA load whose completion lands on the LEADER's
// barrier (a shared::cluster address from mapa)
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   sm100::smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sm100::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}

// GRAD = false: the log-prob epilogue (online max / sum over the row's tiles, rl_lmhead_logprob).
// GRAD = true:  the gradient epilogue (rl_lmhead_loss_bwd): every logits tile is recomputed and
//               turned straight into G = s_t (2^(x k - lse2) - [v == y]) in bf16 (one rounding) —
//               the logits themselves are never written.
// PAIR: launched as clusters of (1, 2, 1) CTAs — consecutive token blocks share every W tile
template <bool GRAD, bool PAIR = false>
__global__ void __launch_bounds__(kLmThreads, 1)
    lmhead_kernel(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w,
                  const LmArgs a) {
  constexpr int STAGES = PAIR ? kLmPairStages : kLmStages;
  constexpr uint32_t BBYTES = PAIR ? kLmPairBBytes : kLmBBytes;
  constexpr uint32_t STAGE = kLmABytes + BBYTES;
  extern __shared__ uint8_t lm_smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  const uint32_t crank = PAIR ? sm100::cluster_ctarank() : 0;
  const bool leader = crank == 0;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = (sm100::smem_u32(lm_smem_raw) + 1023u) & ~1023u;
  // grid (splits, row blocks), split fastest: the CTAs resident together cover few token blocks, so
  // every hidden block re-read (once per vocabulary tile) is an L2 hit shared by its splits
  // PAIR: a 1-D grid of clusters (2, 1, 1), linear index = ((pair * splits + split) * 2 + rank), so
  // the split stays the fastest-varying index (the L2 order of the single-CTA grid) and the two CTAs
  // of a cluster are the pair's token blocks 2 pair and 2 pair + 1
  uint32_t split_idx = blockIdx.x;
  int64_t tblock = blockIdx.y;
  if (PAIR) {
    const uint32_t q = blockIdx.x >> 1;
    split_idx = q % (uint32_t)a.n_splits;
    tblock = (int64_t)(q / (uint32_t)a.n_splits) * 2 + (blockIdx.x & 1);
  }
  const int64_t m0 = tblock * kLmBM;
  // this CTA's vocabulary tiles [jt0, jt1) (split split_idx)
  const int jt0 = (int)split_idx * a.tiles_per_split;
  const int jt1 = min(a.vtiles, jt0 + a.tiles_per_split);
  const int ntiles = max(0, jt1 - jt0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      sm100::mbar_init(&full[i], PAIR ? 2 : 1);  // PAIR: the leader's full[] takes both producers
      sm100::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&acc_full[i], 1);
      sm100::mbar_init(&acc_empty[i], PAIR ? 8 : 4);  // PAIR: both CTAs' epilogue warps, at the leader
    }
    sm100::fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       sm100::smem_u32(&tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       sm100::smem_u32(&tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR) sm100::cluster_sync();  // the peer's barriers exist before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int total = ntiles * a.kblocks;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      for (int it = 0; it < total; ++it) {
        const int st = it % STAGES;
        const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
        sm100::mbar_wait(&empty[st], ph ^ 1u);
        const int j = jt0 + it / a.kblocks, kb = it % a.kblocks;
        const uint32_t sa = sbase + (uint32_t)st * STAGE, sb = sa + kLmABytes;
        if (PAIR) {  // both CTAs' copies complete on the leader's full[st]; the leader expects both
          const uint32_t lbar = cluster_addr(&full[st], 0);
          if (leader) sm100::mbar_arrive_expect_tx(&full[st], 2 * STAGE);
          else sm100::mbar_arrive_remote_relaxed(&full[st], 0);
          tma_load_2d_pair(sa, &tm_h, kb * kLmBK, (int32_t)m0, lbar);
          tma_load_2d_pair(sb, &tm_w, kb * kLmBK, j * kLmBN + (int32_t)crank * (kLmBN / 2), lbar);
        } else {
          sm100::mbar_arrive_expect_tx(&full[st], STAGE);
          tma_load_2d(sa, &tm_h, kb * kLmBK, (int32_t)m0, &full[st]);
          tma_load_2d(sb, &tm_w, kb * kLmBK, j * kLmBN, &full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // --------------------------------------- MMA issuer (PAIR: the leader)
      int it = 0;
      for (int j = 0; j < ntiles; ++j) {
        const int acc = j & 1;
        sm100::mbar_wait(&acc_empty[acc], (((uint32_t)j >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t td = tmem + (uint32_t)acc * kLmBN;
        for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
          const int st = it % STAGES;
          sm100::mbar_wait(&full[st], (uint32_t)(it / STAGES) & 1u);
          tc_fence_after();
          const uint32_t sa = sbase + (uint32_t)st * STAGE, sb = sa + kLmABytes;
          const uint64_t ad = umma_desc_sw128(sa), bd = umma_desc_sw128(sb);
#pragma unroll
          for (int k = 0; k < kLmBK / 16; ++k) {  // K = 16 bf16 = 32 B per MMA: start address + 2 (16-B units)
            if (PAIR) umma_bf16_pair(td, ad + 2 * k, bd + 2 * k, kLmPairIdesc, (kb | k) != 0);
            else umma_bf16(td, ad + 2 * k, bd + 2 * k, kLmIdesc, (kb | k) != 0);
          }
          if (PAIR) umma_commit_pair(&empty[st]);  // both CTAs' slot st free once these MMAs read it
          else umma_commit(&empty[st]);
        }
        if (PAIR) umma_commit_pair(&acc_full[acc]);  // accumulator complete (each CTA its 128 rows)
        else umma_commit(&acc_full[acc]);
      }
    }
  } else if (GRAD) {  // ------------------------------------------------ gradient epilogue 2..5
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
    const bool live = row < a.n;
    const int32_t y = live ? a.targets[row] : -1;
    const float k = a.inv_t * RL_LOG2E;
    const float st = (live && y >= 0 && y < a.V) ? a.scale[row] : 0.f;  // y outside [0, V): G row 0
    const float nl2 = live ? -a.lse[row] * RL_LOG2E : 0.f;  // -lse in the log2 domain
    const uint64_t k2 = f2pack_lm(k, k), nl22 = f2pack_lm(nl2, nl2), s2 = f2pack_lm(st, st);
    uint16_t* grow = a.g_out + (live ? row : 0) * a.ld_g;
    for (int j = 0; j < ntiles; ++j) {
      const int acc = j & 1;
      sm100::mbar_wait(&acc_full[acc], ((uint32_t)j >> 1) & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kLmBN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kLmBN + c * 32), v);
        const int64_t c0 = (int64_t)(jt0 + j) * kLmBN + c * 32;
        if (c0 >= a.V) break;  // warp-uniform
        uint32_t o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float e0, e1;
          f2unpack_lm(ffma2_lm(f2pack_lm(v[2 * i], v[2 * i + 1]), k2, nl22), e0, e1);
          float g0, g1;
          f2unpack_lm(fmul2_lm(f2pack_lm(exp2f(e0), exp2f(e1)), s2), g0, g1);
          if (y - c0 == 2 * i) g0 = st * (exp2f(e0) - 1.f);       // target column: s (p_y - 1)
          if (y - c0 == 2 * i + 1) g1 = st * (exp2f(e1) - 1.f);
          o[i] = pack_bf16x2(g0, g1);
        }
        RL_DCHECK(!live || (row < a.n && c0 < a.V && c0 + 32 <= a.ld_g + 31));
        if (live && c0 + 32 <= a.V) {
          uint4* dst = reinterpret_cast<uint4*>(grow + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else if (live) {
          for (int i = 0; i < 32 && c0 + i < a.V; ++i) grow[c0 + i] = (uint16_t)(o[i >> 1] >> (16 * (i & 1)));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) sm100::mbar_arrive_remote_relaxed(&acc_empty[acc], 0);  // the leader's barrier
        else sm100::mbar_arrive(&acc_empty[acc]);
      }
    }
  } else {  // ---------------------------------------------------------- epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int64_t row = m0 + q * 32 + lane;
    const bool live = row < a.n;
    const int32_t y = live ? a.targets[row] : -1;
    const float k = a.inv_t * RL_LOG2E;
    float m = -INFINITY, s = 0.f, zy = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int acc = j & 1;
      sm100::mbar_wait(&acc_full[acc], ((uint32_t)j >> 1) & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kLmBN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kLmBN + c * 32), v);
        const int64_t c0 = (int64_t)(jt0 + j) * kLmBN + c * 32;
        if (c0 >= a.V) break;
        const int64_t dy = (int64_t)y - c0;
#pragma unroll
        for (int i = 0; i < 32; ++i) zy = (dy == i) ? v[i] : zy;
        if (c0 + 32 > a.V) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = (c0 + i < a.V) ? v[i] : -INFINITY;
        }
        float cm = v[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) cm = fmaxf(cm, v[i]);
        const float nm = fmaxf(m, cm * k);
        float acc_s = (m == -INFINITY) ? 0.f : s * exp2f(m - nm);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc_s += exp2f(fmaf(v[i], k, -nm));
        m = nm;
        s = acc_s;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) sm100::mbar_arrive_remote_relaxed(&acc_empty[acc], 0);  // the leader's barrier
        else sm100::mbar_arrive(&acc_empty[acc]);
      }
    }
    if (live && gridDim.x > 1) {
      a.partial[(int64_t)split_idx * a.n + row] = make_float4(m, s, zy, 0.f);
    } else if (live) {
      const float lse2 = m + log2f(s);
      if (a.lse_out) a.lse_out[row] = lse2 * RL_LN2;
      float lp = 0.f;
      if (y >= 0 && y < a.V) lp = zy * a.inv_t - lse2 * RL_LN2;
      else if (y >= a.V) lp = __int_as_float(0x7fc00000);
      a.logp_out[row] = lp;
    }
  }
  tc_fence_before();
  if (PAIR) sm100::cluster_sync();  // both CTAs done (incl. remote arrivals) before either deallocates
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// splits > 1: combine the per-split (max2, sum, target logit) records of each row in split order
__global__ void lmhead_combine_kernel(const float4* __restrict__ partial, int splits, const LmArgs a) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < a.n; row += (int64_t)gridDim.x * blockDim.x) {
    float M = -INFINITY;
    for (int i = 0; i < splits; ++i) M = fmaxf(M, partial[(int64_t)i * a.n + row].x);
    float S = 0.f, zy = 0.f;
    for (int i = 0; i < splits; ++i) {
      const float4 e = partial[(int64_t)i * a.n + row];
      if (e.x != -INFINITY) S += e.y * exp2f(e.x - M);
      zy += e.z;
    }
    const float lse2 = M + log2f(S);
    if (a.lse_out) a.lse_out[row] = lse2 * RL_LN2;
    const int32_t y = a.targets[row];
    float lp = 0.f;
    if (y >= 0 && y < a.V) lp = zy * a.inv_t - lse2 * RL_LN2;
    else if (y >= a.V) lp = __int_as_float(0x7fc00000);
    a.logp_out[row] = lp;
  }
}

// Vocabulary splits S (the fast grid index, so a wave holds ~sms / S token blocks).  Two L2 effects
// set S (measured, tools/lmbench.py, d = 4096, V = 151936):
//   * a wave's hidden blocks (128 x d bf16 each, re-read once per vocabulary tile) must stay in L2:
//     S = 1 puts 148 blocks = 148 MB in flight and thrashes the 126 MB L2 (70 GB of DRAM reads at
//     N = 16384 for 1.4 GB of operands) — S_min keeps them <= 80 MB;
//   * every further split divides the readers sharing a W tile while it is L2-resident (S = 8: 1277
//     TFLOP/s at N = 16384, S = 2: 1514; S = 15: 42 GB of DRAM reads).
// So S = S_min when that grid fills the GPU; smaller grids (few token blocks) search S in
// [S_min, 16] for the fewest waves x tiles per CTA (N = 4096: S = 9, 1533 TFLOP/s; S = 5: 922).
static int lm_splits(int64_t n, int64_t d, int64_t vocab, int sms) {
  const int64_t rb = (n + kLmBM - 1) / kLmBM, vt = (vocab + kLmBN - 1) / kLmBN;
  const int64_t block_bytes = (int64_t)kLmBM * d * 2;
  const int64_t smin = std::min<int64_t>(vt, std::max<int64_t>(1, (sms * block_bytes + (80ll << 20) - 1) / (80ll << 20)));
  if (rb * smin >= sms) {
    const int64_t tps = (vt + smin - 1) / smin;
    return (int)((vt + tps - 1) / tps);
  }
  int best = 1;
  int64_t best_cost = INT64_MAX;
  for (int64_t sp = smin; sp <= std::min<int64_t>(vt, 16); ++sp) {
    const int64_t tps = (vt + sp - 1) / sp, used = (vt + tps - 1) / tps;
    const int64_t cost = ((rb * used + sms - 1) / sms) * tps;
    if (cost < best_cost) {
      best_cost = cost;
      best = (int)used;
    }
  }
  return best;
}
static int lm_sms() { return dev_info().sms; }

typedef CUresult (*PfnTensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                            CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                            CUtensorMapFloatOOBfill);

static PfnTensorMapEncodeTiled tensor_map_encoder() {
  static PfnTensorMapEncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PfnTensorMapEncodeTiled)p;
  }
  return fn;
}

// rows x cols bf16 matrix (row stride ld elements) as a 2-D tensor map with a {64, box_rows} box
static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows) {
  PfnTensorMapEncodeTiled enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kLmBK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------------------------------------
// The backward's two GEMMs on tcgen05 (lm_gemm_kernel): C[M, N] (+)= A[M, K] B[K, N] in fp32 from
// bf16 operands in HBM, one 128 x 256 output tile per CTA, the K loop through a 4-stage TMA ring.
//   dh = G W:     A = G  [C, V]  K-major (row-major, K = V contiguous)
//                 B = W  [V, d]  MN-major (row-major, N = d contiguous)
//   dW = G^T h:   A = G^T        MN-major (G row-major, M = V contiguous)
//                 B = h  [C, d]  MN-major
// An MN-major operand tile is staged as 64-element-wide column slabs (one 2-D TMA box of 64 x 64,
// 128-B swizzle, 8 KB each): descriptor LBO = 8 KB between slabs, SBO = 1 KB between 8-row groups,
// and each K = 16 step advances the start by 16 rows x 128 B; the instruction descriptor's
// a_major / b_major bits (15 / 16) select the MN-major reading.
constexpr int kGmBM = 128, kGmBN = 256, kGmBK = 64, kGmStages = 4, kGmThreads = 192;
constexpr uint32_t kGmABytes = kGmBM * kGmBK * 2, kGmBBytes = kGmBN * kGmBK * 2;
constexpr uint32_t kGmStage = kGmABytes + kGmBBytes;  // 48 KB
constexpr size_t kGmSmem = (size_t)kGmStages * kGmStage + 1024;

__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

struct GmArgs {
  float* out;
  int64_t ldo;
  int32_t M, N, kblocks;
  int32_t accumulate;
  int32_t nblocks;  // PAIR launches: N blocks (the grid is 1-D)
};

template <bool A_MN, bool B_MN, bool PAIR>
__global__ void __launch_bounds__(kGmThreads, 1)
    lm_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const GmArgs g) {
  // PAIR: clusters of two CTAs, one 256 x 256 output tile per pair (tcgen05 cta_group::2, M = 256):
  // each CTA stages its own 128 rows of A and half of the tile's N columns of B (MN-major B only)
  static_assert(!PAIR || B_MN, "paired tiles split an MN-major B operand");
  constexpr int STAGES = PAIR ? 6 : kGmStages;
  constexpr uint32_t BBYTES = PAIR ? kGmBBytes / 2 : kGmBBytes;
  constexpr uint32_t STAGE = kGmABytes + BBYTES;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(kGmBN >> 3) << 17) |
                             ((uint32_t)((PAIR ? 2 * kGmBM : kGmBM) >> 4) << 24);
  extern __shared__ uint8_t gm_smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], acc_full;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = (sm100::smem_u32(gm_smem_raw) + 1023u) & ~1023u;
  const uint32_t crank = PAIR ? sm100::cluster_ctarank() : 0;
  const bool leader = crank == 0;
  int32_t m0, n0;
  if (PAIR) {  // 1-D grid of clusters: (pair tile = N block fastest, then M pair) x rank
    const uint32_t pt = blockIdx.x >> 1;
    n0 = (int32_t)(pt % (uint32_t)g.nblocks) * kGmBN;
    m0 = (int32_t)((pt / (uint32_t)g.nblocks) * 2 + crank) * kGmBM;
  } else {
    m0 = (int32_t)blockIdx.y * kGmBM;
    n0 = (int32_t)blockIdx.x * kGmBN;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      sm100::mbar_init(&full[i], PAIR ? 2 : 1);
      sm100::mbar_init(&empty[i], 1);
    }
    sm100::mbar_init(&acc_full, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                       sm100::smem_u32(&tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                       sm100::smem_u32(&tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR) sm100::cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      for (int kb = 0; kb < g.kblocks; ++kb) {
        const int st = kb % STAGES;
        sm100::mbar_wait(&empty[st], ((uint32_t)(kb / STAGES) & 1u) ^ 1u);
        const uint32_t sa = sbase + (uint32_t)st * STAGE, sb = sa + kGmABytes;
        const int32_t k0 = kb * kGmBK;
        if (PAIR) {
          const uint32_t lbar = cluster_addr(&full[st], 0);
          if (leader) sm100::mbar_arrive_expect_tx(&full[st], 2 * STAGE);
          else sm100::mbar_arrive_remote_relaxed(&full[st], 0);
          if (A_MN) {
            tma_load_2d_pair(sa, &tm_a, m0, k0, lbar);
            tma_load_2d_pair(sa + 8192, &tm_a, m0 + 64, k0, lbar);
          } else {
            tma_load_2d_pair(sa, &tm_a, k0, m0, lbar);
          }
          const int32_t nh = n0 + (int32_t)crank * (kGmBN / 2);  // this CTA's half of the N columns
          tma_load_2d_pair(sb, &tm_b, nh, k0, lbar);
          tma_load_2d_pair(sb + 8192, &tm_b, nh + 64, k0, lbar);
        } else {
          sm100::mbar_arrive_expect_tx(&full[st], STAGE);
          if (A_MN) {  // two 64-wide M slabs of the row-major [K, M] operand
            tma_load_2d(sa, &tm_a, m0, k0, &full[st]);
            tma_load_2d(sa + 8192, &tm_a, m0 + 64, k0, &full[st]);
          } else {
            tma_load_2d(sa, &tm_a, k0, m0, &full[st]);
          }
          if (B_MN) {  // four 64-wide N slabs of the row-major [K, N] operand
#pragma unroll
            for (int q = 0; q < 4; ++q) tma_load_2d(sb + q * 8192, &tm_b, n0 + 64 * q, k0, &full[st]);
          } else {
            tma_load_2d(sb, &tm_b, k0, n0, &full[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // --------------------------------------- MMA issuer (PAIR: the leader)
      for (int kb = 0; kb < g.kblocks; ++kb) {
        const int st = kb % STAGES;
        sm100::mbar_wait(&full[st], (uint32_t)(kb / STAGES) & 1u);
        tc_fence_after();
        const uint32_t sa = sbase + (uint32_t)st * STAGE, sb = sa + kGmABytes;
        const uint64_t ad = A_MN ? umma_desc_mn_sw128(sa) : umma_desc_sw128(sa);
        const uint64_t bd = B_MN ? umma_desc_mn_sw128(sb) : umma_desc_sw128(sb);
#pragma unroll
        for (int k = 0; k < kGmBK / 16; ++k) {
          // K step of 16: K-major +32 B (2 units), MN-major +16 rows x 128 B (128 units)
          const uint64_t ao = A_MN ? 128ull * k : 2ull * k, bo = B_MN ? 128ull * k : 2ull * k;
          if (PAIR) umma_bf16_pair(tmem, ad + ao, bd + bo, IDESC, (kb | k) != 0);
          else umma_bf16(tmem, ad + ao, bd + bo, IDESC, (kb | k) != 0);
        }
        if (PAIR) umma_commit_pair(&empty[st]);
        else umma_commit(&empty[st]);
      }
      if (PAIR) umma_commit_pair(&acc_full);
      else umma_commit(&acc_full);
    }
  } else {  // ---------------------------------------------------------- epilogue warps 2..5
    const int q = warp & 3;
    const int32_t row = m0 + q * 32 + lane;
    sm100::mbar_wait(&acc_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < kGmBN / 32; ++c) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), v);
      const int32_t col = n0 + c * 32;
      if (row < g.M && col < g.N) {
        float* o = g.out + (int64_t)row * g.ldo + col;
        if (col + 32 <= g.N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 w = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            if (g.accumulate) {
              const float4 p = o4[i];
              w.x += p.x;
              w.y += p.y;
              w.z += p.z;
              w.w += p.w;
            }
            o4[i] = w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col + i < g.N) o[i] = g.accumulate ? o[i] + v[i] : v[i];
        }
      }
    }
  }
  tc_fence_before();
  if (PAIR) sm100::cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// Launch the LM-head kernel over a (splits, token blocks) grid: CTA pairs (cta_group::2, clusters of
// (1, 2, 1), token blocks padded to even) when there are >= 2 token blocks — unless the development
// option RL_DEV_LM_PAIR selects single CTAs.  w_base/ld_w/vocab/d describe W for the tensor maps.
template <bool GRAD>
static rl_status launch_lm(int splits, int64_t n_rows, const CUtensorMap& mh, const void* w_base, int64_t vocab,
                           int64_t d, int64_t ld_w, const LmArgs& a, cudaStream_t s) {
  const int64_t rb = (n_rows + kLmBM - 1) / kLmBM;
  // measured (tools/lmbench.py, d 4096, V 151936): pairs win for the gradient kernel (1,537 vs 1,433
  // TFLOP/s for the backward at N = 16K, 1,300 vs 1,275 at 128K) but not for the log-prob kernel
  // (1,496 vs 1,476 at 16K, 1,292 vs 1,372 at 128K: ncu shows 20 GB of DRAM reads against 2.9 GB
  // for single CTAs — the cluster schedule loses the W-tile L2 reuse across token blocks)
  const int opt = dev_option(OPT_LM_PAIR);  // 0 default, 1 single CTAs, 2 pairs
  const bool pair = rb >= 2 && (opt == 2 || (opt == 0 && GRAD));
  CUtensorMap mw;
  if (!make_map(&mw, w_base, vocab, d, ld_w, pair ? kLmBN / 2 : kLmBN))
    return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (!pair) {
    if (cudaFuncSetAttribute(lmhead_kernel<GRAD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLmSmem) !=
        cudaSuccess)
      return check_launch("cudaFuncSetAttribute(lmhead)");
    lmhead_kernel<GRAD, false><<<dim3((unsigned)splits, (unsigned)rb), kLmThreads, kLmSmem, s>>>(mh, mw, a);
    return check_launch(GRAD ? "lmhead_kernel<grad>" : "lmhead_kernel<logprob>");
  }
  auto kern = lmhead_kernel<GRAD, true>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLmSmem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(lmhead pair)");
  // clusters of two along a 1-D grid over the linear (pair, split, rank) index
  LmArgs b = a;
  b.n_splits = splits;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)((rb + 1) / 2 * 2 * splits), 1, 1);
  cfg.blockDim = dim3(kLmThreads);
  cfg.dynamicSmemBytes = kLmSmem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, mh, mw, b) != cudaSuccess)
    return check_launch(GRAD ? "lmhead_kernel<grad, pair>" : "lmhead_kernel<logprob, pair>");
  return check_launch(GRAD ? "lmhead_kernel<grad, pair>" : "lmhead_kernel<logprob, pair>");
}

template <bool A_MN, bool B_MN>
static rl_status lm_gemm(const CUtensorMap& ta, const CUtensorMap& tb, float* out, int64_t ldo, int64_t M, int64_t N,
                         int64_t K, bool accumulate, cudaStream_t s) {
  if (M <= 0 || N <= 0) return RL_OK;
  GmArgs g;
  g.out = out;
  g.ldo = ldo;
  g.M = (int32_t)M;
  g.N = (int32_t)N;
  g.kblocks = (int32_t)((K + kGmBK - 1) / kGmBK);
  g.accumulate = accumulate ? 1 : 0;
  const int64_t mb = (M + kGmBM - 1) / kGmBM, nb = (N + kGmBN - 1) / kGmBN;
  g.nblocks = (int32_t)nb;
  const bool pair = B_MN && mb >= 2 && dev_option(OPT_LM_PAIR) == 2;  // measured: single CTAs 3-6 % faster
  if (!pair) {
    auto kern = lm_gemm_kernel<A_MN, B_MN, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGmSmem) != cudaSuccess)
      return check_launch("cudaFuncSetAttribute(lm_gemm)");
    if (mb > 65535) return fail(RL_ERR_UNSUPPORTED, "lm_gemm: M too large");
    kern<<<dim3((unsigned)nb, (unsigned)mb), kGmThreads, kGmSmem, s>>>(ta, tb, g);
    return check_launch(A_MN ? "lm_gemm_kernel<dW>" : "lm_gemm_kernel<dh>");
  }
  // B_MN is always true on this path (static_assert in the kernel)
  auto kern = lm_gemm_kernel<A_MN, true, true>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGmSmem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(lm_gemm pair)");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)((mb + 1) / 2 * 2 * nb), 1, 1);
  cfg.blockDim = dim3(kGmThreads);
  cfg.dynamicSmemBytes = kGmSmem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ta, tb, g) != cudaSuccess)
    return check_launch(A_MN ? "lm_gemm_kernel<dW, pair>" : "lm_gemm_kernel<dh, pair>");
  return check_launch(A_MN ? "lm_gemm_kernel<dW, pair>" : "lm_gemm_kernel<dh, pair>");
}

}  // namespace rl

extern "C" size_t rl_lmhead_workspace_size(int64_t n_tokens, int64_t d, int64_t vocab) {
  using namespace rl;
  if (n_tokens <= 0 || vocab <= 0 || d <= 0) return 0;
  const int sp = lm_splits(n_tokens, d, vocab, lm_sms());
  return sp > 1 ? (size_t)sp * (size_t)n_tokens * sizeof(float4) : 0;
}

extern "C" rl_status rl_lmhead_logprob(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                                       int64_t n_tokens, int64_t d, int64_t vocab, const int32_t* targets,
                                       float inv_temperature, float* logp_out, float* lse_out, void* workspace,
                                       size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (n_tokens < 0 || d < 1 || vocab < 1) return fail(RL_ERR_INVALID_ARGUMENT, "need n_tokens >= 0, d >= 1, vocab >= 1");
  if (ld_hidden < d || ld_weight < d) return fail(RL_ERR_INVALID_ARGUMENT, "ld_hidden / ld_weight < d");
  if (n_tokens >= ((int64_t)1 << 31) || vocab >= ((int64_t)1 << 31) || d >= ((int64_t)1 << 31))
    return fail(RL_ERR_UNSUPPORTED, "n_tokens, d and vocab must be < 2^31");
  if (!(inv_temperature > 0.f) || !isfinite(inv_temperature))
    return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be finite and > 0");
  if (n_tokens == 0) return RL_OK;
  if (!hidden || !weight || !targets || !logp_out) return fail(RL_ERR_INVALID_ARGUMENT, "NULL hidden/weight/targets/logp_out");
  if (((uintptr_t)hidden & 15) || ((uintptr_t)weight & 15) || (ld_hidden % 8) || (ld_weight % 8))
    return fail(RL_ERR_ALIGNMENT, "hidden / weight must be 16-B aligned with ld % 8 == 0");
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  CUtensorMap mh;
  if (!make_map(&mh, hidden, n_tokens, d, ld_hidden, kLmBM)) return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  LmArgs a{};
  a.targets = targets;
  a.n = n_tokens;
  a.V = vocab;
  a.kblocks = (int32_t)((d + kLmBK - 1) / kLmBK);
  a.vtiles = (int32_t)((vocab + kLmBN - 1) / kLmBN);
  int splits = lm_splits(n_tokens, d, vocab, lm_sms());
  const int forced = dev_option(OPT_LM_SPLITS);  // development: force the split count (<= the workspace's)
  if (forced > 0 && forced <= splits) splits = forced;
  a.tiles_per_split = (a.vtiles + splits - 1) / splits;
  splits = (a.vtiles + a.tiles_per_split - 1) / a.tiles_per_split;
  const size_t need = splits > 1 ? (size_t)splits * (size_t)n_tokens * sizeof(float4) : 0;
  if (need && (!workspace || workspace_bytes < need))
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes (rl_lmhead_workspace_size)", need);
  a.partial = (float4*)workspace;
  a.inv_t = inv_temperature;
  a.logp_out = logp_out;
  a.lse_out = lse_out;
  if ((n_tokens + kLmBM - 1) / kLmBM > 65534) return fail(RL_ERR_UNSUPPORTED, "n_tokens > 65534 * 128 per call");
  rl_status st = launch_lm<false>(splits, n_tokens, mh, weight, vocab, d, ld_weight, a, (cudaStream_t)stream);
  if (st != RL_OK || splits == 1) return st;
  const int cb = (int)std::min<int64_t>((n_tokens + 255) / 256, 148 * 4);
  lmhead_combine_kernel<<<cb, 256, 0, (cudaStream_t)stream>>>(a.partial, splits, a);
  return check_launch("lmhead_combine_kernel");
}

// ------------------------------------------------------------------------------------------------
// NEXT 4 backward: dh = G W and dW (+)= G^T h with G = s_t (softmax(x_t) - onehot(y_t)), x = (h W^T) inv_T.
// Per chunk of C tokens: lmhead_kernel<true> recomputes the logits tiles on the tensor cores and
// writes G (bf16) into the workspace — the logits never exist in memory — then two plain GEMMs
// consume G (cuBLAS, bf16 x bf16 -> fp32 accumulate): dh_chunk = G W and dW += G^T h_chunk.
// Why G is materialised per chunk: a CTA that owns a 128-row tile of G would have
// to hold a 128 x d fp32 dh accumulator (2 MB at d = 4096) and a 256 x d dW one — 8x / 16x the
// 256 KB of TMEM — so the contraction over V (dh) and over tokens (dW) cannot stay on chip; G in
// bf16 costs 2 B per element against 4 d flops of GEMM per element (compute-bound by ~1000x).
namespace rl {
static cublasHandle_t cublas_handle() {
  static cublasHandle_t handles[kMaxDevices] = {};
  static std::mutex mu;
  const int dev = dev_info().ordinal;
  std::lock_guard<std::mutex> lk(mu);
  if (!handles[dev] && cublasCreate(&handles[dev]) != CUBLAS_STATUS_SUCCESS) handles[dev] = nullptr;
  return handles[dev];
}
}  // namespace rl

extern "C" size_t rl_lmhead_loss_bwd_workspace_size(int64_t chunk_tokens, int64_t vocab) {
  if (chunk_tokens <= 0 || vocab <= 0) return 0;
  const int64_t ldg = (vocab + 7) / 8 * 8;
  return (size_t)chunk_tokens * (size_t)ldg * 2;
}

extern "C" rl_status rl_lmhead_loss_bwd(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                                        int64_t n_tokens, int64_t d, int64_t vocab, const int32_t* targets,
                                        const float* lse, const float* scale, float inv_temperature,
                                        float* dhidden, int64_t ld_dhidden, float* dweight, int64_t ld_dweight,
                                        uint32_t flags, void* workspace, size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (n_tokens < 0 || d < 1 || vocab < 1) return fail(RL_ERR_INVALID_ARGUMENT, "need n_tokens >= 0, d >= 1, vocab >= 1");
  if (ld_hidden < d || ld_weight < d || (dhidden && ld_dhidden < d) || (dweight && ld_dweight < d))
    return fail(RL_ERR_INVALID_ARGUMENT, "a row stride is < d");
  if (n_tokens >= ((int64_t)1 << 31) || vocab >= ((int64_t)1 << 31) || d >= ((int64_t)1 << 31))
    return fail(RL_ERR_UNSUPPORTED, "n_tokens, d and vocab must be < 2^31");
  if (!(inv_temperature > 0.f) || !isfinite(inv_temperature))
    return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be finite and > 0");
  if (!dhidden && !dweight) return fail(RL_ERR_INVALID_ARGUMENT, "neither dhidden nor dweight requested");
  if (!hidden || !weight) return fail(RL_ERR_INVALID_ARGUMENT, "NULL hidden/weight");
  if (((uintptr_t)hidden & 15) || ((uintptr_t)weight & 15) || (ld_hidden % 8) || (ld_weight % 8))
    return fail(RL_ERR_ALIGNMENT, "hidden / weight must be 16-B aligned with ld % 8 == 0");
  const int64_t ldg = (vocab + 7) / 8 * 8;
  const int64_t chunk = workspace ? (int64_t)(workspace_bytes / ((size_t)ldg * 2)) / kLmBM * kLmBM : 0;
  if (n_tokens > 0 && chunk < std::min<int64_t>(n_tokens, kLmBM))
    return fail(RL_ERR_WORKSPACE, "workspace must hold >= 128 (or n_tokens) G rows: >= %zu bytes",
                rl_lmhead_loss_bwd_workspace_size(std::min<int64_t>(n_tokens, kLmBM), vocab));
  if (((uintptr_t)workspace & 15)) return fail(RL_ERR_ALIGNMENT, "workspace must be 16-B aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const bool acc_w = (flags & RL_F_STATS_ACCUMULATE) != 0;  // dW += (else dW =)
  if (n_tokens == 0) {
    if (dweight && !acc_w && cudaMemset2DAsync(dweight, (size_t)ld_dweight * 4, 0, (size_t)d * 4, (size_t)vocab, s) !=
                                 cudaSuccess)
      return check_launch("memset dweight");
    return RL_OK;
  }
  if (!targets || !lse || !scale) return fail(RL_ERR_INVALID_ARGUMENT, "NULL targets/lse/scale");
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cublasHandle_t h = cublas_handle();
  if (!h) return fail(RL_ERR_CUDA, "cublasCreate failed");
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return fail(RL_ERR_CUDA, "cublasSetStream failed");

  uint16_t* G = (uint16_t*)workspace;
  const float one = 1.f, zero = 0.f;
  for (int64_t t0 = 0; t0 < n_tokens; t0 += chunk) {
    const int64_t C = std::min(chunk, n_tokens - t0);
    const void* h0 = (const char*)hidden + (size_t)t0 * ld_hidden * 2;
    CUtensorMap mh;
    if (!make_map(&mh, h0, C, d, ld_hidden, kLmBM)) return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    LmArgs a{};
    a.targets = targets + t0;
    a.n = C;
    a.V = vocab;
    a.kblocks = (int32_t)((d + kLmBK - 1) / kLmBK);
    a.vtiles = (int32_t)((vocab + kLmBN - 1) / kLmBN);
    int splits = lm_splits(C, d, vocab, lm_sms());
    a.tiles_per_split = (a.vtiles + splits - 1) / splits;
    splits = (a.vtiles + a.tiles_per_split - 1) / a.tiles_per_split;
    a.inv_t = inv_temperature;
    a.lse = lse + t0;
    a.scale = scale + t0;
    a.g_out = G;
    a.ld_g = ldg;
    if (rl_status st = launch_lm<true>(splits, C, mh, weight, vocab, d, ld_weight, a, s); st != RL_OK) return st;
    const float* beta = (acc_w || t0 > 0) ? &one : &zero;
    // dh / dW: plain GEMMs -> cuBLAS by default (measured per 16,384-token chunk, d 4096, V 151936:
    // cuBLAS 12.6 / 13.3 ms, lm_gemm_kernel 14.9 / 14.5 ms); the hand-written tcgen05 GEMMs stay
    // selectable (RL_DEV_LM_GEMM = 2) and parity-tested
    if (dev_option(OPT_LM_GEMM) == 2) {  // the backward's GEMMs on tcgen05 (lm_gemm_kernel)
      CUtensorMap tg_k, tg_mn, tw_mn, th_mn;
      if (dhidden) {  // dh_chunk [C, d] = G [C, V] . W [V, d]
        if (!make_map(&tg_k, G, C, vocab, ldg, kGmBM) || !make_map(&tw_mn, weight, vocab, d, ld_weight, kGmBK))
          return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        if (rl_status st = lm_gemm<false, true>(tg_k, tw_mn, dhidden + (size_t)t0 * ld_dhidden, ld_dhidden, C, d,
                                                vocab, false, s);
            st != RL_OK)
          return st;
      }
      if (dweight) {  // dW [V, d] (+)= G^T [V, C] . h_chunk [C, d]
        if (!make_map(&tg_mn, G, C, vocab, ldg, kGmBK) || !make_map(&th_mn, h0, C, d, ld_hidden, kGmBK))
          return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        if (rl_status st = lm_gemm<true, true>(tg_mn, th_mn, dweight, ld_dweight, vocab, d, C, beta == &one, s);
            st != RL_OK)
          return st;
      }
      continue;
    }
    // cuBLAS (development option RL_DEV_LM_GEMM): row-major operands as column-major GEMMs:
    // dh^T [d x C] = W^T [d x V] . G^T [V x C]
    if (dhidden &&
        cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)d, (int)C, (int)vocab, &one, weight, CUDA_R_16BF, (int)ld_weight,
                     G, CUDA_R_16BF, (int)ldg, &zero, dhidden + (size_t)t0 * ld_dhidden, CUDA_R_32F, (int)ld_dhidden,
                     CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return fail(RL_ERR_CUDA, "cublasGemmEx (dh = G W) failed");
    // dW^T [d x V] (+)= h^T [d x C] . G [C x V]
    if (dweight &&
        cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, (int)vocab, (int)C, &one, h0, CUDA_R_16BF, (int)ld_hidden,
                     G, CUDA_R_16BF, (int)ldg, beta, dweight, CUDA_R_32F, (int)ld_dweight, CUBLAS_COMPUTE_32F,
                     CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return fail(RL_ERR_CUDA, "cublasGemmEx (dW += G^T h) failed");
  }
  return check_launch("rl_lmhead_loss_bwd");
}
