// (7) bf16 delta-sparsity scan and sparse encode / apply — NEXT 3 of SURVEY.md §8(f)
// ("the trainer needs to ship only a tiny fraction of its weights",
// sparsity 0.989-0.993; SPEC.md:297-313 compute_delta / apply_delta).
//
// encode: the indices (increasing) and new words of every position where two 16-bit snapshots
// differ — a stream compaction that reads each snapshot once (16-B loads) and writes the ~1 % of
// changes once, HBM-bound on the two reads (two-stage design below).
// apply: base[idx[j]] = word[j] (scatter).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "common.cuh"

namespace rl {

constexpr int kDtThreads = 256;
constexpr int kDtVec = 8;                                     // 16-B vectors per thread per array
constexpr int kDtTile = kDtThreads * kDtVec * 8;              // 16384 words per tile

// bit e of the result: word e of the 8-word vectors a, b differ
__device__ __forceinline__ uint32_t diff8(const uint4& a, const uint4& b) {
  const uint32_t x[4] = {a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w};
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m |= ((x[i] & 0xFFFFu) ? 1u : 0u) << (2 * i) | ((x[i] >> 16) ? 1u : 0u) << (2 * i + 1);
  return m;
}

// ---------------------------------------------------------------------------------------------
// Two-stage encode: (1) a pure streaming pass compares the snapshots tile by tile
// (16,384 words, 16-B loads, no cross-CTA dependency), ranks the tile's changes in word order with
// a block scan and writes them compacted into the tile's own staging slot (capacity kStageCap
// changes: new word + 16-bit index within the tile) plus the tile's change count; a tile with more
// changes writes its change bitmask instead (1 bit per word); (2) an exclusive scan of the tile
// counts (CUB, tiny); (3) a copy of every tile's staged changes to its sorted output position —
// or, for an overflowed tile, a pass over its bitmask that gathers the new words from `next`.
// At sparsity 0.99 every tile stages (~164 changes each): the snapshots are read exactly once and
// stage 3 touches only the changes.
constexpr int kD2Tile = kDtTile;     // 16384 words: 512 u32 mask words, 256 threads x 8 vectors
constexpr int kStageCap = 1024;      // staged changes per tile (6.25 % of its words)

__global__ void __launch_bounds__(kDtThreads, 3) delta_mask_kernel(const uint16_t* __restrict__ prev,
                                                                  const uint16_t* __restrict__ next, int64_t n,
                                                                  int64_t n_tiles, uint32_t* __restrict__ bits,
                                                                  uint64_t* __restrict__ tile_count,
                                                                  uint32_t* __restrict__ stage) {
  __shared__ uint32_t wsum[kDtThreads / 32][kDtVec / 2];  // per warp: packed pairs of row totals
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t wt = tile * kD2Tile;
    // thread t holds vectors v = u * 256 + t (u = 0..7: "row" u of the tile), 8 words each
    uint4 vb[kDtVec];
    uint32_t m[kDtVec];
    if (wt + kD2Tile <= n) {
      const uint4* pa = reinterpret_cast<const uint4*>(prev + wt) + tid;
      const uint4* pb = reinterpret_cast<const uint4*>(next + wt) + tid;
      uint4 va[kDtVec];
#pragma unroll
      for (int u = 0; u < kDtVec; ++u) {
        va[u] = ld_stream_v4(pa + u * kDtThreads);
        vb[u] = ld_stream_v4(pb + u * kDtThreads);
      }
#pragma unroll
      for (int u = 0; u < kDtVec; ++u) m[u] = diff8(va[u], vb[u]);
    } else {
#pragma unroll
      for (int u = 0; u < kDtVec; ++u) {
        m[u] = 0;
        uint16_t wv[8];
        for (int e = 0; e < 8; ++e) {
          const int64_t w = wt + 8 * ((int64_t)u * kDtThreads + tid) + e;
          wv[e] = w < n ? next[w] : 0;
          if (w < n && prev[w] != wv[e]) m[u] |= 1u << e;
        }
        vb[u] = make_uint4(wv[0] | (uint32_t)wv[1] << 16, wv[2] | (uint32_t)wv[3] << 16,
                           wv[4] | (uint32_t)wv[5] << 16, wv[6] | (uint32_t)wv[7] << 16);
      }
    }
    // word-order rank: position of (row u, thread t) = sum of rows < u + sum over threads < t of
    // row u.  Rows are scanned in pairs packed as 16-bit halves (a row holds <= 2048 changes).
    uint32_t incl[kDtVec / 2], cnt[kDtVec / 2];
#pragma unroll
    for (int q = 0; q < kDtVec / 2; ++q) {
      cnt[q] = (uint32_t)__popc(m[2 * q]) | (uint32_t)__popc(m[2 * q + 1]) << 16;
      incl[q] = cnt[q];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl[q], o);
        if (lane >= o) incl[q] += v;
      }
      if (lane == 31) wsum[warp][q] = incl[q];
    }
    __syncthreads();
    uint32_t before[kDtVec / 2], tot[kDtVec / 2];
#pragma unroll
    for (int q = 0; q < kDtVec / 2; ++q) {
      before[q] = 0;
      tot[q] = 0;
    }
#pragma unroll
    for (int w = 0; w < kDtThreads / 32; ++w)
#pragma unroll
      for (int q = 0; q < kDtVec / 2; ++q) {
        const uint32_t x = wsum[w][q];
        tot[q] += x;
        before[q] += w < warp ? x : 0u;
      }
    uint32_t row_base[kDtVec], T = 0;
#pragma unroll
    for (int u = 0; u < kDtVec; ++u) {
      const uint32_t rt = (u & 1) ? tot[u / 2] >> 16 : tot[u / 2] & 0xFFFFu;
      row_base[u] = T;
      T += rt;
    }
    if (T <= (uint32_t)kStageCap) {
      uint32_t* st = stage + (size_t)tile * kStageCap;
#pragma unroll
      for (int u = 0; u < kDtVec; ++u) {
        const uint32_t ex = before[u / 2] + incl[u / 2] - cnt[u / 2];
        uint32_t pos = row_base[u] + ((u & 1) ? ex >> 16 : ex & 0xFFFFu);
        uint32_t mm = m[u];
        const uint32_t wv[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
        while (mm) {
          const int e = __ffs(mm) - 1;
          mm &= mm - 1;
          const uint32_t word = (wv[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
          const uint32_t local = (uint32_t)(8 * (u * kDtThreads + tid) + e);  // < 16384
          st[pos++] = word << 16 | local;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kDtVec; ++u)
        reinterpret_cast<uint8_t*>(bits)[(size_t)tile * (kD2Tile / 8) + (size_t)u * kDtThreads + tid] = (uint8_t)m[u];
    }
    if (tid == 0) tile_count[tile] = T;
    __syncthreads();  // wsum reusable
  }
}

// pass 3: a staged tile is copied (thread j: changes j, j + 256, ...); an overflowed tile: thread t
// owns mask words [t*2, t*2+2) (64 words of the snapshot), ranks its changes with a block scan and
// writes them at tile_offset + rank, the new word gathered from `next`
__global__ void __launch_bounds__(kDtThreads) delta_scatter_kernel(const uint16_t* __restrict__ next, int64_t n,
                                                                     int64_t n_tiles, const uint32_t* __restrict__ bits,
                                                                     const uint64_t* __restrict__ tile_off,
                                                                     const uint64_t* __restrict__ tile_count,
                                                                     const uint32_t* __restrict__ stage,
                                                                     uint32_t* __restrict__ idx_out,
                                                                     uint16_t* __restrict__ word_out, int64_t capacity,
                                                                     unsigned long long* __restrict__ count_out) {
  __shared__ uint32_t wsum[kDtThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t T = (int64_t)tile_count[tile], base = (int64_t)tile_off[tile];
    if (tile == n_tiles - 1 && tid == 0) *count_out = (unsigned long long)(base + T);
    if (T <= kStageCap) {
      const uint32_t* st = stage + (size_t)tile * kStageCap;
      for (int64_t j = tid; j < T; j += kDtThreads) {
        const int64_t off = base + j;
        if (off < capacity) {
          const uint32_t e = st[j];
          idx_out[off] = (uint32_t)(tile * kD2Tile + (e & 0xFFFFu));
          word_out[off] = (uint16_t)(e >> 16);
        }
      }
      continue;  // block-uniform branch: no barrier skipped by a subset of threads
    }
    const uint2 mw = reinterpret_cast<const uint2*>(bits + (size_t)tile * (kD2Tile / 32))[tid];
    const uint32_t c = __popc(mw.x) + __popc(mw.y);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < kDtThreads / 32; ++w) before += w < warp ? wsum[w] : 0;
    int64_t off = base + before + incl - c;
    const int64_t w0 = tile * kD2Tile + (int64_t)tid * 64;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t m = half ? mw.y : mw.x;
      while (m) {
        const int e = __ffs(m) - 1;
        m &= m - 1;
        if (off < capacity) {
          const int64_t w = w0 + half * 32 + e;
          idx_out[off] = (uint32_t)w;
          word_out[off] = next[w];
        }
        ++off;
      }
    }
    __syncthreads();  // wsum reusable
  }
}

__global__ void delta_apply_kernel(uint16_t* __restrict__ base, int64_t n, const uint32_t* __restrict__ idx,
                                   const uint16_t* __restrict__ words, const unsigned long long* __restrict__ count,
                                   int64_t capacity, unsigned long long* __restrict__ bad) {
  const int64_t k = (int64_t)min((unsigned long long)capacity, *count);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[j];
    if (i < n) base[i] = words[j];
    else atomicAdd(bad, 1ull);
  }
}

static int64_t dt_tiles(int64_t n) { return (n + kDtTile - 1) / kDtTile; }

}  // namespace rl

namespace rl {
// workspace: [tile counts: tiles+2 u64][tile offsets: tiles u64]
//            [change bitmask: tiles * 2 KB][staged changes: tiles * kStageCap u32][CUB scan temp]
struct DtLayout {
  size_t status, offs, bits, stage, temp, temp_bytes, total;
};
static DtLayout dt_layout(int64_t n_words) {
  const int64_t tiles = dt_tiles(n_words);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)std::max<int64_t>(tiles, 1));
  DtLayout L;
  size_t off = 0;
  auto al = [&](size_t b) {
    const size_t o = off;
    off += (b + 255) & ~(size_t)255;
    return o;
  };
  L.status = al((size_t)(tiles + 2) * 8);
  L.offs = al((size_t)tiles * 8);
  L.bits = al((size_t)tiles * (kD2Tile / 8));
  L.stage = al((size_t)tiles * kStageCap * 4);
  L.temp_bytes = scan_bytes;
  L.temp = al(scan_bytes);
  L.total = off;
  return L;
}
}  // namespace rl

extern "C" size_t rl_bf16_delta_workspace_size(int64_t n_words) {
  if (n_words < 0) return 0;
  return rl::dt_layout(n_words).total;
}

extern "C" rl_status rl_bf16_delta_encode(const void* prev, const void* next, int64_t n_words, uint32_t* idx_out,
                                          uint16_t* word_out, int64_t capacity, unsigned long long* count_out,
                                          void* workspace, size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (n_words < 0 || n_words > (int64_t)0xFFFFFFFFll) return fail(RL_ERR_INVALID_ARGUMENT, "n_words must be in [0, 2^32)");
  if (capacity < 0) return fail(RL_ERR_INVALID_ARGUMENT, "capacity < 0");
  if (!count_out) return fail(RL_ERR_INVALID_ARGUMENT, "NULL count_out");
  if (n_words > 0 && (!prev || !next)) return fail(RL_ERR_INVALID_ARGUMENT, "NULL prev/next");
  if (capacity > 0 && (!idx_out || !word_out)) return fail(RL_ERR_INVALID_ARGUMENT, "NULL idx_out/word_out");
  if (((uintptr_t)prev & 15) || ((uintptr_t)next & 15)) return fail(RL_ERR_ALIGNMENT, "prev/next must be 16-B aligned");
  if (!workspace || workspace_bytes < rl_bf16_delta_workspace_size(n_words))
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes", rl_bf16_delta_workspace_size(n_words));
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tiles = dt_tiles(n_words);
  const DtLayout L = dt_layout(n_words);
  char* w = (char*)workspace;
  uint64_t* status = (uint64_t*)(w + L.status);
  if (tiles == 0) {
    if (cudaMemsetAsync(count_out, 0, 8, s) != cudaSuccess) return check_launch("delta memset");
    return RL_OK;
  }
  static int sms_tab[kMaxDevices] = {};
  int& sms = dev_slot(sms_tab);
  if (!sms) sms = dev_info().sms;
  uint64_t* counts = status;
  uint64_t* offs = (uint64_t*)(w + L.offs);
  uint32_t* bits = (uint32_t*)(w + L.bits);
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sms * 8);
  uint32_t* stage = (uint32_t*)(w + L.stage);
  delta_mask_kernel<<<grid, kDtThreads, 0, s>>>((const uint16_t*)prev, (const uint16_t*)next, n_words, tiles, bits,
                                                counts, stage);
  rl_status st = check_launch("delta_mask_kernel");
  if (st != RL_OK) return st;
  size_t tb = L.temp_bytes;
  if (cub::DeviceScan::ExclusiveSum(w + L.temp, tb, counts, offs, (int)tiles, s) != cudaSuccess)
    return check_launch("cub scan (delta)");
  delta_scatter_kernel<<<grid, kDtThreads, 0, s>>>((const uint16_t*)next, n_words, tiles, bits, offs, counts, stage,
                                                   idx_out, word_out, capacity, count_out);
  return check_launch("delta_scatter_kernel");
}

extern "C" rl_status rl_bf16_delta_apply(void* base, int64_t n_words, const uint32_t* idx, const uint16_t* words,
                                         const unsigned long long* count, int64_t capacity,
                                         unsigned long long* bad_index_count, rl_stream stream) {
  using namespace rl;
  if (n_words < 0 || capacity < 0) return fail(RL_ERR_INVALID_ARGUMENT, "n_words / capacity < 0");
  if (!count || !bad_index_count) return fail(RL_ERR_INVALID_ARGUMENT, "NULL count / bad_index_count");
  if ((n_words > 0 && !base) || (capacity > 0 && (!idx || !words)))
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL base/idx/words");
  if (capacity == 0) return RL_OK;
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = (int)std::min<int64_t>((capacity + 255) / 256, 148 * 8);
  delta_apply_kernel<<<grid, 256, 0, s>>>((uint16_t*)base, n_words, idx, words, count, capacity, bad_index_count);
  return check_launch("delta_apply_kernel");
}
