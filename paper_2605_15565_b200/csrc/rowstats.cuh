// Streaming per-row softmax statistics over one logits row (c3 of DESIGN.md §3):
// per-thread online (max, sum 2^(t-max)) over 128-bit vectors, t = x * k with
// k = inv_temperature * log2(e), then a block reduction.  Used by the read-only
// log-prob kernel and by the two-pass (L2 re-read) loss kernel.
#pragma once
#include "common.cuh"

namespace rl {

template <typename T>
struct VecTraits;
template <>
struct VecTraits<float> {
  static constexpr int EPV = 4;  // elements per 16-B vector
  __device__ static __forceinline__ void unpack(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
  __device__ static __forceinline__ float load1(const void* row, int64_t c) {
    return reinterpret_cast<const float*>(row)[c];
  }
  __device__ static __forceinline__ void store1(void* row, int64_t c, float v) {
    reinterpret_cast<float*>(row)[c] = v;
  }
};
struct bf16_t {};  // tag type: logits stored as raw bf16 bit patterns
template <>
struct VecTraits<bf16_t> {
  static constexpr int EPV = 8;
  __device__ static __forceinline__ void unpack(const uint4& v, float* f) {
    f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
    f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
  }
  __device__ static __forceinline__ uint4 pack(const float* f) {
    return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                      pack_bf16x2(f[6], f[7]));
  }
  __device__ static __forceinline__ float load1(const void* row, int64_t c) {
    return __uint_as_float(((uint32_t)reinterpret_cast<const uint16_t*>(row)[c]) << 16);
  }
  __device__ static __forceinline__ void store1(void* row, int64_t c, float v) {
    reinterpret_cast<uint16_t*>(row)[c] = (uint16_t)(pack_bf16x2(v, 0.f) & 0xffffu);
  }
};

// f[j] -= s (resp. = v) for the one j == d in [0, N), if any — compile-time indices only, so the
// array is never placed in local memory (a runtime index f[d] would put it there)
template <int N>
__device__ __forceinline__ void onehot_sub(float (&f)[N], int64_t d, float s) {
#pragma unroll
  for (int j = 0; j < N; ++j) f[j] = (d == j) ? f[j] - s : f[j];
}
template <int N>
__device__ __forceinline__ void onehot_set(float (&f)[N], int64_t d, float v) {
#pragma unroll
  for (int j = 0; j < N; ++j) f[j] = (d == j) ? v : f[j];
}

template <typename T>
__device__ __forceinline__ int64_t elem_bytes() {
  return VecTraits<T>::EPV == 8 ? 2 : 4;
}

// Online update of a thread-local (m, s) with a batch of raw values f[0..n), k > 0.
template <int N>
__device__ __forceinline__ void ms_update(MS& st, const float* f, float k) {
  float bm = f[0];
#pragma unroll
  for (int j = 1; j < N; ++j) bm = fmaxf(bm, f[j]);
  const float nm = fmaxf(st.m, bm * k);
  if (nm == -INFINITY) return;  // everything so far is -inf
  float acc = (st.m == -INFINITY) ? 0.f : st.s * fast_exp2(st.m - nm);
#pragma unroll
  for (int j = 0; j < N; ++j) acc += fast_exp2(fmaf(f[j], k, -nm));
  st.m = nm;
  st.s = acc;
}

// Block-wide (m, s) reduction; result broadcast to every thread. smem: >= 2*32 floats.
template <int THREADS>
__device__ __forceinline__ MS block_reduce_ms(MS v, float* smem) {
  v = warp_reduce_ms(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smem[warp] = v.m;
    smem[32 + warp] = v.s;
  }
  __syncthreads();
  MS r{-INFINITY, 0.f};
  if (lane < THREADS / 32) r = MS{smem[lane], smem[32 + lane]};
  r = warp_reduce_ms(r);
  __syncthreads();  // smem reusable after this
  return r;
}

// Per-thread pass over a row: vectors tid, tid+THREADS, ... (U in flight), then the
// scalar tail [nvec*EPV, V).  `pol` is an L2 cache policy (evict_last for a re-read).
// (t = this thread's index among the THREADS sharing the row; threadIdx.x by default)
template <typename T, int THREADS, int U>
__device__ __forceinline__ MS row_stats_thread(const void* row, int64_t V, float k, uint64_t pol,
                                               int t = -1) {
  constexpr int EPV = VecTraits<T>::EPV;
  const uint4* vrow = reinterpret_cast<const uint4*>(row);
  const int64_t nvec = V / EPV;
  if (t < 0) t = threadIdx.x;
  MS st{-INFINITY, 0.f};
  int64_t i = t;
  for (; i + (int64_t)(U - 1) * THREADS < nvec; i += (int64_t)U * THREADS) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_hint_v4(vrow + i + u * THREADS, pol);
    float f[U * EPV];
#pragma unroll
    for (int u = 0; u < U; ++u) VecTraits<T>::unpack(v[u], f + u * EPV);
    ms_update<U * EPV>(st, f, k);
  }
  for (; i < nvec; i += THREADS) {
    float f[EPV];
    VecTraits<T>::unpack(ld_hint_v4(vrow + i, pol), f);
    ms_update<EPV>(st, f, k);
  }
  for (int64_t c = nvec * EPV + t; c < V; c += THREADS) {
    float f[1] = {VecTraits<T>::load1(row, c)};
    ms_update<1>(st, f, k);
  }
  return st;
}

}  // namespace rl
