// Development probe (not part of the library): the achievable HBM rate of the access patterns the
// fused loss kernel could use, with no loss math.  Rows of V = 151936 bf16 (297 KB), N = 131072.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/copy_probe tools/copy_probe.cu
//   copy_probe [mode]   modes: ldg (LDG/STG grid-stride), tma_stg (TMA ring -> LDS -> STG),
//                              tma_tma (TMA ring -> TMA bulk store), all (default)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_copy(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t j = i + (int64_t)u * gridDim.x * blockDim.x;
      if (j < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(in + j));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t j = i + (int64_t)u * gridDim.x * blockDim.x;
      if (j < n) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + j), "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w) : "memory");
    }
  }
}

constexpr int kWarps = 15, kThreads = kWarps * 32 + 32, kChunkVec = kWarps * 32, kChunkBytes = kChunkVec * 16;

// Each CTA streams rows rowsPerCta apart (row = blockIdx.x + t * gridDim.x), columns [0, V) of bf16.
// mode 0: consumers LDS + STG.cs ; mode 1: one thread issues a TMA bulk store of the chunk.
__device__ int g_inflight_cap = 0;
__device__ int g_pace = 0;
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) tma_copy(const char* in, char* out, int64_t nrows, int64_t row_bytes,
                                                        int nslots) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + nslots;
  unsigned char* ring = sm + ((16 * nslots + 127) & ~127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (int)((row_bytes + kChunkBytes - 1) / kChunkBytes);
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(MODE != 1 ? kWarps : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my_rows = blockIdx.x < nrows ? (nrows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_rows * nch;
  if (warp == kWarps) {
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      const int cap = g_inflight_cap;
      for (int64_t g = 0; g < total; ++g) {
        uint32_t ok = 0;
        if (cap > 0 && g >= cap) {  // at most `cap` chunks in flight: chunk g - cap must have landed
          const int64_t gc = g - cap;
          const uint32_t cs = (uint32_t)(gc % nslots), cp = (uint32_t)((gc / nslots) & 1);
          while (!ok)
            asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_u32(&full[cs])), "r"(cp) : "memory");
          ok = 0;
        }
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(smem_u32(&empty[slot])), "r"(ph ^ 1) : "memory");
        const int64_t t = g / nch;
        const int j = (int)(g - t * nch);
        const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * kChunkBytes;
        const uint32_t bytes = (uint32_t)min((int64_t)kChunkBytes, row_bytes - (int64_t)j * kChunkBytes);
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(bytes) : "memory");
        if (MODE == 5) {
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                           smem_u32(ring + (size_t)slot * kChunkBytes)), "l"(in + off), "r"(bytes), "r"(smem_u32(&full[slot])), "l"(pol) : "memory");
        } else {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(ring + (size_t)slot * kChunkBytes)), "l"(in + off), "r"(bytes), "r"(smem_u32(&full[slot])) : "memory");
        }
        if (++slot == (uint32_t)nslots) { slot = 0; ph ^= 1; }
      }
    }
    return;
  }
  uint32_t slot = 0, ph = 0;
  if (MODE == 2 || MODE == 6) {  // whole row resident before it is processed (pass A constraint); 6: paced
    const int pace = g_pace;  // ns of busy work per chunk in the copy-out (MODE 6)
    for (int64_t t = 0; t < my_rows; ++t) {
      uint32_t s2 = slot, p2 = ph;
      for (int j = 0; j < nch; ++j) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(smem_u32(&full[s2])), "r"(p2) : "memory");
        if (++s2 == (uint32_t)nslots) { s2 = 0; p2 ^= 1; }
      }
      for (int j = 0; j < nch; ++j) {
        const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * kChunkBytes;
        const uint32_t bytes = (uint32_t)min((int64_t)kChunkBytes, row_bytes - (int64_t)j * kChunkBytes);
        if ((uint32_t)tid * 16 < bytes) {
          uint4 v = *reinterpret_cast<const uint4*>(ring + (size_t)slot * kChunkBytes + tid * 16);
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + off + tid * 16), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
        if (++slot == (uint32_t)nslots) { slot = 0; ph ^= 1; }
        if (MODE == 6 && pace > 0) {
          unsigned long long t0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          for (;;) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 >= (unsigned long long)pace) break;
          }
        }
      }
    }
    return;
  }
  uint32_t sink = 0;
  for (int64_t g = 0; g < total; ++g) {
    const int64_t t = g / nch;
    const int j = (int)(g - t * nch);
    const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * kChunkBytes;
    const uint32_t bytes = (uint32_t)min((int64_t)kChunkBytes, row_bytes - (int64_t)j * kChunkBytes);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(smem_u32(&full[slot])), "r"(ph) : "memory");
    if (MODE == 7) {  // read only: fold the data into one word per thread
      if ((uint32_t)tid * 16 < bytes) {
        uint4 v = *reinterpret_cast<const uint4*>(ring + (size_t)slot * kChunkBytes + tid * 16);
        sink ^= v.x ^ v.y ^ v.z ^ v.w;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
    } else if (MODE == 0 || MODE >= 3) {
      if ((uint32_t)tid * 16 < bytes) {
        uint4 v = *reinterpret_cast<const uint4*>(ring + (size_t)slot * kChunkBytes + tid * 16);
        if (MODE == 0 || MODE == 5)
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + off + tid * 16), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        else if (MODE == 3)
          asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + off + tid * 16), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        else
          asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + off + tid * 16), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
    } else {
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + off),
                     "r"(smem_u32(ring + (size_t)slot * kChunkBytes)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
      }
    }
    if (++slot == (uint32_t)nslots) { slot = 0; ph ^= 1; }
  }
  if (MODE == 7 && sink == 0x12345678u) out[tid] = 1;
}

// LDG read only: 4 independent 16-B loads in flight per thread, folded into one word.
__global__ void ldg_read(const uint4* __restrict__ in, uint32_t* out, int64_t n) {
  uint32_t sink = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t j = i + (int64_t)u * gridDim.x * blockDim.x;
      v[u] = make_uint4(0, 0, 0, 0);
      if (j < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(in + j));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) sink ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (sink == 0x12345678u) out[threadIdx.x] = 1;
}

// Per-thread cp.async (LDGSTS) ring: every consumer thread streams ITS OWN 16-B vectors of the
// CTA's rows D chunks ahead into its own smem slots (no producer warp, no mbarriers); COPY =
// also store them (st.global.cs), else read only.
template <int D, bool COPY>
__global__ void __launch_bounds__(kWarps * 32, 1) ldgsts_stream(const char* in, char* out, int64_t nrows, int64_t row_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int tid = threadIdx.x;
  const int nch = (int)((row_bytes + kChunkBytes - 1) / kChunkBytes);
  const int64_t my_rows = blockIdx.x < nrows ? (nrows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_rows * nch;
  auto src = [&](int64_t g, uint32_t& ok) -> int64_t {
    const int64_t t = g / nch;
    const int j = (int)(g - t * nch);
    const int64_t o = (int64_t)j * kChunkBytes + tid * 16;
    ok = g < total && o < row_bytes;
    return (blockIdx.x + t * gridDim.x) * row_bytes + o;
  };
  const uint32_t my = smem_u32(sm) + tid * 16;
  for (int d = 0; d < D; ++d) {
    uint32_t ok;
    const int64_t o = src(d, ok);
    if (ok) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(my + d * kChunkBytes), "l"(in + o) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  uint32_t sink = 0;
  int slot = 0;
  for (int64_t g = 0; g < total; ++g) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    uint32_t ok;
    const int64_t o = src(g, ok);
    if (ok) {
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(my + slot * kChunkBytes));
      if (COPY) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + o), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      else sink ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    uint32_t ok2;
    const int64_t o2 = src(g + D, ok2);
    if (ok2) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(my + slot * kChunkBytes), "l"(in + o2) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (++slot == D) slot = 0;
  }
  if (!COPY && sink == 0x12345678u) out[tid] = 1;
}

__global__ void fill_hash(uint32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 0x9E3779B9u ^ (uint32_t)(i >> 32);
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    p[i] = x & 0xBFFFBFFFu;  // finite bf16 pairs
  }
}

// Row streams: each CTA reads whole rows (row = blockIdx.x + t * gridDim.x), U loads in flight
// per thread — the access pattern of the token_logprob kernel.  STREAMS rows per CTA at a time
// (interleaved) when STREAMS > 1.
template <int THREADS, int U, int STREAMS>
__global__ void __launch_bounds__(THREADS) ldg_rows(const char* in, uint32_t* out, int64_t nrows, int64_t row_bytes) {
  uint32_t sink = 0;
  const int64_t nvec = row_bytes / 16;
  for (int64_t r0 = blockIdx.x * STREAMS; r0 < nrows; r0 += (int64_t)gridDim.x * STREAMS) {
    for (int64_t i = threadIdx.x; i < nvec; i += (int64_t)U * THREADS) {
      uint4 v[STREAMS][U];
#pragma unroll
      for (int st = 0; st < STREAMS; ++st)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = i + u * THREADS;
          v[st][u] = make_uint4(0, 0, 0, 0);
          if (j < nvec && r0 + st < nrows)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[st][u].x), "=r"(v[st][u].y), "=r"(v[st][u].z), "=r"(v[st][u].w) : "l"(in + (r0 + st) * row_bytes + j * 16));
        }
#pragma unroll
      for (int st = 0; st < STREAMS; ++st)
#pragma unroll
        for (int u = 0; u < U; ++u) sink ^= v[st][u].x ^ v[st][u].y ^ v[st][u].z ^ v[st][u].w;
    }
  }
  if (sink == 0x12345678u) out[threadIdx.x] = 1;
}

// TMA read (COPY: + STG) with VPT 16-B vectors per consumer thread per slot, i.e. one bulk copy
// of VPT * 7.5 KB per slot: does a larger bulk transfer raise the per-SM TMA read rate?
template <int VPT, bool COPY>
__global__ void __launch_bounds__(kThreads, 1) tma_sz(const char* in, char* out, int64_t nrows, int64_t row_bytes, int nslots) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int SB = VPT * kChunkBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + nslots;
  unsigned char* ring = sm + ((16 * nslots + 127) & ~127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (int)((row_bytes + SB - 1) / SB);
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(kWarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my_rows = blockIdx.x < nrows ? (nrows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_rows * nch;
  if (warp == kWarps) {
    if (lane == 0) {
      uint32_t slot = 0, ph = 0;
      for (int64_t g = 0; g < total; ++g) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(smem_u32(&empty[slot])), "r"(ph ^ 1) : "memory");
        const int64_t t = g / nch;
        const int j = (int)(g - t * nch);
        const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * SB;
        const uint32_t bytes = (uint32_t)min((int64_t)SB, row_bytes - (int64_t)j * SB);
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + (size_t)slot * SB)), "l"(in + off), "r"(bytes), "r"(smem_u32(&full[slot])) : "memory");
        if (++slot == (uint32_t)nslots) { slot = 0; ph ^= 1; }
      }
    }
    return;
  }
  uint32_t slot = 0, ph = 0, sink = 0;
  for (int64_t g = 0; g < total; ++g) {
    const int64_t t = g / nch;
    const int j = (int)(g - t * nch);
    const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * SB;
    const uint32_t bytes = (uint32_t)min((int64_t)SB, row_bytes - (int64_t)j * SB);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(smem_u32(&full[slot])), "r"(ph) : "memory");
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const uint32_t o = (uint32_t)(u * kChunkVec + tid) * 16;
      if (o < bytes) {
        uint4 v = *reinterpret_cast<const uint4*>(ring + (size_t)slot * SB + o);
        if (COPY) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + off + o), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        else sink ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
    if (++slot == (uint32_t)nslots) { slot = 0; ph ^= 1; }
  }
  if (!COPY && sink == 0x12345678u) out[tid] = 1;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "all";
  const int64_t N = 131072, V = 151936, row_bytes = V * 2;
  const size_t bytes = (size_t)N * row_bytes;
  char *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  if (getenv("PROBE_MEMSET")) CK(cudaMemset(in, 1, bytes));
  else fill_hash<<<1184, 256>>>((uint32_t*)in, (int64_t)(bytes / 4));
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* name, float ms) { printf("%-28s %8.3f ms  %8.1f GB/s (R+W)\n", name, ms, 2.0 * bytes / ms / 1e6); };
  if (!strcmp(mode, "cap")) {
    for (int rep = 0; rep < 2; ++rep)
      for (int nslots : {28}) for (int cap : {0, 6, 8, 10, 12, 16}) for (int m : {0, 2}) {
        CK(cudaMemcpyToSymbol(g_inflight_cap, &cap, sizeof(int)));
        const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
        auto k = m == 0 ? tma_copy<0> : tma_copy<2>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEventRecord(a);
        if (m == 0) k<<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
        else k<<<sms, kThreads, smem>>>(in, out, 2 * N, row_bytes / 2, nslots);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "%s slots=%d cap=%d", m == 0 ? "tma_stg" : "burst", nslots, cap);
        if (rep) report(nm, ms);
      }
    return 0;
  }
  if (!strcmp(mode, "read")) {
    auto rreport = [&](const char* name, float ms, double mult) { printf("%-28s %8.3f ms  %8.1f GB/s (%s)\n", name, ms, mult * bytes / ms / 1e6, mult > 1 ? "R+W" : "read"); };
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      for (int per : {2, 4}) {
        cudaEventRecord(a);
        ldg_read<<<sms * per, 512>>>((const uint4*)in, (uint32_t*)out, (int64_t)(bytes / 16));
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "ldg read %d CTA/SM", per);
        if (rep) rreport(nm, ms, 1);
      }
      for (int nslots : {10, 28}) {
        const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
        CK(cudaFuncSetAttribute(tma_copy<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEventRecord(a);
        tma_copy<7><<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "tma read nslots=%d", nslots);
        if (rep) rreport(nm, ms, 1);
        CK(cudaFuncSetAttribute(tma_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEventRecord(a);
        tma_copy<0><<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        snprintf(nm, 64, "tma copy nslots=%d", nslots);
        if (rep) rreport(nm, ms, 2);
      }
#define LDGSTS_RUN(D)                                                                                     \
      {                                                                                                   \
        const int smem = (D) * kChunkBytes;                                                               \
        CK(cudaFuncSetAttribute(ldgsts_stream<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
        CK(cudaFuncSetAttribute(ldgsts_stream<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));  \
        cudaEventRecord(a);                                                                               \
        ldgsts_stream<D, false><<<sms, kWarps * 32, smem>>>(in, out, N, row_bytes);                       \
        cudaEventRecord(b);                                                                               \
        CK(cudaEventSynchronize(b));                                                                      \
        CK(cudaGetLastError());                                                                           \
        cudaEventElapsedTime(&ms, a, b);                                                                  \
        char nm[64];                                                                                      \
        snprintf(nm, 64, "ldgsts read D=%d", D);                                                          \
        if (rep) rreport(nm, ms, 1);                                                                      \
        cudaEventRecord(a);                                                                               \
        ldgsts_stream<D, true><<<sms, kWarps * 32, smem>>>(in, out, N, row_bytes);                        \
        cudaEventRecord(b);                                                                               \
        CK(cudaEventSynchronize(b));                                                                      \
        cudaEventElapsedTime(&ms, a, b);                                                                  \
        snprintf(nm, 64, "ldgsts copy D=%d", D);                                                          \
        if (rep) rreport(nm, ms, 2);                                                                      \
      }
      LDGSTS_RUN(4) LDGSTS_RUN(8) LDGSTS_RUN(16) LDGSTS_RUN(28)
#define ROWS_RUN(TH, U, ST, PER)                                                           \
      {                                                                                    \
        cudaEventRecord(a);                                                                \
        ldg_rows<TH, U, ST><<<sms * PER, TH>>>(in, (uint32_t*)out, N, row_bytes);          \
        cudaEventRecord(b);                                                                \
        CK(cudaEventSynchronize(b));                                                       \
        CK(cudaGetLastError());                                                            \
        cudaEventElapsedTime(&ms, a, b);                                                   \
        char nm[64];                                                                       \
        snprintf(nm, 64, "rows th=%d U=%d st=%d x%d/SM", TH, U, ST, PER);                   \
        if (rep) rreport(nm, ms, 1);                                                       \
      }
      ROWS_RUN(256, 4, 1, 8) ROWS_RUN(256, 4, 1, 4) ROWS_RUN(256, 4, 1, 1) ROWS_RUN(512, 4, 1, 1)
      ROWS_RUN(512, 8, 1, 1) ROWS_RUN(512, 2, 4, 1) ROWS_RUN(512, 4, 2, 1) ROWS_RUN(256, 4, 1, 2)
    }
    return 0;
  }
  if (!strcmp(mode, "cluster")) {  // the same TMA copy, plain vs cluster launches
    for (int rep = 0; rep < 2; ++rep)
      for (int cl : {1, 2, 4})
        for (int half : {0, 1}) {
          const int nslots = 10;
          const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
          CK(cudaFuncSetAttribute(tma_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          if (cl > 1) CK(cudaFuncSetAttribute(tma_copy<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
          cudaLaunchConfig_t cfg = {};
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cl;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.gridDim = dim3(sms / cl * cl);
          if (cl == 4) cfg.gridDim = dim3(132);
          cfg.blockDim = dim3(kThreads);
          cfg.dynamicSmemBytes = smem;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaEventRecord(a);
          if (half) CK(cudaLaunchKernelEx(&cfg, tma_copy<0>, (const char*)in, out, 2 * N, row_bytes / 2, nslots));
          else CK(cudaLaunchKernelEx(&cfg, tma_copy<0>, (const char*)in, out, N, row_bytes, nslots));
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          char nm[64];
          snprintf(nm, 64, "tma copy cluster=%d %s grid=%d", cl, half ? "half-rows" : "rows", cfg.gridDim.x);
          if (rep) report(nm, ms);
        }
    return 0;
  }
  if (!strcmp(mode, "tmasize")) {
    auto rreport = [&](const char* name, float ms, double mult) { printf("%-28s %8.3f ms  %8.1f GB/s (%s)\n", name, ms, mult * bytes / ms / 1e6, mult > 1 ? "R+W" : "read"); };
#define SZ_RUN(VPT, COPY, NS)                                                                      \
    {                                                                                            \
      const int smem = ((16 * (NS) + 127) & ~127) + (NS) * (VPT) * kChunkBytes;                  \
      CK(cudaFuncSetAttribute(tma_sz<VPT, COPY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
      cudaEventRecord(a);                                                                        \
      tma_sz<VPT, COPY><<<sms, kThreads, smem>>>(in, out, N, row_bytes, NS);                     \
      cudaEventRecord(b);                                                                        \
      CK(cudaEventSynchronize(b));                                                               \
      CK(cudaGetLastError());                                                                    \
      float ms;                                                                                  \
      cudaEventElapsedTime(&ms, a, b);                                                           \
      char nm[64];                                                                               \
      snprintf(nm, 64, "tma %s %dKB x %d slots", COPY ? "copy" : "read", (VPT) * 15 / 2, NS);    \
      if (rep) rreport(nm, ms, COPY ? 2 : 1);                                                    \
    }
    for (int rep = 0; rep < 2; ++rep) {
      SZ_RUN(1, false, 10) SZ_RUN(1, false, 28) SZ_RUN(2, false, 6) SZ_RUN(2, false, 14) SZ_RUN(4, false, 3)
      SZ_RUN(4, false, 7) SZ_RUN(8, false, 3) SZ_RUN(1, true, 10) SZ_RUN(2, true, 6) SZ_RUN(4, true, 3)
      SZ_RUN(4, true, 7) SZ_RUN(8, true, 3)
    }
    return 0;
  }
  if (!strcmp(mode, "paced")) {
    for (int rep = 0; rep < 2; ++rep)
      for (int pace : {0, 100, 200, 250, 300}) {
        CK(cudaMemcpyToSymbol(g_pace, &pace, sizeof(int)));
        const int nslots = 28;
        const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
        CK(cudaFuncSetAttribute(tma_copy<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEventRecord(a);
        tma_copy<6><<<sms, kThreads, smem>>>(in, out, 2 * N, row_bytes / 2, nslots);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "burst paced %d ns/chunk", pace);
        if (rep) report(nm, ms);
      }
    return 0;
  }
  if (!strcmp(mode, "hints")) {
    for (int rep = 0; rep < 2; ++rep)
      for (int nslots : {10, 28}) {
        const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
        const char* names[] = {"st.cs", "", "", "st.wb", "st.L1::no_alloc", "st.cs + tma evict_first"};
        for (int m : {0, 3, 4, 5}) {
          cudaFuncAttributes fa;
          void (*k)(const char*, char*, int64_t, int64_t, int) = m == 0 ? tma_copy<0> : m == 3 ? tma_copy<3> : m == 4 ? tma_copy<4> : tma_copy<5>;
          (void)fa;
          CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          cudaEventRecord(a);
          k<<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          char nm[64];
          snprintf(nm, 64, "%s nslots=%d", names[m], nslots);
          if (rep) report(nm, ms);
        }
      }
    return 0;
  }
  for (int rep = 0; rep < 2; ++rep) {
    if (!strcmp(mode, "all") || !strcmp(mode, "ldg")) {
      for (int per : {2, 4, 8}) {
        cudaEventRecord(a);
        ldg_copy<<<sms * per, 512>>>((const uint4*)in, (uint4*)out, (int64_t)(bytes / 16));
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "ldg/stg %d CTA/SM", per);
        if (rep) report(nm, ms);
      }
    }
    for (int m = 0; m < 3; ++m) {
      if (strcmp(mode, "all") && strcmp(mode, m == 0 ? "tma_stg" : m == 1 ? "tma_tma" : "burst")) continue;
      for (int nslots : {10, 20, 28}) {
        if (m == 2 && nslots < 21) continue;
        const int smem = ((16 * nslots + 127) & ~127) + nslots * kChunkBytes;
        if (m == 0) {
          CK(cudaFuncSetAttribute(tma_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          cudaEventRecord(a);
          tma_copy<0><<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
        } else if (m == 2) {
          // per-CTA half rows (the loss kernel's cluster slice): row_bytes/2, 2N rows
          CK(cudaFuncSetAttribute(tma_copy<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          cudaEventRecord(a);
          tma_copy<2><<<sms, kThreads, smem>>>(in, out, 2 * N, row_bytes / 2, nslots);
        } else {
          CK(cudaFuncSetAttribute(tma_copy<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          cudaEventRecord(a);
          tma_copy<1><<<sms, kThreads, smem>>>(in, out, N, row_bytes, nslots);
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        char nm[64];
        snprintf(nm, 64, "%s nslots=%d", m == 0 ? "tma->lds->stg" : m == 1 ? "tma->tma_store" : "burst(half row)", nslots);
        if (rep) report(nm, ms);
      }
    }
  }
  return 0;
}
