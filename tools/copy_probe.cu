// Development probe (not part of the library): the achievable HBM rate of the access patterns the
// fused loss kernel could use, with no loss math.  Rows of V = 151936 bf16 (297 KB), N = 131072.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/copy_probe tools/copy_probe.cu
//   copy_probe [mode]   modes: ldg (LDG/STG grid-stride), tma_stg (TMA ring -> LDS -> STG),
//                              tma_tma (TMA ring -> TMA bulk store), all (default)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

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
  for (int64_t g = 0; g < total; ++g) {
    const int64_t t = g / nch;
    const int j = (int)(g - t * nch);
    const int64_t off = (blockIdx.x + t * gridDim.x) * row_bytes + (int64_t)j * kChunkBytes;
    const uint32_t bytes = (uint32_t)min((int64_t)kChunkBytes, row_bytes - (int64_t)j * kChunkBytes);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(smem_u32(&full[slot])), "r"(ph) : "memory");
    if (MODE == 0 || MODE >= 3) {
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
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "all";
  const int64_t N = 131072, V = 151936, row_bytes = V * 2;
  const size_t bytes = (size_t)N * row_bytes;
  char *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
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
