// Thin inline-PTX wrappers for the sm_100a features the row-resident kernel uses:
// mbarriers, cp.async.bulk (TMA bulk copy global -> shared), cluster rank / DSMEM mapping,
// remote mbarrier arrive and cluster barriers.
#pragma once
#include <stdint.h>

namespace rl {
namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// arrive + set expected transaction bytes (producer, before issuing the bulk copy)
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on the barrier at the same smem offset in CTA `rank` of this cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// relaxed remote arrive: no release fence (a cluster-scope release compiles to MEMBAR.ALL.GPU);
// for arrivals that order nothing but async-proxy / tensor-memory work tracked by the barrier itself
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// acquire at cluster scope (for barriers that remote CTAs arrive on)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// TMA bulk copy global -> shared (this CTA), completion signalled on `bar` (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// store 16 bytes into the same smem offset of CTA `rank` (DSMEM)
__device__ __forceinline__ void st_remote_v4(void* local_addr, uint32_t rank, float a, float b, float c,
                                             float d) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// 16-B store into the same smem offset of cluster CTA `rank`, completing 16 tx bytes on that CTA's
// mbarrier at the offset of `bar` (st.async: no release fence, so the sender does not wait for its
// own earlier global stores — the receiver arms its barrier with mbar_arrive_expect_tx).
__device__ __forceinline__ void st_async_v4(void* local_addr, uint64_t* bar, uint32_t rank, float a, float b,
                                            float c, float d) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_addr)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(rb)
               : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

}  // namespace sm100
}  // namespace rl

// ---- 32-bit shared-address variants (keep the hot loops free of generic->shared conversions)
namespace rl {
namespace sm100 {
__device__ __forceinline__ bool mbar_try_wait_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait_a(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint4 lds128_a(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
}  // namespace sm100
}  // namespace rl

namespace rl {
namespace sm100 {
// A consumer thread releases a TMA ring slot (the slot's empty barrier counts every consumer
// THREAD).  The arrive must not take effect before this thread's ld.shared of the slot has read
// it, or the producer may refill the slot under the load.  On sm_100a an
// mbarrier.arrive.release issued right after ld.shared — by lane 0 for its warp or by each lane
// for itself — was measured to overtake the load when the warp's loads queue behind global
// traffic (rare wrong row statistics in back-to-back 4-GPU vocab-parallel calls: tools/race_check.py).
// So the arrive's predicate depends on the loaded data: `dep` = bits of the vectors this thread
// read from the slot, `zero` = a runtime 0 that ptxas cannot fold; (dep != zero || zero == 0) is
// always true, but the arrive issues only once the loads have returned.
constexpr int kRelPerWarp = 32;  // every consumer thread arrives for itself
__device__ __forceinline__ void mbar_release_after(uint32_t bar, uint32_t dep, uint32_t zero) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, %2;\n\tsetp.eq.u32 q, %2, 0;\n\tor.pred p, p, q;\n\t"
      "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n\t}" ::"r"(bar),
      "r"(dep), "r"(zero)
      : "memory");
}
}  // namespace sm100
}  // namespace rl

namespace rl {
namespace sm100 {
// bulk L2 prefetch of [src, src+bytes) (bytes % 16 == 0): pulls a future row slice into L2 so the
// later TMA load of each chunk is an L2 hit (lookahead beyond the shared-memory ring).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}
}  // namespace sm100
}  // namespace rl

namespace rl {
namespace sm100 {
// shared-memory atomic add with acquire-release semantics at CTA scope; returns the old value
__device__ __forceinline__ uint32_t atom_add_acqrel(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
}  // namespace sm100
}  // namespace rl

namespace rl {
namespace sm100 {
// TMA bulk copy global -> shared without an L2 cache hint (measured 3-4 % faster than evict_first
// for this streaming pattern, tools/copy_probe.cu "hints")
__device__ __forceinline__ void bulk_g2s_nohint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// polite polling wait (test_wait + nanosleep): for a lane that shares its warp with another
// lane's loop, so the other divergent path keeps getting issue slots
__device__ __forceinline__ void mbar_wait_polite(uint64_t* bar, uint32_t parity, bool cluster_acquire) {
  for (;;) {
    uint32_t ok;
    if (cluster_acquire)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}
}  // namespace sm100
}  // namespace rl
