// (6) M2PO second-moment trust mask — NEXT 1 of SURVEY.md §8(f), reading M1 of DESIGN.md §3
// ("M2PO ... with m²-threshold 0.01"; the paper gives no formula).
//
// Per valid token m_t = (logp_t - old_t)^2 (fp32: the kernel's precision takes the decision);
// drop the fewest largest-m tokens so that the mean m of the kept ones is <= tau.  Equivalently
// keep the j* smallest, j* = max{ j : sum of the j smallest <= tau * j }, ties of equal m ordered
// by token index (the larger index is kept first, matching the oracle's descending order with
// ties by ascending index).  The selection is global over the ranks of `comm` (its keys are
// all-gathered: every rank sorts the same array and derives the same cut).
//
//   keys: fp32 bit pattern of m (order-preserving for m >= 0); invalid tokens 0xFFFFFFFF (last)
//   array position i holds global token g = G - 1 - i, so the stable ascending radix sort keeps
//   ties in descending g
//   prefix sums of the sorted m in fp64 (small first: no cancellation near the cut)
//   j* by atomicMax over the j that satisfy the bound (the mean is monotone in j)
#include <cub/cub.cuh>
#include <nccl.h>

#include "common.cuh"

namespace rl {

ncclComm_t comm_nccl(rl_comm* c);
int32_t comm_rank(const rl_comm* c);
int32_t comm_size(const rl_comm* c);

constexpr uint32_t kInvalidKey = 0xFFFFFFFFu;

__global__ void m2po_keys_kernel(const float* __restrict__ logp, const float* __restrict__ old,
                                 const uint8_t* __restrict__ valid, int64_t n, uint32_t* __restrict__ keys) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const bool v = valid == nullptr || valid[t] != 0;
    const float d = __fsub_rn(logp[t], old[t]);
    const float m = __fmul_rn(d, d);
    keys[t] = v ? __float_as_uint(m) : kInvalidKey;  // m >= 0 (or NaN: sorts after +inf)
  }
}

// reverse the gathered keys into sort order (position i <- global token G-1-i) and set the values
__global__ void m2po_reverse_kernel(const uint32_t* __restrict__ keys, int64_t G, uint32_t* __restrict__ kin,
                                    uint32_t* __restrict__ vin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = G - 1 - i;
    kin[i] = keys[g];
    vin[i] = (uint32_t)g;
  }
}

__global__ void m2po_values_kernel(const uint32_t* __restrict__ ksorted, int64_t G, double* __restrict__ mval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ksorted[i];
    mval[i] = k == kInvalidKey ? 0.0 : (double)__uint_as_float(k);
  }
}

// j* = max { j in [1, nv] : P_j <= tau j } (P_j = inclusive prefix at position j-1); nv = number of
// valid keys (they precede the invalid ones)
__global__ void m2po_cut_kernel(const uint32_t* __restrict__ ksorted, const double* __restrict__ prefix, int64_t G,
                                double tau, unsigned long long* __restrict__ jstar, unsigned long long* __restrict__ nvalid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < G; i += (int64_t)gridDim.x * blockDim.x) {
    const bool valid = ksorted[i] != kInvalidKey;
    if (valid && (i + 1 == G || ksorted[i + 1] == kInvalidKey)) *nvalid = (unsigned long long)(i + 1);
    if (valid && prefix[i] <= tau * (double)(i + 1)) atomicMax(jstar, (unsigned long long)(i + 1));
  }
}

// this rank's tokens among the kept sorted positions [0, j*)
__global__ void m2po_mask_kernel(const uint32_t* __restrict__ vsorted, const unsigned long long* __restrict__ jstar,
                                 int64_t g0, int64_t n, uint8_t* __restrict__ mask) {
  const int64_t j = (int64_t)*jstar;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < j; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)vsorted[i] - g0;
    if (g >= 0 && g < n) mask[g] = 1;
  }
}

__global__ void m2po_stats_kernel(const double* __restrict__ prefix, const unsigned long long* __restrict__ jstar,
                                  const unsigned long long* __restrict__ nvalid, double* __restrict__ out) {
  const double nv = (double)*nvalid, j = (double)*jstar;
  out[0] = nv;
  out[1] = nv - j;                                           // k*: tokens masked by M2PO
  out[2] = nv > 0 ? prefix[(int64_t)nv - 1] / nv : 0.0;     // mean m before
  out[3] = j > 0 ? prefix[(int64_t)j - 1] / j : 0.0;         // mean m of the kept tokens
  out[4] = j;                                                // kept tokens (the loss's N_active)
}

struct M2poLayout {
  size_t keys, kin, vin, kout, vout, prefix, scal, temp, total;
};

static M2poLayout m2po_layout(int64_t n, int32_t P) {
  const int64_t G = n * P;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)G);
  cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (double*)nullptr, (double*)nullptr, (int)G);
  M2poLayout L;
  size_t off = 0;
  auto al = [&](size_t b) {
    const size_t o = off;
    off += (b + 255) & ~(size_t)255;
    return o;
  };
  L.keys = al((size_t)G * 4);
  L.kin = al((size_t)G * 4);
  L.vin = al((size_t)G * 4);
  L.kout = al((size_t)G * 4);
  L.vout = al((size_t)G * 4);
  L.prefix = al((size_t)G * 8);
  L.scal = al(64);
  L.temp = al(std::max(sort_bytes, scan_bytes));
  L.total = off;
  return L;
}

}  // namespace rl

extern "C" size_t rl_m2po_workspace_size(int64_t n_tokens, int32_t nranks) {
  if (n_tokens < 0 || nranks < 1 || n_tokens * (int64_t)nranks >= ((int64_t)1 << 31)) return 0;
  return rl::m2po_layout(std::max<int64_t>(n_tokens, 1), nranks).total;
}

extern "C" rl_status rl_m2po_mask(const float* logp, const float* old_logp, const uint8_t* valid, int64_t n_tokens,
                                  float tau, rl_comm* comm, uint8_t* mask_out, double* stats_out, void* workspace,
                                  size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (n_tokens < 0) return fail(RL_ERR_INVALID_ARGUMENT, "n_tokens < 0");
  if (!(tau >= 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "tau must be >= 0");
  const int32_t P = comm ? comm_size(comm) : 1;
  const int32_t rank = comm ? comm_rank(comm) : 0;
  if (n_tokens * (int64_t)P >= ((int64_t)1 << 31)) return fail(RL_ERR_UNSUPPORTED, "n_tokens * nranks >= 2^31");
  if (n_tokens > 0 && (!logp || !old_logp || !mask_out)) return fail(RL_ERR_INVALID_ARGUMENT, "NULL logp/old_logp/mask_out");
  if (!stats_out) return fail(RL_ERR_INVALID_ARGUMENT, "NULL stats_out");
  const int64_t n = std::max<int64_t>(n_tokens, 1);
  const M2poLayout L = m2po_layout(n, P);
  if (!workspace || workspace_bytes < L.total)
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes", L.total);
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)workspace;
  uint32_t* keys = (uint32_t*)(w + L.keys);
  uint32_t *kin = (uint32_t*)(w + L.kin), *vin = (uint32_t*)(w + L.vin);
  uint32_t *kout = (uint32_t*)(w + L.kout), *vout = (uint32_t*)(w + L.vout);
  double* prefix = (double*)(w + L.prefix);
  unsigned long long* scal = (unsigned long long*)(w + L.scal);  // [0] j*, [1] n_valid
  const int64_t G = n * P;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((G + threads - 1) / threads, 148 * 8);
  // this rank's keys (a rank with no tokens contributes one invalid key: every rank sends n)
  if (n_tokens > 0) {
    m2po_keys_kernel<<<blocks, threads, 0, s>>>(logp, old_logp, valid, n_tokens, keys + (size_t)rank * n);
  } else if (cudaMemsetAsync(keys + (size_t)rank * n, 0xFF, 4, s) != cudaSuccess) {
    return check_launch("m2po memset");
  }
  rl_status st = check_launch("m2po_keys_kernel");
  if (st != RL_OK) return st;
  if (P > 1) {
    ncclResult_t r = ncclAllGather(keys + (size_t)rank * n, keys, (size_t)n, ncclUint32, comm_nccl(comm), s);
    if (r != ncclSuccess) return fail(RL_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  }
  m2po_reverse_kernel<<<blocks, threads, 0, s>>>(keys, G, kin, vin);
  size_t temp_bytes = L.total - L.temp;
  if (cub::DeviceRadixSort::SortPairs(w + L.temp, temp_bytes, kin, kout, vin, vout, (int)G, 0, 32, s) != cudaSuccess)
    return check_launch("cub radix sort");
  m2po_values_kernel<<<blocks, threads, 0, s>>>(kout, G, prefix);
  temp_bytes = L.total - L.temp;
  if (cub::DeviceScan::InclusiveSum(w + L.temp, temp_bytes, prefix, prefix, (int)G, s) != cudaSuccess)
    return check_launch("cub scan");
  if (cudaMemsetAsync(scal, 0, 16, s) != cudaSuccess) return check_launch("m2po memset");
  m2po_cut_kernel<<<blocks, threads, 0, s>>>(kout, prefix, G, (double)tau, scal, scal + 1);
  if (n_tokens > 0) {
    if (cudaMemsetAsync(mask_out, 0, (size_t)n_tokens, s) != cudaSuccess) return check_launch("m2po memset");
    m2po_mask_kernel<<<blocks, threads, 0, s>>>(vout, scal, (int64_t)rank * n, n_tokens, mask_out);
  }
  m2po_stats_kernel<<<1, 1, 0, s>>>(prefix, scal, scal + 1, stats_out);
  return check_launch("m2po kernels");
}
