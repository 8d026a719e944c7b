// (1) GRPO group-relative advantages — c1 of DESIGN.md §3.
// PAPER.md:572 "group-level reward normalization", PAPER.md:580 GRPO, 8 rollouts per prompt
// (PAPER.md:574); zero-variance predicate SPEC.md:56-64 (exact equality, singleton -> zero,
// SPEC.md:232); optional batch-level advantage normalization (reading Z6).
//
// Bit-exact to the fp64 definition: every floating-point step uses the explicitly rounded
// intrinsics (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn), so no FMA contraction can
// change the rounding order; sums are sequential in member order (reading Z7).
// Work is tiny (8 B per sequence): one CTA, groups spread over its threads; the batch-norm
// sums are done by one thread sequentially (their order is part of the definition).
#include "common.cuh"

namespace rl {

__global__ void __launch_bounds__(1024) group_advantage_kernel(
    const double* __restrict__ rewards, const int32_t* __restrict__ cu_groups, int32_t n_groups,
    int32_t n_seq, int32_t std_mode, double eps, int32_t batch_norm, double bn_eps,
    const int32_t* __restrict__ seq_weight, double* __restrict__ adv64, float* __restrict__ adv_out,
    uint8_t* __restrict__ zero_var_out) {
  for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
    const int lo = cu_groups[g], hi = cu_groups[g + 1];
    const int n = hi - lo;
    if (n <= 0 || lo < 0 || hi > n_seq) {  // empty group -> invalid-argument
      if (zero_var_out) zero_var_out[g] = 2;
      continue;
    }
    const double first = rewards[lo];
    bool allequal = true;
    for (int i = lo; i < hi; ++i) allequal = allequal && (rewards[i] == first);
    if (zero_var_out) zero_var_out[g] = allequal ? 1 : 0;
    if (allequal) {
      for (int i = lo; i < hi; ++i) {
        if (batch_norm) adv64[i] = 0.0;
        else adv_out[i] = 0.0f;
      }
      continue;
    }
    double acc = 0.0;
    for (int i = lo; i < hi; ++i) acc = __dadd_rn(acc, rewards[i]);
    const double mu = __ddiv_rn(acc, (double)n);
    double q = 0.0;
    for (int i = lo; i < hi; ++i) {
      const double d = __dadd_rn(rewards[i], -mu);
      q = __dadd_rn(q, __dmul_rn(d, d));
    }
    double den = 1.0;
    const bool use_std = std_mode != RL_STD_NONE;
    if (std_mode == RL_STD_UNBIASED) den = __dadd_rn(__dsqrt_rn(__ddiv_rn(q, (double)(n - 1))), eps);
    else if (std_mode == RL_STD_BIASED) den = __dadd_rn(__dsqrt_rn(__ddiv_rn(q, (double)n)), eps);
    for (int i = lo; i < hi; ++i) {
      const double d = __dadd_rn(rewards[i], -mu);
      const double a = use_std ? __ddiv_rn(d, den) : d;
      if (batch_norm) adv64[i] = a;
      else adv_out[i] = __double2float_rn(a);
    }
  }
  if (!batch_norm) return;
  __syncthreads();
  __shared__ double s_mu, s_den;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    // W = sum L_i (exact integer); mu_B = (sum L_i*A_i)/W; v_B = (sum L_i*((A_i-mu_B)^2))/W
    long long W = 0;
    for (int i = 0; i < n_seq; ++i) W += seq_weight[i];
    s_skip = (W <= 0);
    if (W > 0) {
      double s = 0.0;
      for (int i = 0; i < n_seq; ++i) s = __dadd_rn(s, __dmul_rn((double)seq_weight[i], adv64[i]));
      const double mu = __ddiv_rn(s, (double)W);
      double v = 0.0;
      for (int i = 0; i < n_seq; ++i) {
        const double e = __dadd_rn(adv64[i], -mu);
        v = __dadd_rn(v, __dmul_rn((double)seq_weight[i], __dmul_rn(e, e)));
      }
      s_mu = mu;
      s_den = __dadd_rn(__dsqrt_rn(__ddiv_rn(v, (double)W)), bn_eps);
    }
  }
  __syncthreads();
  // members of invalid groups were never written to adv64: only touch valid groups
  for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
    const int lo = cu_groups[g], hi = cu_groups[g + 1];
    if (hi - lo <= 0 || lo < 0 || hi > n_seq) continue;
    for (int i = lo; i < hi; ++i) {
      const double a = s_skip ? adv64[i] : __ddiv_rn(__dadd_rn(adv64[i], -s_mu), s_den);
      adv_out[i] = __double2float_rn(a);
    }
  }
}

}  // namespace rl

extern "C" size_t rl_group_advantage_workspace_size(int32_t n_seq) {
  return n_seq > 0 ? (size_t)n_seq * sizeof(double) : 0;
}

extern "C" rl_status rl_group_advantage(const double* rewards, const int32_t* cu_groups,
                                        int32_t n_groups, int32_t n_seq, int32_t std_mode,
                                        double eps, int32_t batch_norm, double bn_eps,
                                        const int32_t* seq_weight, void* workspace,
                                        size_t workspace_bytes, float* adv_out,
                                        uint8_t* zero_var_out, rl_stream stream) {
  using namespace rl;
  if (n_groups < 0 || n_seq < 0) return fail(RL_ERR_INVALID_ARGUMENT, "n_groups/n_seq < 0");
  if (std_mode < RL_STD_UNBIASED || std_mode > RL_STD_NONE)
    return fail(RL_ERR_INVALID_ARGUMENT, "bad std_mode %d", std_mode);
  if (n_groups == 0 && n_seq == 0) return RL_OK;
  if (!rewards || !cu_groups || !adv_out) return fail(RL_ERR_INVALID_ARGUMENT, "NULL rewards/cu_groups/adv_out");
  if (n_groups == 0) return fail(RL_ERR_INVALID_ARGUMENT, "n_seq > 0 but no groups");
  if (batch_norm) {
    if (!seq_weight) return fail(RL_ERR_INVALID_ARGUMENT, "batch_norm needs seq_weight");
    if (!workspace || workspace_bytes < rl_group_advantage_workspace_size(n_seq))
      return fail(RL_ERR_WORKSPACE, "batch_norm needs %zu workspace bytes",
                  rl_group_advantage_workspace_size(n_seq));
  }
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  group_advantage_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      rewards, cu_groups, n_groups, n_seq, std_mode, eps, batch_norm, bn_eps, seq_weight,
      (double*)workspace, adv_out, zero_var_out);
  return check_launch("group_advantage_kernel");
}
