/*
 * rl_policy_dev.h — development hooks of librlpolicy.so (NOT part of the product ABI in
 * rl_policy.h).  The tests and tools use them to A/B alternative kernels that are kept for
 * parity coverage; the library never reads environment variables.
 *
 * rl_dev_set_option(key, value): sets a process-wide option and returns its previous value
 * (-1 for an unknown key).  Keys:
 *   0 RL_DEV_LOSS_KERNEL  rl_policy_loss_fwd_bwd kernel: 0 = single-visit cluster kernel
 *                         (default), 1 = exact max-referenced two-pass kernel for every row
 *   1 RL_DEV_VP_PATH      fused rl_vocab_parallel_logprob: 0 = in-kernel peer exchange when
 *                         rl_comm_enable_peer_exchange succeeded (default), 1 = NCCL path
 *   2 RL_DEV_LM_SPLITS    rl_lmhead_logprob vocabulary splits: 0 = cost model (default), else
 *                         the split count (clamped to what the workspace holds)
 *   3 RL_DEV_VP_KERNEL    peer-exchange vocab-parallel kernel: 0 = default (the L2 re-read ring
 *                         kernel on more than one rank; on one rank the register-cache kernel when
 *                         the shard fits it), 1 = the ring kernel, 2 = the register-cache kernel
 *                         whenever the shard fits it
 *   4 RL_DEV_VC_GROUPS    vp_cache_kernel collector groups (0 = min(8, 32 / P))
 *   5 RL_DEV_VC_ROWS      vp_cache_kernel rows parked in shared memory + 1 (0 = default)
 *   6 RL_DEV_VC_PUB       vp_cache_kernel record send + 1: 0 collector (strong stores), 1 last
 *                         consumer warp (weak stores; default), 2 collector (weak stores)
 *   7 RL_DEV_LM_PAIR      LM-head kernels: 0 = CTA pairs (cta_group::2) for the backward's gradient
 *                         kernel, single CTAs for the log-prob kernel (default); 1 = single CTAs;
 *                         2 = pairs for both (pairs need >= 2 token blocks)
 *   8 RL_DEV_LM_GEMM      rl_lmhead_loss_bwd's dh / dW GEMMs: 0 / 1 = cuBLAS (default), 2 = the
 *                         hand-written lm_gemm_kernel on tcgen05 (with RL_DEV_LM_PAIR = 2: CTA pairs)
 *   9 RL_DEV_VR_DELAY     vp_ring_kernel rows between the two reads of a row slice (0 = the L2-window
 *                         rule, default; else that many, with one row per service group)
 *  10 RL_DEV_VC_TMEM     vp_cache_kernel: where the rows awaiting their scale are parked: 0 = default
 *                         (tensor memory for shards of <= 2,688 vectors on more than one rank, else
 *                         shared memory), 1 = shared memory, 2 = tensor memory (2 rows at the wide,
 *                         4 at the narrow widths)
 * Options are read at launch time; set them before the calls they should affect.
 */
#ifndef RL_POLICY_DEV_H_
#define RL_POLICY_DEV_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
#define RL_DEV_LOSS_KERNEL 0
#define RL_DEV_VP_PATH 1
#define RL_DEV_LM_SPLITS 2
#define RL_DEV_VP_KERNEL 3
#define RL_DEV_VC_GROUPS 4
#define RL_DEV_VC_ROWS 5
#define RL_DEV_VC_PUB 6
#define RL_DEV_LM_PAIR 7
#define RL_DEV_LM_GEMM 8
#define RL_DEV_VR_DELAY 9
#define RL_DEV_VC_TMEM 10
int32_t rl_dev_set_option(int32_t key, int32_t value);
#ifdef __cplusplus
}
#endif
#endif
