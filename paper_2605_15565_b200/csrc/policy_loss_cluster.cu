// Row-resident cluster kernel "R" of the fused loss — placeholder until the
// kernel lands; the entry point falls back to the two-pass kernel on RL_ERR_UNSUPPORTED.
#include "loss_common.cuh"

namespace rl {
rl_status launch_loss_cluster(const void*, int32_t, int64_t, int64_t, int64_t, const int32_t*,
                              const float*, const uint8_t*, const int32_t*, const float*,
                              const int32_t*, const int32_t*, const Knobs&, void*, float*,
                              uint8_t*, double*, int*, cudaStream_t) {
  return RL_ERR_UNSUPPORTED;
}
}  // namespace rl
