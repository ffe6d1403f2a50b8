// rgb_blocked.cu -- placeholder until the tensor-core blocked kernel lands.
#include "rgb_common.cuh"

namespace rgb {
bool blocked_supports(const rgb_config&) { return false; }
int launch_blocked(const rgb_config&, rgb_state&, const void*, int64_t, const void*, int64_t, int64_t,
                   const rgb_logs&, cudaStream_t, int) {
  return RGB_E_UNSUPPORTED;
}
}  // namespace rgb
