// Explicit instance fast_hdmr_kernel<0, 1, 0> (kExact = 0, kCarry = 1, kOrder3 = 0).
#include "fast_hdmr_device.cuh"

namespace ddsg_b200 {
namespace fast {
DDSG_FAST_INSTANCE(0, 1, 0)
}  // namespace fast
}  // namespace ddsg_b200
