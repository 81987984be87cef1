// Explicit instance fast_hdmr_kernel<0, 1, 1> (kExact = 0, kCarry = 1, kOrder3 = 1).
#include "fast_hdmr_device.cuh"

namespace ddsg_b200 {
namespace fast {
DDSG_FAST_INSTANCE(0, 1, 1)
}  // namespace fast
}  // namespace ddsg_b200
