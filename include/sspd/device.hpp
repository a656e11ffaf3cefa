// sspd/device.hpp -- B200 extension of the sspd API: which GPU new grids
// live on.  Grids are created on the calling thread's current sspd device
// (default: $SSPD_DEVICE, else 0).  There is no CPU fallback: constructing a
// grid without a usable sm_100 device throws std::runtime_error.
#pragma once

#include <vector>

namespace sspd {

void set_device(int device);
int current_device();
int device_count();
// CUDA ordinals of the usable (sm_100) devices, ascending; what
// RunConfig::devices > 1 spreads routers over.
std::vector<int> device_ordinals();

}  // namespace sspd
