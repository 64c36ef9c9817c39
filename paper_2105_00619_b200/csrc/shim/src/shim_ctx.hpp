// shim_ctx.hpp -- per-thread C-ABI context for the C++ drop-in shim.
#pragma once

#include "optb_cuda.h"

namespace optb::shim {

// One optb_ctx per host thread on device $OPTB_DEVICE (default 0): the
// reference functions are reentrant and so is the shim.
optb_ctx* context();

// Throws the errors.hpp class matching a non-zero C-ABI status.
void check(int status);

}  // namespace optb::shim
