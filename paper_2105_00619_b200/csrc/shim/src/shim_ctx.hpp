// shim_ctx.hpp -- per-thread C-ABI context for the C++ drop-in shim.
#pragma once

#include <cstdint>

#include "optb/codec.hpp"
#include "optb_cuda.h"

namespace optb::shim {

// One optb_ctx per host thread on device $OPTB_DEVICE (default 0): the
// reference functions are reentrant and so is the shim.
optb_ctx* context();

// Throws the errors.hpp class matching a non-zero C-ABI status.
void check(int status);

// An EncodedBatch of n images from one chunk's device-layout plane (P words
// of container_value_bytes, little-endian) and parity plane (nullable).
codec::EncodedBatch make_encoded(codec::CodecMode mode, const codec::ImageShape& shape, std::size_t n,
                                 const uint8_t* plane, const uint8_t* offsets);

}  // namespace optb::shim
