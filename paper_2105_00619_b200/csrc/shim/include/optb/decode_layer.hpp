// optb/decode_layer.hpp -- the decode layer's input transform (nn.cpp:153-192)
// as a free function over encoded chunks, for callers of the reference's
// nn::decode_input whose network lives elsewhere (optb::nn is out of scope of
// the B200 path).  Validation and messages follow nn.cpp:158-175; the values
// are float(q) * scale (nn.cpp:186), optionally stored as binary16 like the
// MixedPrecision tape (nn.cpp:141-146, 235).  Output is (rows, pixels) row-major.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "optb/codec.hpp"

namespace optb::nn {

std::vector<float> decode_input(std::span<const codec::EncodedBatch> chunks, codec::CodecMode mode,
                                std::size_t n_images, float scale);
std::vector<std::uint16_t> decode_input_half(std::span<const codec::EncodedBatch> chunks,
                                             codec::CodecMode mode, std::size_t n_images,
                                             float scale);

}  // namespace optb::nn
