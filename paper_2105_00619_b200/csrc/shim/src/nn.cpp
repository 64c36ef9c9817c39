// shim/src/nn.cpp -- decode-layer input transform (nn.cpp:153-192) over the C
// ABI: chunk validation with the reference's messages (nn.cpp:158-175), then
// one optb_decode_host call per run of equally sized chunks with the fused
// float(q)*scale epilogue (fp32, or the binary16 tape store).
#include <cstring>
#include <string>

#include "optb/decode_layer.hpp"
#include "optb_cuda.h"
#include "shim_ctx.hpp"

namespace optb::nn {
namespace {

template <typename T>
std::vector<T> run(std::span<const codec::EncodedBatch> chunks, codec::CodecMode mode,
                   std::size_t n_images, float scale, int dtype) {
  if (chunks.empty()) throw ShapeError("layer 0: no encoded batches supplied");
  std::size_t rows = 0;
  for (const auto& enc : chunks) {
    if (enc.mode != mode)
      throw ShapeError(std::string("layer 0: decode expects mode ") + codec::mode_name(mode) +
                       " but batch uses " + codec::mode_name(enc.mode));
    if (!(enc.shape == chunks[0].shape)) throw ShapeError("layer 0: encoded chunks disagree on image shape");
    rows += enc.n_images;
  }
  if (n_images != 0 && rows != n_images)
    throw ShapeError("layer 0: decode expects " + std::to_string(n_images) + " images, got " +
                     std::to_string(rows));
  const std::size_t P = chunks[0].pixel_count();
  const std::size_t wc = codec::container_value_bytes(mode);
  std::vector<T> out(rows * P);
  std::size_t row = 0;
  for (std::size_t k = 0; k < chunks.size();) {
    const std::size_t n = chunks[k].n_images;
    std::size_t j = k;
    while (j < chunks.size() && chunks[j].n_images == n) ++j;
    optb_layout L{static_cast<int32_t>(mode), static_cast<uint32_t>(n), P, n, j - k};
    const uint64_t ost = optb_offsets_stride(L.mode, P, L.per_chunk);
    std::vector<uint8_t> planes((j - k) * P * wc);
    std::vector<uint8_t> offs(std::max<uint64_t>((j - k) * ost, 16));
    for (std::size_t c = k; c < j; ++c) {
      const auto& enc = chunks[c];
      if (n == 0) throw FormatError("decode: empty encoded batch");
      if (mode == codec::CodecMode::Float64Faithful) {
        if (enc.packed_f64.size() != P) throw FormatError("decode: container plane size mismatch");
        std::memcpy(planes.data() + (c - k) * P * wc, enc.packed_f64.data(), P * 8);
      } else {
        if (enc.packed.size() != P) throw FormatError("decode: container plane size mismatch");
        for (std::size_t p = 0; p < P; ++p) std::memcpy(planes.data() + ((c - k) * P + p) * wc, &enc.packed[p], wc);
      }
      std::copy(enc.offsets.begin(), enc.offsets.end(), offs.begin() + static_cast<std::ptrdiff_t>((c - k) * ost));
    }
    const optb_epilogue E{dtype, scale, nullptr, nullptr, nullptr, 0};
    shim::check(optb_decode_host(shim::context(), &L, planes.data(), offs.data(), &E, out.data() + row * P));
    row += n * (j - k);
    k = j;
  }
  return out;
}

}  // namespace

std::vector<float> decode_input(std::span<const codec::EncodedBatch> chunks, codec::CodecMode mode,
                                std::size_t n_images, float scale) {
  return run<float>(chunks, mode, n_images, scale, OPTB_OUT_F32);
}

std::vector<std::uint16_t> decode_input_half(std::span<const codec::EncodedBatch> chunks,
                                             codec::CodecMode mode, std::size_t n_images, float scale) {
  return run<std::uint16_t>(chunks, mode, n_images, scale, OPTB_OUT_F16);
}

}  // namespace optb::nn
