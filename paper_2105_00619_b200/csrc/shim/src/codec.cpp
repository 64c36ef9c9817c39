// shim/src/codec.cpp -- optb::codec (reference API, codec.hpp) over the C ABI.
// Host-side: argument validation with the reference's messages
// (codec.cpp:79-97, 150-158), marshalling between std::vector<u128> and the
// [P][Wc] device layout, and the OPTB byte format (codec.cpp:228-381).  All
// packing / unpacking runs on the GPU (optb_encode_host / optb_decode_host).
#include "optb/codec.hpp"

#include <bit>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <string>

#include "optb_cuda.h"
#include "shim_ctx.hpp"

namespace optb {

void throw_status(int status, const std::string& message) {
  switch (status) {
    case OPTB_ERR_SHAPE: throw ShapeError(message);
    case OPTB_ERR_CAPACITY: throw CapacityError(message);
    case OPTB_ERR_FORMAT: throw FormatError(message);
    default: throw Error(message);
  }
}

namespace shim {

optb_ctx* context() {
  thread_local struct Holder {
    optb_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) optb_ctx_destroy(ctx);
    }
  } holder;
  if (!holder.ctx) {
    const char* env = std::getenv("OPTB_DEVICE");
    check(optb_ctx_create(env ? std::atoi(env) : 0, &holder.ctx));
  }
  return holder.ctx;
}

void check(int status) {
  if (status != OPTB_OK) throw_status(status, optb_last_error());
}

}  // namespace shim
}  // namespace optb

namespace optb::shim {

codec::EncodedBatch make_encoded(codec::CodecMode mode, const codec::ImageShape& shape, std::size_t n,
                                 const uint8_t* plane, const uint8_t* offsets) {
  using namespace codec;
  const std::size_t P = shape.pixel_count(), wc = container_value_bytes(mode);
  EncodedBatch enc;
  enc.mode = mode;
  enc.shape = shape;
  enc.n_images = static_cast<uint8_t>(n);
  if (mode == CodecMode::Float64Faithful) {
    enc.packed_f64.resize(P);
    std::memcpy(enc.packed_f64.data(), plane, P * 8);
    return enc;
  }
  enc.packed.resize(P);
  for (std::size_t p = 0; p < P; ++p) {
    u128 v = 0;
    std::memcpy(&v, plane + p * wc, wc);  // little-endian low bytes
    enc.packed[p] = v;
  }
  if (mode_has_offsets(mode)) enc.offsets.assign(offsets, offsets + (n * P + 7) / 8);
  return enc;
}

}  // namespace optb::shim

namespace optb::codec {

std::size_t capacity(CodecMode mode) {
  const uint32_t c = optb_capacity(static_cast<int32_t>(mode));
  if (c == 0) throw Error("unknown codec mode");
  return c;
}
bool capacity_is_hard(CodecMode mode) { return optb_capacity_is_hard(static_cast<int32_t>(mode)) != 0; }
const char* mode_name(CodecMode mode) { return optb_mode_name(static_cast<int32_t>(mode)); }
bool mode_has_offsets(CodecMode mode) { return optb_mode_has_offsets(static_cast<int32_t>(mode)) != 0; }
std::size_t container_value_bytes(CodecMode mode) {
  return optb_container_value_bytes(static_cast<int32_t>(mode));
}

bool EncodedBatch::offset_bit(std::size_t image, std::size_t pixel) const {
  const std::size_t bit = image * pixel_count() + pixel;
  return (offsets[bit / 8] >> (bit % 8)) & 1u;
}

namespace {

void check_images(std::span<const Image> images) {
  if (images.empty()) throw Error("encode: batch must contain at least one image");
  const ImageShape shape = images[0].shape;
  if (shape.pixel_count() == 0) throw ShapeError("encode: image extents must be positive");
  for (std::size_t i = 0; i < images.size(); ++i) {
    if (!(images[i].shape == shape))
      throw ShapeError("encode: image " + std::to_string(i) + " shape differs from image 0");
    if (images[i].pixels.size() != shape.pixel_count())
      throw ShapeError("encode: image " + std::to_string(i) + " pixel buffer does not match shape");
  }
}

optb_layout one_chunk(CodecMode mode, std::size_t n, std::size_t pixels) {
  optb_layout L{};
  L.mode = static_cast<int32_t>(mode);
  L.per_chunk = static_cast<uint32_t>(n);
  L.pixels = pixels;
  L.batch = n;
  L.n_batches = 1;
  return L;
}

}  // namespace

EncodedBatch encode(std::span<const Image> images, CodecMode mode) {
  check_images(images);
  const std::size_t n = images.size(), P = images[0].shape.pixel_count();
  const optb_layout L = one_chunk(mode, n, P);
  shim::check(optb_layout_check(&L));  // capacity message (codec.cpp:94-96)
  std::vector<uint8_t> rows(n * P);
  for (std::size_t i = 0; i < n; ++i) std::memcpy(rows.data() + i * P, images[i].pixels.data(), P);
  const std::size_t wc = container_value_bytes(mode);
  std::vector<uint8_t> plane(P * wc);
  std::vector<uint8_t> offs(std::max<uint64_t>(optb_layout_offsets_bytes(&L), 16));
  shim::check(optb_encode_host(shim::context(), &L, rows.data(), plane.data(), offs.data()));
  return shim::make_encoded(mode, images[0].shape, n, plane.data(), offs.data());
}

std::vector<Image> decode(const EncodedBatch& enc) {
  const std::size_t P = enc.pixel_count(), n = enc.n_images;
  if (n == 0 || P == 0) throw FormatError("decode: empty encoded batch");
  const bool f64 = enc.mode == CodecMode::Float64Faithful;
  if ((f64 ? enc.packed_f64.size() : enc.packed.size()) != P)
    throw FormatError("decode: container plane size mismatch");
  if (mode_has_offsets(enc.mode) && enc.offsets.size() != (n * P + 7) / 8)
    throw FormatError("decode: offset plane size mismatch");
  const std::size_t wc = container_value_bytes(enc.mode);
  std::vector<uint8_t> plane(P * wc);
  if (f64) {
    std::memcpy(plane.data(), enc.packed_f64.data(), P * 8);
  } else {
    for (std::size_t p = 0; p < P; ++p) std::memcpy(plane.data() + p * wc, &enc.packed[p], wc);
  }
  const optb_layout L = one_chunk(enc.mode, n, P);
  std::vector<uint8_t> offs(std::max<uint64_t>(optb_layout_offsets_bytes(&L), 16));
  std::copy(enc.offsets.begin(), enc.offsets.end(), offs.begin());
  std::vector<uint8_t> out(n * P);
  const optb_epilogue E{OPTB_OUT_U8, 1.0f, nullptr, nullptr, nullptr, 0};
  shim::check(optb_decode_host(shim::context(), &L, plane.data(), offs.data(), &E, out.data()));
  std::vector<Image> images(n);
  for (std::size_t i = 0; i < n; ++i) {
    images[i].shape = enc.shape;
    images[i].pixels.assign(out.begin() + i * P, out.begin() + (i + 1) * P);
  }
  return images;
}

std::vector<int> roundtrip_error(std::span<const Image> images, CodecMode mode) {
  const std::vector<Image> back = decode(encode(images, mode));
  std::vector<int> errs(images.size(), 0);
  for (std::size_t i = 0; i < images.size(); ++i) {
    int worst = 0;
    for (std::size_t p = 0; p < images[i].pixels.size(); ++p) {
      const int d = std::abs(int(images[i].pixels[p]) - int(back[i].pixels[p]));
      worst = d > worst ? d : worst;
    }
    errs[i] = worst;
  }
  return errs;
}

// ---------------------------------------------------------------- OPTB format
// "OPTB", u16 version 1, u8 mode, u8 n_images, u32 H, W, C (little-endian),
// then P words of container_value_bytes (binary64 bits for f64), then the
// parity plane for the offset modes (codec.cpp:283-317).
namespace {

void put_le(std::ostream& out, uint64_t v, int bytes) {
  char b[8];
  for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>(v >> (8 * i));
  out.write(b, bytes);
}

uint64_t get_le(std::istream& in, int bytes) {
  unsigned char b[8];
  in.read(reinterpret_cast<char*>(b), bytes);
  if (in.gcount() != bytes) throw FormatError("optb: truncated stream");
  uint64_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}

}  // namespace

void write_optb(std::ostream& out, const EncodedBatch& enc) {
  if (enc.n_images == 0) throw Error("optb: refusing to write an empty batch");
  out.write("OPTB", 4);
  put_le(out, 1, 2);
  put_le(out, static_cast<uint8_t>(enc.mode), 1);
  put_le(out, enc.n_images, 1);
  put_le(out, enc.shape.height, 4);
  put_le(out, enc.shape.width, 4);
  put_le(out, enc.shape.channels, 4);
  const std::size_t P = enc.pixel_count();
  if (enc.mode == CodecMode::Float64Faithful) {
    for (std::size_t p = 0; p < P; ++p) put_le(out, std::bit_cast<uint64_t>(enc.packed_f64[p]), 8);
  } else {
    const bool wide = container_value_bytes(enc.mode) == 16;
    for (std::size_t p = 0; p < P; ++p) {
      put_le(out, static_cast<uint64_t>(enc.packed[p]), 8);
      if (wide) put_le(out, static_cast<uint64_t>(enc.packed[p] >> 64), 8);
    }
  }
  if (mode_has_offsets(enc.mode))
    out.write(reinterpret_cast<const char*>(enc.offsets.data()), static_cast<std::streamsize>(enc.offsets.size()));
  if (!out) throw FormatError("optb: stream write failed");
}

EncodedBatch read_optb(std::istream& in) {
  char magic[4];
  in.read(magic, 4);
  if (in.gcount() != 4) throw FormatError("optb: truncated stream");
  if (std::memcmp(magic, "OPTB", 4) != 0) throw FormatError("optb: bad magic");
  const uint64_t version = get_le(in, 2);
  if (version != 1) throw FormatError("optb: unsupported version " + std::to_string(version));
  const uint64_t tag = get_le(in, 1);
  const uint64_t n = get_le(in, 1);
  if (tag > 4) throw FormatError("optb: unknown mode tag " + std::to_string(tag));
  EncodedBatch enc;
  enc.mode = static_cast<CodecMode>(tag);
  enc.n_images = static_cast<uint8_t>(n);
  enc.shape.height = static_cast<uint32_t>(get_le(in, 4));
  enc.shape.width = static_cast<uint32_t>(get_le(in, 4));
  enc.shape.channels = static_cast<uint32_t>(get_le(in, 4));
  const std::size_t P = enc.pixel_count();
  if (n == 0 || P == 0) throw FormatError("optb: empty batch header");
  const std::size_t limit = capacity_is_hard(enc.mode) ? capacity(enc.mode) : kFloat64AcceptLimit;
  if (n > limit)
    throw FormatError("optb: image count " + std::to_string(n) + " exceeds " + mode_name(enc.mode) + " capacity");
  if (enc.mode == CodecMode::Float64Faithful) {
    enc.packed_f64.resize(P);
    for (std::size_t p = 0; p < P; ++p) enc.packed_f64[p] = std::bit_cast<double>(get_le(in, 8));
  } else {
    const bool wide = container_value_bytes(enc.mode) == 16;
    enc.packed.resize(P);
    for (std::size_t p = 0; p < P; ++p) {
      const uint64_t lo = get_le(in, 8);
      const uint64_t hi = wide ? get_le(in, 8) : 0;
      enc.packed[p] = (static_cast<u128>(hi) << 64) | lo;
    }
  }
  if (mode_has_offsets(enc.mode)) {
    enc.offsets.resize((n * P + 7) / 8);
    in.read(reinterpret_cast<char*>(enc.offsets.data()), static_cast<std::streamsize>(enc.offsets.size()));
    if (static_cast<std::size_t>(in.gcount()) != enc.offsets.size()) throw FormatError("optb: truncated stream");
  }
  return enc;
}

void write_optb_file(const std::filesystem::path& path, const EncodedBatch& enc) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw FormatError("optb: cannot open for writing: " + path.string());
  write_optb(out, enc);
  out.flush();
  if (!out) throw FormatError("optb: write failed: " + path.string());
}

EncodedBatch read_optb_file(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw FormatError("optb: cannot open: " + path.string());
  return read_optb(in);
}

}  // namespace optb::codec
