// ref_capi.cpp -- C-linkage wrapper over the REFERENCE optb library, compiled
// from its own sources under /root/reference/proj/src with -Doptb=optb_ref
// (recipe: oracle/Makefile; output only into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY.  Used (a) by tests/golden/make_golden.py and the
// CPU tests to pin the C restatement (optb_oracle.c) against the reference
// itself, and (b) by bench.py's cpu_baseline leg / `--impl reference` arm to
// time the reference's own CPU path.  Nothing here is on the product path.
//
// The reference headers are included from /root/reference/proj/include; the
// macro renames their namespace so this TU never collides with anything else.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "optb/codec.hpp"
#include "optb/dataset.hpp"
#include "optb/errors.hpp"
#include "optb/nn.hpp"
#include "optb/rng.hpp"
#include "optb/sampler.hpp"
#include "optb/tensor.hpp"

namespace R = optb_ref;
namespace RC = optb_ref::codec;

namespace {

int put_msg(char* msg, size_t cap, const char* what) {
  if (msg && cap) {
    std::strncpy(msg, what, cap - 1);
    msg[cap - 1] = 0;
  }
  return 0;
}

template <typename F>
int guarded(char* msg, size_t cap, F&& f) {
  try {
    f();
    return 0;
  } catch (const R::CapacityError& e) {
    put_msg(msg, cap, e.what());
    return 3;
  } catch (const R::ShapeError& e) {
    put_msg(msg, cap, e.what());
    return 2;
  } catch (const R::FormatError& e) {
    put_msg(msg, cap, e.what());
    return 4;
  } catch (const R::Error& e) {
    put_msg(msg, cap, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_msg(msg, cap, e.what());
    return 9;
  }
}

RC::ImageShape shape_of(uint32_t h, uint32_t w, uint32_t c) { return RC::ImageShape{h, w, c}; }

std::vector<RC::Image> make_images(const uint8_t* images, uint32_t n, RC::ImageShape s) {
  const size_t P = s.pixel_count();
  std::vector<RC::Image> v(n);
  for (uint32_t i = 0; i < n; ++i) {
    v[i].shape = s;
    v[i].pixels.assign(images + size_t(i) * P, images + size_t(i + 1) * P);
  }
  return v;
}

// EncodedBatch.packed is u128 in memory (codec.hpp:71); the device layout keeps
// the low Wc bytes little-endian, which is also the on-disk order (codec.cpp:298-312).
void export_plane(const RC::EncodedBatch& enc, uint8_t* plane) {
  const size_t P = enc.pixel_count();
  if (enc.mode == RC::CodecMode::Float64Faithful) {
    std::memcpy(plane, enc.packed_f64.data(), P * 8);
    return;
  }
  const size_t wc = RC::container_value_bytes(enc.mode);
  for (size_t p = 0; p < P; ++p) {
    RC::u128 v = enc.packed[p];
    for (size_t b = 0; b < wc; ++b) {
      plane[p * wc + b] = static_cast<uint8_t>(v);
      v >>= 8;
    }
  }
}

RC::EncodedBatch import_plane(int mode, const uint8_t* plane, const uint8_t* offsets, uint32_t n,
                              RC::ImageShape s) {
  RC::EncodedBatch enc;
  enc.mode = static_cast<RC::CodecMode>(mode);
  enc.shape = s;
  enc.n_images = static_cast<uint8_t>(n);
  const size_t P = s.pixel_count();
  if (enc.mode == RC::CodecMode::Float64Faithful) {
    enc.packed_f64.resize(P);
    std::memcpy(enc.packed_f64.data(), plane, P * 8);
  } else {
    const size_t wc = RC::container_value_bytes(enc.mode);
    enc.packed.resize(P);
    for (size_t p = 0; p < P; ++p) {
      RC::u128 v = 0;
      for (int b = int(wc) - 1; b >= 0; --b) v = (v << 8) | plane[p * wc + b];
      enc.packed[p] = v;
    }
    if (RC::mode_has_offsets(enc.mode)) {
      enc.offsets.assign(offsets, offsets + (size_t(n) * P + 7) / 8);
    }
  }
  return enc;
}

struct RefCursor {
  std::unique_ptr<R::sampler::BatchCursor> cursor;
};

}  // namespace

extern "C" {

int ref_capacity(int mode) { return int(RC::capacity(static_cast<RC::CodecMode>(mode))); }

int ref_encode(int mode, const uint8_t* images, uint32_t n, uint32_t h, uint32_t w, uint32_t c,
               uint8_t* plane, uint8_t* offsets, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const auto imgs = make_images(images, n, shape_of(h, w, c));
    const RC::EncodedBatch enc = RC::encode(imgs, static_cast<RC::CodecMode>(mode));
    export_plane(enc, plane);
    if (offsets && !enc.offsets.empty())
      std::memcpy(offsets, enc.offsets.data(), enc.offsets.size());
  });
}

int ref_decode(int mode, const uint8_t* plane, const uint8_t* offsets, uint32_t n, uint32_t h,
               uint32_t w, uint32_t c, uint8_t* images, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const RC::EncodedBatch enc = import_plane(mode, plane, offsets, n, shape_of(h, w, c));
    const auto back = RC::decode(enc);
    const size_t P = enc.pixel_count();
    for (size_t i = 0; i < back.size(); ++i) std::memcpy(images + i * P, back[i].pixels.data(), P);
  });
}

int ref_roundtrip_error(int mode, const uint8_t* images, uint32_t n, uint32_t h, uint32_t w,
                        uint32_t c, int32_t* errs, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const auto imgs = make_images(images, n, shape_of(h, w, c));
    const auto e = RC::roundtrip_error(imgs, static_cast<RC::CodecMode>(mode));
    for (size_t i = 0; i < e.size(); ++i) errs[i] = e[i];
  });
}

// OPTB stream bytes of one encoded chunk (codec.cpp:283-317).
int ref_write_optb(int mode, const uint8_t* images, uint32_t n, uint32_t h, uint32_t w,
                   uint32_t c, uint8_t* out, size_t out_cap, size_t* out_len, char* msg,
                   size_t cap) {
  return guarded(msg, cap, [&] {
    const auto imgs = make_images(images, n, shape_of(h, w, c));
    std::ostringstream os;
    RC::write_optb(os, RC::encode(imgs, static_cast<RC::CodecMode>(mode)));
    const std::string s = os.str();
    *out_len = s.size();
    if (s.size() <= out_cap) std::memcpy(out, s.data(), s.size());
  });
}

// nn::decode_input over a list of chunks (nn.cpp:153-192), optionally followed
// by the MixedPrecision binary16 tape store (nn.cpp:141-146, 235).
// chunk k holds ns[k] images; planes are [P][Wc] at plane + k*P*Wc.
int ref_decode_input(int mode, const uint8_t* planes, const uint8_t* offsets, uint64_t ostride,
                     const uint32_t* ns, uint32_t n_chunks, uint32_t h, uint32_t w, uint32_t c,
                     float scale, int half, void* out, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const RC::ImageShape s = shape_of(h, w, c);
    const size_t P = s.pixel_count();
    const size_t wc = RC::container_value_bytes(static_cast<RC::CodecMode>(mode));
    std::vector<RC::EncodedBatch> chunks;
    size_t rows = 0;
    for (uint32_t k = 0; k < n_chunks; ++k) {
      chunks.push_back(import_plane(mode, planes + size_t(k) * P * wc,
                                    offsets ? offsets + k * ostride : nullptr, ns[k], s));
      rows += ns[k];
    }
    const std::vector<R::nn::LayerSpec> specs = {
        R::nn::DecodeSpec{static_cast<RC::CodecMode>(mode), rows, scale}};
    const R::nn::Network net = R::nn::Network::make(
        specs, half ? R::nn::Precision::MixedPrecision : R::nn::Precision::SinglePrecision, 1);
    const R::Tensor t = R::nn::decode_input(net, chunks);
    if (half) {
      const R::Tensor stored = R::nn::boundary_storage(net, t);
      const auto hb = stored.half_bits();
      std::memcpy(out, hb.data(), hb.size() * 2);
    } else {
      const auto v = t.values();
      std::memcpy(out, v.data(), v.size() * 4);
    }
  });
}

uint16_t ref_float_to_half(float v) { return R::float_to_half(v); }

int ref_sbs_plan(const double* weights, uint64_t n_classes, uint64_t batch, uint64_t seed,
                 uint64_t* counts, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const auto p = R::sampler::plan(std::span<const double>(weights, n_classes), batch, seed);
    for (size_t i = 0; i < p.counts.size(); ++i) counts[i] = p.counts[i];
  });
}

int ref_class_index(const int32_t* labels, uint64_t n, uint64_t n_classes, uint64_t* offsets,
                    int64_t* members, char* msg, size_t cap) {
  return guarded(msg, cap, [&] {
    const auto idx =
        R::sampler::ClassIndex::from_labels(std::span<const int>(labels, n), n_classes);
    uint64_t o = 0;
    for (size_t c = 0; c < idx.by_class.size(); ++c) {
      offsets[c] = o;
      for (size_t e : idx.by_class[c]) members[o++] = int64_t(e);
    }
    offsets[idx.by_class.size()] = o;
  });
}

void* ref_cursor_create(const double* weights, uint64_t n_classes, uint64_t batch, uint64_t seed,
                        const uint64_t* class_offsets, const int64_t* members, int* status,
                        char* msg, size_t cap) {
  RefCursor* rc = nullptr;
  *status = guarded(msg, cap, [&] {
    auto p = R::sampler::plan(std::span<const double>(weights, n_classes), batch, seed);
    R::sampler::ClassIndex idx;
    idx.by_class.resize(n_classes);
    for (uint64_t c = 0; c < n_classes; ++c)
      for (uint64_t k = class_offsets[c]; k < class_offsets[c + 1]; ++k)
        idx.by_class[c].push_back(size_t(members[k]));
    auto cur = std::make_unique<R::sampler::BatchCursor>(std::move(p), std::move(idx));
    rc = new RefCursor{std::move(cur)};
  });
  return rc;
}

void ref_cursor_next(void* h, uint64_t n_batches, int64_t* examples, int32_t* classes) {
  auto* rc = static_cast<RefCursor*>(h);
  size_t r = 0;
  for (uint64_t b = 0; b < n_batches; ++b) {
    for (const auto& d : rc->cursor->next()) {
      examples[r] = int64_t(d.example);
      if (classes) classes[r] = int32_t(d.cls);
      ++r;
    }
  }
}

void ref_cursor_destroy(void* h) { delete static_cast<RefCursor*>(h); }

uint64_t ref_splitmix(uint64_t* state) {
  R::Rng rng(*state);
  const uint64_t v = rng.next_u64();
  *state += 0x9e3779b97f4a7c15ull;
  return v;
}

// ---------------------------------------------------------------- CPU baseline
// A reference dataset (dataset.hpp:14-20) built once, outside any timing.
void* ref_dataset_create(const uint8_t* pixels, uint64_t n_rows, uint32_t h, uint32_t w,
                         uint32_t c) {
  auto* ds = new R::data::Dataset();
  ds->shape = shape_of(h, w, c);
  ds->num_classes = 1;
  ds->pixels.assign(pixels, pixels + n_rows * ds->shape.pixel_count());
  ds->labels.assign(n_rows, 0);
  return ds;
}

void ref_dataset_destroy(void* h) { delete static_cast<R::data::Dataset*>(h); }

// One bench step of the reference path on `threads` host threads: for every
// batch, the draw's images are gathered with Dataset::image_of and packed
// chunk by chunk with codec::encode (runner.cpp:77-90), then every chunk is
// unpacked with codec::decode (decode_kind 0) or nn::decode_input at scale
// 1/255 (decode_kind 1, nn.cpp:153-192).  Batches are split across threads in
// contiguous shards (the functions are reentrant).  Returns the
// wall seconds; *checksum gets a checksum of the decoded first pixels.
double ref_bench_roundtrip(void* ds_handle, int mode, const int64_t* examples, uint64_t n_batches,
                           uint64_t batch, int threads, int decode_kind, uint64_t* checksum) {
  const auto& ds = *static_cast<const R::data::Dataset*>(ds_handle);
  const auto cm = static_cast<RC::CodecMode>(mode);
  const size_t cap = RC::capacity(cm);
  if (threads < 1) threads = 1;
  std::vector<uint64_t> sums(threads, 0);
  auto work = [&](int t) {
    const uint64_t b0 = n_batches * t / threads, b1 = n_batches * (t + 1) / threads;
    const std::vector<R::nn::LayerSpec> specs = {
        R::nn::DecodeSpec{cm, batch, 1.0f / 255.0f}};
    const R::nn::Network net =
        R::nn::Network::make(specs, R::nn::Precision::SinglePrecision, 1);
    for (uint64_t b = b0; b < b1; ++b) {
      std::vector<RC::EncodedBatch> chunks;
      for (size_t base = 0; base < batch; base += cap) {
        const size_t n = std::min(cap, size_t(batch) - base);
        std::vector<RC::Image> images;
        images.reserve(n);
        for (size_t i = 0; i < n; ++i)
          images.push_back(ds.image_of(size_t(examples[b * batch + base + i])));
        chunks.push_back(RC::encode(images, cm));
      }
      if (decode_kind == 0) {
        for (const auto& enc : chunks) {
          const auto back = RC::decode(enc);
          sums[t] += back[0].pixels[0];
        }
      } else {
        const R::Tensor out = R::nn::decode_input(net, chunks);
        sums[t] += uint64_t(out.values()[0] * 255.0f);
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t s = 0;
  for (auto v : sums) s += v;
  if (checksum) *checksum = s;
  return secs;
}

}  // extern "C"
