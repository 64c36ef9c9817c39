// shim_api_bench.cpp -- the reference runner's call pattern through the
// public C++ API only, so the same source builds against either library:
//   * the B200 drop-in (paper_2105_00619_b200/csrc/shim headers,
//     liboptb_shim.so + liboptb_cuda.so)  -> paper_2105_00619_b200/optb_shim_api_bench
//   * the reference itself, compiled from /root/reference/proj/src by
//     oracle/Makefile                     -> oracle/_ref/ref_api_bench
//
// Per batch, as runner.cpp does it:
//   draw_stream     runner.cpp:45-59  one BatchCursor::next() per batch
//   encode_chunks   runner.cpp:77-90  image_of copies (dataset.cpp:16-22) +
//                                     one codec::encode per 16-image chunk
//   consumer        codec::decode of every chunk (the decode under
//                                     nn::decode_input, nn.cpp:153-192)
// Dataset: N x 32x32x3 u8 counter-based pixels, labels e % 100; uniform
// weights, B = 512, seed 1234 (the C2 configuration).
//
//   <bin> [n_examples] [n_batches]   -> one JSON line
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "optb/codec.hpp"
#include "optb/sampler.hpp"

namespace {

uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

int main(int argc, char** argv) {
  using namespace optb;
  const std::size_t N = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 50000;
  const std::size_t n_batches = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 20;
  const std::size_t C = 100, B = 512, P = 32 * 32 * 3;
  const codec::CodecMode mode = codec::CodecMode::ExactInt128;
  const codec::ImageShape shape{32, 32, 3};
  std::vector<uint8_t> pixels(N * P);
  for (std::size_t i = 0; i < pixels.size() / 8; ++i) {
    const uint64_t w = mix(7 + (i + 1) * 0x9e3779b97f4a7c15ull);
    for (int k = 0; k < 8; ++k) pixels[i * 8 + k] = static_cast<uint8_t>(w >> (8 * k));
  }
  std::vector<int> labels(N);
  for (std::size_t i = 0; i < N; ++i) labels[i] = static_cast<int>(i % C);

  const double t0 = now_s();
  const std::vector<double> weights(C, 1.0 / C);
  sampler::BatchCursor cursor(sampler::plan(weights, B, 1234), sampler::ClassIndex::from_labels(labels, C));
  const double t_ctor = now_s() - t0;

  auto run = [&](std::size_t nb, double* t_draw, double* t_enc, double* t_dec, uint64_t* sum) {
    const std::size_t cap = codec::capacity(mode);
    for (std::size_t b = 0; b < nb; ++b) {
      double a = now_s();
      const std::vector<sampler::Draw> draws = cursor.next();
      double z = now_s();
      *t_draw += z - a;
      std::vector<codec::EncodedBatch> chunks;
      for (std::size_t base = 0; base < draws.size(); base += cap) {
        const std::size_t n = std::min(cap, draws.size() - base);
        std::vector<codec::Image> images;
        images.reserve(n);
        for (std::size_t i = 0; i < n; ++i) {
          codec::Image img;
          img.shape = shape;
          const uint8_t* row = pixels.data() + draws[base + i].example * P;
          img.pixels.assign(row, row + P);
          images.push_back(std::move(img));
        }
        chunks.push_back(codec::encode(images, mode));
      }
      a = now_s();
      *t_enc += a - z;
      for (const codec::EncodedBatch& enc : chunks) {
        const std::vector<codec::Image> back = codec::decode(enc);
        *sum += back.front().pixels[0] + back.back().pixels[P - 1];
      }
      *t_dec += now_s() - a;
    }
  };
  double d = 0, e = 0, x = 0;
  uint64_t sum = 0;
  run(2, &d, &e, &x, &sum);  // warm-up (allocations, staging, first launches)
  d = e = x = 0;
  const double t1 = now_s();
  run(n_batches, &d, &e, &x, &sum);
  const double secs = now_s() - t1;
  std::printf(
      "{\"images_per_s\": %.1f, \"batches\": %zu, \"batch\": %zu, \"dataset\": %zu, \"us_per_batch\": %.1f, "
      "\"next_us_per_batch\": %.2f, \"encode_us_per_chunk\": %.2f, \"decode_us_per_chunk\": %.2f, "
      "\"cursor_ctor_ms\": %.2f, \"checksum\": %llu}\n",
      n_batches * B / secs, n_batches, B, N, secs / n_batches * 1e6, d / n_batches * 1e6,
      e / (n_batches * (B / 16)) * 1e6, x / (n_batches * (B / 16)) * 1e6, t_ctor * 1e3,
      static_cast<unsigned long long>(sum));
  return 0;
}
