// shim_extra.cpp -- drop-in checks beyond the reference's unit suites, in the
// reference's own test idiom (doctest), against the C++ shim over the GPU:
//   * BatchCursor copy semantics (sampler.hpp:45-68: the class is copyable and
//     a copy continues the identical stream) and the hook's emission order
//     across the shim's drawn-ahead ring refills (sampler.cpp:99);
//   * acceptance.cpp criteria 1 (codec losslessness, :58-87), 6 (pipeline
//     overlap, :254-282) and 8 (sampler exactness, :317-352), restated over
//     the same public API with the same seeds and bounds (acceptance.cpp
//     itself also needs the out-of-scope trainer and checkpoint planner).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <vector>

#include "optb/codec.hpp"
#include "optb/pipeline.hpp"
#include "optb/rng.hpp"
#include "optb/sampler.hpp"

using namespace optb;

namespace {

std::vector<int> labels_mod(std::size_t n, int classes) {
  std::vector<int> l(n);
  for (std::size_t i = 0; i < n; ++i) l[i] = static_cast<int>(i % classes);
  return l;
}

std::vector<std::size_t> examples_of(const std::vector<sampler::Draw>& d) {
  std::vector<std::size_t> e;
  for (const auto& x : d) e.push_back(x.example);
  return e;
}

std::vector<codec::Image> random_images(Rng& rng, std::size_t n) {
  const codec::ImageShape shape{static_cast<std::uint32_t>(1 + rng.next_below(6)),
                                static_cast<std::uint32_t>(1 + rng.next_below(6)),
                                static_cast<std::uint32_t>(1 + rng.next_below(3))};
  std::vector<codec::Image> images(n);
  for (auto& img : images) {
    img.shape = shape;
    img.pixels.resize(shape.pixel_count());
    for (auto& p : img.pixels) p = static_cast<std::uint8_t>(rng.next_below(256));
  }
  return images;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

TEST_SUITE_BEGIN("shim");

TEST_CASE("a copied cursor continues the identical stream independently") {
  const auto labels = labels_mod(700, 7);
  const std::vector<double> w(7, 1.0 / 7);
  sampler::BatchCursor a(sampler::plan(w, 32, 5), sampler::ClassIndex::from_labels(labels, 7));
  sampler::BatchCursor fresh(sampler::plan(w, 32, 5), sampler::ClassIndex::from_labels(labels, 7));
  for (int i = 0; i < 3; ++i) CHECK(examples_of(a.next()) == examples_of(fresh.next()));
  sampler::BatchCursor b = a;  // copy mid-ring (the shim drew ahead)
  sampler::BatchCursor c(a);
  for (int i = 0; i < 40; ++i) {  // several lazy reshuffles of every class
    const auto want = examples_of(fresh.next());
    CHECK(examples_of(a.next()) == want);
    CHECK(examples_of(b.next()) == want);
  }
  for (int i = 0; i < 40; ++i) c.next();
  CHECK(examples_of(c.next()) == examples_of(b.next()));
  sampler::BatchCursor d(sampler::plan(w, 32, 6), sampler::ClassIndex::from_labels(labels, 7));
  d = b;  // copy assignment replaces the stream
  CHECK(examples_of(d.next()) == examples_of(b.next()));
}

TEST_CASE("the preprocess hook sees every draw in emission order across ring refills") {
  const auto labels = labels_mod(500, 5);
  const std::vector<double> w(5, 0.2);
  sampler::BatchCursor cur(sampler::plan(w, 20, 9), sampler::ClassIndex::from_labels(labels, 5));
  std::vector<std::pair<std::size_t, std::size_t>> seen;
  cur.set_preprocess_hook([&](std::size_t c, std::size_t e) { seen.emplace_back(c, e); });
  std::vector<std::pair<std::size_t, std::size_t>> want;
  for (int i = 0; i < 37; ++i)
    for (const auto& d : cur.next()) want.emplace_back(d.cls, d.example);
  CHECK(seen == want);
}

TEST_CASE("acceptance criterion 1: randomized round trips are bit-exact within 10 s") {
  const auto t0 = std::chrono::steady_clock::now();
  const std::pair<codec::CodecMode, std::size_t> cases[] = {{codec::CodecMode::ExactInt64, 8},
                                                            {codec::CodecMode::ExactInt128, 16},
                                                            {codec::CodecMode::Float64Faithful, 6},
                                                            {codec::CodecMode::LosslessOffset64, 9}};
  Rng rng(0xACCE551);
  std::size_t trips = 0;
  for (const auto& [mode, max_n] : cases) {
    for (int it = 0; it < 1000; ++it) {
      const std::size_t n = 1 + rng.next_below(max_n);
      const auto images = random_images(rng, n);
      const auto back = codec::decode(codec::encode(images, mode));
      REQUIRE(back.size() == n);
      for (std::size_t i = 0; i < n; ++i) REQUIRE(back[i] == images[i]);
      ++trips;
    }
  }
  const double secs = seconds_since(t0);
  std::printf("criterion 1: %zu round trips in %.2f s\n", trips, secs);
  CHECK(trips == 4000);
  CHECK(secs < 10.0);
}

TEST_CASE("acceptance criterion 8: every batch is exactly [8,4,4] and the stream is reproducible") {
  std::vector<int> labels;
  for (int i = 0; i < 48; ++i) labels.push_back(0);
  for (int i = 0; i < 24; ++i) labels.push_back(1);
  for (int i = 0; i < 24; ++i) labels.push_back(2);
  const std::vector<double> w = {0.5, 0.25, 0.25};
  auto stream = [&](std::uint64_t seed) {
    sampler::BatchCursor cur(sampler::plan(w, 16, seed), sampler::ClassIndex::from_labels(labels, 3));
    std::vector<std::vector<sampler::Draw>> out;
    for (int b = 0; b < 6; ++b) out.push_back(cur.next());
    return out;
  };
  const auto s1 = stream(11), s2 = stream(11);
  for (std::size_t b = 0; b < s1.size(); ++b) {
    std::size_t counts[3] = {0, 0, 0};
    for (const auto& d : s1[b]) ++counts[d.cls];
    CHECK(counts[0] == 8);
    CHECK(counts[1] == 4);
    CHECK(counts[2] == 4);
    CHECK(examples_of(s1[b]) == examples_of(s2[b]));
  }
}

TEST_CASE("acceptance criterion 6: E-D wall clock is at most 0.85 of serialized") {
  std::vector<double> ratios;
  for (int r = 0; r < 3; ++r) {
    pipeline::PipelineConfig cfg;
    cfg.epochs = 10;
    cfg.batches_per_epoch = 1;
    cfg.mode = codec::CodecMode::ExactInt64;
    cfg.injected_prepare_ms = 25.0;  // P = 0.25 T
    Rng rng(7);
    const auto images = random_images(rng, 4);
    const pipeline::TimingReport rep = pipeline::run(
        cfg, [&](std::size_t, std::size_t) { return images; },
        [&](const pipeline::EpochBuffer&) { std::this_thread::sleep_for(std::chrono::milliseconds(100)); });
    double serialized = 0.0;
    for (const auto& e : rep.epochs) serialized += e.prepare_ms + e.train_ms;
    ratios.push_back(rep.total_ms / serialized);
  }
  std::sort(ratios.begin(), ratios.end());
  std::printf("criterion 6: median E-D / serialized %.3f\n", ratios[1]);
  CHECK(ratios[1] <= 0.85);
}

TEST_CASE("pipeline: one device call per epoch decodes back to the built batches") {
  pipeline::PipelineConfig cfg;
  cfg.epochs = 3;
  cfg.batches_per_epoch = 40;
  cfg.mode = codec::CodecMode::LosslessOffset128;
  auto build = [](std::size_t e, std::size_t b) {
    Rng rng(1000 * e + b);
    std::vector<codec::Image> imgs(18);
    for (auto& im : imgs) {
      im.shape = codec::ImageShape{8, 8, 3};
      im.pixels.resize(192);
      for (auto& p : im.pixels) p = static_cast<std::uint8_t>(rng.next_below(256));
    }
    return imgs;
  };
  std::size_t epochs = 0;
  pipeline::run(cfg, build, [&](const pipeline::EpochBuffer& buf) {
    REQUIRE(buf.batches.size() == 40);
    for (std::size_t b = 0; b < 40; ++b) {
      const auto want = codec::encode(build(buf.epoch_id, b), cfg.mode);  // per-batch call
      CHECK(buf.batches[b].packed == want.packed);
      CHECK(buf.batches[b].offsets == want.offsets);
      CHECK(codec::decode(buf.batches[b]) == build(buf.epoch_id, b));
    }
    ++epochs;
  });
  CHECK(epochs == 3);
}

TEST_SUITE_END();
