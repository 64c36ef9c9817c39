// shim/src/sampler.cpp -- optb::sampler (reference API, sampler.hpp) over the
// C ABI: plan (host arithmetic, optb_sbs_plan), from_labels (GPU stable
// partition, optb_class_index_host), BatchCursor (GPU permutations and chain,
// optb_sbs_*).  next() runs the preprocessing hook host-side, in emission
// order, after the draws come back (sampler.cpp:99).
#include "optb/sampler.hpp"

#include <algorithm>
#include <string>

#include "optb_cuda.h"
#include "shim_ctx.hpp"

namespace optb::sampler {

SamplerPlan plan(std::span<const double> class_weights, std::size_t batch_size, std::uint64_t seed) {
  std::vector<uint64_t> counts(class_weights.size() ? class_weights.size() : 1);
  shim::check(optb_sbs_plan(class_weights.data(), class_weights.size(), batch_size, counts.data()));
  SamplerPlan p;
  p.class_weights.assign(class_weights.begin(), class_weights.end());
  p.batch_size = batch_size;
  p.seed = seed;
  p.counts.assign(counts.begin(), counts.begin() + class_weights.size());
  return p;
}

ClassIndex ClassIndex::from_labels(std::span<const int> labels, std::size_t num_classes) {
  std::vector<uint64_t> offsets(num_classes + 1, 0);
  std::vector<int64_t> members(labels.size());
  static_assert(sizeof(int) == sizeof(int32_t));
  shim::check(optb_class_index_host(shim::context(), reinterpret_cast<const int32_t*>(labels.data()),
                                    labels.size(), num_classes, offsets.data(), members.data()));
  ClassIndex idx;
  idx.by_class.resize(num_classes);
  for (std::size_t c = 0; c < num_classes; ++c)
    idx.by_class[c].assign(members.begin() + static_cast<std::ptrdiff_t>(offsets[c]),
                           members.begin() + static_cast<std::ptrdiff_t>(offsets[c + 1]));
  return idx;
}

BatchCursor::BatchCursor(SamplerPlan plan, ClassIndex index) : plan_(std::move(plan)) {
  if (index.num_classes() != plan_.num_classes()) {  // sampler.cpp:69-72
    throw Error("sampler: index has " + std::to_string(index.num_classes()) + " classes, plan has " +
                std::to_string(plan_.num_classes()));
  }
  const std::size_t C = plan_.num_classes();
  std::vector<uint64_t> counts(plan_.counts.begin(), plan_.counts.end());
  std::vector<uint64_t> offsets(C + 1, 0);
  for (std::size_t c = 0; c < C; ++c) offsets[c + 1] = offsets[c] + index.by_class[c].size();
  std::vector<int64_t> members;
  members.reserve(offsets[C]);
  for (const auto& v : index.by_class)
    for (std::size_t e : v) members.push_back(static_cast<int64_t>(e));
  shim::check(optb_sbs_create(shim::context(), counts.data(), C, plan_.batch_size, plan_.seed,
                              offsets.data(), members.data(), 0, &handle_));
}

BatchCursor::~BatchCursor() {
  if (handle_) optb_sbs_destroy(handle_);
}

BatchCursor::BatchCursor(const BatchCursor& other)
    : plan_(other.plan_), hook_(other.hook_), ring_ex_(other.ring_ex_), ring_cls_(other.ring_cls_),
      ring_pos_(other.ring_pos_), ring_len_(other.ring_len_), refill_(other.refill_) {
  if (other.handle_) shim::check(optb_sbs_clone(other.handle_, &handle_));
}

BatchCursor& BatchCursor::operator=(const BatchCursor& other) {
  if (this != &other) {
    BatchCursor copy(other);
    *this = std::move(copy);
  }
  return *this;
}

BatchCursor::BatchCursor(BatchCursor&& other) noexcept
    : plan_(std::move(other.plan_)), handle_(other.handle_), hook_(std::move(other.hook_)),
      ring_ex_(std::move(other.ring_ex_)), ring_cls_(std::move(other.ring_cls_)), ring_pos_(other.ring_pos_),
      ring_len_(other.ring_len_), refill_(other.refill_) {
  other.handle_ = nullptr;
  other.ring_pos_ = other.ring_len_ = 0;
}

BatchCursor& BatchCursor::operator=(BatchCursor&& other) noexcept {
  if (this != &other) {
    if (handle_) optb_sbs_destroy(handle_);
    plan_ = std::move(other.plan_);
    handle_ = other.handle_;
    hook_ = std::move(other.hook_);
    ring_ex_ = std::move(other.ring_ex_);
    ring_cls_ = std::move(other.ring_cls_);
    ring_pos_ = other.ring_pos_;
    ring_len_ = other.ring_len_;
    refill_ = other.refill_;
    other.handle_ = nullptr;
    other.ring_pos_ = other.ring_len_ = 0;
  }
  return *this;
}

std::vector<Draw> BatchCursor::next() {
  const std::size_t B = plan_.batch_size;
  if (ring_pos_ == ring_len_) {  // refill: one device call draws refill_ batches
    ring_ex_.resize(refill_ * B);
    ring_cls_.resize(refill_ * B);
    shim::check(optb_sbs_next_host(handle_, refill_, ring_ex_.data(), ring_cls_.data()));
    ring_pos_ = 0;
    ring_len_ = refill_;
    // grow geometrically: a caller drawing a handful of batches pays for
    // few extra, a long stream amortises the device round trip
    refill_ = std::min<std::size_t>(refill_ * 2, std::max<std::size_t>(1, (std::size_t{1} << 16) / (B ? B : 1)));
  }
  std::vector<Draw> batch(B);
  const int64_t* ex = ring_ex_.data() + ring_pos_ * B;
  const int32_t* cls = ring_cls_.data() + ring_pos_ * B;
  ++ring_pos_;
  for (std::size_t r = 0; r < B; ++r) {
    batch[r] = Draw{static_cast<std::size_t>(ex[r]), static_cast<std::size_t>(cls[r])};
    if (hook_) hook_(batch[r].cls, batch[r].example);
  }
  return batch;
}

}  // namespace optb::sampler
