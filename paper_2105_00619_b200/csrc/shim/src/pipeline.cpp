// shim/src/pipeline.cpp -- optb::pipeline for the drop-in (reference API,
// pipeline.hpp:15-92), the encode-while-train loop of pipeline.cpp:181-244
// with the encoding on the GPU.
//
// Design.  The trainer thread consumes epochs from a one-deep mailbox that a
// producer thread fills.  The producer builds an epoch's batches with the
// caller's BatchBuilder (host callback), then encodes the WHOLE epoch with a
// single optb_encode_host call when every batch has the same image shape and
// count (the common case: capacity-sized chunks of one dataset) -- one H2D,
// one kernel, one D2H per epoch instead of a device round trip per batch --
// and cuts the container planes back into per-batch EncodedBatch values.
// Mixed batches fall back to codec::encode per batch (same results, same
// errors).  Contract kept from the reference:
//   * at most two epochs alive (the one training, the one ready/preparing);
//   * epochs delivered in order, exactly once, status Ready;
//   * a producer error is rethrown to the trainer before the affected epoch;
//   * a trainer error stops the producer before it starts another epoch;
//   * warm start: load the dumped epoch 0 once and train on it every epoch;
//   * serialize: prepare and train strictly in turn.
#include "optb/pipeline.hpp"

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <mutex>
#include <ostream>
#include <thread>

#include "optb_cuda.h"
#include "shim_ctx.hpp"

namespace optb::pipeline {

namespace {

using Clock = std::chrono::steady_clock;
using metering::Category;

double elapsed_ms(Clock::time_point from, Clock::time_point to) {
  return std::chrono::duration<double, std::milli>(to - from).count();
}

// The one-deep hand-off.  `put` blocks while an epoch is waiting (that is
// what bounds the live epochs to two); `take` blocks until an epoch or the
// producer's error arrives and rethrows the error.  `shut` (trainer failed)
// releases a blocked producer, which then drops its epoch.
class Mailbox {
public:
  bool wait_room() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !full_ || shut_; });
    return !shut_;
  }
  bool put(EpochBuffer&& b) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !full_ || shut_; });
    if (shut_) return false;
    slot_ = std::move(b);
    full_ = true;
    cv_.notify_all();
    return true;
  }
  void fail(std::exception_ptr e) {
    std::lock_guard<std::mutex> lk(mu_);
    err_ = std::move(e);
    cv_.notify_all();
  }
  EpochBuffer take() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return full_ || err_; });
    if (!full_) std::rethrow_exception(err_);
    full_ = false;
    EpochBuffer b = std::move(slot_);
    cv_.notify_all();
    return b;
  }
  void shut() {
    std::lock_guard<std::mutex> lk(mu_);
    shut_ = true;
    cv_.notify_all();
  }

private:
  std::mutex mu_;
  std::condition_variable cv_;
  EpochBuffer slot_;
  bool full_ = false, shut_ = false;
  std::exception_ptr err_;
};

// Every batch of the epoch as one device call when they share shape and
// image count; per-batch codec::encode otherwise (or when the count is over
// capacity, so the reference's CapacityError is raised by encode itself).
std::vector<codec::EncodedBatch> encode_epoch(const std::vector<std::vector<codec::Image>>& epoch,
                                              codec::CodecMode mode) {
  bool uniform = !epoch.empty() && !epoch[0].empty();
  const std::size_t n = uniform ? epoch[0].size() : 0;
  const codec::ImageShape shape = uniform ? epoch[0][0].shape : codec::ImageShape{};
  const std::size_t P = shape.pixel_count();
  uniform = uniform && P > 0 && n <= optb_accept_limit(static_cast<int32_t>(mode));
  for (std::size_t b = 0; uniform && b < epoch.size(); ++b) {
    uniform = epoch[b].size() == n;
    for (std::size_t i = 0; uniform && i < n; ++i)
      uniform = epoch[b][i].shape == shape && epoch[b][i].pixels.size() == P;
  }
  std::vector<codec::EncodedBatch> out;
  out.reserve(epoch.size());
  if (!uniform) {
    for (const auto& batch : epoch) out.push_back(codec::encode(batch, mode));
    return out;
  }
  optb_layout L{};
  L.mode = static_cast<int32_t>(mode);
  L.per_chunk = static_cast<uint32_t>(n);
  L.pixels = P;
  L.batch = n;
  L.n_batches = epoch.size();
  shim::check(optb_layout_check(&L));
  std::vector<uint8_t> rows(epoch.size() * n * P);
  for (std::size_t b = 0; b < epoch.size(); ++b)
    for (std::size_t i = 0; i < n; ++i) std::memcpy(rows.data() + (b * n + i) * P, epoch[b][i].pixels.data(), P);
  const std::size_t plane = P * codec::container_value_bytes(mode);
  const uint64_t ostride = optb_offsets_stride(L.mode, P, L.per_chunk);
  std::vector<uint8_t> cont(plane * epoch.size());
  std::vector<uint8_t> offs(std::max<std::size_t>(ostride * epoch.size(), 16));
  shim::check(optb_encode_host(shim::context(), &L, rows.data(), cont.data(), offs.data()));
  for (std::size_t b = 0; b < epoch.size(); ++b)
    out.push_back(shim::make_encoded(mode, shape, n, cont.data() + b * plane, offs.data() + b * ostride));
  return out;
}

EpochBuffer prepare(const PipelineConfig& cfg, const BatchBuilder& build, std::size_t epoch) {
  EpochBuffer buf;
  buf.epoch_id = epoch;
  std::vector<std::vector<codec::Image>> images(cfg.batches_per_epoch);
  for (std::size_t b = 0; b < cfg.batches_per_epoch; ++b) images[b] = build(epoch, b);
  buf.batches = encode_epoch(images, cfg.mode);
  if (cfg.injected_prepare_ms > 0.0)
    std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(cfg.injected_prepare_ms));
  if (cfg.dump_to_disk) dump(buf.batches, cfg.dump_dir, epoch);
  buf.status = BufferStatus::Ready;
  return buf;
}

// Trains one epoch and accounts its bytes as freed afterwards.
double train_one(const TrainEpoch& train, EpochBuffer& buf, metering::MemoryLedger* ledger) {
  const auto t0 = Clock::now();
  train(buf);
  buf.status = BufferStatus::Consumed;
  const double ms = elapsed_ms(t0, Clock::now());
  if (ledger) ledger->track_free(Category::EncodedBatches, buf.byte_size(), "epoch_buffer");
  return ms;
}

TimingReport run_warm(const PipelineConfig& cfg, const TrainEpoch& train, metering::MemoryLedger* ledger) {
  TimingReport rep;
  const auto t_begin = Clock::now();
  const std::vector<codec::EncodedBatch> epoch0 = load(cfg.dump_dir, 0);
  for (std::size_t e = 0; e < cfg.epochs; ++e) {
    EpochBuffer buf;
    buf.epoch_id = e;
    buf.batches = epoch0;
    buf.status = BufferStatus::Ready;
    if (ledger) ledger->track_alloc(Category::EncodedBatches, buf.byte_size(), "epoch_buffer");
    EpochTiming t;
    t.epoch = e;
    t.train_ms = train_one(train, buf, ledger);
    rep.epochs.push_back(t);
  }
  rep.total_ms = elapsed_ms(t_begin, Clock::now());
  return rep;
}

TimingReport run_serial(const PipelineConfig& cfg, const BatchBuilder& build, const TrainEpoch& train,
                        metering::MemoryLedger* ledger) {
  TimingReport rep;
  const auto t_begin = Clock::now();
  for (std::size_t e = 0; e < cfg.epochs; ++e) {
    EpochTiming t;
    t.epoch = e;
    const auto p0 = Clock::now();
    EpochBuffer buf = prepare(cfg, build, e);
    if (ledger) ledger->track_alloc(Category::EncodedBatches, buf.byte_size(), "epoch_buffer");
    t.prepare_ms = elapsed_ms(p0, Clock::now());
    if (e == 0) rep.cold_prepare_ms = t.prepare_ms;
    t.train_ms = train_one(train, buf, ledger);
    rep.epochs.push_back(t);
  }
  rep.total_ms = elapsed_ms(t_begin, Clock::now());
  return rep;
}

}  // namespace

std::size_t EpochBuffer::byte_size() const {
  std::size_t total = 0;
  for (const codec::EncodedBatch& b : batches) total += b.byte_size();
  return total;
}

void TimingReport::write_csv(std::ostream& out) const {
  out << "epoch,prepare_ms,train_ms,overlap_ms\n";
  for (const EpochTiming& e : epochs)
    out << e.epoch << ',' << e.prepare_ms << ',' << e.train_ms << ',' << e.overlap_ms << '\n';
}

TimingReport run(const PipelineConfig& cfg, const BatchBuilder& build, const TrainEpoch& train,
                 metering::MemoryLedger* ledger) {
  if (cfg.epochs == 0 || cfg.batches_per_epoch == 0)  // pipeline.cpp:178-180 message
    throw Error("pipeline: epochs and batches_per_epoch must be positive");
  if (cfg.warm_start) return run_warm(cfg, train, ledger);
  if (cfg.serialize) return run_serial(cfg, build, train, ledger);

  TimingReport rep;
  rep.epochs.resize(cfg.epochs);
  // [begin, end) of every prepare and every train, for the overlap column
  std::vector<std::pair<Clock::time_point, Clock::time_point>> prep(cfg.epochs), fit(cfg.epochs);
  Mailbox box;
  const auto t_begin = Clock::now();
  std::thread producer([&] {
    try {
      for (std::size_t e = 0; e < cfg.epochs && box.wait_room(); ++e) {
        const auto p0 = Clock::now();
        EpochBuffer buf = prepare(cfg, build, e);
        prep[e] = {p0, Clock::now()};
        rep.epochs[e].prepare_ms = elapsed_ms(p0, prep[e].second);
        const std::size_t bytes = buf.byte_size();
        if (ledger) ledger->track_alloc(Category::EncodedBatches, bytes, "epoch_buffer");
        if (!box.put(std::move(buf))) {  // the trainer has stopped
          if (ledger) ledger->track_free(Category::EncodedBatches, bytes, "epoch_buffer");
          return;
        }
      }
    } catch (...) {
      box.fail(std::current_exception());
    }
  });
  try {
    for (std::size_t e = 0; e < cfg.epochs; ++e) {
      EpochBuffer buf = box.take();
      const auto t0 = Clock::now();
      if (e == 0) rep.cold_prepare_ms = elapsed_ms(t_begin, t0);
      rep.epochs[e].epoch = e;
      rep.epochs[e].train_ms = train_one(train, buf, ledger);
      fit[e] = {t0, Clock::now()};
    }
  } catch (...) {
    box.shut();
    producer.join();
    throw;
  }
  producer.join();
  rep.total_ms = elapsed_ms(t_begin, Clock::now());
  for (std::size_t e = 0; e + 1 < cfg.epochs; ++e) {  // training of e against preparing e+1
    const auto lo = std::max(fit[e].first, prep[e + 1].first);
    const auto hi = std::min(fit[e].second, prep[e + 1].second);
    rep.epochs[e].overlap_ms = hi > lo ? elapsed_ms(lo, hi) : 0.0;
  }
  return rep;
}

void dump(std::span<const codec::EncodedBatch> batches, const std::filesystem::path& dir, std::size_t epoch) {
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  if (ec) throw FormatError("dump: cannot create directory " + dir.string());
  for (std::size_t i = 0; i < batches.size(); ++i)
    codec::write_optb_file(dir / ("batch_" + std::to_string(epoch) + "_" + std::to_string(i) + ".optb"),
                           batches[i]);
}

std::vector<codec::EncodedBatch> load(const std::filesystem::path& dir, std::size_t epoch) {
  std::vector<codec::EncodedBatch> out;
  for (std::size_t i = 0;; ++i) {
    const auto path = dir / ("batch_" + std::to_string(epoch) + "_" + std::to_string(i) + ".optb");
    if (!std::filesystem::exists(path)) break;
    out.push_back(codec::read_optb_file(path));
  }
  if (out.empty())
    throw FormatError("load: no batch files for epoch " + std::to_string(epoch) + " in " + dir.string());
  return out;
}

}  // namespace optb::pipeline
