// pipeline.cu -- the encode-while-train data path as a device pipeline.
//
// Replaces the reference's producer/consumer hand-off (pipeline.cpp:37-97
// HandoffSlot, :116-129 prepare_epoch, :181-244 run) for the E-D path: instead
// of a producer thread encoding whole epochs into host buffers behind a mutex,
// each step is enqueued on CUDA streams with event hand-offs:
//   side stream   : SBS draws (optb_sbs_next_dev) of the next `steps_per_draw`
//                   steps into draw buffer (call+1)%2, once the encodes of the
//                   call that last used that buffer are done;
//   caller stream : wait for the step's draws -> gather-encode + decode with
//                   the fused epilogue into the caller's layer-input buffer:
//                   one optb_roundtrip_dev launch, or (split_kernels)
//                   optb_encode_dev then optb_decode_dev.
// Reference invariants kept: at most two live draw buffers (pipeline.hpp:19-20),
// in-order delivery, and errors surfacing before the affected step is consumed
// (device-side format errors latch in the context, optb_ctx_sync).
// optb_pipeline_step_host is the same step on HOST buffers: the epoch's
// dataset is uploaded into one of two device buffers on a copy stream (while
// the previous step computes and downloads), the step runs, and the decoded
// rows are copied back on a second copy stream -- both PCIe directions and
// the kernels overlap across consecutive calls.
// Built only on the public C ABI (include/optb_cuda.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>

#include "internal.h"
#include "optb_cuda.h"

namespace {
constexpr int kTimingRing = 64;

// every failure sets optb_last_error() (the cause of a CUDA failure included)
int arg_fail(const char* what) { return optb_b200::set_error_text(OPTB_ERR_ARG, std::string("pipeline: ") + what); }
int cuda_fail(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return optb_b200::set_error_text(OPTB_ERR_CUDA, std::string("pipeline: ") + what + ": " + cudaGetErrorString(e));
}
}

struct optb_pipeline {
  optb_ctx* ctx = nullptr;
  optb_pipeline_desc d{};
  uint32_t spd = 1;       // steps per SBS call
  uint64_t rows = 0;      // rows per step
  cudaStream_t side = nullptr;
  // draw buffers: nbuf - 1 sampler calls run ahead of the step being
  // computed (1 normally; 2 when every rank draws the stream of >= 4 ranks,
  // whose sampler work no longer fits in one call's worth of steps)
  static constexpr int kMaxBufs = 3;
  int nbuf = 2;
  int64_t* ex[kMaxBufs] = {};
  int32_t* cls[kMaxBufs] = {};
  void* cont = nullptr;
  uint8_t* offs = nullptr;
  cudaEvent_t sbs_done[kMaxBufs] = {}, enc_done[kMaxBufs] = {};
  cudaEvent_t t_s0[kTimingRing] = {}, t_s1[kTimingRing] = {}, t_e0[kTimingRing] = {},
              t_e1[kTimingRing] = {}, t_d1[kTimingRing] = {};
  uint64_t step = 0;   // next step to deliver
  uint64_t calls = 0;  // SBS calls enqueued
  // the previous fused step's stream and that stream's launch tag after it
  // (stream_tag): the next step may gather early if nothing that can trigger
  // its dependents early was launched there since (RowSrc::early)
  cudaStream_t last_stream = nullptr;
  uint64_t last_tag = 0;
  uintptr_t last_out = 0;  // the previous step's output range (what it wrote)
  uint64_t last_out_bytes = 0;
  bool timing = false;
  bool warm = false;     // warm start: decode the loaded epoch every step
  uint32_t tstride = 1;  // time every tstride-th step (and sampler call)
  // host leg (optb_pipeline_step_host): double-buffered device copies of the
  // host dataset and of the decoded rows, with their own copy streams
  struct Host {
    cudaStream_t up = nullptr, down = nullptr;
    uint8_t* ds[2] = {};
    uint8_t* out[2] = {};
    uint64_t ds_cap = 0, out_cap = 0;
    cudaEvent_t up_done[2] = {}, used[2] = {}, down_done[2] = {};
    uint64_t k = 0;  // host steps enqueued
  } host;
};

namespace {

int enqueue_draws(optb_pipeline* p) {
  const uint64_t c = p->calls;
  const int b = static_cast<int>(c % p->nbuf);
  if (c >= static_cast<uint64_t>(p->nbuf) && cudaStreamWaitEvent(p->side, p->enc_done[b], 0) != cudaSuccess)
    return cuda_fail("stream wait");
  const int r = static_cast<int>(c % kTimingRing);
  const bool timed = p->timing;  // side stream: its events never sit between two round trips
  if (timed) cudaEventRecord(p->t_s0[r], p->side);
  const uint64_t n = p->d.layout.n_batches * p->d.n_shards * p->spd;
  int st = optb_sbs_next_dev(p->d.sbs, n, p->d.shard, p->d.n_shards, p->ex[b], p->cls[b], p->side);
  if (st) return st;
  if (timed) cudaEventRecord(p->t_s1[r], p->side);
  if (cudaEventRecord(p->sbs_done[b], p->side) != cudaSuccess) return cuda_fail("event record");
  ++p->calls;
  return OPTB_OK;
}

}  // namespace

extern "C" {

int optb_pipeline_create(optb_ctx* ctx, const optb_pipeline_desc* d, optb_pipeline** out) {
  if (!ctx || !d || !out || !d->sbs || !d->dataset) return arg_fail("create: null ctx, descriptor, sampler or dataset");
  *out = nullptr;
  int st = optb_layout_check(&d->layout);
  if (st) return st;
  if (d->n_shards == 0 || d->shard >= d->n_shards) return arg_fail("create: shard must be < n_shards");
  auto* p = new optb_pipeline();
  p->ctx = ctx;
  p->d = *d;
  p->spd = d->steps_per_draw ? d->steps_per_draw : 1;
  p->timing = d->record_timings != 0;
  p->tstride = d->timing_stride ? d->timing_stride : 1;
  p->rows = optb_layout_rows(&d->layout);
  p->nbuf = d->n_shards >= 4 ? 3 : 2;
  bool ok = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) == cudaSuccess;
  for (int b = 0; b < p->nbuf && ok; ++b) {
    ok = cudaMalloc(&p->ex[b], p->rows * p->spd * sizeof(int64_t)) == cudaSuccess &&
         cudaMalloc(&p->cls[b], p->rows * p->spd * sizeof(int32_t)) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->sbs_done[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->enc_done[b], cudaEventDisableTiming) == cudaSuccess;
  }
  if (ok) ok = cudaMalloc(&p->cont, optb_layout_container_bytes(&d->layout) + 16) == cudaSuccess;
  const uint64_t ob = optb_layout_offsets_bytes(&d->layout);
  if (ok && ob) ok = cudaMalloc(&p->offs, ob) == cudaSuccess;
  for (int r = 0; r < kTimingRing && ok && p->timing; ++r) {
    ok = cudaEventCreate(&p->t_s0[r]) == cudaSuccess && cudaEventCreate(&p->t_s1[r]) == cudaSuccess &&
         cudaEventCreate(&p->t_e0[r]) == cudaSuccess && cudaEventCreate(&p->t_e1[r]) == cudaSuccess &&
         cudaEventCreate(&p->t_d1[r]) == cudaSuccess;
  }
  if (!ok) {
    optb_pipeline_destroy(p);
    return cuda_fail("CUDA call failed");
  }
  // the sampler's generation pool for one call (growing it mid-stream would
  // synchronise the side stream with the step in flight)
  st = optb_b200::sbs_reserve(d->sbs, d->layout.n_batches * d->n_shards * p->spd);
  if (st) {
    optb_pipeline_destroy(p);
    return st;
  }
  for (int c = 0; c + 1 < p->nbuf; ++c) {  // the first calls' draws start right away
    st = enqueue_draws(p);
    if (st) {
      optb_pipeline_destroy(p);
      return st;
    }
  }
  *out = p;
  return OPTB_OK;
}

int optb_pipeline_create_warm(optb_ctx* ctx, const optb_layout* layout, uint32_t h, uint32_t w, uint32_t c,
                              const char* dir, uint64_t epoch, const optb_epilogue* epilogue, int32_t record_timings,
                              optb_pipeline** out) {
  if (!ctx || !layout || !dir || !epilogue || !out) return arg_fail("create_warm: null argument");
  *out = nullptr;
  int st = optb_layout_check(layout);
  if (st) return st;
  if ((epilogue->class_scale || epilogue->class_bias) && !epilogue->row_class)
    return arg_fail("create_warm: class tables need row_class (a warm start has no draws)");
  auto* p = new optb_pipeline();
  p->ctx = ctx;
  p->d.layout = *layout;
  p->d.epilogue = *epilogue;
  p->d.n_shards = 1;
  p->warm = true;
  p->timing = record_timings != 0;
  p->rows = optb_layout_rows(layout);
  bool ok = cudaMalloc(&p->cont, optb_layout_container_bytes(layout) + 16) == cudaSuccess;
  const uint64_t ob = optb_layout_offsets_bytes(layout);
  if (ok && ob) ok = cudaMalloc(&p->offs, ob) == cudaSuccess;
  for (int r = 0; r < kTimingRing && ok && p->timing; ++r)
    ok = cudaEventCreate(&p->t_e0[r]) == cudaSuccess && cudaEventCreate(&p->t_e1[r]) == cudaSuccess &&
         cudaEventCreate(&p->t_d1[r]) == cudaSuccess;
  if (!ok) {
    optb_pipeline_destroy(p);
    return cuda_fail("CUDA call failed");
  }
  // the dumped epoch is read and validated once (pipeline.cpp:154-177 run_warm)
  st = optb_load_dev(ctx, layout, h, w, c, dir, epoch, p->cont, p->offs);
  if (st) {
    optb_pipeline_destroy(p);
    return st;
  }
  *out = p;
  return OPTB_OK;
}

int optb_pipeline_step(optb_pipeline* p, void* out, void* stream) {
  if (!p || !out) return arg_fail("step: null pipeline or output");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t k = p->step;
  if (p->warm) {  // no sampler, no encode: the loaded containers decode into `out`
    const int r = static_cast<int>(k % kTimingRing);
    if (p->timing) {
      cudaEventRecord(p->t_e0[r], s);
      cudaEventRecord(p->t_e1[r], s);
    }
    const int st = optb_decode_dev(p->ctx, &p->d.layout, p->cont, p->offs, &p->d.epilogue, out, s);
    if (st) return st;
    if (p->timing) cudaEventRecord(p->t_d1[r], s);
    ++p->step;
    return OPTB_OK;
  }
  const uint64_t call = k / p->spd, sub = k % p->spd;
  const int b = static_cast<int>(call % p->nbuf);
  const int r = static_cast<int>((k / p->tstride) % kTimingRing);
  const bool timed = p->timing && k % p->tstride == 0;
  int st;
  if (sub == 0) {
    st = enqueue_draws(p);  // the next call's draws overlap this call's steps
    if (st) return st;
    if (cudaStreamWaitEvent(s, p->sbs_done[b], 0) != cudaSuccess) return cuda_fail("stream wait");
  }
  optb_epilogue e = p->d.epilogue;
  if (e.class_scale && !e.row_class) e.row_class = p->cls[b] + sub * p->rows;
  if (timed) cudaEventRecord(p->t_e0[r], s);
  // early gather (RowSrc::early): before its griddepcontrol.wait the step
  // reads only the dataset rows and its draws.  Allowed when the kernel right
  // before it in the stream is this pipeline's previous step (stream tag
  // unchanged since), which wrote only the containers and the previous `out`
  // -- so the dataset must be disjoint from that `out` and from this one.  A
  // kernel launched from outside the library in between does not trigger its
  // dependents early (or, if a caller's kernel does, it must not write the
  // dataset after its trigger).
  const uint64_t ds_bytes = optb_b200::sbs_examples(p->d.sbs) * p->d.row_stride;
  const uint64_t out_row = e.out_row_stride ? e.out_row_stride : p->d.layout.pixels;
  const uint64_t out_bytes = p->rows * out_row * (e.out_dtype == OPTB_OUT_U8 ? 1 : e.out_dtype == OPTB_OUT_F32 ? 4 : 2);
  const uintptr_t o0 = reinterpret_cast<uintptr_t>(out), d0 = reinterpret_cast<uintptr_t>(p->d.dataset);
  auto apart = [&](uintptr_t a, uint64_t na) { return a + na <= d0 || d0 + ds_bytes <= a; };
  const bool disjoint = ds_bytes && apart(o0, out_bytes) && apart(p->last_out, p->last_out_bytes);
  const bool early = disjoint && p->last_tag && p->last_stream == s && optb_b200::stream_tag(s) == p->last_tag;
  if (p->d.split_kernels) {
    st = optb_b200::encode_dev(p->ctx, &p->d.layout, p->d.dataset, p->d.row_stride, p->ex[b] + sub * p->rows,
                               p->cont, p->offs, s, early);
    if (st) return st;
    if (timed) cudaEventRecord(p->t_e1[r], s);
    // the draw buffer is free for the side stream once nothing reads it: the
    // encode reads the examples, the decode reads the classes when the
    // per-class epilogue takes them from this step's draws
    const bool dec_reads_cls = e.class_scale && !p->d.epilogue.row_class;
    if (!dec_reads_cls && sub + 1 == p->spd && cudaEventRecord(p->enc_done[b], s) != cudaSuccess)
      return cuda_fail("event record");
    st = optb_decode_dev(p->ctx, &p->d.layout, p->cont, p->offs, &e, out, s);
    if (st) return st;
    if (dec_reads_cls && sub + 1 == p->spd && cudaEventRecord(p->enc_done[b], s) != cudaSuccess)
      return cuda_fail("event record");
  } else {
    st = optb_b200::roundtrip_dev(p->ctx, &p->d.layout, p->d.dataset, p->d.row_stride, p->ex[b] + sub * p->rows,
                                  p->cont, p->offs, &e, out, s, early);
    if (st) return st;
    if (timed) cudaEventRecord(p->t_e1[r], s);
    if (sub + 1 == p->spd && cudaEventRecord(p->enc_done[b], s) != cudaSuccess) return cuda_fail("event record");
  }
  if (timed && p->d.split_kernels) cudaEventRecord(p->t_d1[r], s);  // fused: the launch ends at t_e1
  p->last_stream = s;
  p->last_tag = optb_b200::stream_tag(s);
  p->last_out = o0;
  p->last_out_bytes = out_bytes;
  ++p->step;
  return OPTB_OK;
}

int optb_pipeline_set_dataset(optb_pipeline* p, const uint8_t* dataset, uint64_t row_stride) {
  if (!p || !dataset) return arg_fail("set_dataset: null pipeline or dataset");
  if (p->warm) return arg_fail("set_dataset: a warm-start pipeline has no dataset");
  p->d.dataset = dataset;
  p->d.row_stride = row_stride;
  return OPTB_OK;
}

int optb_pipeline_draws(const optb_pipeline* p, uint64_t step, const int64_t** examples,
                        const int32_t** classes) {
  if (!p || step >= p->calls * p->spd) return arg_fail("draws: step not drawn yet");
  const uint64_t call = step / p->spd;
  if (call + static_cast<uint64_t>(p->nbuf) < p->calls) return arg_fail("draws: step's draw buffer already reused");
  const uint64_t sub = step % p->spd;
  if (examples) *examples = p->ex[call % p->nbuf] + sub * p->rows;
  if (classes) *classes = p->cls[call % p->nbuf] + sub * p->rows;
  return OPTB_OK;
}

const void* optb_pipeline_containers(const optb_pipeline* p) { return p ? p->cont : nullptr; }

int optb_pipeline_timings(const optb_pipeline* p, uint64_t step, float* sbs_ms, float* enc_ms,
                          float* dec_ms) {
  if (!p || !p->timing || step >= p->step || step % p->tstride ||
      (p->step - 1 - step) / p->tstride >= static_cast<uint64_t>(kTimingRing))
    return arg_fail("timings: not recorded for that step (record_timings, timing_stride, last 64 timed steps)");
  const int r = static_cast<int>((step / p->tstride) % kTimingRing);
  const int rc = static_cast<int>((step / p->spd) % kTimingRing);
  const bool two = p->d.split_kernels || p->warm;  // a separate decode interval
  cudaEvent_t last = two ? p->t_d1[r] : p->t_e1[r];
  if (cudaEventSynchronize(last) != cudaSuccess) return cuda_fail("synchronize");
  if (sbs_ms && p->warm) {
    *sbs_ms = 0.0f;
  } else if (sbs_ms) {  // the SBS call that produced this step's draws, per step
    if (cudaEventElapsedTime(sbs_ms, p->t_s0[rc], p->t_s1[rc]) != cudaSuccess) return cuda_fail("event timing");
    *sbs_ms /= static_cast<float>(p->spd);
  }
  if (enc_ms && cudaEventElapsedTime(enc_ms, p->t_e0[r], p->t_e1[r]) != cudaSuccess) return cuda_fail("event timing");
  if (dec_ms) {
    if (!two) {
      *dec_ms = 0.0f;  // one fused launch: all of it is in enc_ms
    } else if (cudaEventElapsedTime(dec_ms, p->t_e1[r], p->t_d1[r]) != cudaSuccess) {
      return cuda_fail("CUDA call failed");
    }
  }
  return OPTB_OK;
}

int optb_pipeline_step_host(optb_pipeline* p, const uint8_t* dataset_host, uint64_t n_rows, uint64_t row_stride,
                            void* out_host, void* stream) {
  if (!p || !dataset_host || !out_host || !n_rows) return arg_fail("step_host: null buffer or empty dataset");
  if (p->warm) return arg_fail("step_host: a warm-start pipeline has no dataset");
  if (row_stride == 0) row_stride = p->d.layout.pixels;
  if (row_stride < p->d.layout.pixels) return arg_fail("step_host: row_stride < pixels");
  // the draws index every example of the sampler's class index
  if (n_rows < optb_b200::sbs_examples(p->d.sbs))
    return arg_fail(("step_host: " + std::to_string(n_rows) + " dataset rows, the sampler draws from " +
                     std::to_string(optb_b200::sbs_examples(p->d.sbs)) + " examples").c_str());
  auto& h = p->host;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t es = p->d.epilogue.out_dtype == OPTB_OUT_U8 ? 1 : p->d.epilogue.out_dtype == OPTB_OUT_F32 ? 4 : 2;
  const uint64_t ors = p->d.epilogue.out_row_stride ? p->d.epilogue.out_row_stride : p->d.layout.pixels;
  const uint64_t ds_bytes = n_rows * row_stride, out_bytes = p->rows * ors * es;
  if (!h.up) {
    bool ok = cudaStreamCreateWithFlags(&h.up, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&h.down, cudaStreamNonBlocking) == cudaSuccess;
    for (int b = 0; b < 2 && ok; ++b)
      ok = cudaEventCreateWithFlags(&h.up_done[b], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h.used[b], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h.down_done[b], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return cuda_fail("CUDA call failed");
  }
  if (h.ds_cap < ds_bytes || h.out_cap < out_bytes) {  // (re)size: drain the leg first
    if (cudaStreamSynchronize(h.up) != cudaSuccess || cudaStreamSynchronize(h.down) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return cuda_fail("CUDA call failed");
    for (int b = 0; b < 2; ++b) {
      if (h.ds_cap < ds_bytes) {
        if (h.ds[b]) cudaFree(h.ds[b]);
        h.ds[b] = nullptr;
        if (cudaMalloc(&h.ds[b], ds_bytes) != cudaSuccess) return cuda_fail("device allocation");
      }
      if (h.out_cap < out_bytes) {
        if (h.out[b]) cudaFree(h.out[b]);
        h.out[b] = nullptr;
        if (cudaMalloc(&h.out[b], out_bytes) != cudaSuccess) return cuda_fail("device allocation");
      }
    }
    h.ds_cap = h.ds_cap < ds_bytes ? ds_bytes : h.ds_cap;
    h.out_cap = h.out_cap < out_bytes ? out_bytes : h.out_cap;
    h.k = 0;  // fresh buffers: nothing in flight to wait for
  }
  const int b = static_cast<int>(h.k % 2);
  // H2D of this step's dataset once step k-2 no longer reads buffer b; it
  // runs on the copy engine while step k-1 computes and copies out
  if (h.k >= 2 && cudaStreamWaitEvent(h.up, h.used[b], 0) != cudaSuccess) return cuda_fail("stream wait");
  if (cudaMemcpyAsync(h.ds[b], dataset_host, ds_bytes, cudaMemcpyHostToDevice, h.up) != cudaSuccess ||
      cudaEventRecord(h.up_done[b], h.up) != cudaSuccess || cudaStreamWaitEvent(s, h.up_done[b], 0) != cudaSuccess)
    return cuda_fail("CUDA call failed");
  if (h.k >= 2 && cudaStreamWaitEvent(s, h.down_done[b], 0) != cudaSuccess) return cuda_fail("stream wait");
  const uint8_t* prev_ds = p->d.dataset;
  const uint64_t prev_stride = p->d.row_stride;
  p->d.dataset = h.ds[b];
  p->d.row_stride = row_stride;
  int st = optb_pipeline_step(p, h.out[b], stream);
  p->d.dataset = prev_ds;
  p->d.row_stride = prev_stride;
  if (st) return st;
  if (cudaEventRecord(h.used[b], s) != cudaSuccess || cudaStreamWaitEvent(h.down, h.used[b], 0) != cudaSuccess ||
      cudaMemcpyAsync(out_host, h.out[b], out_bytes, cudaMemcpyDeviceToHost, h.down) != cudaSuccess ||
      cudaEventRecord(h.down_done[b], h.down) != cudaSuccess)
    return cuda_fail("CUDA call failed");
  ++h.k;
  return OPTB_OK;
}

int optb_pipeline_host_wait(optb_pipeline* p, void* stream) {
  if (!p) return arg_fail("null pipeline");
  auto& h = p->host;
  if (!h.up || h.k == 0) return OPTB_OK;
  if (!stream) {  // host wait: every upload and download enqueued so far
    if (cudaStreamSynchronize(h.up) != cudaSuccess || cudaStreamSynchronize(h.down) != cudaSuccess)
      return cuda_fail("CUDA call failed");
    return OPTB_OK;
  }
  // device wait: the last download (it follows every earlier step's work)
  const int b = static_cast<int>((h.k - 1) % 2);
  return cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), h.down_done[b], 0) == cudaSuccess ? OPTB_OK
                                                                                                : OPTB_ERR_CUDA;
}

void optb_pipeline_destroy(optb_pipeline* p) {
  if (!p) return;
  if (p->side) cudaStreamSynchronize(p->side);
  cudaDeviceSynchronize();
  {
    auto& h = p->host;
    for (int b = 0; b < 2; ++b) {
      if (h.ds[b]) cudaFree(h.ds[b]);
      if (h.out[b]) cudaFree(h.out[b]);
      if (h.up_done[b]) cudaEventDestroy(h.up_done[b]);
      if (h.used[b]) cudaEventDestroy(h.used[b]);
      if (h.down_done[b]) cudaEventDestroy(h.down_done[b]);
    }
    if (h.up) cudaStreamDestroy(h.up);
    if (h.down) cudaStreamDestroy(h.down);
  }
  for (int b = 0; b < p->kMaxBufs; ++b) {
    if (p->ex[b]) cudaFree(p->ex[b]);
    if (p->cls[b]) cudaFree(p->cls[b]);
    if (p->sbs_done[b]) cudaEventDestroy(p->sbs_done[b]);
    if (p->enc_done[b]) cudaEventDestroy(p->enc_done[b]);
  }
  for (int r = 0; r < kTimingRing; ++r) {
    cudaEvent_t* evs[5] = {&p->t_s0[r], &p->t_s1[r], &p->t_e0[r], &p->t_e1[r], &p->t_d1[r]};
    for (cudaEvent_t* e : evs)
      if (*e) cudaEventDestroy(*e);
  }
  if (p->cont) cudaFree(p->cont);
  if (p->offs) cudaFree(p->offs);
  if (p->side) cudaStreamDestroy(p->side);
  delete p;
}

}  // extern "C"
