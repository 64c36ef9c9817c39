// capi.cu -- the C ABI (include/optb_cuda.h): validation with the reference's
// error messages, contexts, the host staging pipeline, and the SBS host-side
// event planner.  Kernels live in codec.cu and sbs.cu.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "optb_cuda.h"

using namespace optb_b200;

// ------------------------------------------------------------------ errors
namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace

int optb_b200::set_error_text(int code, const std::string& message) {
  g_err = message;
  return code;
}

namespace {

int cuda_err(cudaError_t e, const char* where) {
  return set_err(OPTB_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call, where)                          \
  do {                                           \
    cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return cuda_err(_e, where); \
  } while (0)

bool valid_mode(int32_t m) { return m >= 0 && m <= 4; }

}  // namespace

// ------------------------------------------------------------------ metadata
extern "C" {

uint32_t optb_abi_version(void) { return OPTB_ABI_VERSION; }

uint32_t optb_capacity(int32_t mode) {  // codec.cpp:13-27
  switch (mode) {
    case OPTB_EXACT64: return 8;
    case OPTB_EXACT128: return 16;
    case OPTB_F64: return 6;
    case OPTB_LOSSLESS64: return 9;
    case OPTB_LOSSLESS128: return 18;
  }
  return 0;
}

uint32_t optb_accept_limit(int32_t mode) {
  return mode == OPTB_F64 ? 16u : optb_capacity(mode);
}

int32_t optb_capacity_is_hard(int32_t mode) { return mode != OPTB_F64; }

const char* optb_mode_name(int32_t mode) {  // codec.cpp:31-45
  switch (mode) {
    case OPTB_EXACT64: return "exact64";
    case OPTB_EXACT128: return "exact128";
    case OPTB_F64: return "f64";
    case OPTB_LOSSLESS64: return "lossless64";
    case OPTB_LOSSLESS128: return "lossless128";
  }
  return "?";
}

int32_t optb_mode_has_offsets(int32_t mode) {
  return mode == OPTB_LOSSLESS64 || mode == OPTB_LOSSLESS128;
}

uint32_t optb_container_value_bytes(int32_t mode) {  // codec.cpp:51-62
  switch (mode) {
    case OPTB_EXACT64:
    case OPTB_F64:
    case OPTB_LOSSLESS64: return 8;
    case OPTB_EXACT128:
    case OPTB_LOSSLESS128: return 16;
  }
  return 0;
}

uint64_t optb_offsets_plane_bytes(uint32_t n, uint64_t pixels) {
  return (static_cast<uint64_t>(n) * pixels + 7) / 8;
}

uint64_t optb_offsets_stride(int32_t mode, uint64_t pixels, uint32_t per_chunk) {
  if (!optb_mode_has_offsets(mode)) return 0;
  return (optb_offsets_plane_bytes(per_chunk, pixels) + 15) / 16 * 16;
}

uint64_t optb_layout_chunks(const optb_layout* L) {
  if (!L || L->per_chunk == 0) return 0;
  return L->n_batches * ((L->batch + L->per_chunk - 1) / L->per_chunk);
}

uint64_t optb_layout_rows(const optb_layout* L) { return L ? L->batch * L->n_batches : 0; }

uint64_t optb_layout_container_bytes(const optb_layout* L) {
  return optb_layout_chunks(L) * (L ? L->pixels : 0) * optb_container_value_bytes(L ? L->mode : -1);
}

uint64_t optb_layout_offsets_bytes(const optb_layout* L) {
  if (!L) return 0;
  return optb_layout_chunks(L) * optb_offsets_stride(L->mode, L->pixels, L->per_chunk);
}

int optb_layout_check(const optb_layout* L) {  // codec.cpp:79-97
  if (!L) return set_err(OPTB_ERR_ARG, "layout: null");
  if (!valid_mode(L->mode)) return set_err(OPTB_ERR, "unknown codec mode");
  if (L->per_chunk == 0) return set_err(OPTB_ERR, "encode: batch must contain at least one image");
  if (L->pixels == 0) return set_err(OPTB_ERR_SHAPE, "encode: image extents must be positive");
  const uint32_t limit = optb_accept_limit(L->mode);
  if (L->per_chunk > limit)
    return set_err(OPTB_ERR_CAPACITY, "encode: %u images exceed %s capacity of %u", L->per_chunk,
                   optb_mode_name(L->mode), limit);
  if (L->batch == 0) return set_err(OPTB_ERR_ARG, "layout: batch must be positive");
  g_err.clear();
  return OPTB_OK;
}

const char* optb_last_error(void) { return g_err.c_str(); }

}  // extern "C"

// ------------------------------------------------------------------ context
struct optb_ctx {
  int device = 0;
  int sms = 148;
  DevError* d_err = nullptr;
  uint64_t launches = 0;
  cudaStream_t s_compute = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  // host-API staging (2 slots)
  static constexpr int kSlots = 2;
  size_t slot_in = 0, slot_out = 0, slot_off = 0;
  uint8_t* pin_in[kSlots] = {};
  uint8_t* pin_out[kSlots] = {};
  uint8_t* pin_off[kSlots] = {};
  uint8_t* dev_in[kSlots] = {};
  uint8_t* dev_out[kSlots] = {};
  uint8_t* dev_off[kSlots] = {};
  cudaEvent_t ev_h2d[kSlots] = {}, ev_kern[kSlots] = {}, ev_d2h[kSlots] = {};
  // scratch for class index / sbs host outputs
  uint32_t* ci_scratch = nullptr;
  uint64_t ci_words = 0;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  // pinned error-latch words for the small-call host path: [0] the reset
  // value, [1] the read-back (both stream ordered, no extra synchronisation)
  DevError* pin_err = nullptr;
  DevError* d_err_small = nullptr;  // the small host calls' own latch (synchronous calls)
};

namespace {


// The reference message of a latched device error (optb_ctx_sync).
int latch_status(const DevError& h) {
  const unsigned n = static_cast<unsigned>(h.key & 0xff);
  switch (h.kind) {
    case kErrIntRange:  // codec.cpp:191-194
      return set_err(OPTB_ERR_FORMAT, "decode: container value exceeds range of %u packed images", n);
    case kErrF64Range:  // codec.cpp:165-170
      return set_err(OPTB_ERR_FORMAT, "decode: container value out of range for %u images", n);
    case kErrLabel:  // sampler.cpp:58-61
      return set_err(OPTB_ERR, "sampler: label %lld outside %llu classes", static_cast<long long>(h.label),
                     static_cast<unsigned long long>(h.aux));
  }
  return set_err(OPTB_ERR, "device error %u", h.kind);
}

int reset_err(optb_ctx* c, cudaStream_t s) {
  DevError z{0, 0, ~0ull, 0, 0};
  CK(cudaMemcpyAsync(c->d_err, &z, sizeof z, cudaMemcpyHostToDevice, s), "reset error latch");
  CK(cudaStreamSynchronize(s), "reset error latch");
  return OPTB_OK;
}

Geom make_geom(const optb_layout* L) {
  Geom g;
  g.mode = L->mode;
  g.per_chunk = L->per_chunk;
  g.wc = optb_container_value_bytes(L->mode);
  g.cpb = static_cast<uint32_t>((L->batch + L->per_chunk - 1) / L->per_chunk);
  g.P = L->pixels;
  g.B = L->batch;
  g.chunks = optb_layout_chunks(L);
  g.ostride = optb_offsets_stride(L->mode, L->pixels, L->per_chunk);
  g.chunk_base = 0;
  return g;
}

int check_epilogue(const optb_epilogue* E) {
  if (!E) return set_err(OPTB_ERR_ARG, "decode: null epilogue");
  if (E->out_dtype < OPTB_OUT_U8 || E->out_dtype > OPTB_OUT_BF16)
    return set_err(OPTB_ERR_ARG, "decode: unknown output dtype %d", E->out_dtype);
  if ((E->class_scale || E->class_bias) && !E->row_class)
    return set_err(OPTB_ERR_ARG, "decode: class tables need row_class");
  if (E->class_bias && !E->class_scale)
    return set_err(OPTB_ERR_ARG, "decode: class_bias needs class_scale");
  return OPTB_OK;
}

Epi make_epi(const optb_epilogue* E, uint64_t P) {
  Epi e;
  e.dtype = E->out_dtype;
  e.scale = E->scale;
  e.class_scale = E->class_scale;
  e.class_bias = E->class_bias;
  e.row_class = E->row_class;
  e.row_stride = E->out_row_stride ? E->out_row_stride : P;
  return e;
}

// Decode layout validation mirrors codec.cpp:150-158 (empty batch) and the
// capacity header checks of read_optb (codec.cpp:338-344).
int check_decode_layout(const optb_layout* L) {
  if (!L) return set_err(OPTB_ERR_ARG, "layout: null");
  if (!valid_mode(L->mode)) return set_err(OPTB_ERR, "unknown codec mode");
  if (L->per_chunk == 0 || L->pixels == 0)
    return set_err(OPTB_ERR_FORMAT, "decode: empty encoded batch");
  if (L->per_chunk > optb_accept_limit(L->mode))
    return set_err(OPTB_ERR_FORMAT, "optb: image count %u exceeds %s capacity", L->per_chunk,
                   optb_mode_name(L->mode));
  if (L->batch == 0) return set_err(OPTB_ERR_ARG, "layout: batch must be positive");
  return OPTB_OK;
}

size_t out_elem_bytes(int dtype) {
  return dtype == OPTB_OUT_U8 ? 1 : dtype == OPTB_OUT_F32 ? 4 : 2;
}

}  // namespace

extern "C" {

int optb_ctx_create(int device, optb_ctx** out) {
  if (!out) return set_err(OPTB_ERR_ARG, "ctx: null output");
  *out = nullptr;
  int n = 0;
  CK(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n)
    return set_err(OPTB_ERR_CUDA, "ctx: device %d not present (%d devices)", device, n);
  CK(cudaSetDevice(device), "cudaSetDevice");
  auto* c = new optb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->d_err, sizeof(DevError)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->s_compute, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) != cudaSuccess) {
    optb_ctx_destroy(c);
    return cuda_err(cudaGetLastError(), "ctx create");
  }
  for (int i = 0; i < optb_ctx::kSlots; ++i) {
    cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_kern[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming);
  }
  if (cudaHostAlloc(&c->pin_err, 2 * sizeof(DevError), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    optb_ctx_destroy(c);
    return cuda_err(cudaGetLastError(), "ctx create");
  }
  c->pin_err[0] = DevError{0, 0, ~0ull, 0, 0};
  if (cudaMalloc(&c->d_err_small, sizeof(DevError)) != cudaSuccess ||
      cudaMemcpy(c->d_err_small, &c->pin_err[0], sizeof(DevError), cudaMemcpyHostToDevice) != cudaSuccess) {
    optb_ctx_destroy(c);
    return cuda_err(cudaGetLastError(), "ctx create");
  }
  int st = reset_err(c, c->s_compute);
  if (st) {
    optb_ctx_destroy(c);
    return st;
  }
  *out = c;
  g_err.clear();
  return OPTB_OK;
}

void optb_ctx_destroy(optb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < optb_ctx::kSlots; ++i) {
    if (c->pin_in[i]) cudaFreeHost(c->pin_in[i]);
    if (c->pin_out[i]) cudaFreeHost(c->pin_out[i]);
    if (c->pin_off[i]) cudaFreeHost(c->pin_off[i]);
    if (c->dev_in[i]) cudaFree(c->dev_in[i]);
    if (c->dev_out[i]) cudaFree(c->dev_out[i]);
    if (c->dev_off[i]) cudaFree(c->dev_off[i]);
    if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
    if (c->ev_kern[i]) cudaEventDestroy(c->ev_kern[i]);
    if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
  }
  if (c->ci_scratch) cudaFree(c->ci_scratch);
  if (c->tmp) cudaFree(c->tmp);
  if (c->d_err) cudaFree(c->d_err);
  if (c->pin_err) cudaFreeHost(c->pin_err);
  if (c->d_err_small) cudaFree(c->d_err_small);
  if (c->s_compute) cudaStreamDestroy(c->s_compute);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  delete c;
}

uint64_t optb_ctx_launches(const optb_ctx* c) { return c ? c->launches : 0; }

int optb_ctx_sync(optb_ctx* c, void* stream) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevError h{};
  CK(cudaStreamSynchronize(s), "stream synchronize");
  CK(cudaMemcpyAsync(&h, c->d_err, sizeof h, cudaMemcpyDeviceToHost, c->s_compute), "read error latch");
  CK(cudaStreamSynchronize(c->s_compute), "read error latch");
  if (h.kind == kErrNone) {
    g_err.clear();
    return OPTB_OK;
  }
  int st = reset_err(c, c->s_compute);
  if (st) return st;
  return latch_status(h);
}

// ------------------------------------------------------------------ codec, device
int optb_encode_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
                    const int64_t* row_index, void* containers, uint8_t* offsets, void* stream) {
  return optb_b200::encode_dev(c, L, images, row_stride, row_index, containers, offsets, stream, false);
}

int optb_encode_rows_dev(optb_ctx* c, const optb_layout* L, const uint64_t* row_ptrs, int32_t rows_aligned16,
                         void* containers, uint8_t* offsets, void* stream) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = optb_layout_check(L);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  if (!row_ptrs || !containers || (optb_mode_has_offsets(L->mode) && !offsets))
    return set_err(OPTB_ERR_ARG, "encode: null buffer");
  const Geom g = make_geom(L);
  const RowSrc rs{nullptr, 0, nullptr, row_ptrs, rows_aligned16};
  cudaError_t e = launch_encode(g, rs, containers, offsets, static_cast<cudaStream_t>(stream), c->sms, &c->launches);
  if (e != cudaSuccess) return cuda_err(e, "encode launch");
  return OPTB_OK;
}

int optb_decode_dev(optb_ctx* c, const optb_layout* L, const void* containers,
                    const uint8_t* offsets, const optb_epilogue* E, void* out, void* stream) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = check_decode_layout(L);
  if (st) return st;
  st = check_epilogue(E);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  if (!containers || !out || (optb_mode_has_offsets(L->mode) && !offsets))
    return set_err(OPTB_ERR_ARG, "decode: null buffer");
  const Epi ep = make_epi(E, L->pixels);
  if (ep.row_stride < L->pixels) return set_err(OPTB_ERR_ARG, "decode: out_row_stride < pixels");
  const Geom g = make_geom(L);
  cudaError_t e = launch_decode(g, containers, offsets, ep, out, c->d_err,
                                static_cast<cudaStream_t>(stream), c->sms, &c->launches);
  if (e != cudaSuccess) return cuda_err(e, "decode launch");
  return OPTB_OK;
}

namespace {

int roundtrip(optb_ctx* c, const optb_layout* L, const RowSrc& rs, void* containers, uint8_t* offsets,
              const optb_epilogue* E, void* out, void* stream) {
  const Epi ep = make_epi(E, L->pixels);
  if (ep.row_stride < L->pixels) return set_err(OPTB_ERR_ARG, "decode: out_row_stride < pixels");
  const Geom g = make_geom(L);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_roundtrip(g, rs, containers, offsets, ep, out, c->d_err, s, c->sms, &c->launches);
  if (e == cudaErrorNotSupported) {
    e = launch_encode(g, rs, containers, offsets, s, c->sms, &c->launches);
    if (e != cudaSuccess) return cuda_err(e, "encode launch");
    e = launch_decode(g, containers, offsets, ep, out, c->d_err, s, c->sms, &c->launches);
    if (e != cudaSuccess) return cuda_err(e, "decode launch");
    return OPTB_OK;
  }
  if (e != cudaSuccess) return cuda_err(e, "roundtrip launch");
  return OPTB_OK;
}

int roundtrip_checks(optb_ctx* c, const optb_layout* L, const optb_epilogue* E) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = optb_layout_check(L);
  if (st) return st;
  st = check_decode_layout(L);
  if (st) return st;
  return check_epilogue(E);
}

}  // namespace

int optb_roundtrip_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
                       const int64_t* row_index, void* containers, uint8_t* offsets, const optb_epilogue* E,
                       void* out, void* stream) {
  return optb_b200::roundtrip_dev(c, L, images, row_stride, row_index, containers, offsets, E, out, stream, false);
}

int optb_roundtrip_rows_dev(optb_ctx* c, const optb_layout* L, const uint64_t* row_ptrs, int32_t rows_aligned16,
                            void* containers, uint8_t* offsets, const optb_epilogue* E, void* out, void* stream) {
  int st = roundtrip_checks(c, L, E);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  if (!row_ptrs || !containers || !out || (optb_mode_has_offsets(L->mode) && !offsets))
    return set_err(OPTB_ERR_ARG, "roundtrip: null buffer");
  return roundtrip(c, L, RowSrc{nullptr, 0, nullptr, row_ptrs, rows_aligned16}, containers, offsets, E, out,
                   stream);
}

int optb_last_roundtrip_kind(void) { return optb_b200::g_rt_kind; }

int optb_synth_pixels_dev(optb_ctx* c, uint64_t seed, uint64_t first_row, uint64_t n_rows,
                          uint64_t pixels, uint8_t* out, uint64_t row_stride, void* stream) {
  if (!c || !out) return set_err(OPTB_ERR_ARG, "synth: null");
  if (row_stride == 0) row_stride = pixels;
  cudaError_t e = launch_synth(seed, first_row, n_rows, pixels, out, row_stride,
                               static_cast<cudaStream_t>(stream), c->sms, &c->launches);
  if (e != cudaSuccess) return cuda_err(e, "synth launch");
  return OPTB_OK;
}

}  // extern "C"

int optb_b200::encode_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
                           const int64_t* row_index, void* containers, uint8_t* offsets, void* stream, bool early) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = optb_layout_check(L);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  if (!images || !containers || (optb_mode_has_offsets(L->mode) && !offsets))
    return set_err(OPTB_ERR_ARG, "encode: null buffer");
  if (row_stride == 0) row_stride = L->pixels;
  if (row_stride < L->pixels) return set_err(OPTB_ERR_ARG, "encode: row_stride < pixels");
  const Geom g = make_geom(L);
  const RowSrc rs{images, row_stride, row_index, nullptr, 0, early ? 1 : 0};
  cudaError_t e = launch_encode(g, rs, containers, offsets, static_cast<cudaStream_t>(stream), c->sms, &c->launches);
  if (e != cudaSuccess) return cuda_err(e, "encode launch");
  return OPTB_OK;
}


int optb_b200::roundtrip_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
                             const int64_t* row_index, void* containers, uint8_t* offsets, const optb_epilogue* E,
                             void* out, void* stream, bool early) {
  int st = roundtrip_checks(c, L, E);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  if (!images || !containers || !out || (optb_mode_has_offsets(L->mode) && !offsets))
    return set_err(OPTB_ERR_ARG, "roundtrip: null buffer");
  if (row_stride == 0) row_stride = L->pixels;
  if (row_stride < L->pixels) return set_err(OPTB_ERR_ARG, "encode: row_stride < pixels");
  return roundtrip(c, L, RowSrc{images, row_stride, row_index, nullptr, 0, early ? 1 : 0}, containers, offsets, E,
                   out, stream);
}


// ------------------------------------------------------------------ host pipeline
namespace {

struct Slice {
  uint64_t row0, rows;       // stream rows [row0, row0 + rows)
  uint64_t chunk0, chunks;   // chunks [chunk0, chunk0 + chunks)
  optb_layout L;             // layout of the slice on its own
};

// Split a stream into slices of about `target` input bytes.  Whole batches
// when a batch is small; otherwise runs of whole chunks inside one batch (a
// run starting at a chunk boundary re-chunks identically).
std::vector<Slice> plan_slices(const optb_layout* L, uint64_t bytes_per_row, uint64_t target) {
  std::vector<Slice> out;
  const uint64_t pc = L->per_chunk;
  const uint64_t cpb = (L->batch + pc - 1) / pc;
  const uint64_t batch_bytes = L->batch * bytes_per_row;
  if (batch_bytes <= target) {
    const uint64_t per = std::max<uint64_t>(1, target / batch_bytes);
    for (uint64_t b = 0; b < L->n_batches; b += per) {
      const uint64_t nb = std::min(per, L->n_batches - b);
      Slice s;
      s.row0 = b * L->batch;
      s.rows = nb * L->batch;
      s.chunk0 = b * cpb;
      s.chunks = nb * cpb;
      s.L = *L;
      s.L.n_batches = nb;
      out.push_back(s);
    }
    return out;
  }
  const uint64_t chunk_bytes = pc * bytes_per_row;
  const uint64_t per_chunks = std::max<uint64_t>(1, target / chunk_bytes);
  for (uint64_t b = 0; b < L->n_batches; ++b) {
    for (uint64_t j = 0; j < cpb; j += per_chunks) {
      const uint64_t nj = std::min(per_chunks, cpb - j);
      const uint64_t r_begin = j * pc, r_end = std::min((j + nj) * pc, L->batch);
      Slice s;
      s.row0 = b * L->batch + r_begin;
      s.rows = r_end - r_begin;
      s.chunk0 = b * cpb + j;
      s.chunks = nj;
      s.L = *L;
      s.L.batch = s.rows;
      s.L.n_batches = 1;
      out.push_back(s);
    }
  }
  return out;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_slots(optb_ctx* c, size_t in_b, size_t out_b, size_t off_b) {
  if (c->slot_in < in_b || c->slot_out < out_b || c->slot_off < off_b) {
    cudaDeviceSynchronize();
    for (int i = 0; i < optb_ctx::kSlots; ++i) {
      if (c->pin_in[i]) cudaFreeHost(c->pin_in[i]);
      if (c->pin_out[i]) cudaFreeHost(c->pin_out[i]);
      if (c->pin_off[i]) cudaFreeHost(c->pin_off[i]);
      if (c->dev_in[i]) cudaFree(c->dev_in[i]);
      if (c->dev_out[i]) cudaFree(c->dev_out[i]);
      if (c->dev_off[i]) cudaFree(c->dev_off[i]);
      c->pin_in[i] = c->pin_out[i] = c->pin_off[i] = nullptr;
      c->dev_in[i] = c->dev_out[i] = c->dev_off[i] = nullptr;
    }
    c->slot_in = std::max(c->slot_in, in_b);
    c->slot_out = std::max(c->slot_out, out_b);
    c->slot_off = std::max<size_t>(std::max(c->slot_off, off_b), 16);
    for (int i = 0; i < optb_ctx::kSlots; ++i) {
      CK(cudaHostAlloc(&c->pin_in[i], c->slot_in, cudaHostAllocMapped | cudaHostAllocPortable), "pinned staging");
      CK(cudaHostAlloc(&c->pin_out[i], c->slot_out, cudaHostAllocMapped | cudaHostAllocPortable), "pinned staging");
      CK(cudaHostAlloc(&c->pin_off[i], c->slot_off, cudaHostAllocMapped | cudaHostAllocPortable), "pinned staging");
      CK(cudaMalloc(&c->dev_in[i], c->slot_in), "device staging");
      CK(cudaMalloc(&c->dev_out[i], c->slot_out), "device staging");
      CK(cudaMalloc(&c->dev_off[i], c->slot_off), "device staging");
    }
  }
  return OPTB_OK;
}

constexpr uint64_t kSliceTarget = 32ull << 20;

// Small host calls (the drop-in API encodes / decodes one chunk per call,
// runner.cpp:77-90, nn.cpp:182): latency is the cost, and every dependent
// copy adds a DMA <-> SM hand-off of several microseconds.  Where the vector
// kernels apply, the kernel runs ZERO-COPY on the context's pinned staging
// (mapped into the device address space): 16-byte cp.async gathers of the
// rows over PCIe, per-lane stores of its results straight into pinned memory
// (g_sysmem: no tensor-map transfers) -- one launch and one synchronisation;
// the decode's error latch is copied out by a second tiny kernel (a kernel to
// kernel hand-off, not a DMA).  Other geometries stage through device memory:
// H2D, kernel, D2H, still on one stream with one synchronisation.
constexpr uint64_t kSmallCall = 4ull << 20;

__global__ void k_latch_out(const DevError* __restrict__ d, DevError* __restrict__ h) {
  if (threadIdx.x == 0) *h = *d;
}

template <typename T>
T* mapped(T* host) {
  void* d = nullptr;
  return cudaHostGetDevicePointer(&d, host, 0) == cudaSuccess ? static_cast<T*>(d) : nullptr;
}

bool small_vec(const optb_layout* L) {
  const bool lossless = L->mode == OPTB_LOSSLESS64 || L->mode == OPTB_LOSSLESS128;
  return L->pixels % (lossless ? 32 : 16) == 0;
}

struct SysmemScope {  // the launches inside read / write mapped host memory
  SysmemScope() { g_sysmem = true; }
  ~SysmemScope() { g_sysmem = false; }
};

int small_encode(optb_ctx* c, const optb_layout* L, const uint8_t* images, void* containers, uint8_t* offsets) {
  const uint64_t P = L->pixels, rows = optb_layout_rows(L);
  const uint64_t cb = optb_layout_container_bytes(L), ob = optb_layout_offsets_bytes(L);
  int st = ensure_slots(c, rows * P, cb, ob);
  if (st) return st;
  cudaStream_t s = c->s_compute;
  memcpy(c->pin_in[0], images, rows * P);
  const Geom g = make_geom(L);
  cudaError_t e;
  if (small_vec(L)) {
    uint8_t *src = mapped(c->pin_in[0]), *dst = mapped(c->pin_out[0]), *odst = mapped(c->pin_off[0]);
    if (!src || !dst || !odst) return cuda_err(cudaGetLastError(), "mapped staging");
    SysmemScope scope;
    e = launch_encode(g, RowSrc{src, P, nullptr, nullptr, 0}, dst, odst, s, c->sms, &c->launches);
  } else {
    CK(cudaMemcpyAsync(c->dev_in[0], c->pin_in[0], rows * P, cudaMemcpyHostToDevice, s), "H2D");
    e = launch_encode(g, RowSrc{c->dev_in[0], P, nullptr, nullptr, 0}, c->dev_out[0], c->dev_off[0], s, c->sms,
                      &c->launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->pin_out[0], c->dev_out[0], cb, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && ob) e = cudaMemcpyAsync(c->pin_off[0], c->dev_off[0], ob, cudaMemcpyDeviceToHost, s);
  }
  if (e != cudaSuccess) return cuda_err(e, "encode launch");
  CK(cudaStreamSynchronize(s), "sync");
  memcpy(containers, c->pin_out[0], cb);
  if (ob) memcpy(offsets, c->pin_off[0], ob);
  g_err.clear();
  return OPTB_OK;
}

int small_decode(optb_ctx* c, const optb_layout* L, const void* containers, const uint8_t* offsets,
                 const optb_epilogue* E, void* out) {
  const uint64_t P = L->pixels, rows = optb_layout_rows(L);
  const uint64_t cb = optb_layout_container_bytes(L), ob = optb_layout_offsets_bytes(L);
  const uint64_t outb = rows * P * out_elem_bytes(E->out_dtype);
  int st = ensure_slots(c, cb, outb, ob);
  if (st) return st;
  cudaStream_t s = c->s_compute;
  memcpy(c->pin_in[0], containers, cb);
  if (ob) memcpy(c->pin_off[0], offsets, ob);
  const Geom g = make_geom(L);
  const Epi ep = make_epi(E, P);
  DevError* h_latch = mapped(&c->pin_err[1]);
  if (!h_latch) return cuda_err(cudaGetLastError(), "mapped latch");
  cudaError_t e;
  if (small_vec(L)) {
    uint8_t *src = mapped(c->pin_in[0]), *dst = mapped(c->pin_out[0]), *osrc = mapped(c->pin_off[0]);
    if (!src || !dst || !osrc) return cuda_err(cudaGetLastError(), "mapped staging");
    SysmemScope scope;
    e = launch_decode(g, src, osrc, ep, dst, c->d_err_small, s, c->sms, &c->launches);
  } else {
    CK(cudaMemcpyAsync(c->dev_in[0], c->pin_in[0], cb, cudaMemcpyHostToDevice, s), "H2D");
    if (ob) CK(cudaMemcpyAsync(c->dev_off[0], c->pin_off[0], ob, cudaMemcpyHostToDevice, s), "H2D");
    e = launch_decode(g, c->dev_in[0], c->dev_off[0], ep, c->dev_out[0], c->d_err_small, s, c->sms, &c->launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->pin_out[0], c->dev_out[0], outb, cudaMemcpyDeviceToHost, s);
  }
  if (e != cudaSuccess) return cuda_err(e, "decode launch");
  k_latch_out<<<1, 32, 0, s>>>(c->d_err_small, h_latch);
  ++c->launches;
  CK(cudaGetLastError(), "latch copy");
  CK(cudaStreamSynchronize(s), "sync");
  const DevError h = c->pin_err[1];
  if (h.kind != kErrNone) {  // rare: report, and clear the latch for the next call
    CK(cudaMemcpy(c->d_err_small, &c->pin_err[0], sizeof(DevError), cudaMemcpyHostToDevice), "error latch");
    return latch_status(h);
  }
  memcpy(out, c->pin_out[0], outb);
  g_err.clear();
  return OPTB_OK;
}

}  // namespace

extern "C" {

// Host encode: images (host) -> containers/offsets (host).  Slices are
// double-buffered: H2D on s_h2d, kernels on s_compute, D2H on s_d2h.
int optb_encode_host(optb_ctx* c, const optb_layout* L, const uint8_t* images, void* containers,
                     uint8_t* offsets) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = optb_layout_check(L);
  if (st) return st;
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const uint64_t P = L->pixels;
  if (optb_layout_rows(L) * P + optb_layout_container_bytes(L) <= kSmallCall)
    return small_encode(c, L, images, containers, offsets);
  const uint32_t wc = optb_container_value_bytes(L->mode);
  const uint64_t ost = optb_offsets_stride(L->mode, P, L->per_chunk);
  const auto slices = plan_slices(L, P, kSliceTarget);
  uint64_t max_rows = 0, max_chunks = 0;
  for (const auto& s : slices) {
    max_rows = std::max(max_rows, s.rows);
    max_chunks = std::max(max_chunks, s.chunks);
  }
  st = ensure_slots(c, max_rows * P, max_chunks * P * wc, max_chunks * ost);
  if (st) return st;
  const bool pin_src = is_pinned(images), pin_dst = is_pinned(containers) &&
                                                   (!ost || is_pinned(offsets));
  auto copy_out = [&](size_t i) -> int {
    const Slice& s = slices[i];
    const int k = static_cast<int>(i % optb_ctx::kSlots);
    CK(cudaEventSynchronize(c->ev_d2h[k]), "D2H");
    if (!pin_dst) {
      memcpy(static_cast<uint8_t*>(containers) + s.chunk0 * P * wc, c->pin_out[k], s.chunks * P * wc);
      if (ost) memcpy(offsets + s.chunk0 * ost, c->pin_off[k], s.chunks * ost);
    }
    return OPTB_OK;
  };
  for (size_t i = 0; i < slices.size(); ++i) {
    const Slice& s = slices[i];
    const int k = static_cast<int>(i % optb_ctx::kSlots);
    const uint8_t* src = images + s.row0 * P;
    if (!pin_src) {
      CK(cudaEventSynchronize(c->ev_h2d[k]), "H2D");
      memcpy(c->pin_in[k], src, s.rows * P);
      src = c->pin_in[k];
    }
    CK(cudaStreamWaitEvent(c->s_h2d, c->ev_kern[k], 0), "wait");
    CK(cudaMemcpyAsync(c->dev_in[k], src, s.rows * P, cudaMemcpyHostToDevice, c->s_h2d), "H2D");
    CK(cudaEventRecord(c->ev_h2d[k], c->s_h2d), "event");
    CK(cudaStreamWaitEvent(c->s_compute, c->ev_h2d[k], 0), "wait");
    CK(cudaStreamWaitEvent(c->s_compute, c->ev_d2h[k], 0), "wait");
    const Geom g = make_geom(&s.L);
    cudaError_t e = launch_encode(g, RowSrc{c->dev_in[k], P, nullptr, nullptr, 0}, c->dev_out[k], c->dev_off[k],
                                  c->s_compute, c->sms, &c->launches);
    if (e != cudaSuccess) return cuda_err(e, "encode launch");
    CK(cudaEventRecord(c->ev_kern[k], c->s_compute), "event");
    CK(cudaStreamWaitEvent(c->s_d2h, c->ev_kern[k], 0), "wait");
    uint8_t* dst = pin_dst ? static_cast<uint8_t*>(containers) + s.chunk0 * P * wc : c->pin_out[k];
    CK(cudaMemcpyAsync(dst, c->dev_out[k], s.chunks * P * wc, cudaMemcpyDeviceToHost, c->s_d2h), "D2H");
    if (ost) {
      uint8_t* od = pin_dst ? offsets + s.chunk0 * ost : c->pin_off[k];
      CK(cudaMemcpyAsync(od, c->dev_off[k], s.chunks * ost, cudaMemcpyDeviceToHost, c->s_d2h), "D2H");
    }
    CK(cudaEventRecord(c->ev_d2h[k], c->s_d2h), "event");
    if (i >= 1) {
      st = copy_out(i - 1);
      if (st) return st;
    }
  }
  st = copy_out(slices.size() - 1);
  if (st) return st;
  CK(cudaStreamSynchronize(c->s_d2h), "sync");
  g_err.clear();
  return OPTB_OK;
}

int optb_decode_host(optb_ctx* c, const optb_layout* L, const void* containers,
                     const uint8_t* offsets, const optb_epilogue* E, void* out) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  int st = check_decode_layout(L);
  if (st) return st;
  st = check_epilogue(E);
  if (st) return st;
  if (E->class_scale || E->row_class)
    return set_err(OPTB_ERR_ARG, "decode_host: class tables are device-side; use optb_decode_dev");
  if (optb_layout_rows(L) == 0) return OPTB_OK;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  const uint64_t P = L->pixels;
  const uint32_t wc = optb_container_value_bytes(L->mode);
  const uint64_t ost = optb_offsets_stride(L->mode, P, L->per_chunk);
  const size_t es = out_elem_bytes(E->out_dtype);
  const uint64_t ors = E->out_row_stride ? E->out_row_stride : P;
  if (ors != P) return set_err(OPTB_ERR_ARG, "decode_host: out_row_stride must be 0 or P");
  if (optb_layout_container_bytes(L) + optb_layout_rows(L) * P * es <= kSmallCall)
    return small_decode(c, L, containers, offsets, E, out);
  // slice on container bytes per row (one chunk of per_chunk rows is P*wc)
  const auto slices = plan_slices(L, (P * wc + L->per_chunk - 1) / L->per_chunk, kSliceTarget);
  uint64_t max_rows = 0, max_chunks = 0;
  for (const auto& s : slices) {
    max_rows = std::max(max_rows, s.rows);
    max_chunks = std::max(max_chunks, s.chunks);
  }
  st = ensure_slots(c, max_chunks * P * wc, max_rows * P * es, max_chunks * ost);
  if (st) return st;
  st = reset_err(c, c->s_compute);
  if (st) return st;
  const bool pin_src = is_pinned(containers) && (!ost || is_pinned(offsets));
  const bool pin_dst = is_pinned(out);
  auto copy_out = [&](size_t i) -> int {
    const Slice& s = slices[i];
    const int k = static_cast<int>(i % optb_ctx::kSlots);
    CK(cudaEventSynchronize(c->ev_d2h[k]), "D2H");
    if (!pin_dst) memcpy(static_cast<uint8_t*>(out) + s.row0 * P * es, c->pin_out[k], s.rows * P * es);
    return OPTB_OK;
  };
  for (size_t i = 0; i < slices.size(); ++i) {
    const Slice& s = slices[i];
    const int k = static_cast<int>(i % optb_ctx::kSlots);
    const uint8_t* src = static_cast<const uint8_t*>(containers) + s.chunk0 * P * wc;
    const uint8_t* osrc = ost ? offsets + s.chunk0 * ost : nullptr;
    if (!pin_src) {
      CK(cudaEventSynchronize(c->ev_h2d[k]), "H2D");
      memcpy(c->pin_in[k], src, s.chunks * P * wc);
      src = c->pin_in[k];
      if (ost) {
        memcpy(c->pin_off[k], osrc, s.chunks * ost);
        osrc = c->pin_off[k];
      }
    }
    CK(cudaStreamWaitEvent(c->s_h2d, c->ev_kern[k], 0), "wait");
    CK(cudaMemcpyAsync(c->dev_in[k], src, s.chunks * P * wc, cudaMemcpyHostToDevice, c->s_h2d), "H2D");
    if (ost)
      CK(cudaMemcpyAsync(c->dev_off[k], osrc, s.chunks * ost, cudaMemcpyHostToDevice, c->s_h2d), "H2D");
    CK(cudaEventRecord(c->ev_h2d[k], c->s_h2d), "event");
    CK(cudaStreamWaitEvent(c->s_compute, c->ev_h2d[k], 0), "wait");
    CK(cudaStreamWaitEvent(c->s_compute, c->ev_d2h[k], 0), "wait");
    Geom g = make_geom(&s.L);
    g.chunk_base = s.chunk0;
    Epi ep = make_epi(E, P);
    cudaError_t e = launch_decode(g, c->dev_in[k], c->dev_off[k], ep, c->dev_out[k], c->d_err,
                                  c->s_compute, c->sms, &c->launches);
    if (e != cudaSuccess) return cuda_err(e, "decode launch");
    CK(cudaEventRecord(c->ev_kern[k], c->s_compute), "event");
    CK(cudaStreamWaitEvent(c->s_d2h, c->ev_kern[k], 0), "wait");
    uint8_t* dst = pin_dst ? static_cast<uint8_t*>(out) + s.row0 * P * es : c->pin_out[k];
    CK(cudaMemcpyAsync(dst, c->dev_out[k], s.rows * P * es, cudaMemcpyDeviceToHost, c->s_d2h), "D2H");
    CK(cudaEventRecord(c->ev_d2h[k], c->s_d2h), "event");
    if (i >= 1) {
      st = copy_out(i - 1);
      if (st) return st;
    }
  }
  st = copy_out(slices.size() - 1);
  if (st) return st;
  return optb_ctx_sync(c, c->s_d2h);
}

}  // extern "C"

// ------------------------------------------------------------------ SBS
// ------------------------------------------------------------------ SBS
// Host side of the GPU BatchCursor: it only plans.  Per call it lists the
// reshuffle events (class, generation) in the reference's chain order
// (sampler.cpp:91-104: batch, then class, then draw), lays out the
// generation pool, and uploads one small block; the kernels do the rest.
struct optb_sbs {
  optb_ctx* ctx = nullptr;
  uint64_t C = 0, B = 0, N = 0;
  std::vector<uint64_t> counts, m, off, prefix, gen;
  uint64_t batches = 0;
  int force_serial = 0;
  bool prof = false;               // optb_sbs_set_profiling
  cudaEvent_t pe[4] = {};          // call start, uploaded, reshuffled, gathered
  bool small_ids = true;  // every example id < 2^32 (shared-memory shuffle)
  uint32_t max_m = 0;
  // device
  int64_t* d_pool = nullptr;  // [N current permutations][generation area]
  uint64_t pool_cap = 0;      // elements
  unsigned long long* d_chain = nullptr;
  // host mirror of the chain state after every enqueued call (the seeds of a
  // call's events are walked here, one mix each); a device-side serial redo
  // that ends elsewhere bumps *diverged_h and the next call resyncs
  uint64_t host_chain = 0;
  unsigned int* diverged_h = nullptr;  // mapped pinned counter
  unsigned int* diverged_d = nullptr;
  unsigned int diverged_seen = 0;
  uint8_t* d_static = nullptr;  // counts[C] prefix[C+1] size[C] row_cls[B]
  uint64_t* d_recip = nullptr;  // [max_m + 1] reciprocals for the Fisher-Yates reductions (launch_recip_table)
  uint8_t* d_call = nullptr;    // per-call block (stream ordered reuse)
  size_t call_cap = 0;
  static constexpr int kRing = 4;  // pinned upload buffers in flight
  uint8_t* h_call[kRing] = {};
  size_t h_call_cap[kRing] = {};
  cudaEvent_t uploaded[kRing] = {};
  int ring = 0;
  // scratch for next_host
  int64_t* d_ex = nullptr;
  int32_t* d_cl = nullptr;
  int64_t* h_ex = nullptr;  // pinned bounce buffers of optb_sbs_next_host
  int32_t* h_cl = nullptr;
  uint64_t ex_cap = 0;
};

uint64_t optb_b200::sbs_examples(const optb_sbs* s) { return s ? s->N : 0; }
namespace {
int ensure_pool(optb_sbs* s, uint64_t elems, cudaStream_t st);
int ensure_call_slot(optb_sbs* s, int r, size_t bytes, cudaStream_t st);
}
// Pool size for any call of up to n batches: class c starts at most
// floor(n * count_c / m_c) + 1 generations in it and gets one more slot for
// its pre-call permutation (run_events layout).  Growing the pool inside a
// call synchronises the call's stream, which in a pipeline waits for the
// step that last used the draw buffer -- so the pipeline reserves up front.
int optb_b200::sbs_reserve(optb_sbs* s, uint64_t n) {
  if (!s) return OPTB_OK;
  uint64_t need = s->N, events = 0;
  for (uint64_t c = 0; c < s->C; ++c) {
    if (!s->counts[c]) continue;
    const uint64_t e = n * s->counts[c] / std::max<uint64_t>(s->m[c], 1) + 1;
    events += e;
    if (s->m[c] >= 2) need += (e + 1) * s->m[c];
  }
  int rc = ensure_pool(s, std::max<uint64_t>(need, 1), s->ctx->s_compute);
  if (rc) return rc;
  // the call block: event records, seeds, per-class lists and the gather
  // tables (run_events / optb_sbs_next_dev), 16-byte padded pieces
  const size_t block = events * (sizeof(SbsEvent) + 8 + 4) + s->C * (4 + 8 + 8 + 32) + 1024;
  for (int r = 0; r < optb_sbs::kRing; ++r) {
    rc = ensure_call_slot(s, r, block, s->ctx->s_compute);
    if (rc) return rc;
  }
  return OPTB_OK;
}

namespace {

// SplitMix64 finaliser (rng.hpp:16-21), host side.
uint64_t host_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Packs per-call arrays into one 16-byte aligned block.
struct Packer {
  std::vector<uint8_t> buf;
  template <typename T>
  size_t put(const T* p, size_t n) {
    size_t at = (buf.size() + 15) / 16 * 16;
    buf.resize(at + n * sizeof(T));
    if (n) memcpy(buf.data() + at, p, n * sizeof(T));
    return at;
  }
  size_t reserve(size_t bytes) {
    size_t at = (buf.size() + 15) / 16 * 16;
    buf.resize(at + bytes, 0);
    return at;
  }
};

// Pinned slot r and the device block hold at least `bytes` (growing the
// device block waits for the calls in flight on `st`).
int ensure_call_slot(optb_sbs* s, int r, size_t bytes, cudaStream_t st) {
  if (s->h_call_cap[r] < bytes) {
    if (s->h_call[r]) cudaFreeHost(s->h_call[r]);
    s->h_call[r] = nullptr;
    CK(cudaHostAlloc(&s->h_call[r], bytes * 2 + 16, cudaHostAllocMapped | cudaHostAllocPortable), "sbs pinned");
    s->h_call_cap[r] = bytes * 2;
  }
  if (s->call_cap < bytes) {
    if (s->d_call) {
      CK(cudaStreamSynchronize(st), "sbs sync");
      cudaFree(s->d_call);
    }
    s->d_call = nullptr;
    CK(cudaMalloc(&s->d_call, bytes * 2), "sbs call block");
    s->call_cap = bytes * 2;
  }
  return OPTB_OK;
}

int upload_call(optb_sbs* s, const Packer& pk, cudaStream_t st) {
  const size_t bytes = std::max<size_t>(pk.buf.size(), 16);
  const int r = s->ring;
  s->ring = (s->ring + 1) % optb_sbs::kRing;
  CK(cudaEventSynchronize(s->uploaded[r]), "sbs upload");  // this pinned slot is free again
  int rc = ensure_call_slot(s, r, bytes, st);
  if (rc) return rc;
  memcpy(s->h_call[r], pk.buf.data(), pk.buf.size());
  // A kernel pulls the block over PCIe from the mapped pinned slot instead of
  // a cudaMemcpyAsync: an H2D copy would queue on the copy engine behind any
  // bulk upload in flight (the e2e leg streams a 153.6 MB dataset per step)
  // and stall the draws for milliseconds.
  void* src = nullptr;
  CK(cudaHostGetDevicePointer(&src, s->h_call[r], 0), "sbs mapped slot");
  CK(launch_copy_in(src, s->d_call, bytes, st, &s->ctx->launches), "sbs upload");
  CK(cudaEventRecord(s->uploaded[r], st), "sbs upload");
  return OPTB_OK;
}

int ensure_pool(optb_sbs* s, uint64_t elems, cudaStream_t st) {
  if (s->pool_cap >= elems) return OPTB_OK;
  const uint64_t cap = std::max<uint64_t>(elems, s->pool_cap * 2);
  int64_t* p = nullptr;
  CK(cudaStreamSynchronize(st), "sbs pool");
  CK(cudaMalloc(&p, cap * sizeof(int64_t)), "sbs pool");
  if (s->d_pool) {
    CK(cudaMemcpyAsync(p, s->d_pool, s->N * sizeof(int64_t), cudaMemcpyDeviceToDevice, st), "sbs pool");
    CK(cudaStreamSynchronize(st), "sbs pool");
    cudaFree(s->d_pool);
  }
  s->d_pool = p;
  s->pool_cap = cap;
  return OPTB_OK;
}

struct EvKey {
  uint64_t beta, cls, g;
  uint64_t t;  // 1-based index of the event among its class's events in this call
};

// Lazy reshuffles of the next n batches (sampler.cpp:97): class c's draw D
// (counted from the constructor) starts generation D / m_c when
// D % m_c == 0 and D > 0.  Chain order is (batch, class, generation); the
// classes are enumerated in order and each class's generations in order, so
// a stable counting sort by batch gives the whole order in O(events +
// batches) (N-GPU runs plan N x 97 batches per step; a comparison sort
// dominated the host time).
std::vector<EvKey> plan_events(uint64_t C, const uint64_t* counts, const uint64_t* m, const uint64_t* gen,
                               uint64_t batches, uint64_t n, std::vector<uint64_t>* ev_count) {
  std::vector<EvKey> gen_order;
  ev_count->assign(C, 0);
  std::vector<uint64_t> at(n + 2, 0);
  for (uint64_t c = 0; c < C; ++c) {
    const uint64_t cnt = counts[c], mm = m[c];
    if (cnt == 0 || mm == 0) continue;
    const uint64_t D1 = (batches + n) * cnt;
    for (uint64_t g = gen[c] + 1; g * mm < D1; ++g) {
      const uint64_t beta = (g * mm) / cnt;  // in [batches, batches + n)
      gen_order.push_back({beta, c, g, g - gen[c]});
      ++at[beta - batches + 1];
      ++(*ev_count)[c];
    }
  }
  for (uint64_t b = 0; b <= n; ++b) at[b + 1] += at[b];
  std::vector<EvKey> keys(gen_order.size());
  for (const EvKey& k : gen_order) keys[at[k.beta - batches]++] = k;
  return keys;
}

// Lays out the generation pool for `keys` (already in chain order) starting at
// element N: a reshuffling class c with E_c events gets E_c + 1 slots of m_c
// (slot 0 = copy of its pre-call permutation).  Fills the event records and
// the per-class K9 lists, packs them and launches K9 + K8.  `gen_base` gets,
// per class, the pool offset of the pre-call permutation the gather reads.
int run_events(optb_sbs* s, const std::vector<EvKey>& keys, Packer& pk,
               std::vector<uint64_t>* gen_base, size_t* o_extra, const std::vector<uint64_t>* extra,
               cudaStream_t st) {
  const uint64_t C = s->C, E = keys.size();
  std::vector<uint64_t> ev_count(C, 0);
  for (const auto& k : keys) ++ev_count[k.cls];
  std::vector<uint64_t> base(C, 0);
  uint64_t cursor = s->N;
  for (uint64_t c = 0; c < C; ++c) {
    if (ev_count[c] == 0 || s->m[c] < 2) continue;
    base[c] = cursor;
    cursor += (ev_count[c] + 1) * s->m[c];
  }
  int rc = ensure_pool(s, std::max<uint64_t>(cursor, 1), st);
  if (rc) return rc;
  std::vector<SbsEvent> evs(E);
  std::vector<std::vector<uint32_t>> per(C);
  for (uint64_t e = 0; e < E; ++e) {
    const uint64_t c = keys[e].cls, mm = s->m[c], t = keys[e].t;
    evs[e].cls = static_cast<uint32_t>(c);
    evs[e].m = static_cast<uint32_t>(mm);
    if (mm >= 2) {
      evs[e].slot = base[c] + t * mm;
      evs[e].src = (t == 1) ? s->off[c] : base[c] + (t - 1) * mm;
      per[c].push_back(static_cast<uint32_t>(e));
    } else {
      evs[e].slot = evs[e].src = s->off[c];
    }
  }
  std::vector<uint32_t> begin{0}, list;
  std::vector<uint64_t> ccopy, cfinal;
  for (uint64_t c = 0; c < C; ++c) {
    if (per[c].empty()) continue;
    for (uint32_t e : per[c]) list.push_back(e);
    begin.push_back(static_cast<uint32_t>(list.size()));
    ccopy.push_back(base[c]);
    cfinal.push_back(s->off[c]);
  }
  if (gen_base) {
    gen_base->assign(C, 0);
    for (uint64_t c = 0; c < C; ++c) (*gen_base)[c] = per[c].empty() ? s->off[c] : base[c];
  }
  // the chain seeds of this call's events, walked on the host from its mirror
  // of the device state (resynced first if a serial redo diverged from it)
  if (*reinterpret_cast<volatile unsigned int*>(s->diverged_h) != s->diverged_seen) {
    CK(cudaDeviceSynchronize(), "sbs resync");
    unsigned long long dev_chain = 0;
    CK(cudaMemcpy(&dev_chain, s->d_chain, 8, cudaMemcpyDeviceToHost), "sbs resync");
    s->host_chain = dev_chain;
    s->diverged_seen = *reinterpret_cast<volatile unsigned int*>(s->diverged_h);
  }
  std::vector<uint64_t> seeds(std::max<uint64_t>(E, 1), 0);
  const uint64_t expect_start = s->host_chain;
  uint64_t chain = expect_start;
  for (uint64_t e = 0; e < E; ++e) {  // K = m-1 draws + next_u64 (sampler.cpp:84-88), one mix
    seeds[e] = chain;
    chain = host_mix64(chain + (evs[e].m >= 2 ? static_cast<uint64_t>(evs[e].m) : 1ull) * 0x9e3779b97f4a7c15ull);
  }
  s->host_chain = chain;
  const size_t o_ev = pk.put(evs.data(), E);
  const size_t o_seeds = pk.put(seeds.data(), seeds.size());
  const size_t o_flag = pk.reserve(16);
  const size_t o_begin = pk.put(begin.data(), begin.size());
  const size_t o_list = pk.put(list.data(), list.size());
  const size_t o_copy = pk.put(ccopy.data(), ccopy.size());
  const size_t o_final = pk.put(cfinal.data(), cfinal.size());
  if (extra) *o_extra = pk.put(extra->data(), extra->size());
  if (s->prof) cudaEventRecord(s->pe[0], st);
  rc = upload_call(s, pk, st);
  if (s->prof) cudaEventRecord(s->pe[1], st);
  if (rc) return rc;
  if (E == 0) {
    if (s->prof) cudaEventRecord(s->pe[2], st);
    return OPTB_OK;
  }
  uint8_t* d = s->d_call;
  ChainArgs a;
  a.ev = reinterpret_cast<const SbsEvent*>(d + o_ev);
  a.E = E;
  a.cls_begin = reinterpret_cast<const uint32_t*>(d + o_begin);
  a.cls_list = reinterpret_cast<const uint32_t*>(d + o_list);
  a.cls_copy = reinterpret_cast<const uint64_t*>(d + o_copy);
  a.cls_final = reinterpret_cast<const uint64_t*>(d + o_final);
  a.seeds = reinterpret_cast<uint64_t*>(d + o_seeds);
  a.flag = reinterpret_cast<uint32_t*>(d + o_flag);
  a.chain = s->d_chain;
  a.pool = s->d_pool;
  a.expect_start = expect_start;
  a.expect_final = chain;
  a.diverged = s->diverged_d;
  a.recip = s->d_recip;
  uint64_t max_gen_words = 0;
  for (uint64_t c = 0; c < C; ++c)
    if (!per[c].empty()) max_gen_words = std::max<uint64_t>(max_gen_words, per[c].size() * s->m[c]);
  cudaError_t e = launch_sbs_events(a, static_cast<uint32_t>(ccopy.size()), static_cast<uint32_t>(list.size()),
                                    s->small_ids ? s->max_m : 0xffffffffu, max_gen_words, s->force_serial, st,
                                    &s->ctx->launches);
  if (e != cudaSuccess) return cuda_err(e, "sbs events");
  if (s->prof) cudaEventRecord(s->pe[2], st);
  return OPTB_OK;
}

}  // namespace

extern "C" {

int optb_sbs_plan(const double* w, uint64_t C, uint64_t B, uint64_t* counts) {
  // sampler.cpp:11-51
  if (C == 0) return set_err(OPTB_ERR, "sampler: at least one class weight required");
  if (B == 0) return set_err(OPTB_ERR, "sampler: batch size must be positive");
  if (!w || !counts) return set_err(OPTB_ERR_ARG, "sampler: null buffer");
  double sum = 0.0;
  for (uint64_t c = 0; c < C; ++c) {
    if (w[c] < 0.0)
      return set_err(OPTB_ERR, "sampler: negative weight for class %llu", (unsigned long long)c);
    sum += w[c];
  }
  if (std::abs(sum - 1.0) > 1e-9)
    return set_err(OPTB_ERR, "sampler: class weights sum to %s, expected 1",
                   std::to_string(sum).c_str());
  std::vector<double> rem(C);
  std::vector<uint64_t> order(C);
  uint64_t assigned = 0;
  for (uint64_t c = 0; c < C; ++c) {
    const double exact = w[c] * static_cast<double>(B);
    counts[c] = static_cast<uint64_t>(std::floor(exact));
    rem[c] = exact - std::floor(exact);
    assigned += counts[c];
    order[c] = c;
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](uint64_t a, uint64_t b) { return rem[a] > rem[b]; });
  for (uint64_t k = 0; assigned < B; ++k) {
    counts[order[k % C]] += 1;
    ++assigned;
  }
  g_err.clear();
  return OPTB_OK;
}

int optb_class_index_dev(optb_ctx* c, const int32_t* labels, uint64_t n, uint64_t C,
                         uint64_t* class_offsets, int64_t* members, void* stream) {
  if (!c) return set_err(OPTB_ERR_ARG, "ctx: null");
  if (C == 0) return set_err(OPTB_ERR_ARG, "class index: no classes");
  if (C > 50000) return set_err(OPTB_ERR_ARG, "class index: more than 50000 classes unsupported");
  if (n >= (1ull << 32)) return set_err(OPTB_ERR_ARG, "class index: n >= 2^32 unsupported");
  const uint64_t words = std::max<uint64_t>(class_index_scratch_words(n, C), 1);
  if (c->ci_words < words) {
    if (c->ci_scratch) cudaFree(c->ci_scratch);
    c->ci_scratch = nullptr;
    c->ci_words = 0;
    CK(cudaMalloc(&c->ci_scratch, words * sizeof(uint32_t)), "class index scratch");
    c->ci_words = words;
  }
  cudaError_t e = launch_class_index(labels, n, C, class_offsets, members, c->ci_scratch,
                                     c->ci_words, c->d_err, static_cast<cudaStream_t>(stream),
                                     &c->launches);
  if (e != cudaSuccess) return cuda_err(e, "class index launch");
  return OPTB_OK;
}


int optb_class_index_host(optb_ctx* c, const int32_t* labels, uint64_t n, uint64_t C,
                          uint64_t* class_offsets, int64_t* members) {
  if (!c || (!labels && n) || !class_offsets || (!members && n)) return set_err(OPTB_ERR_ARG, "class index: null");
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  int32_t* d_lab = nullptr;
  uint64_t* d_off = nullptr;
  int64_t* d_mem = nullptr;
  auto release = [&] {
    if (d_lab) cudaFree(d_lab);
    if (d_off) cudaFree(d_off);
    if (d_mem) cudaFree(d_mem);
  };
  if (cudaMalloc(&d_lab, std::max<uint64_t>(n, 1) * 4) != cudaSuccess ||
      cudaMalloc(&d_off, (C + 1) * 8) != cudaSuccess ||
      cudaMalloc(&d_mem, std::max<uint64_t>(n, 1) * 8) != cudaSuccess) {
    release();
    return cuda_err(cudaGetLastError(), "class index buffers");
  }
  cudaStream_t st = c->s_compute;
  int rc = OPTB_OK;
  if (n && cudaMemcpyAsync(d_lab, labels, n * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = cuda_err(cudaGetLastError(), "class index upload");
  if (!rc) rc = optb_class_index_dev(c, d_lab, n, C, d_off, d_mem, st);
  if (!rc) rc = optb_ctx_sync(c, st);
  if (!rc && (cudaMemcpy(class_offsets, d_off, (C + 1) * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
              (n && cudaMemcpy(members, d_mem, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess)))
    rc = cuda_err(cudaGetLastError(), "class index download");
  release();
  return rc;
}

namespace {
// the reciprocal table of the parallel Fisher-Yates (one per sampler)
int build_recip(optb_sbs* s, cudaStream_t st) {
  if (!s->small_ids || s->max_m < 2) return OPTB_OK;
  if (cudaMalloc(&s->d_recip, (static_cast<size_t>(s->max_m) + 1) * 8) != cudaSuccess)
    return cuda_err(cudaGetLastError(), "sbs reciprocals");
  const cudaError_t e = launch_recip_table(s->d_recip, s->max_m, st);
  return e == cudaSuccess ? OPTB_OK : cuda_err(e, "sbs reciprocals");
}
}  // namespace

int optb_sbs_create(optb_ctx* c, const uint64_t* counts, uint64_t C, uint64_t B, uint64_t seed,
                    const uint64_t* class_offsets, const int64_t* members, int32_t on_dev,
                    optb_sbs** out) {
  if (!c || !out || !counts || !class_offsets) return set_err(OPTB_ERR_ARG, "sbs: null argument");
  *out = nullptr;
  if (C == 0) return set_err(OPTB_ERR, "sampler: at least one class weight required");
  uint64_t total = 0;
  for (uint64_t k = 0; k < C; ++k) total += counts[k];
  if (total != B)
    return set_err(OPTB_ERR_ARG, "sbs: counts sum to %llu, batch is %llu", (unsigned long long)total,
                   (unsigned long long)B);
  for (uint64_t k = 0; k < C; ++k) {  // sampler.cpp:75-79
    if (class_offsets[k + 1] < class_offsets[k]) return set_err(OPTB_ERR_ARG, "sbs: offsets not monotone");
    if (counts[k] > 0 && class_offsets[k + 1] == class_offsets[k])
      return set_err(OPTB_ERR, "sampler: class %llu has no examples but a positive batch count",
                     (unsigned long long)k);
  }
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  auto* s = new optb_sbs();
  s->ctx = c;
  s->C = C;
  s->B = B;
  s->N = class_offsets[C];
  s->counts.assign(counts, counts + C);
  s->off.assign(class_offsets, class_offsets + C + 1);
  s->m.resize(C);
  s->gen.assign(C, 0);
  s->prefix.assign(C + 1, 0);
  for (uint64_t k = 0; k < C; ++k) {
    s->m[k] = s->off[k + 1] - s->off[k];
    s->prefix[k + 1] = s->prefix[k] + counts[k];
    if (s->m[k] >= (1ull << 32)) s->small_ids = false;
    else if (s->m[k] >= 2) s->max_m = std::max<uint32_t>(s->max_m, static_cast<uint32_t>(s->m[k]));
  }
  if (s->N >= (1ull << 32)) s->small_ids = false;
  cudaStream_t st = c->s_compute;
  auto fail = [&](int code) {
    optb_sbs_destroy(s);
    return code;
  };
  for (int r = 0; r < optb_sbs::kRing; ++r)
    if (cudaEventCreateWithFlags(&s->uploaded[r], cudaEventDisableTiming) != cudaSuccess)
      return fail(cuda_err(cudaGetLastError(), "sbs event"));
  if (cudaMalloc(&s->d_chain, sizeof(unsigned long long)) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs chain"));
  if (cudaHostAlloc(&s->diverged_h, 16, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->diverged_d), s->diverged_h, 0) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs mapped counter"));
  *s->diverged_h = 0;
  int rc = ensure_pool(s, std::max<uint64_t>(s->N, 1), st);
  if (rc) return fail(rc);
  if (s->N) {
    if (on_dev) {
      // device members may still be in flight on the caller's stream
      if (cudaDeviceSynchronize() != cudaSuccess) return fail(cuda_err(cudaGetLastError(), "sbs members"));
      if (cudaMemcpyAsync(s->d_pool, members, s->N * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return fail(cuda_err(cudaGetLastError(), "sbs members"));
    } else {
      for (uint64_t i = 0; i < s->N; ++i)
        if (members[i] < 0 || static_cast<uint64_t>(members[i]) >= (1ull << 32)) s->small_ids = false;
      if (cudaMemcpy(s->d_pool, members, s->N * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(cuda_err(cudaGetLastError(), "sbs members"));
    }
  }
  {  // static device arrays: counts, prefix, class sizes, row -> class
    std::vector<uint32_t> row_cls(B);
    for (uint64_t k = 0; k < C; ++k)
      for (uint64_t r = s->prefix[k]; r < s->prefix[k + 1]; ++r) row_cls[r] = static_cast<uint32_t>(k);
    Packer pk;
    pk.put(s->counts.data(), C);
    pk.put(s->prefix.data(), C + 1);
    pk.put(s->m.data(), C);
    pk.put(row_cls.data(), B);
    if (cudaMalloc(&s->d_static, pk.buf.size() + 16) != cudaSuccess ||
        cudaMemcpy(s->d_static, pk.buf.data(), pk.buf.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(cuda_err(cudaGetLastError(), "sbs static"));
  }
  rc = build_recip(s, st);
  if (rc) return fail(rc);
  // pool and call blocks sized once for calls of up to 64 Ki draws (the
  // drop-in cursor's largest ring refill): a growing caller then pays no
  // synchronising reallocation inside a call (C2 stream: a 128-batch refill
  // 2.5-11 ms -> the draw time)
  rc = optb_b200::sbs_reserve(s, std::max<uint64_t>(1, (1ull << 16) / std::max<uint64_t>(B, 1)));
  if (rc) return fail(rc);
  const unsigned long long seed64 = seed;
  if (cudaMemcpy(s->d_chain, &seed64, 8, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs seed"));
  s->host_chain = seed64;
  // constructor: reshuffle every class in class order (sampler.cpp:73-81),
  // including empty and single-example classes (they still consume a draw)
  std::vector<EvKey> keys(C);
  for (uint64_t k = 0; k < C; ++k) keys[k] = {0, k, 0, 1};
  Packer pk;
  rc = run_events(s, keys, pk, nullptr, nullptr, nullptr, st);
  if (rc) return fail(rc);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(cuda_err(cudaGetLastError(), "sbs ctor"));
  *out = s;
  g_err.clear();
  return OPTB_OK;
}

int optb_sbs_clone(const optb_sbs* src, optb_sbs** out) {
  if (!src || !out) return set_err(OPTB_ERR_ARG, "sbs: null argument");
  *out = nullptr;
  optb_ctx* c = src->ctx;
  CK(cudaSetDevice(c->device), "cudaSetDevice");
  // every call enqueued on the source (any stream) has finished: its device
  // chain and permutations are the state after its last call
  CK(cudaDeviceSynchronize(), "sbs clone");
  auto* s = new optb_sbs();
  s->ctx = c;
  s->C = src->C;
  s->B = src->B;
  s->N = src->N;
  s->counts = src->counts;
  s->m = src->m;
  s->off = src->off;
  s->prefix = src->prefix;
  s->gen = src->gen;
  s->batches = src->batches;
  s->force_serial = src->force_serial;
  s->small_ids = src->small_ids;
  s->max_m = src->max_m;
  auto fail = [&](int code) {
    optb_sbs_destroy(s);
    return code;
  };
  for (int r = 0; r < optb_sbs::kRing; ++r)
    if (cudaEventCreateWithFlags(&s->uploaded[r], cudaEventDisableTiming) != cudaSuccess)
      return fail(cuda_err(cudaGetLastError(), "sbs event"));
  if (cudaMalloc(&s->d_chain, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemcpy(s->d_chain, src->d_chain, 8, cudaMemcpyDeviceToDevice) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs chain"));
  unsigned long long chain = 0;
  if (cudaMemcpy(&chain, src->d_chain, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs chain"));
  s->host_chain = chain;  // the device chain is authoritative (a serial redo may have moved it)
  if (cudaHostAlloc(&s->diverged_h, 16, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->diverged_d), s->diverged_h, 0) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs mapped counter"));
  *s->diverged_h = 0;
  int rc = ensure_pool(s, std::max<uint64_t>(s->N, 1), c->s_compute);
  if (rc) return fail(rc);
  if (s->N && cudaMemcpy(s->d_pool, src->d_pool, s->N * 8, cudaMemcpyDeviceToDevice) != cudaSuccess)
    return fail(cuda_err(cudaGetLastError(), "sbs permutations"));
  {  // static arrays: same bytes as the source's (layout of optb_sbs_create)
    size_t bytes = 0;
    auto add = [&](size_t b) { bytes = (bytes + 15) / 16 * 16 + b; };
    add(s->C * 8);
    add((s->C + 1) * 8);
    add(s->C * 8);
    add(s->B * 4);
    if (cudaMalloc(&s->d_static, bytes + 16) != cudaSuccess ||
        cudaMemcpy(s->d_static, src->d_static, bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
      return fail(cuda_err(cudaGetLastError(), "sbs static"));
  }
  rc = build_recip(s, c->s_compute);
  if (rc) return fail(rc);
  rc = optb_b200::sbs_reserve(s, std::max<uint64_t>(1, (1ull << 16) / std::max<uint64_t>(s->B, 1)));
  if (rc) return fail(rc);
  if (cudaStreamSynchronize(c->s_compute) != cudaSuccess) return fail(cuda_err(cudaGetLastError(), "sbs clone"));
  *out = s;
  g_err.clear();
  return OPTB_OK;
}

void optb_sbs_destroy(optb_sbs* s) {
  if (!s) return;
  cudaDeviceSynchronize();
  if (s->d_pool) cudaFree(s->d_pool);
  if (s->d_chain) cudaFree(s->d_chain);
  if (s->diverged_h) cudaFreeHost(s->diverged_h);
  if (s->d_static) cudaFree(s->d_static);
  if (s->d_recip) cudaFree(s->d_recip);
  if (s->d_call) cudaFree(s->d_call);
  for (int r = 0; r < optb_sbs::kRing; ++r) {
    if (s->h_call[r]) cudaFreeHost(s->h_call[r]);
    if (s->uploaded[r]) cudaEventDestroy(s->uploaded[r]);
  }
  if (s->d_ex) cudaFree(s->d_ex);
  if (s->d_cl) cudaFree(s->d_cl);
  if (s->h_ex) cudaFreeHost(s->h_ex);
  if (s->h_cl) cudaFreeHost(s->h_cl);
  for (auto& e : s->pe)
    if (e) cudaEventDestroy(e);
  delete s;
}

uint64_t optb_sbs_batches_drawn(const optb_sbs* s) { return s ? s->batches : 0; }

int optb_sbs_set_profiling(optb_sbs* s, int32_t on) {
  if (!s) return set_err(OPTB_ERR_ARG, "sbs: null");
  if (on && !s->pe[0])
    for (auto& e : s->pe) CK(cudaEventCreate(&e), "sbs profiling events");
  s->prof = on != 0;
  return OPTB_OK;
}

int optb_sbs_profile(optb_sbs* s, float* upload_ms, float* reshuffle_ms, float* gather_ms) {
  if (!s || !s->prof) return set_err(OPTB_ERR_ARG, "sbs: profiling is off");
  CK(cudaEventSynchronize(s->pe[3]), "sbs profile");
  if (upload_ms) CK(cudaEventElapsedTime(upload_ms, s->pe[0], s->pe[1]), "sbs profile");
  if (reshuffle_ms) CK(cudaEventElapsedTime(reshuffle_ms, s->pe[1], s->pe[2]), "sbs profile");
  if (gather_ms) CK(cudaEventElapsedTime(gather_ms, s->pe[2], s->pe[3]), "sbs profile");
  return OPTB_OK;
}

int optb_sbs_plan_call(uint64_t n_classes, const uint64_t* counts, const uint64_t* class_sizes,
                       const uint64_t* gen, uint64_t batches_before, uint64_t n, uint64_t chain, uint64_t max_events,
                       uint64_t* ev_class, uint64_t* ev_gen, uint64_t* ev_seed, uint64_t* n_events,
                       uint64_t* chain_after) {
  if (!counts || !class_sizes || !gen || !n_events) return set_err(OPTB_ERR_ARG, "sbs plan: null argument");
  for (uint64_t c = 0; c < n_classes; ++c)  // every generation started by the draws so far is counted
    if (counts[c] && class_sizes[c] && (gen[c] + 1) * class_sizes[c] < batches_before * counts[c])
      return set_err(OPTB_ERR_ARG, "sbs plan: generation of class %llu behind its draws",
                     static_cast<unsigned long long>(c));
  std::vector<uint64_t> ev_count;
  const std::vector<EvKey> keys = plan_events(n_classes, counts, class_sizes, gen, batches_before, n, &ev_count);
  *n_events = keys.size();
  if (keys.size() > max_events) return set_err(OPTB_ERR_ARG, "sbs plan: %llu events > max_events",
                                               static_cast<unsigned long long>(keys.size()));
  for (size_t e = 0; e < keys.size(); ++e) {  // the host's walk of the chain (run_events)
    if (ev_class) ev_class[e] = keys[e].cls;
    if (ev_gen) ev_gen[e] = keys[e].g;
    if (ev_seed) ev_seed[e] = chain;
    const uint64_t mm = class_sizes[keys[e].cls];
    chain = host_mix64(chain + (mm >= 2 ? mm : 1ull) * 0x9e3779b97f4a7c15ull);
  }
  if (chain_after) *chain_after = chain;
  return OPTB_OK;
}

int optb_sbs_set_force_serial(optb_sbs* s, int32_t on) {
  if (!s) return set_err(OPTB_ERR_ARG, "sbs: null");
  s->force_serial = on ? 1 : 0;
  return OPTB_OK;
}

int optb_sbs_next_dev(optb_sbs* s, uint64_t n, uint32_t shard, uint32_t n_shards,
                      int64_t* examples, int32_t* classes, void* stream) {
  if (!s) return set_err(OPTB_ERR_ARG, "sbs: null");
  if (n_shards == 0 || shard >= n_shards)
    return set_err(OPTB_ERR_ARG, "sbs: bad shard %u of %u", shard, n_shards);
  if (n == 0) return OPTB_OK;
  if (!examples) return set_err(OPTB_ERR_ARG, "sbs: null examples");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t C = s->C;
  // Lazy reshuffles (sampler.cpp:97): class c's draw D (counted from the
  // constructor) starts generation D / m_c when D % m_c == 0 and D > 0.
  std::vector<uint64_t> ev_count;
  const std::vector<EvKey> keys = plan_events(C, s->counts.data(), s->m.data(), s->gen.data(), s->batches, n,
                                              &ev_count);
  // gather tables: drawn_before, generation at pool slot 0, its offset, stride
  std::vector<uint64_t> ga(4 * C);
  for (uint64_t c = 0; c < C; ++c) {
    ga[c] = s->batches * s->counts[c];
    ga[C + c] = s->gen[c];
    ga[3 * C + c] = s->m[c] >= 2 ? s->m[c] : 0;  // stride 0: the permutation never changes
  }
  // the pool offsets are known only after layout; run_events fills gen_base
  // and the packed copy of `ga` is patched before the upload
  std::vector<uint64_t> gen_base;
  Packer pk;
  size_t o_ga = 0;
  {
    // lay out first to learn gen_base, then pack ga with it
    uint64_t cursor = s->N;
    gen_base.assign(C, 0);
    for (uint64_t c = 0; c < C; ++c) {
      if (ev_count[c] == 0 || s->m[c] < 2) {
        gen_base[c] = s->off[c];
        continue;
      }
      gen_base[c] = cursor;
      cursor += (ev_count[c] + 1) * s->m[c];
    }
    for (uint64_t c = 0; c < C; ++c) ga[2 * C + c] = gen_base[c];
  }
  int rc = run_events(s, keys, pk, nullptr, &o_ga, &ga, st);
  if (rc) return rc;
  const uint64_t* d_ga = reinterpret_cast<const uint64_t*>(s->d_call + o_ga);
  SbsGatherArgs a;
  const uint8_t* stat = s->d_static;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = (o + 15) / 16 * 16;
    o = at + bytes;
    return stat + at;
  };
  a.counts = reinterpret_cast<const uint64_t*>(take(C * 8));
  a.prefix = reinterpret_cast<const uint64_t*>(take((C + 1) * 8));
  a.class_size = reinterpret_cast<const uint64_t*>(take(C * 8));
  a.row_cls = reinterpret_cast<const uint32_t*>(take(s->B * 4));
  a.drawn_before = d_ga;
  a.gen_base_gen = d_ga + C;
  a.gen_base_off = d_ga + 2 * C;
  a.gen_stride = d_ga + 3 * C;
  a.pool = s->d_pool;
  a.C = C;
  a.B = s->B;
  a.n_batches = n;
  a.shard = shard;
  a.n_shards = n_shards;
  cudaError_t e = launch_sbs_gather(a, examples, classes, st, &s->ctx->launches);
  if (e != cudaSuccess) return cuda_err(e, "sbs gather");
  if (s->prof) cudaEventRecord(s->pe[3], st);
  for (uint64_t c = 0; c < C; ++c) s->gen[c] += ev_count[c];
  s->batches += n;
  return OPTB_OK;
}

int optb_sbs_next_host(optb_sbs* s, uint64_t n, int64_t* examples, int32_t* classes) {
  if (!s) return set_err(OPTB_ERR_ARG, "sbs: null");
  if (n == 0) return OPTB_OK;
  const uint64_t rows = n * s->B;
  if (s->ex_cap < rows) {
    // sized once for the drop-in cursor's largest refill (64 Ki draws): a
    // growing caller does not pay a synchronising cudaMalloc per refill
    const uint64_t cap = rows > (1ull << 16) ? rows : (1ull << 16);
    if (s->d_ex) cudaFree(s->d_ex);
    if (s->d_cl) cudaFree(s->d_cl);
    if (s->h_ex) cudaFreeHost(s->h_ex);
    if (s->h_cl) cudaFreeHost(s->h_cl);
    s->d_ex = nullptr;
    s->d_cl = nullptr;
    s->h_ex = nullptr;
    s->h_cl = nullptr;
    s->ex_cap = 0;
    CK(cudaMalloc(&s->d_ex, cap * 8), "sbs scratch");
    CK(cudaMalloc(&s->d_cl, cap * 4), "sbs scratch");
    CK(cudaHostAlloc(&s->h_ex, cap * 8, cudaHostAllocDefault), "sbs pinned scratch");
    CK(cudaHostAlloc(&s->h_cl, cap * 4, cudaHostAllocDefault), "sbs pinned scratch");
    s->ex_cap = cap;
  }
  cudaStream_t st = s->ctx->s_compute;
  int rc = optb_sbs_next_dev(s, n, 0, 1, s->d_ex, s->d_cl, st);
  if (rc) return rc;
  // pinned bounce buffers: an async DMA instead of the driver's staged
  // pageable copy; the caller's arrays are filled by memcpy
  CK(cudaMemcpyAsync(s->h_ex, s->d_ex, rows * 8, cudaMemcpyDeviceToHost, st), "sbs D2H");
  if (classes) CK(cudaMemcpyAsync(s->h_cl, s->d_cl, rows * 4, cudaMemcpyDeviceToHost, st), "sbs D2H");
  CK(cudaStreamSynchronize(st), "sbs sync");
  memcpy(examples, s->h_ex, rows * 8);
  if (classes) memcpy(classes, s->h_cl, rows * 4);
  g_err.clear();
  return OPTB_OK;
}

}  // extern "C"
