// io.cu -- OPTB epoch dump / load for device streams (optb_dump_dev,
// optb_load_dev).  Replaces pipeline::dump / pipeline::load
// (pipeline.cpp:246-271) over codec::write_optb / read_optb
// (codec.cpp:283-367) for the GPU path: the container planes are already in
// OPTB payload order, so no pack/unpack kernel is needed -- each chunk is a
// header plus a D2H (or H2D) copy staged through a ring of pinned buffers,
// with file I/O of chunk k overlapping the copy of chunk k+1.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>

#include <string>
#include <vector>

#include "internal.h"
#include "optb_cuda.h"

namespace {

int io_fail(int code, const std::string& msg) { return optb_b200::set_error_text(code, msg); }

std::string chunk_path(const char* dir, uint64_t epoch, uint64_t k) {
  return std::string(dir) + "/batch_" + std::to_string(epoch) + "_" + std::to_string(k) + ".optb";
}

void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

struct ChunkGeom {
  uint64_t n;       // images in chunk k
  uint64_t bytes;   // plane bytes
  uint64_t obytes;  // parity plane bytes (exact, ceil(n*P/8))
};

ChunkGeom chunk_geom(const optb_layout* L, uint64_t k) {
  const uint64_t cpb = (L->batch + L->per_chunk - 1) / L->per_chunk;
  const uint64_t j = k % cpb;
  const uint64_t left = L->batch - j * L->per_chunk;
  ChunkGeom g;
  g.n = left < L->per_chunk ? left : L->per_chunk;
  g.bytes = L->pixels * optb_container_value_bytes(L->mode);
  g.obytes = optb_mode_has_offsets(L->mode) ? optb_offsets_plane_bytes(static_cast<uint32_t>(g.n), L->pixels) : 0;
  return g;
}

struct Staging {
  static constexpr int kRing = 4;
  uint8_t* buf[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  size_t cap = 0;
  cudaStream_t s = nullptr;
  ~Staging() {
    for (int i = 0; i < kRing; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    if (s) cudaStreamDestroy(s);
  }
  bool init(size_t bytes) {
    cap = bytes;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return false;
    for (int i = 0; i < kRing; ++i)
      if (cudaHostAlloc(&buf[i], bytes, cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
        return false;
    return true;
  }
};

}  // namespace

extern "C" {

int optb_dump_dev(optb_ctx* ctx, const optb_layout* L, const void* containers, const uint8_t* offsets,
                  uint32_t h, uint32_t w, uint32_t c, const char* dir, uint64_t epoch) {
  if (!ctx || !L || !containers || !dir) return io_fail(OPTB_ERR_ARG, "dump: null argument");
  int st = optb_layout_check(L);
  if (st) return st;
  if (static_cast<uint64_t>(h) * w * c != L->pixels) return io_fail(OPTB_ERR_SHAPE, "dump: h*w*c != pixels");
  if (optb_mode_has_offsets(L->mode) && !offsets) return io_fail(OPTB_ERR_ARG, "dump: null offsets");
  // synchronous: the planes may still be written by kernels queued on any stream
  if (cudaDeviceSynchronize() != cudaSuccess) return io_fail(OPTB_ERR_CUDA, "dump: device synchronize");
  mkdir(dir, 0755);  // create_directories for the last level (pipeline.cpp:248-250)
  struct stat sb;
  if (stat(dir, &sb) != 0 || !S_ISDIR(sb.st_mode))
    return io_fail(OPTB_ERR_FORMAT, std::string("dump: cannot create directory ") + dir);
  const uint64_t chunks = optb_layout_chunks(L);
  const uint64_t ostride = optb_offsets_stride(L->mode, L->pixels, L->per_chunk);
  const ChunkGeom full = chunk_geom(L, 0);
  Staging stg;
  if (!stg.init(20 + full.bytes + (full.obytes ? ostride : 0)))
    return io_fail(OPTB_ERR_CUDA, "dump: pinned staging");
  auto write_out = [&](uint64_t k) -> int {
    const int r = static_cast<int>(k % Staging::kRing);
    if (cudaEventSynchronize(stg.ev[r]) != cudaSuccess) return io_fail(OPTB_ERR_CUDA, "dump: D2H");
    const ChunkGeom g = chunk_geom(L, k);
    uint8_t* b = stg.buf[r];
    memcpy(b, "OPTB", 4);
    put_le(b + 4, 1, 2);
    put_le(b + 6, static_cast<uint64_t>(L->mode), 1);
    put_le(b + 7, g.n, 1);
    put_le(b + 8, h, 4);
    put_le(b + 12, w, 4);
    put_le(b + 16, c, 4);
    const std::string path = chunk_path(dir, epoch, k);
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) return io_fail(OPTB_ERR_FORMAT, "optb: cannot open for writing: " + path);
    const size_t total = 20 + g.bytes + g.obytes;
    const size_t wr = fwrite(b, 1, total, f);
    const int cl = fclose(f);
    if (wr != total || cl != 0) return io_fail(OPTB_ERR_FORMAT, "optb: write failed: " + path);
    return OPTB_OK;
  };
  for (uint64_t k = 0; k < chunks; ++k) {
    const int r = static_cast<int>(k % Staging::kRing);
    if (k >= Staging::kRing) {
      st = write_out(k - Staging::kRing);
      if (st) return st;
    }
    const ChunkGeom g = chunk_geom(L, k);
    if (cudaMemcpyAsync(stg.buf[r] + 20, static_cast<const uint8_t*>(containers) + k * g.bytes, g.bytes,
                        cudaMemcpyDeviceToHost, stg.s) != cudaSuccess ||
        (g.obytes && cudaMemcpyAsync(stg.buf[r] + 20 + g.bytes, offsets + k * ostride, g.obytes,
                                     cudaMemcpyDeviceToHost, stg.s) != cudaSuccess) ||
        cudaEventRecord(stg.ev[r], stg.s) != cudaSuccess)
      return io_fail(OPTB_ERR_CUDA, "dump: D2H");
  }
  for (uint64_t k = chunks > Staging::kRing ? chunks - Staging::kRing : 0; k < chunks; ++k) {
    st = write_out(k);
    if (st) return st;
  }
  return OPTB_OK;
}

int optb_load_dev(optb_ctx* ctx, const optb_layout* L, uint32_t h, uint32_t w, uint32_t c,
                  const char* dir, uint64_t epoch, void* containers, uint8_t* offsets) {
  if (!ctx || !L || !containers || !dir) return io_fail(OPTB_ERR_ARG, "load: null argument");
  int st = optb_layout_check(L);
  if (st) return st;
  if (static_cast<uint64_t>(h) * w * c != L->pixels) return io_fail(OPTB_ERR_SHAPE, "load: h*w*c != pixels");
  if (optb_mode_has_offsets(L->mode) && !offsets) return io_fail(OPTB_ERR_ARG, "load: null offsets");
  // synchronous: queued kernels may still read the destination planes
  if (cudaDeviceSynchronize() != cudaSuccess) return io_fail(OPTB_ERR_CUDA, "load: device synchronize");
  const uint64_t chunks = optb_layout_chunks(L);
  const uint64_t ostride = optb_offsets_stride(L->mode, L->pixels, L->per_chunk);
  const ChunkGeom full = chunk_geom(L, 0);
  Staging stg;
  if (!stg.init(20 + full.bytes + (full.obytes ? ostride : 0)))
    return io_fail(OPTB_ERR_CUDA, "load: pinned staging");
  if (chunks == 0) return OPTB_OK;
  for (uint64_t k = 0; k < chunks; ++k) {
    const int r = static_cast<int>(k % Staging::kRing);
    if (cudaEventSynchronize(stg.ev[r]) != cudaSuccess) return io_fail(OPTB_ERR_CUDA, "load: H2D");
    const ChunkGeom g = chunk_geom(L, k);
    const std::string path = chunk_path(dir, epoch, k);
    FILE* f = fopen(path.c_str(), "rb");
    if (!f)
      return io_fail(OPTB_ERR_FORMAT, "load: missing batch file " + path + " for epoch " + std::to_string(epoch));
    uint8_t* b = stg.buf[r];
    const size_t want = 20 + g.bytes + g.obytes;
    const size_t got = fread(b, 1, want, f);
    const bool extra = fgetc(f) != EOF;
    fclose(f);
    // read_optb's checks, in its order (codec.cpp:319-344)
    if (got < 4) return io_fail(OPTB_ERR_FORMAT, "optb: truncated stream");
    if (memcmp(b, "OPTB", 4) != 0) return io_fail(OPTB_ERR_FORMAT, "optb: bad magic");
    if (got < 6) return io_fail(OPTB_ERR_FORMAT, "optb: truncated stream");
    const uint64_t version = get_le(b + 4, 2);
    if (version != 1) return io_fail(OPTB_ERR_FORMAT, "optb: unsupported version " + std::to_string(version));
    if (got < 20) return io_fail(OPTB_ERR_FORMAT, "optb: truncated stream");
    const uint64_t tag = b[6], n = b[7];
    if (tag > 4) return io_fail(OPTB_ERR_FORMAT, "optb: unknown mode tag " + std::to_string(tag));
    if (tag != static_cast<uint64_t>(L->mode) || n != g.n || get_le(b + 8, 4) != h || get_le(b + 12, 4) != w ||
        get_le(b + 16, 4) != c)
      return io_fail(OPTB_ERR_FORMAT, "load: " + path + " does not match the expected layout");
    if (got != want) return io_fail(OPTB_ERR_FORMAT, "optb: truncated stream");
    (void)extra;  // like read_optb_file, bytes after the parity plane are ignored
    if (cudaMemcpyAsync(static_cast<uint8_t*>(containers) + k * g.bytes, b + 20, g.bytes, cudaMemcpyHostToDevice,
                        stg.s) != cudaSuccess ||
        (g.obytes && cudaMemcpyAsync(offsets + k * ostride, b + 20 + g.bytes, g.obytes, cudaMemcpyHostToDevice,
                                     stg.s) != cudaSuccess) ||
        cudaEventRecord(stg.ev[r], stg.s) != cudaSuccess)
      return io_fail(OPTB_ERR_CUDA, "load: H2D");
  }
  if (cudaStreamSynchronize(stg.s) != cudaSuccess) return io_fail(OPTB_ERR_CUDA, "load: H2D");
  return OPTB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- records
namespace {

// One CTA per record at a time: the record (1 + C*H*W bytes, not aligned) is
// staged in shared memory with coalesced byte loads, then written out
// channel-interleaved with coalesced byte stores (dataset.cpp:84-91).
__global__ void k_records_to_hwc(const uint8_t* __restrict__ src, uint64_t n_rec, uint32_t hw, uint32_t ch,
                                 uint32_t n_classes, uint8_t* __restrict__ dst, int32_t* __restrict__ labels,
                                 unsigned long long* bad) {
  extern __shared__ uint8_t rec[];
  const uint64_t P = static_cast<uint64_t>(hw) * ch;
  for (uint64_t r = blockIdx.x; r < n_rec; r += gridDim.x) {
    const uint8_t* s = src + r * (P + 1);
    for (uint64_t i = threadIdx.x; i < P + 1; i += blockDim.x) rec[i] = s[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      labels[r] = rec[0];
      if (rec[0] >= n_classes) atomicMin(bad, static_cast<unsigned long long>(r));
    }
    for (uint64_t o = threadIdx.x; o < P; o += blockDim.x) {
      const uint64_t px = o / ch, cc = o - px * ch;
      dst[r * P + o] = rec[1 + cc * hw + px];
    }
    __syncthreads();
  }
}

// Records too large to stage whole (P + 1 beyond the shared-memory budget,
// e.g. 299x299x3): one CTA per (record, pixel tile).  The tile's bytes of
// every channel plane are staged with coalesced loads, then written
// channel-interleaved.
__global__ void k_records_to_hwc_tiled(const uint8_t* __restrict__ src, uint64_t n_rec, uint32_t hw, uint32_t ch,
                                       uint32_t tile, uint32_t n_classes, uint8_t* __restrict__ dst,
                                       int32_t* __restrict__ labels, unsigned long long* bad) {
  extern __shared__ uint8_t rec[];
  const uint64_t P = static_cast<uint64_t>(hw) * ch;
  const uint64_t tiles = (hw + tile - 1) / tile;
  for (uint64_t w = blockIdx.x; w < n_rec * tiles; w += gridDim.x) {
    const uint64_t r = w / tiles, px0 = (w - r * tiles) * tile;
    const uint32_t npx = static_cast<uint32_t>(hw - px0 < tile ? hw - px0 : tile);
    const uint8_t* s = src + r * (P + 1);
    if (px0 == 0 && threadIdx.x == 0) {
      labels[r] = s[0];
      if (s[0] >= n_classes) atomicMin(bad, static_cast<unsigned long long>(r));
    }
    for (uint32_t i = threadIdx.x; i < npx * ch; i += blockDim.x) {
      const uint32_t cc = i / npx, px = i - cc * npx;
      rec[i] = s[1 + static_cast<uint64_t>(cc) * hw + px0 + px];
    }
    __syncthreads();
    uint8_t* d = dst + r * P + px0 * ch;
    for (uint32_t o = threadIdx.x; o < npx * ch; o += blockDim.x) {
      const uint32_t px = o / ch, cc = o - px * ch;
      d[o] = rec[cc * npx + px];
    }
    __syncthreads();
  }
}

constexpr uint64_t kRecordStageBytes = 96 * 1024;  // whole-record staging up to this size

}  // namespace

extern "C" int optb_load_records_dev(optb_ctx* ctx, const char* path, uint32_t h, uint32_t w, uint32_t c,
                                     uint32_t n_classes, uint8_t* pixels, int32_t* labels, uint64_t max_records,
                                     uint64_t* n_records) {
  if (!ctx || !path || !pixels || !labels || !n_records) return io_fail(OPTB_ERR_ARG, "records: null argument");
  const uint64_t P = static_cast<uint64_t>(h) * w * c;
  if (P == 0) return io_fail(OPTB_ERR_SHAPE, "records: image extents must be positive");
  FILE* f = fopen(path, "rb");
  if (!f) return io_fail(OPTB_ERR_FORMAT, std::string("records: cannot open ") + path);
  fseek(f, 0, SEEK_END);
  const long size = ftell(f);
  fseek(f, 0, SEEK_SET);
  const uint64_t n = static_cast<uint64_t>(size) / (P + 1);
  if (static_cast<uint64_t>(size) % (P + 1) != 0) {
    fclose(f);
    return io_fail(OPTB_ERR_FORMAT, std::string("records: trailing partial record in ") + path);
  }
  if (n == 0) {
    fclose(f);
    return io_fail(OPTB_ERR_FORMAT, std::string("records: no records in ") + path);
  }
  if (n > max_records) {
    fclose(f);
    return io_fail(OPTB_ERR_ARG, "records: " + std::to_string(n) + " records exceed the output capacity");
  }
  uint8_t* host = nullptr;
  uint8_t* dev = nullptr;
  unsigned long long* bad = nullptr;
  auto release = [&] {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    if (bad) cudaFree(bad);
  };
  if (cudaHostAlloc(&host, size, cudaHostAllocDefault) != cudaSuccess || cudaMalloc(&dev, size) != cudaSuccess ||
      cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess) {
    fclose(f);
    release();
    return io_fail(OPTB_ERR_CUDA, "records: staging buffers");
  }
  const size_t got = fread(host, 1, size, f);
  fclose(f);
  if (got != static_cast<size_t>(size)) {
    release();
    return io_fail(OPTB_ERR_FORMAT, std::string("records: cannot read ") + path);
  }
  const unsigned long long none = ~0ull;
  cudaError_t e = cudaMemcpy(bad, &none, sizeof none, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dev, host, size, cudaMemcpyHostToDevice);
  if (P + 1 <= kRecordStageBytes) {
    const unsigned grid = static_cast<unsigned>(n < 148 * 8 ? n : 148 * 8);
    if (e == cudaSuccess && P + 1 > 48 * 1024)
      e = cudaFuncSetAttribute(k_records_to_hwc, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P + 1));
    if (e == cudaSuccess) k_records_to_hwc<<<grid, 256, P + 1>>>(dev, n, h * w, c, n_classes, pixels, labels, bad);
  } else {
    // tile of pixels whose bytes over all channels fit the staging budget
    const uint64_t hw = static_cast<uint64_t>(h) * w;
    const uint64_t t = (32 * 1024) / c ? (32 * 1024) / c : 1;
    const uint32_t tile = static_cast<uint32_t>(t < hw ? t : hw);
    const uint64_t smem = static_cast<uint64_t>(tile) * c;
    if (smem > kRecordStageBytes) {
      release();
      return io_fail(OPTB_ERR_SHAPE, "records: " + std::to_string(c) + " channels exceed the staging budget");
    }
    if (e == cudaSuccess && smem > 48 * 1024)
      e = cudaFuncSetAttribute(k_records_to_hwc_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
    const uint64_t work = n * ((hw + tile - 1) / tile);
    const unsigned grid = static_cast<unsigned>(work < 148 * 8 ? work : 148 * 8);
    if (e == cudaSuccess)
      k_records_to_hwc_tiled<<<grid, 256, smem>>>(dev, n, static_cast<uint32_t>(hw), c, tile, n_classes, pixels,
                                                  labels, bad);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    release();
    return io_fail(OPTB_ERR_CUDA, std::string("records: kernel launch: ") + cudaGetErrorString(e));
  }
  unsigned long long first_bad = none;
  e = cudaMemcpy(&first_bad, bad, sizeof first_bad, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    release();
    return io_fail(OPTB_ERR_CUDA, std::string("records: ") + cudaGetErrorString(e));
  }
  int rc = OPTB_OK;
  if (first_bad != none) {  // dataset.cpp:78-82 names the first offending label
    const int label = host[first_bad * (P + 1)];
    rc = io_fail(OPTB_ERR_FORMAT, "records: label " + std::to_string(label) + " outside " +
                                      std::to_string(n_classes) + " classes in " + path);
  }
  release();
  *n_records = n;
  return rc;
}

// ---------------------------------------------------------------- sharded dataset helpers
namespace {

// One warp per row; 16-byte copies when both rows are 16-byte aligned.
__global__ void k_gather_rows(const uint8_t* __restrict__ src, uint64_t src_stride,
                              const int64_t* __restrict__ index, uint64_t n, int64_t bias, uint64_t P,
                              uint8_t* __restrict__ dst, uint64_t dst_stride) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += warps) {
    const uint8_t* s = src + static_cast<uint64_t>(index[i] - bias) * src_stride;
    uint8_t* d = dst + i * dst_stride;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    uint64_t done = 0;
    if (vec) {
      const uint64_t v = P / 16;
      for (uint64_t k = lane; k < v; k += 32)
        reinterpret_cast<uint4*>(d)[k] = __ldg(reinterpret_cast<const uint4*>(s) + k);
      done = v * 16;
    }
    for (uint64_t k = done + lane; k < P; k += 32) d[k] = s[k];
  }
}

__global__ void k_inverse_perm(const int64_t* __restrict__ perm, uint64_t n, int64_t* __restrict__ inv) {
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    inv[perm[j]] = static_cast<int64_t>(j);
}

__global__ void k_owner_labels(const int64_t* __restrict__ ex, uint64_t n, uint64_t per, uint32_t shards,
                               int32_t* __restrict__ owner) {
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t o = static_cast<uint64_t>(ex[j]) / per;
    owner[j] = static_cast<int32_t>(o < shards ? o : shards - 1);
  }
}

unsigned grid_of(uint64_t work, unsigned per_block) {
  const uint64_t g = (work + per_block - 1) / per_block;
  return static_cast<unsigned>(g < 148 * 8 ? (g ? g : 1) : 148 * 8);
}

}  // namespace

extern "C" int optb_gather_rows_dev(optb_ctx* ctx, const uint8_t* src, uint64_t src_stride, const int64_t* index,
                                    uint64_t n, int64_t bias, uint64_t pixels, uint8_t* dst, uint64_t dst_stride,
                                    void* stream) {
  if (!ctx || (!n)) return ctx ? OPTB_OK : io_fail(OPTB_ERR_ARG, "gather_rows: null ctx");
  if (!src || !index || !dst) return io_fail(OPTB_ERR_ARG, "gather_rows: null buffer");
  k_gather_rows<<<grid_of(n * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, src_stride ? src_stride : pixels, index, n, bias, pixels, dst, dst_stride ? dst_stride : pixels);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OPTB_OK : io_fail(OPTB_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int optb_inverse_perm_dev(optb_ctx* ctx, const int64_t* perm, uint64_t n, int64_t* inv, void* stream) {
  if (!ctx || (n && (!perm || !inv))) return io_fail(OPTB_ERR_ARG, "inverse_perm: null argument");
  if (!n) return OPTB_OK;
  k_inverse_perm<<<grid_of(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(perm, n, inv);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OPTB_OK : io_fail(OPTB_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int optb_owner_labels_dev(optb_ctx* ctx, const int64_t* examples, uint64_t n, uint64_t per,
                                     uint32_t shards, int32_t* owner, void* stream) {
  if (!ctx || !shards || !per || (n && (!examples || !owner))) return io_fail(OPTB_ERR_ARG, "owner_labels: bad argument");
  if (!n) return OPTB_OK;
  k_owner_labels<<<grid_of(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(examples, n, per, shards, owner);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OPTB_OK : io_fail(OPTB_ERR_CUDA, cudaGetErrorString(e));
}
