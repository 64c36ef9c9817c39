// codec.cu -- dispatch of the optb codec kernels (the kernels themselves are in
// codec_impl.cuh, instantiated per mode variant by codec_v<N>.cu), the
// synthetic-data kernel, and the shared launch helpers.
#include <mutex>
#include <unordered_map>

#include "codec_impl.cuh"

namespace optb_b200 {
namespace {

// ------------------------------------------------------------------ synth
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_synth(uint64_t seed, uint64_t first_row, uint64_t n_rows, uint64_t P,
                        uint8_t* out, uint64_t row_stride) {
  const uint64_t words = (P + 7) / 8;
  const uint64_t total = n_rows * words;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = t / words, q = t - r * words;
    const uint64_t w = mix64(seed + ((first_row + r) * words + q + 1) * 0x9e3779b97f4a7c15ull);
    uint8_t* dst = out + r * row_stride + q * 8;
    if (q * 8 + 8 <= P && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
      *reinterpret_cast<uint64_t*>(dst) = w;
    } else {
      for (uint64_t b = 0; b < 8 && q * 8 + b < P; ++b) dst[b] = static_cast<uint8_t>(w >> (8 * b));
    }
  }
}

}  // namespace


// Row sources qualify for the vector path when every row is 16-byte aligned:
// index mode checks base and stride, pointer mode trusts the caller's flag.
bool rows_vec_ok(const RowSrc& rs) {
  return rs.ptrs ? rs.ptrs_aligned16 != 0 : (rs.stride % 16 == 0 && aligned16(rs.images));
}

cudaError_t launch_encode(const Geom& g, const RowSrc& rs, void* containers, uint8_t* offsets, cudaStream_t s,
                          int sms, uint64_t* launches) {
  const bool vec = vec_ok(g) && rows_vec_ok(rs) && aligned16(containers);
  switch (g.mode) {
    case OPTB_EXACT64: return encode_v0(g, rs, vec, containers, offsets, s, sms, launches);
    case OPTB_EXACT128: return encode_v1(g, rs, vec, containers, offsets, s, sms, launches);
    case OPTB_F64:
      if (vec && g.per_chunk <= 8) return encode_v5(g, rs, true, containers, offsets, s, sms, launches);
      return encode_v2(g, rs, vec, containers, offsets, s, sms, launches);
    case OPTB_LOSSLESS64: return encode_v3(g, rs, vec, containers, offsets, s, sms, launches);
    default: return encode_v4(g, rs, vec, containers, offsets, s, sms, launches);
  }
}

cudaError_t launch_decode(const Geom& g, const void* containers, const uint8_t* offsets,
                          const Epi& e, void* out, DevError* err, cudaStream_t s, int sms,
                          uint64_t* launches) {
  const int es = e.dtype == OPTB_OUT_U8 ? 1 : e.dtype == OPTB_OUT_F32 ? 4 : 2;
  const bool vec = vec_ok(g) && aligned16(containers) && aligned16(out) && (e.row_stride * es) % 16 == 0;
  switch (g.mode) {
    case OPTB_EXACT64: return decode_v0(g, containers, offsets, e, vec, out, err, s, sms, launches);
    case OPTB_EXACT128: return decode_v1(g, containers, offsets, e, vec, out, err, s, sms, launches);
    case OPTB_F64:
      if (vec && g.per_chunk <= 8) return decode_v5(g, containers, offsets, e, true, out, err, s, sms, launches);
      return decode_v2(g, containers, offsets, e, vec, out, err, s, sms, launches);
    case OPTB_LOSSLESS64: return decode_v3(g, containers, offsets, e, vec, out, err, s, sms, launches);
    default: return decode_v4(g, containers, offsets, e, vec, out, err, s, sms, launches);
  }
}

// The plain grid-stride kernels, whatever the alignment: the small host
// calls run them straight on mapped pinned memory (zero-copy over PCIe).
cudaError_t launch_encode_generic(const Geom& g, const RowSrc& rs, void* containers, uint8_t* offsets,
                                  cudaStream_t s, int sms, uint64_t* launches) {
  switch (g.mode) {
    case OPTB_EXACT64: return encode_v0(g, rs, false, containers, offsets, s, sms, launches);
    case OPTB_EXACT128: return encode_v1(g, rs, false, containers, offsets, s, sms, launches);
    case OPTB_F64: return encode_v2(g, rs, false, containers, offsets, s, sms, launches);
    case OPTB_LOSSLESS64: return encode_v3(g, rs, false, containers, offsets, s, sms, launches);
    default: return encode_v4(g, rs, false, containers, offsets, s, sms, launches);
  }
}

cudaError_t launch_decode_generic(const Geom& g, const void* containers, const uint8_t* offsets, const Epi& e,
                                  void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  switch (g.mode) {
    case OPTB_EXACT64: return decode_v0(g, containers, offsets, e, false, out, err, s, sms, launches);
    case OPTB_EXACT128: return decode_v1(g, containers, offsets, e, false, out, err, s, sms, launches);
    case OPTB_F64: return decode_v2(g, containers, offsets, e, false, out, err, s, sms, launches);
    case OPTB_LOSSLESS64: return decode_v3(g, containers, offsets, e, false, out, err, s, sms, launches);
    default: return decode_v4(g, containers, offsets, e, false, out, err, s, sms, launches);
  }
}

thread_local int g_rt_kind = OPTB_RT_NONE;
thread_local bool g_sysmem = false;

namespace {
std::mutex g_tag_mu;
std::unordered_map<cudaStream_t, uint64_t> g_tags;
uint64_t g_tag_next = 1;
}  // namespace

uint64_t stream_tag(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_tag_mu);
  auto it = g_tags.find(s);
  return it == g_tags.end() ? 0 : it->second;
}
void bump_stream_tag(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_tag_mu);
  g_tags[s] = g_tag_next++;
}

cudaError_t launch_roundtrip(const Geom& g, const RowSrc& rs, void* containers, uint8_t* offsets, const Epi& e,
                             void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  g_rt_kind = OPTB_RT_SPLIT;  // unless a fused launcher below takes it
  const int es = e.dtype == OPTB_OUT_U8 ? 1 : e.dtype == OPTB_OUT_F32 ? 4 : 2;
  const bool vec = vec_ok(g) && rows_vec_ok(rs) && aligned16(containers) && aligned16(out) &&
                   (e.row_stride * es) % 16 == 0;
  // lossless: the decode half stages parity bits with 16-byte L2 copies, which
  // needs whole tiles per chunk (P % 512) and a 16-byte aligned plane
  const bool lossless = g.mode == OPTB_LOSSLESS64 || g.mode == OPTB_LOSSLESS128;
  const bool fusable = !lossless || (g.P % 512 == 0 && aligned16(offsets));
  CUtensorMap cm;
  if (!vec || !fusable || !tma_decode_enabled() ||
      !container_map(&cm, containers, g.chunks * g.P * g.wc, g.wc))
    return cudaErrorNotSupported;  // caller: separate encode + decode launches
  switch (g.mode) {
    case OPTB_EXACT64: return roundtrip_v0(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
    case OPTB_EXACT128: return roundtrip_v1(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
    case OPTB_LOSSLESS64: return roundtrip_v3(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
    case OPTB_LOSSLESS128: return roundtrip_v4(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
    default:
      if (g.per_chunk <= 8) return roundtrip_v5(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
      return roundtrip_v2(cm, g, rs, containers, offsets, e, out, err, s, sms, launches);
  }
}

cudaError_t launch_synth(uint64_t seed, uint64_t first_row, uint64_t n_rows, uint64_t P,
                         uint8_t* out, uint64_t row_stride, cudaStream_t s, int sms,
                         uint64_t* launches) {
  const uint64_t words = n_rows * ((P + 7) / 8);
  const int grid = grid_for(k_synth, 256, 0, sms, words);
  k_synth<<<grid, 256, 0, s>>>(seed, first_row, n_rows, P, out, row_stride);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t ensure_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(kernel, dev, bytes);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

}  // namespace optb_b200
