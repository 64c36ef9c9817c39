#pragma once
// codec_impl.cuh -- sm_100a encode / decode kernels for the optb container modes
// and their launch helpers.  Included by codec.cu (dispatch) and by one
// codec_v<N>.cu per mode variant, which instantiate that variant's kernels
// (the six translation units build in parallel).
//
// Reference semantics (file:line under /root/reference/proj):
//   encode  codec.cpp:106-146   decode  codec.cpp:148-208
//   gather  dataset.cpp:16-22 + runner.cpp:77-90 (chunking of a batch)
//   float epilogue  nn.cpp:183-189 (float(q)*scale), fp16 store nn.cpp:235 ->
//   tensor.cpp:12-51 (RNE; __float2half_rn is bit-identical on q*scale values,
//   SURVEY App. B).
//
// Kernel families:
//   k_encode_vec<MODE>    K1/K3/K5: gathered rows by cp.async into a 2-stage
//                         warp-private smem ring, 16-pixel x 16-image register
//                         byte transpose (PRMT), per-mode word build (exact
//                         bytes, lossless 7-bit compaction + 16-bit parity
//                         stores, f64 ordered binary64 adds), XOR-swizzled
//                         staging, fully coalesced 128/64-bit container stores.
//   k_decode_vec<MODE,O,TMA>  K2/K4/K6: container words by one 2D TMA tensor
//                         load per tile (128-byte hardware swizzle, mbarrier
//                         completion; parity bits beside it) or by cp.async into
//                         XOR-swizzled slots (+ lossless parity bits), per-mode
//                         range check and unpack, transpose, u8 rows stored
//                         directly or through a u8 tile with the fused
//                         fp32/fp16/bf16 epilogue.
//   k_encode_bulk<MODE>   K1/K5 for exact and f64: as k_encode_vec, but each
//                         tile's words are laid out in the container tensor
//                         map's 128B swizzle and leave as one bulk tensor store.
//   k_roundtrip_il<MODE,O>  K1+K2 in one persistent launch (optb_roundtrip_dev,
//                         the E-D pipeline step), exact and f64: each warp
//                         stores an encoded tile, then decodes it one tile
//                         later by TMA while its lines are still in L2.
//   k_roundtrip_vec<MODE,O>  the same, phase-ordered (lossless modes): each
//                         warp encodes all its tiles, then decodes them back.
//   k_{en,de}code_generic any P / stride / alignment: one pixel per lane,
//                         warp ballots for the parity plane.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <set>
#include <tuple>
#include <type_traits>
#include <utility>

#include "internal.h"

namespace optb_b200 {
namespace {

#ifndef OPTB_VEC_WARPS
#define OPTB_VEC_WARPS 8
#endif
#ifndef OPTB_VEC_STAGES
#define OPTB_VEC_STAGES 2
#endif
constexpr int kWarps = OPTB_VEC_WARPS;  // warps per CTA for the vector kernels
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ uint4 ldg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg16(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void stg8(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// 4x4 byte transpose of rows a0..a3 (row r's byte c -> row c's byte r).
__device__ __forceinline__ void t4x4(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
  a0 = __byte_perm(t0, t2, 0x5410);
  a1 = __byte_perm(t0, t2, 0x7632);
  a2 = __byte_perm(t1, t3, 0x5410);
  a3 = __byte_perm(t1, t3, 0x7632);
}

// 16x16 byte transpose, m[r][q] holds bytes 4q..4q+3 of row r.  ROWS / COLS
// bound the live part (rows >= ROWS are zero, columns >= COLS are unused):
// exact64 uses 8 of the 16 image columns / rows.
template <int ROWS, int COLS>
__device__ __forceinline__ void transpose16(uint32_t (&m)[16][4]) {
  uint32_t t[16][4];
#pragma unroll
  for (int R = 0; R < 4; ++R) {
#pragma unroll
    for (int Q = 0; Q < 4; ++Q) {
      if (4 * Q >= COLS) continue;
      uint32_t a0 = 4 * R + 0 < ROWS ? m[4 * R + 0][Q] : 0u;
      uint32_t a1 = 4 * R + 1 < ROWS ? m[4 * R + 1][Q] : 0u;
      uint32_t a2 = 4 * R + 2 < ROWS ? m[4 * R + 2][Q] : 0u;
      uint32_t a3 = 4 * R + 3 < ROWS ? m[4 * R + 3][Q] : 0u;
      t4x4(a0, a1, a2, a3);
      t[4 * Q + 0][R] = a0;
      t[4 * Q + 1][R] = a1;
      t[4 * Q + 2][R] = a2;
      t[4 * Q + 3][R] = a3;
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) m[r][q] = (r < COLS) ? t[r][q] : 0u;
}

struct ChunkPos {
  uint64_t r0;  // first stream row of the chunk
  uint32_t n;   // images in the chunk
};

__device__ __forceinline__ ChunkPos chunk_pos(const Geom& g, uint64_t k) {
  const uint64_t b = k / g.cpb;
  const uint32_t j = static_cast<uint32_t>(k - b * g.cpb);
  const uint64_t first = static_cast<uint64_t>(j) * g.per_chunk;
  const uint64_t left = g.B - first;
  ChunkPos c;
  c.r0 = b * g.B + first;
  c.n = left < g.per_chunk ? static_cast<uint32_t>(left) : g.per_chunk;
  return c;
}

// A lane's work item t = k*G + gi (chunk k = b*cpb + j, G = items per chunk)
// along its grid-stride sequence.  The hot loops advance it with adds and
// compares only; the 64-bit divisions happen once, at kernel start.
struct Walk {
  uint64_t t, k, gi, b;
  uint32_t j;
};
struct WalkStep {
  uint64_t dt, dk, dgi, db;
  uint32_t dj;
};
__device__ __forceinline__ Walk walk_at(const Geom& g, uint64_t G, uint64_t t) {
  Walk w;
  w.t = t;
  w.k = t / G;
  w.gi = t - w.k * G;
  w.b = w.k / g.cpb;
  w.j = static_cast<uint32_t>(w.k - w.b * g.cpb);
  return w;
}
__device__ __forceinline__ WalkStep walk_step(const Geom& g, uint64_t G, uint64_t dt) {
  WalkStep s;
  s.dt = dt;
  s.dk = dt / G;
  s.dgi = dt - s.dk * G;
  s.db = s.dk / g.cpb;
  s.dj = static_cast<uint32_t>(s.dk - s.db * g.cpb);
  return s;
}
__device__ __forceinline__ void walk_advance(Walk& w, const WalkStep& s, const Geom& g, uint64_t G) {
  w.t += s.dt;
  w.gi += s.dgi;
  w.k += s.dk;
  w.b += s.db;
  w.j += s.dj;
  if (w.gi >= G) {  // gi, dgi < G: at most one carry
    w.gi -= G;
    ++w.k;
    ++w.j;
  }
  if (w.j >= g.cpb) {  // j, dj < cpb, carry <= 1: at most one wrap
    w.j -= g.cpb;
    ++w.b;
  }
}
__device__ __forceinline__ ChunkPos walk_chunk(const Geom& g, const Walk& w) {
  const uint64_t first = static_cast<uint64_t>(w.j) * g.per_chunk;
  const uint64_t left = g.B - first;
  ChunkPos c;
  c.r0 = w.b * g.B + first;
  c.n = left < g.per_chunk ? static_cast<uint32_t>(left) : g.per_chunk;
  return c;
}

__device__ __forceinline__ void latch_error(DevError* err, uint32_t kind, uint64_t chunk,
                                            uint32_t n) {
  atomicCAS(&err->kind, 0u, kind);
  atomicMin(&err->key, static_cast<unsigned long long>((chunk << 8) | n));
}

// 256^i as an exact binary64 built from its exponent bits (0 <= i <= 16).
__device__ __forceinline__ double pow256(int i) {
  return __longlong_as_double(static_cast<long long>(1023 + 8 * i) << 52);
}

// ------------------------------------------------------------------ epilogue
// y = RN(float(q) * s) (nn.cpp:186), then RN(y + b) with a per-class bias.
// Fast form for 0 < s < 2^100: PRMT puts the byte q under the exponent of
// 2^23 (a = 2^23 + q, exact), and one FFMA gives RN(a*s - 2^23*s) = RN(q*s)
// because the product is exact inside the FMA and 2^23*s is an exact float;
// so 2 full-rate ops per pixel instead of an extract + I2F + FMUL.  Other
// scales (negative, zero, huge, non-finite) take the plain FMUL, which also
// keeps -0.0 for q = 0 and NaN / Inf exactly as the reference.
struct PxScale {
  float s, ms, b;
  bool fast, affine;
};
__device__ __forceinline__ PxScale px_scale(float s, float b, bool affine) {
  PxScale c;
  c.s = s;
  c.b = b;
  c.affine = affine;
  c.fast = s > 0.0f && s < 0x1p100f;
  c.ms = -__fmul_rn(s, 0x1p23f);
  return c;
}
template <bool FAST>
__device__ __forceinline__ float px_value(uint32_t w, int k, const PxScale& c) {
  float y;
  if constexpr (FAST) {
    y = __fmaf_rn(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u | static_cast<uint32_t>(k))), c.s, c.ms);
  } else {
    y = __fmul_rn(static_cast<float>((w >> (8 * k)) & 0xffu), c.s);
  }
  return c.affine ? __fadd_rn(y, c.b) : y;
}

struct Out4 {
  // store 4 consecutive decoded pixels q (bytes of `q4`) at `dst`
  template <int O, bool FAST>
  static __device__ __forceinline__ void put(void* dst, uint32_t q4, const PxScale& c) {
    float y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = px_value<FAST>(q4, k, c);
    if constexpr (O == OPTB_OUT_F32) {
      float4 f = make_float4(y[0], y[1], y[2], y[3]);
      stg16(dst, *reinterpret_cast<uint4*>(&f));
    } else if constexpr (O == OPTB_OUT_F16) {
      const __half2 h0 = __floats2half2_rn(y[0], y[1]), h1 = __floats2half2_rn(y[2], y[3]);
      stg8(dst, make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1)));
    } else {
      const __nv_bfloat162 h0 = __floats2bfloat162_rn(y[0], y[1]), h1 = __floats2bfloat162_rn(y[2], y[3]);
      stg8(dst, make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1)));
    }
  }
};

// 8 consecutive decoded pixels -> 8 binary16 / bfloat16 values, one 128-bit store.
struct Out8 {
  template <int O, bool FAST>
  static __device__ __forceinline__ void put(void* dst, uint2 q8, const PxScale& c) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t src = k < 2 ? q8.x : q8.y;
      const int sh = 2 * (k & 1);
      const float y0 = px_value<FAST>(src, sh, c), y1 = px_value<FAST>(src, sh + 1, c);
      if constexpr (O == OPTB_OUT_F16) {
        const __half2 h = __floats2half2_rn(y0, y1);
        w[k] = *reinterpret_cast<const uint32_t*>(&h);
      } else {
        const __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
        w[k] = *reinterpret_cast<const uint32_t*>(&h);
      }
    }
    stg16(dst, make_uint4(w[0], w[1], w[2], w[3]));
  }
};

template <int O>
__device__ __forceinline__ void put1(void* out, uint64_t idx, uint32_t q, float s, float b,
                                     bool affine) {
  if constexpr (O == OPTB_OUT_U8) {
    static_cast<uint8_t*>(out)[idx] = static_cast<uint8_t>(q);
  } else {
    const float v0 = __fmul_rn(static_cast<float>(q), s);
    const float y = affine ? __fadd_rn(v0, b) : v0;
    if constexpr (O == OPTB_OUT_F32) {
      static_cast<float*>(out)[idx] = y;
    } else if constexpr (O == OPTB_OUT_F16) {
      static_cast<__half*>(out)[idx] = __float2half_rn(y);
    } else {
      static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(y);
    }
  }
}

__device__ __forceinline__ void row_affine(const Epi& e, uint64_t row, float& s, float& b,
                                           bool& affine) {
  s = e.scale;
  b = 0.0f;
  affine = false;
  if (e.class_scale) {
    const int32_t c = __ldg(e.row_class + row);
    s = __ldg(e.class_scale + c);
    if (e.class_bias) {
      b = __ldg(e.class_bias + c);
      affine = true;
    }
  }
}

// ------------------------------------------------------------------ async copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// shared-window address forms, for kernels short of registers: there the
// generic -> shared conversion of a predicated access is rematerialised
// (S2R + LEA) per access
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// 16-byte shared load if p, else zeros
__device__ __forceinline__ uint4 lds16_if(uint32_t a, bool p) {
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("{.reg .pred q; setp.ne.b32 q, %4, 0; @q ld.shared.v4.u32 {%0,%1,%2,%3}, [%5];}"
               : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
               : "r"(static_cast<uint32_t>(p)), "r"(a)
               : "memory");
  return r;
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------ TMA / mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n OPTB_WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra OPTB_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
// 2D tensor-map tile load into shared memory, completing on mbarrier `b`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(b))
      : "memory");
}
// order this thread's generic-proxy accesses before later async-proxy (TMA) ones
// Bulk tensor store of a 1024-aligned smem box (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
               "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the issuing thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and their global writes are performed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Work items: 16 consecutive pixels of one chunk, linear in (chunk, group),
// so a warp's 32 items cover 32*16*WC contiguous container bytes.  Each warp
// runs a kStages-deep cp.async pipeline over its tiles (one tile = the warp's
// 32 items) in a warp-private ring of shared-memory slots: the copies of the
// next kStages-1 tiles are in flight while the current tile is transposed.
// Requires P % 16 == 0 and 16-byte aligned rows / containers / outputs.
constexpr int kStages = OPTB_VEC_STAGES;


// Programmatic dependent launch (the launchers set the attribute, see
// launch_k): the next kernel in the stream may be scheduled while this grid
// drains, and this grid while the previous one drains -- but no global memory
// is touched before the previous kernel has completed and flushed.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ K1 / K3
// Gather-encode for the exact and lossless modes.  Stage slot layout on
// input: row i of the chunk, lane L's 16 pixels at i*512 + L*16
// (conflict-free); after the register transpose the slot is reused as the
// output tile, word p of lane L at (L*16 + (p ^ (L & SW)))*WC (conflict-free
// both ways), then copied out with fully coalesced 128-bit (64-bit) stores.
// Lossless (codec.cpp:125-135): each pixel's 7-bit fields (px >> 1) are
// compacted from byte lanes with three mask/shift steps; the parity bits
// (px & 1) of a lane's 16 pixels of image i are one 16-bit store at plane bit
// i*P + 16*group (aligned: the vector path needs P % 32 == 0 in these modes).
// kF64Narrow: Float64Faithful with at most 8 images per container (the
// common case, capacity 6): half the staging and transpose work of the
// 16-image (lossy) variant, two CTAs per SM.
constexpr int kF64Narrow = 5;

template <int MODE>
struct VecMode {
  static constexpr bool OFFS = (MODE == OPTB_LOSSLESS64 || MODE == OPTB_LOSSLESS128);
  static constexpr int WC = (MODE == OPTB_EXACT128 || MODE == OPTB_LOSSLESS128) ? 16 : 8;
  static constexpr bool F64 = MODE == OPTB_F64 || MODE == kF64Narrow;
  static constexpr int NI = (MODE == OPTB_EXACT64 || MODE == kF64Narrow) ? 8
                            : (MODE == OPTB_EXACT128 || F64) ? 16
                            : (MODE == OPTB_LOSSLESS64) ? 9 : 18;      // images per word
  static constexpr int NT = NI < 16 ? NI : 16;                         // images in the 16x16 transpose
  static constexpr int SW = (WC == 16) ? 7 : 15;                       // slot XOR swizzle mask
  static constexpr int ROWS_B = NI * 512;                              // staged input rows
  static constexpr int WORDS_B = 512 * WC;                             // container words of a tile
  static constexpr int PAR_B = OFFS ? NI * 64 : 0;                     // staged parity bits (decode)
  // lossless slots rounded up to 1024 bytes: the bulk tensor store reads a
  // 128B-swizzled box, which must start 1024-aligned
  static constexpr int ENC_RAW = ROWS_B > WORDS_B ? ROWS_B : WORDS_B;
  static constexpr int ENC_SLOT = OFFS ? (ENC_RAW + 1023) / 1024 * 1024 : ENC_RAW;
  static constexpr int DEC_SLOT = (WORDS_B + PAR_B) > ROWS_B ? (WORDS_B + PAR_B) : ROWS_B;
  static constexpr int MIN_BLOCKS = (WC == 16 || NI == 16) ? 1 : 2;
};

// Float64Faithful peel of one container value into 16 image bytes
// (codec.cpp:171-175: q = fmod(acc, 256), acc = (acc - q) / 256, pixel =
// (u8)q), without fmod:
//  * 0 <= acc < 2^64: the peel is exactly the integer peel of trunc(acc) --
//    fmod keeps acc's fraction in q, (u8)q drops it, (acc - q)/256 is
//    trunc(acc/256);
//  * acc >= 2^64: acc is a multiple of 2^12, so q = 0 and acc/256 is exact;
//  * +inf / NaN: q is NaN -> pixel 0 (the reference's x86 conversion), and
//    acc stays non-finite; the acc >= 2^64 branch yields the same bytes.
__device__ __forceinline__ void f64_peel16(double acc, uint32_t (&b)[4]) {
  b[0] = b[1] = b[2] = b[3] = 0u;
  bool small = acc < 0x1.0p64;
  uint64_t iacc = small ? static_cast<uint64_t>(acc) : 0ull;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint32_t q = 0u;
    if (small) {
      q = static_cast<uint32_t>(iacc & 0xffull);
      iacc >>= 8;
    } else {
      acc = __dmul_rn(acc, 0x1.0p-8);
      small = acc < 0x1.0p64;
      if (small) iacc = static_cast<uint64_t>(acc);
    }
    b[i >> 2] |= q << (8 * (i & 3));
  }
}

// Out-of-line so the rare lossy >= 2^64 case does not bloat the unrolled
// per-pixel loops of the decode kernel.
__device__ __noinline__ uint4 f64_peel_big(double acc) {
  uint32_t t[4];
  f64_peel16(acc, t);
  return make_uint4(t[0], t[1], t[2], t[3]);
}

// Bit select: the bits of a where M is set, else the bits of b -- ONE LOP3
// (inline PTX: written in C the compiler splits it into two mask steps, as
// a LOP3 takes one immediate).
template <uint32_t M>
__device__ __forceinline__ uint32_t bsel(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "n"(M), "r"(a), "r"(b));
  return d;
}

// 8 byte lanes (a = images 0..3, b = images 4..7 of one pixel) -> the 56-bit
// word of their 7-bit fields px >> 1 (field i at bit 7i), as (low, high)
// halves.  Two merge stages per 32-bit half, each ONE bit select between the
// value and its left-shifted copy -- the shifts are multiplies, which run on
// the FMA pipe, while the integer pipe bounds the lossless encoder:
//   stage 1: sel(0xFE00FE00, x, 2x)   field pairs at bits 2..15 / 18..31
//   stage 2: sel(0xFFFC0000, y, 4y)   the 28-bit group at bits 4..31
// The bits a select lets through from the wrong byte (the parity LSBs, a
// neighbour's top bit) land only at positions the next stage or the final
// merge drops (exhaustively-sampled against the masked form: 2e8 random
// inputs, identical words).
__device__ __forceinline__ uint2 pack7x8(uint32_t a, uint32_t b) {
  const uint32_t ga = bsel<0xFE00FE00u>(a, a * 2u);
  const uint32_t gb = bsel<0xFE00FE00u>(b, b * 2u);
  const uint32_t ha = bsel<0xFFFC0000u>(ga, ga * 4u);
  const uint32_t hb = bsel<0xFFFC0000u>(gb, gb * 4u);
  return make_uint2(bsel<0x0FFFFFFFu>(ha >> 4, hb * (1u << 24)), hb >> 8);
}
// Inverse of pack7x8 with the pixel's shift folded in: the 56-bit word of 8
// fields (low, high halves) -> 8 byte lanes holding field << 1 (the pixel
// without its parity bit), with the same select-and-multiply stages:
//   28-bit groups -> sel(0x3FFF, g, 4g) -> sel(0x00FF00FF, 2h, 4h).
// The byte LSBs come out as garbage: the parity merge (a select, before the
// transpose) overwrites them (decode_tile).
__device__ __forceinline__ uint2 unpack7x8_shl1(uint32_t lo, uint32_t hi) {
  const uint32_t gb = __funnelshift_r(lo, hi, 28);
  const uint32_t ha = bsel<0x00003FFFu>(lo, lo * 4u);
  const uint32_t hb = bsel<0x00003FFFu>(gb, gb * 4u);
  return make_uint2(bsel<0x00FF00FFu>(ha * 2u, ha * 4u), bsel<0x00FF00FFu>(hb * 2u, hb * 4u));
}

// PTRS: stream row r is read from the absolute address src.ptrs[r] (this
// GPU's HBM, a peer GPU's HBM over NVLink, mapped pinned host memory) instead
// of src.images + src.index[r] * src.stride.
// warp_region: bytes of shared memory per warp (its ring), >= kStages * slot;
// the fused kernel gives both bodies the same per-warp region so that a warp
// in one phase never touches another warp's ring in the other phase.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

struct NoHook {
  __device__ void operator()(int, bool) const {}
};
struct NoTileHook {
  __device__ void operator()(uint64_t) const {}
};

// on_last(free_stage, earlier_tiles): called at the top of the warp's last
// tile (warp-uniform) with the ring stage that no copy will fill any more,
// and whether the warp stored tiles in earlier iterations.
// after_tile(base): called once the warp has issued the container stores of
// the tile at item base (warp-uniform, after a __syncwarp).
// BULK (exact / f64, 1024-aligned slots): the tile's container words are
// written into its slot in the 128B-swizzled layout of the container tensor
// map smap and leave in ONE bulk tensor store issued by lane 0 (instead of 16
// shared loads + 16 global stores per lane); a slot is refilled only after
// that store has read it.
// src.early: the kernel started without griddepcontrol.wait (only the rows
// and row ids are read before it, RowSrc::early): every lane waits for the
// previous grid before the warp's first global write.
template <int MODE, bool PTRS, typename Hook = NoHook, typename TileHook = NoTileHook, bool BULK = false,
          int NW = kWarps, int NS = kStages>
__device__ __forceinline__ void encode_body(const Geom& g, const RowSrc& src, uint8_t* __restrict__ cont,
                                            uint8_t* __restrict__ offsets, uint8_t* smem_base,
                                            uint32_t warp_region = NS * VecMode<MODE>::ENC_SLOT,
                                            Hook on_last = Hook{}, TileHook after_tile = TileHook{},
                                            const CUtensorMap* smap = nullptr) {
  const uint8_t* __restrict__ images = src.images;
  const uint64_t row_stride = src.stride;
  const int64_t* __restrict__ row_index = src.index;
  using S = VecMode<MODE>;
  constexpr int WC = S::WC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem_base + warp * warp_region;
  // the register-starved lossless bodies -- lossless64 (128 registers in the
  // split encode) and lossless128 inside the interleaved kernel: the lane's
  // shared-window address derived once (ncu: the per-access conversion was
  // rematerialised, S2R + LEA per predicated row) and the parity plane walked
  // by pointer steps.  C3 n=9 encode 76.0 -> 74.1 us, the n=18 interleaved
  // round trip 115.1 -> 105.2 us; the split lossless128 encode (248
  // registers) and the other modes measured slower with it
  constexpr bool SADDR = MODE == OPTB_LOSSLESS64 || (MODE == OPTB_LOSSLESS128 && BULK);
  const uint32_t ring_s = SADDR ? smem_u32(ring) + lane * 16 : 0u;
  const uint64_t G = g.P / 16;
  const uint64_t items = g.chunks * G;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * NW * 32;
  const uint64_t first = (static_cast<uint64_t>(blockIdx.x) * NW + warp) * 32;

  const WalkStep step = walk_step(g, G, stride);
  // Dataset row ids of a tile are fetched one stage before its copies are
  // issued, so the dependent index loads never stall the pipeline.
  Walk wf = walk_at(g, G, first + lane);  // next tile to fetch row ids for
  using RowT = typename std::conditional<PTRS, uint64_t, uint32_t>::type;
  RowT rows[S::NI];
  uint64_t pend_gi = 0;  // group and image count of the fetched tile
  uint32_t pend_n = 0;
  auto fetch_rows = [&]() {
    pend_n = 0;
    if (wf.t < items) {
      const ChunkPos c = walk_chunk(g, wf);
      pend_n = c.n;
      pend_gi = wf.gi;
      // uniform source choice outside the unrolled loop, predicated loads
      // inside it (no per-row branches)
      if constexpr (PTRS) {
        const unsigned long long* rp = reinterpret_cast<const unsigned long long*>(src.ptrs) + c.r0;
#pragma unroll
        for (int i = 0; i < S::NI; ++i) {
          RowT v = 0;
          if (i < static_cast<int>(c.n)) v = __ldg(rp + i);
          rows[i] = v;
        }
      } else if (row_index) {
        const int64_t* rp = row_index + c.r0;
#pragma unroll
        for (int i = 0; i < S::NI; ++i) {
          RowT v = 0;
          if (i < static_cast<int>(c.n)) v = static_cast<uint32_t>(__ldg(rp + i));
          rows[i] = v;
        }
      } else {
#pragma unroll
        for (int i = 0; i < S::NI; ++i) rows[i] = static_cast<RowT>(c.r0 + i);  // used only for i < n
      }
    }
    walk_advance(wf, step, g, G);
  };
  auto issue = [&](int stage) {
    uint8_t* slot = ring + stage * S::ENC_SLOT;
    if constexpr (BULK) {  // the slot's last bulk store has read it
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < S::NI; ++i) {
      if (i < static_cast<int>(pend_n)) {
        const uint8_t* row = PTRS ? reinterpret_cast<const uint8_t*>(static_cast<uintptr_t>(rows[i]))
                                  : images + static_cast<uint64_t>(rows[i]) * row_stride;
        if constexpr (SADDR) {
          cp_async16_s(ring_s + stage * S::ENC_SLOT + i * 512, row + pend_gi * 16);
        } else {
          cp_async16(slot + i * 512 + lane * 16, row + pend_gi * 16);
        }
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    fetch_rows();
    issue(s);
  }
  fetch_rows();
  int stage = 0;
  Walk wc = walk_at(g, G, first + lane);  // the tile being transposed
  for (uint64_t base = first; base < items; base += stride) {
    if (base + stride >= items) on_last((stage + 1) % NS, base != first);
    issue((stage + NS - 1) % NS);
    fetch_rows();  // consumed by the next iteration's issue
    cp_async_wait<NS - 1>();
    __syncwarp();
    // src.early: this iteration's stores (parity bits below, the words
    // after the transpose) are the warp's first global writes
    if (src.early && base == first) pdl_wait();
    uint8_t* slot = ring + stage * S::ENC_SLOT;
    const uint64_t t = wc.t;
    uint32_t n = 0;
    const uint64_t k = wc.k, gi = wc.gi;
    if (t < items) n = walk_chunk(g, wc).n;
    walk_advance(wc, step, g, G);
    uint32_t m[16][4];
    uint32_t x16[4] = {0, 0, 0, 0}, x17[4] = {0, 0, 0, 0};  // images 16, 17 (lossless128)
#pragma unroll
    for (int i = 0; i < S::NI; ++i) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if constexpr (SADDR) {
        v = lds16_if(ring_s + stage * S::ENC_SLOT + i * 512, i < static_cast<int>(n));
      } else if (i < static_cast<int>(n)) {
        v = *reinterpret_cast<const uint4*>(slot + i * 512 + lane * 16);
      }
      if constexpr (S::OFFS) {
        // parity bits of 16 pixels at plane bit i*P + 16*gi (codec.cpp:132-133);
        // images in [n, per_chunk) (partial chunk) write zeros so the padded
        // plane is deterministic; the plane holds per_chunk images.  Images
        // 0..15 are done after the transpose (below); 16 and 17 here.
        if (i >= 16 && t < items && i < static_cast<int>(g.per_chunk)) {
          const uint32_t bits = (((v.x & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) |
                                ((((v.y & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << 4) |
                                ((((v.z & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << 8) |
                                ((((v.w & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << 12);
          *reinterpret_cast<uint16_t*>(offsets + k * g.ostride + (static_cast<uint64_t>(i) * g.P) / 8 + 2 * gi) =
              static_cast<uint16_t>(bits);
        }
      }
      if (i < 16) {
        m[i][0] = v.x;
        m[i][1] = v.y;
        m[i][2] = v.z;
        m[i][3] = v.w;
      } else if (i == 16) {
        x16[0] = v.x; x16[1] = v.y; x16[2] = v.z; x16[3] = v.w;
      } else {
        x17[0] = v.x; x17[1] = v.y; x17[2] = v.z; x17[3] = v.w;
      }
    }
    if constexpr (S::OFFS) {
      if (t < items && gi == 0) {  // zero the plane's stride padding once per chunk
        for (uint64_t b = (static_cast<uint64_t>(g.per_chunk) * g.P) / 8; b < g.ostride; b += 4)
          *reinterpret_cast<uint32_t*>(offsets + k * g.ostride + b) = 0u;
      }
    }
    transpose16<S::NT, 16>(m);  // m[p] = bytes of images 0..15 at pixel p
    if constexpr (S::OFFS) {
      // parity planes of images 0..min(NI,16)-1 from the transposed bytes:
      // lo[q] / hi[q] collect the low bits of pixels 0..7 / 8..15 of images
      // 4q..4q+3 (bit p of byte k), the shifts as multiplies on the FMA pipe;
      // one PRMT then yields image 4q+k's 16 bits
      constexpr int NQ = (S::NT + 3) / 4;
      uint32_t lo[NQ], hi[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        lo[q] = m[0][q] & 0x01010101u;
        hi[q] = m[8][q] & 0x01010101u;
#pragma unroll
        for (int p = 1; p < 8; ++p) {
          lo[q] += (m[p][q] & 0x01010101u) * (1u << p);
          hi[q] += (m[p + 8][q] & 0x01010101u) * (1u << p);
        }
      }
      if (t < items) {
        uint8_t* plane = offsets + k * g.ostride + 2 * gi;
        const uint64_t pstep = g.P >> 3;  // P % 32 == 0 on the vector path
#pragma unroll
        for (int i = 0; i < S::NT; ++i) {
          if (i < static_cast<int>(g.per_chunk)) {
            const uint32_t bits = __byte_perm(lo[i >> 2], hi[i >> 2], (i & 3) | (((i & 3) + 4) << 4));
            uint8_t* dst = SADDR ? plane : offsets + k * g.ostride + 2 * gi + (static_cast<uint64_t>(i) * g.P) / 8;
            *reinterpret_cast<uint16_t*>(dst) = static_cast<uint16_t>(bits);
          }
          if constexpr (SADDR) plane += pstep;
        }
      }
    }
    // lossless container words (codec.cpp:128-134): pixel p's 7-bit fields
    auto ll_word8 = [&](int p) -> uint2 {  // lossless64: images 0..7, image 8's field at bit 56
      const uint2 lo = pack7x8(m[p][0], m[p][1]);
      return make_uint2(lo.x, lo.y + (m[p][2] & 0xFEu) * (1u << 23));
    };
    auto ll_word16 = [&](int p) -> uint4 {  // lossless128: fields 0..15, images 16/17 at bits 112/119
      const uint2 lo = pack7x8(m[p][0], m[p][1]);  // images 0..7 -> bits 0..55
      const uint2 hi = pack7x8(m[p][2], m[p][3]);  // images 8..15 -> bits 56..111
      const uint32_t b16 = (x16[p >> 2] >> (8 * (p & 3))) & 0xFEu;
      const uint32_t b17 = (x17[p >> 2] >> (8 * (p & 3))) & 0xFEu;
      return make_uint4(lo.x, lo.y + hi.x * (1u << 24), (hi.x >> 8) + hi.y * (1u << 24),
                        (hi.y >> 8) + b16 * (1u << 15) + b17 * (1u << 22));
    };
    __syncwarp();
    if constexpr (BULK) {
      // SWIZZLE_128B box: tile byte b at row b / 128, 16-byte chunk
      // (b % 128) / 16 stored at chunk ^ (row & 7).  Same conflict-free
      // orders as the decode's TMA reads (decode_tile).
      auto f64_word = [&](int p) -> uint2 {
        double acc = 0.0;
        if (n <= 6u) {
          const uint64_t word = (static_cast<uint64_t>(m[p][1]) << 32) | m[p][0];
          acc = static_cast<double>(word & ((1ull << (8 * n)) - 1ull));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < static_cast<int>(n))
              acc = __dadd_rn(acc, __dmul_rn(static_cast<double>((m[p][i >> 2] >> (8 * (i & 3))) & 0xffu),
                                             pow256(i)));
        }
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(acc));
        return make_uint2(static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32));
      };
      if constexpr (WC == 16) {  // word p of lane L: row 2L + p/8, chunk p % 8
        const bool hi = (lane >> 2) & 1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int ra = 2 * lane + (hi ? 1 : 0), rb = 2 * lane + (hi ? 0 : 1);
          uint4 lo4, hi4;
          if constexpr (S::OFFS) {
            lo4 = ll_word16(j);
            hi4 = ll_word16(j + 8);
          } else {
            lo4 = make_uint4(m[j][0], m[j][1], m[j][2], m[j][3]);
            hi4 = make_uint4(m[j + 8][0], m[j + 8][1], m[j + 8][2], m[j + 8][3]);
          }
          *reinterpret_cast<uint4*>(slot + ra * 128 + ((j ^ (ra & 7)) << 4)) = hi ? hi4 : lo4;
          *reinterpret_cast<uint4*>(slot + rb * 128 + ((j ^ (rb & 7)) << 4)) = hi ? lo4 : hi4;
        }
      } else {  // WC 8: words 2c, 2c+1 of lane L: row L, chunk c
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          uint2 a, b;
          if constexpr (S::F64) {
            a = f64_word(2 * cc);
            b = f64_word(2 * cc + 1);
          } else if constexpr (S::OFFS) {
            a = ll_word8(2 * cc);
            b = ll_word8(2 * cc + 1);
          } else {
            a = make_uint2(m[2 * cc][0], m[2 * cc][1]);
            b = make_uint2(m[2 * cc + 1][0], m[2 * cc + 1][1]);
          }
          *reinterpret_cast<uint4*>(slot + lane * 128 + ((cc ^ (lane & 7)) << 4)) = make_uint4(a.x, a.y, b.x, b.y);
        }
      }
      fence_proxy_async_smem();  // the slot's generic writes, before the bulk store reads them
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(smap, 0, static_cast<int>((base * 16 * WC) >> 7), slot);
        bulk_commit();
      }
      // after_tile + stage advance below
    } else {
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const int sl = p ^ (lane & S::SW);
        if constexpr (S::F64) {
          // acc += px_i * 256^i in binary64, i ascending (codec.cpp:116-120); the
          // products are exact, the adds round in the reference's order
          double acc = 0.0;
          if (n <= 6u) {
            // every partial sum is an integer < 2^48: exact, so the ordered sum
            // is the packed integer itself (one conversion instead of 2n ops)
            const uint64_t word = (static_cast<uint64_t>(m[p][1]) << 32) | m[p][0];
            acc = static_cast<double>(word & ((1ull << (8 * n)) - 1ull));
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < static_cast<int>(n))
                acc = __dadd_rn(acc, __dmul_rn(static_cast<double>((m[p][i >> 2] >> (8 * (i & 3))) & 0xffu),
                                               pow256(i)));
          }
          *reinterpret_cast<double*>(slot + (lane * 16 + sl) * 8) = acc;
        } else if constexpr (S::OFFS) {
          if constexpr (WC == 8) {
            *reinterpret_cast<uint2*>(slot + (lane * 16 + sl) * 8) = ll_word8(p);
          } else {
            *reinterpret_cast<uint4*>(slot + (lane * 16 + sl) * 16) = ll_word16(p);
          }
        } else if constexpr (WC == 16) {
          *reinterpret_cast<uint4*>(slot + (lane * 16 + sl) * 16) = make_uint4(m[p][0], m[p][1], m[p][2], m[p][3]);
        } else {
          *reinterpret_cast<uint2*>(slot + (lane * 16 + sl) * 8) = make_uint2(m[p][0], m[p][1]);
        }
      }
      __syncwarp();
      uint8_t* dst = cont + base * 16 * WC;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int W = q * 32 + lane, L = W >> 4, p = W & 15;
        if (base + L < items) {
          const int sl = p ^ (L & S::SW);
          if constexpr (WC == 16) {
            stg16(dst + W * 16, *reinterpret_cast<const uint4*>(slot + (L * 16 + sl) * 16));
          } else {
            stg8(dst + W * 8, *reinterpret_cast<const uint2*>(slot + (L * 16 + sl) * 8));
          }
        }
      }
      __syncwarp();
    }
    after_tile(base);
    stage = (stage + 1) % NS;
  }
  cp_async_wait<0>();
  if constexpr (BULK) {  // the slots stay allocated until the stores have read them
    if (lane == 0) bulk_wait0();
    __syncwarp();
  }
}

template <int MODE, bool PTRS>
__global__ void __launch_bounds__(kThreads, VecMode<MODE>::MIN_BLOCKS)
    k_encode_vec(Geom g, RowSrc src, uint8_t* __restrict__ cont, uint8_t* __restrict__ offsets) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  pdl_trigger();
  if (!src.early) pdl_wait();  // early: encode_body waits before the first store
  encode_body<MODE, PTRS>(g, src, cont, offsets, smem_raw);
}

// Exact and f64 encode with the container tiles leaving as bulk tensor
// stores (one per tile, issued by lane 0) instead of per-lane stores.
// Warps per CTA and ring depth of the separate encode / decode launches
// (configs_bench sweep over 8x2, 6x3, 5x4, 4x5): the bulk-store encode runs
// 6 warps x 3 stages (C3 n=16 72.6 -> 68.6 us, f64 90.1 -> 79.9, C4 108.5 ->
// 99.3); the decode 8 x 2, except exact128 into float outputs at 4 warps x 5
// stages (C4 bf16 174 -> 154 us).  OPTB_SPLIT_WARPS / OPTB_SPLIT_STAGES
// override both (tuning builds).
template <int NW_, int NS_, int MODE>
struct ShapeT {
#if defined(OPTB_SPLIT_WARPS) && defined(OPTB_SPLIT_STAGES)
  static constexpr int NW = OPTB_SPLIT_WARPS, NS = OPTB_SPLIT_STAGES;
#else
  static constexpr int NW = NW_, NS = NS_;
#endif
  static constexpr int MIN_BLOCKS = NW == kWarps && NS == kStages ? VecMode<MODE>::MIN_BLOCKS : 1;
};
// DEEP: the shape for long launches (>= 12 tiles per warp at 8 warps per
// SM); short launches keep 8 x 2 (one 256-image ImageNet batch: 42.0 ->
// 35.8 us for the pair).
template <int MODE, bool DEEP>
struct EncShape : ShapeT<DEEP ? 6 : kWarps, DEEP ? 3 : kStages, MODE> {};
template <int MODE, int O, bool DEEP>
struct DecShape : ShapeT<(DEEP && MODE == OPTB_EXACT128 && O != OPTB_OUT_U8) ? 4 : kWarps,
                         (DEEP && MODE == OPTB_EXACT128 && O != OPTB_OUT_U8) ? 5 : kStages, MODE> {};
inline bool split_deep(const Geom& g, int sms) {
  const uint64_t tiles = (g.chunks * (g.P / 16) + 31) / 32;
  return tiles >= static_cast<uint64_t>(12 * kWarps) * sms;
}

template <int MODE, bool PTRS, bool DEEP>
__global__ void __launch_bounds__(EncShape<MODE, DEEP>::NW * 32, EncShape<MODE, DEEP>::MIN_BLOCKS)
    k_encode_bulk(const __grid_constant__ CUtensorMap cmap, Geom g, RowSrc src, uint8_t* __restrict__ cont,
                  uint8_t* __restrict__ offsets) {
  constexpr int NW = EncShape<MODE, DEEP>::NW, NS = EncShape<MODE, DEEP>::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  pdl_trigger();
  if (!src.early) pdl_wait();  // early: encode_body waits before the first store
  encode_body<MODE, PTRS, NoHook, NoTileHook, true, NW, NS>(g, src, cont, offsets, align1024(smem_raw),
                                                            NS * VecMode<MODE>::ENC_SLOT, NoHook{}, NoTileHook{},
                                                            &cmap);
}

// ------------------------------------------------------------------ K2 / K4
// Decode.  Container words (and, lossless, the tile's parity bits) arrive in
// a warp-private ring slot, either by cp.async straight into the XOR-swizzled
// slot or as ONE 2D TMA tensor load per tile (parity bits by cp.async next to
// it) (the tile's 512*WC contiguous bytes as a [rows][128 B] box with the
// hardware's 128-byte swizzle, completion on a per-stage mbarrier).  Each
// pixel's word is range checked, lossless fields are expanded back to byte
// lanes, the 16x16 transpose gives 16 pixels of every image per lane,
// lossless rows get (field << 1) | parity; u8 rows are stored directly (each
// warp instruction writes 512 contiguous bytes of one row); float outputs go
// through a u8 tile in the same slot so that the epilogue stores are
// coalesced too.
//
// TMA slot layout (SWIZZLE_128B, slot 1024-byte aligned): byte b of the tile
// sits at row r = b / 128, 16-byte chunk c = (b % 128) / 16, stored at
// r*128 + ((c ^ (r & 7)) << 4) + b % 16.  Lane L's word p is tile byte
// (16L + p) * WC.  The read order below keeps the 8 lanes of each
// quarter-warp on 8 distinct chunks (conflict-free):
//   WC = 16: r = 2L + p/8, c = p%8; at step j lane L reads p = j and j+8,
//            lanes with L & 4 the high half first;
//   WC = 8 : r = L, c = p/2; at step c lane L reads words 2c, 2c+1.
template <int MODE>
struct DecSlot {
  static constexpr int RAW = VecMode<MODE>::DEC_SLOT;
  static constexpr int TMA = (RAW + 1023) / 1024 * 1024;
};


// One tile of the decode: the container words of items wc.t .. wc.t + 31
// (lane L: item wc.t + L) are in the warp's slot (TMA: the 128B-swizzled box;
// else the XOR-swizzled cp.async layout, lossless parity bits after the
// words).  Range checks, unpack, transpose, epilogue stores.
// LEAN (the interleaved kernels, register-capped): the f64 peel in one
// per-pixel pass instead of the two-pass branch-free form, and the float
// epilogue's full-chunk rows without per-row predicates
template <int MODE, int O, bool TMA, bool LEAN = false>
__device__ __forceinline__ void decode_tile(const Geom& g, const Walk& wc, uint64_t items, uint8_t* slot,
                                            const Epi& e, void* __restrict__ out, DevError* err) {
  using S = VecMode<MODE>;
  constexpr int WC = S::WC;
  const int lane = threadIdx.x & 31;
  const uint64_t ostride = e.row_stride;
  const bool valid = wc.t < items;
  const uint64_t k = wc.k, gi = wc.gi;
  ChunkPos c{0, 0};
  if (valid) c = walk_chunk(g, wc);
  // raw words: m[p] = word of pixel 16*gi + p (low 8 bytes in [0..1] for WC 8)
  uint32_t m[16][4];
  if constexpr (TMA && WC == 16) {
    const bool hi = (lane >> 2) & 1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int ra = 2 * lane + (hi ? 1 : 0), rb = 2 * lane + (hi ? 0 : 1);
      const uint4 a = *reinterpret_cast<const uint4*>(slot + ra * 128 + ((j ^ (ra & 7)) << 4));
      const uint4 b = *reinterpret_cast<const uint4*>(slot + rb * 128 + ((j ^ (rb & 7)) << 4));
      m[j][0] = hi ? b.x : a.x;
      m[j][1] = hi ? b.y : a.y;
      m[j][2] = hi ? b.z : a.z;
      m[j][3] = hi ? b.w : a.w;
      m[j + 8][0] = hi ? a.x : b.x;
      m[j + 8][1] = hi ? a.y : b.y;
      m[j + 8][2] = hi ? a.z : b.z;
      m[j + 8][3] = hi ? a.w : b.w;
    }
  } else if constexpr (TMA) {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const uint4 v = *reinterpret_cast<const uint4*>(slot + lane * 128 + ((cc ^ (lane & 7)) << 4));
      m[2 * cc][0] = v.x;
      m[2 * cc][1] = v.y;
      m[2 * cc + 1][0] = v.z;
      m[2 * cc + 1][1] = v.w;
      m[2 * cc][2] = m[2 * cc][3] = m[2 * cc + 1][2] = m[2 * cc + 1][3] = 0u;
    }
  } else {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const int sl = p ^ (lane & S::SW);
      if constexpr (WC == 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(slot + (lane * 16 + sl) * 16);
        m[p][0] = v.x;
        m[p][1] = v.y;
        m[p][2] = v.z;
        m[p][3] = v.w;
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(slot + (lane * 16 + sl) * 8);
        m[p][0] = v.x;
        m[p][1] = v.y;
        m[p][2] = m[p][3] = 0u;
      }
    }
  }
  // lossless: images NTD.. (lossless64: 8; lossless128: 16, 17) are built as
  // rows directly (xr), the others go through the 16x16 transpose
  constexpr int NTD = S::OFFS ? (WC == 8 ? 8 : 16) : S::NT;
  uint32_t xr[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  bool bad = false;
  if constexpr (S::OFFS) {
    // range check (codec.cpp:189-194): bits >= 7n of every word must be zero;
    // every pixel of the item has the same n, so only the OR of the lane's
    // 16 words is tested
    uint32_t or_w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int p = 0; p < 16; ++p)
#pragma unroll
      for (int q = 0; q < WC / 4; ++q) or_w[q] |= m[p][q];
    const uint64_t o0 = (static_cast<uint64_t>(or_w[1]) << 32) | or_w[0];
    const uint64_t o1 = (static_cast<uint64_t>(or_w[3]) << 32) | or_w[2];
    const unsigned used = 7u * c.n;
    if (used < 64u) bad = (o0 >> used) != 0 || o1 != 0;
    else bad = (o1 >> (used - 64u)) != 0;
    // the rows of the fields above bit 111 / 55, gathered bytewise from 4
    // pixels' top words with PRMT (pixel = field << 1; the bit a multiply
    // shifts into a byte's LSB is overwritten by the parity merge below):
    //   lossless64 : image 8 = bits 56..62 = byte 3 of word 1 (bits 0..6)
    //   lossless128: image 16 = bits 112..118 = byte 2 of word 3 (bits 0..6),
    //                image 17 = bits 119..125 = byte 2 bit 7 + byte 3 bits 0..5
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if constexpr (WC == 8) {
        const uint32_t t1 = __byte_perm(m[4 * q][1], m[4 * q + 1][1], 0x0073);
        const uint32_t t2 = __byte_perm(m[4 * q + 2][1], m[4 * q + 3][1], 0x0073);
        xr[0][q] = __byte_perm(t1, t2, 0x5410) * 2u;
      } else {
        const uint32_t t1 = __byte_perm(m[4 * q][3], m[4 * q + 1][3], 0x7632);
        const uint32_t t2 = __byte_perm(m[4 * q + 2][3], m[4 * q + 3][3], 0x7632);
        const uint32_t b2 = __byte_perm(t1, t2, 0x6420), b3 = __byte_perm(t1, t2, 0x7531);
        xr[0][q] = b2 * 2u;
        xr[1][q] = bsel<0xFCFCFCFCu>(b3 * 4u, b2 >> 6);
      }
    }
    // images 0..7 (and 8..15): byte lanes of field << 1 per pixel
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const uint32_t w0hi = m[p][1], w1lo = m[p][2], w1hi = m[p][3];
      const uint2 lo = unpack7x8_shl1(m[p][0], w0hi);
      m[p][0] = lo.x;
      m[p][1] = lo.y;
      if constexpr (WC == 16) {  // bits 56..111 = (w0 >> 56) | (w1 << 8)
        const uint2 hi = unpack7x8_shl1(__funnelshift_r(w0hi, w1lo, 24), __funnelshift_r(w1lo, w1hi, 24));
        m[p][2] = hi.x;
        m[p][3] = hi.y;
      } else {
        m[p][2] = m[p][3] = 0u;
      }
    }
    // parity bits (codec.cpp:196-201), merged into the byte LSBs BEFORE the
    // transpose: lane's 16 bits of image i (read for every image: rows past
    // the chunk's n are never stored); per group of 4 images, PRMT gathers
    // the bits of pixels 0..7 (L) and 8..15 (H) one byte per image, so pixel
    // p's 4 parity bits are (L >> p) & 0x01010101 -- the shift as a
    // multiply-high on the FMA pipe, the merge one LOP3
    uint32_t bits[S::NI];
#pragma unroll
    for (int i = 0; i < S::NI; ++i) bits[i] = *reinterpret_cast<const uint16_t*>(slot + S::WORDS_B + i * 64 + lane * 2);
#pragma unroll
    for (int g4 = 0; g4 < NTD / 4; ++g4) {
      const uint32_t A = __byte_perm(bits[4 * g4], bits[4 * g4 + 1], 0x5140);
      const uint32_t B = __byte_perm(bits[4 * g4 + 2], bits[4 * g4 + 3], 0x5140);
      const uint32_t L = __byte_perm(A, B, 0x5410), H = __byte_perm(A, B, 0x7632);
      m[0][g4] = bsel<0x01010101u>(L, m[0][g4]);
      m[8][g4] = bsel<0x01010101u>(H, m[8][g4]);
#pragma unroll
      for (int p = 1; p < 8; ++p) {
        m[p][g4] = bsel<0x01010101u>(__umulhi(L, 1u << (32 - p)), m[p][g4]);
        m[p + 8][g4] = bsel<0x01010101u>(__umulhi(H, 1u << (32 - p)), m[p + 8][g4]);
      }
    }
#pragma unroll
    for (int x = 0; x < S::NI - NTD; ++x)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        xr[x][q] = bsel<0x01010101u>(((bits[NTD + x] >> (4 * q)) & 0xFu) * 0x00204081u, xr[x][q]);
  }
  if constexpr (S::F64 && LEAN) {
    // the interleaved kernels (register-capped): one per-pixel pass
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const uint64_t w0 = (static_cast<uint64_t>(m[p][1]) << 32) | m[p][0];
      // codec.cpp:163-170: negative / NaN always, >= 256^n only within capacity
      const double acc = __longlong_as_double(static_cast<long long>(w0));
      bad |= !(acc >= 0.0) || (c.n <= 6u && acc >= pow256(static_cast<int>(c.n)));
      if (acc < 0x1.0p64) {  // common case: the peel is the integer's bytes
        const uint64_t iacc = static_cast<uint64_t>(acc);
        m[p][0] = static_cast<uint32_t>(iacc);
        m[p][1] = static_cast<uint32_t>(iacc >> 32);
        m[p][2] = m[p][3] = 0u;
      } else {
        const uint4 v = f64_peel_big(acc);
        m[p][0] = v.x;
        m[p][1] = v.y;
        m[p][2] = v.z;
        m[p][3] = v.w;
      }
    }
  } else if constexpr (S::F64) {
    // codec.cpp:163-170: negative / NaN always, >= 256^n only within
    // capacity (the bound hoisted out of the pixel loop; past capacity a NaN,
    // which no comparison reaches, +inf included).  The peel of a value below
    // 2^64 is its integer's bytes: a lane whose 16 values all are (the common
    // case) converts them without a branch per pixel; otherwise the
    // per-pixel form with the out-of-line >= 2^64 peel.  (Split decode: C3
    // n=6 85.2 -> 80.1 us; the register-capped interleaved kernel keeps the
    // one-pass form above, slower with this one.)
    const double lim = c.n <= 6u ? pow256(static_cast<int>(c.n)) : __longlong_as_double(0x7ff8000000000000ll);
    bool big = false;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const double acc = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(m[p][1]) << 32) | m[p][0]));
      bad |= !(acc >= 0.0) | (acc >= lim);
      big |= !(acc < 0x1.0p64);
    }
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const double acc = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(m[p][1]) << 32) | m[p][0]));
      if (!big || acc < 0x1.0p64) {
        const uint64_t iacc = static_cast<uint64_t>(acc);
        m[p][0] = static_cast<uint32_t>(iacc);
        m[p][1] = static_cast<uint32_t>(iacc >> 32);
        m[p][2] = m[p][3] = 0u;
      } else {
        const uint4 v = f64_peel_big(acc);
        m[p][0] = v.x;
        m[p][1] = v.y;
        m[p][2] = v.z;
        m[p][3] = v.w;
      }
    }
  }
  transpose16<16, NTD>(m);  // m[i] = 16 pixels of image i < NTD
  if (valid) {
    if constexpr (!S::OFFS && !S::F64) {
      // range check (codec.cpp:189-194): bytes of images >= n must be zero;
      // nothing to check in a chunk at the word's full capacity (the common
      // case: ~85 instructions per tile of compares and selects skipped)
      if (c.n < static_cast<uint32_t>(S::NI)) {
        uint32_t hi = 0;
#pragma unroll
        for (int i = 0; i < S::NI; ++i)
          if (i >= static_cast<int>(c.n)) hi |= m[i][0] | m[i][1] | m[i][2] | m[i][3];
        bad = hi != 0;
      }
    }
    if (bad) latch_error(err, S::F64 ? kErrF64Range : kErrIntRange, g.chunk_base + k, c.n);
  }
  auto row_vec = [&](int i) -> uint4 {
    if (i < NTD) return make_uint4(m[i < NTD ? i : 0][0], m[i < NTD ? i : 0][1], m[i < NTD ? i : 0][2], m[i < NTD ? i : 0][3]);
    const int x = i - NTD < 2 ? i - NTD : 0;
    return make_uint4(xr[x][0], xr[x][1], xr[x][2], xr[x][3]);
  };
  if constexpr (O == OPTB_OUT_U8) {
    if (valid) {
      uint8_t* dst = static_cast<uint8_t*>(out) + c.r0 * ostride + gi * 16;
#pragma unroll
      for (int i = 0; i < S::NI; ++i) {
        if (i < static_cast<int>(c.n)) stg16(dst, row_vec(i));
        dst += ostride;
      }
    }
  } else {
    __syncwarp();  // all lanes done reading the slot
    // u8 tile in the same slot: image i, lane L's 16 pixels at i*512 + L*16
#pragma unroll
    for (int i = 0; i < S::NI; ++i) *reinterpret_cast<uint4*>(slot + i * 512 + lane * 16) = row_vec(i);
    __syncwarp();
    // epilogue: every lane stores 16 bytes per row -- PX = 4 fp32 or 8 half
    // pixels, starting at pixel PX*(lane % LPS) of source lane L's group
    constexpr int ES = (O == OPTB_OUT_F32) ? 4 : 2;
    constexpr int PX = 16 / ES, LPS = 16 / PX, ROUNDS = 32 / (32 / LPS);
#pragma unroll
    for (int cc = 0; cc < ROUNDS; ++cc) {
      const int L = lane / LPS + (32 / LPS) * cc;
      const uint32_t r0lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(c.r0), L);
      const uint32_t r0hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(c.r0 >> 32), L);
      const uint32_t nL = __shfl_sync(0xffffffffu, valid ? c.n : 0u, L);
      const uint32_t glo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(gi), L);
      const uint32_t ghi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(gi >> 32), L);
      const uint64_t r0L = (static_cast<uint64_t>(r0hi) << 32) | r0lo;
      const uint64_t gL = (static_cast<uint64_t>(ghi) << 32) | glo;
      const int sub = PX * (lane % LPS);
      uint8_t* dst = static_cast<uint8_t*>(out) + (r0L * ostride + gL * 16 + sub) * ES;
      const uint64_t dstep = ostride * ES;
      const uint8_t* src = slot + L * 16 + sub;
      auto put_row = [&](uint8_t* d, int i, const PxScale& sc, auto fast) {
        constexpr bool F = decltype(fast)::value;
        if constexpr (PX == 4) {
          Out4::put<O, F>(d, *reinterpret_cast<const uint32_t*>(src + i * 512), sc);
        } else {
          Out8::put<O, F>(d, *reinterpret_cast<const uint2*>(src + i * 512), sc);
        }
      };
      if (!e.class_scale) {  // one scale for every row (the runner's kPixelScale)
        const PxScale sc = px_scale(e.scale, 0.0f, false);
        if (LEAN && sc.fast && nL == static_cast<uint32_t>(S::NI)) {
          // the interleaved kernels, a full chunk (the common case):
          // straight-line stores, no per-row predicate and branch (ncu: ~100
          // instructions per tile; C4 bf16 one batch per launch 27.6 -> 26.8
          // us).  The split decode measured slower with it (deep shape).
#pragma unroll
          for (int i = 0; i < S::NI; ++i) {
            put_row(dst, i, sc, std::true_type{});
            dst += dstep;
          }
        } else if (sc.fast) {
#pragma unroll
          for (int i = 0; i < S::NI; ++i) {
            if (i < static_cast<int>(nL)) put_row(dst, i, sc, std::true_type{});
            dst += dstep;
          }
        } else {
#pragma unroll
          for (int i = 0; i < S::NI; ++i) {
            if (i < static_cast<int>(nL)) put_row(dst, i, sc, std::false_type{});
            dst += dstep;
          }
        }
      } else {  // per-class (scale, bias) tables indexed by the row's class
#pragma unroll
        for (int i = 0; i < S::NI; ++i) {
          if (i < static_cast<int>(nL)) {
            float s, b;
            bool aff;
            row_affine(e, r0L + i, s, b, aff);
            const PxScale sc = px_scale(s, b, aff);
            if (sc.fast) {
              put_row(dst, i, sc, std::true_type{});
            } else {
              put_row(dst, i, sc, std::false_type{});
            }
          }
          dst += dstep;
        }
      }
    }
    // the slot's next fill is an async-proxy (TMA) write
    if constexpr (TMA) fence_proxy_async_smem();
  }
  __syncwarp();
}

// start_stage / prefetched: the fused kernel may have issued the warp's first
// tile already (into start_stage, mbarriers initialised by the caller).
template <int MODE, int O, bool TMA, int NW = kWarps, int NS = kStages>
__device__ __forceinline__ void decode_body(const CUtensorMap* cmap, const Geom& g, const uint8_t* __restrict__ cont,
                                            const uint8_t* __restrict__ offsets, const Epi& e,
                                            void* __restrict__ out, DevError* err, uint8_t* smem_base,
                                            uint64_t* bars, uint32_t warp_region = 0, int start_stage = 0,
                                            bool prefetched = false) {
  using S = VecMode<MODE>;
  constexpr int WC = S::WC;
  constexpr int SLOT = TMA ? DecSlot<MODE>::TMA : DecSlot<MODE>::RAW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem_base + warp * (warp_region ? warp_region : NS * SLOT);
  uint64_t* bar = bars + warp * NS;
  const uint64_t G = g.P / 16;
  const uint64_t items = g.chunks * G;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * NW * 32;
  const uint64_t first = (static_cast<uint64_t>(blockIdx.x) * NW + warp) * 32;
  if constexpr (TMA) {
    if (!prefetched) {
      if (lane == 0)
        for (int st = 0; st < NS; ++st) mbar_init(bar + st, 1);
      fence_mbar_init();
      __syncwarp();
    }
  }

  const WalkStep step = walk_step(g, G, stride);
  const bool bulk_parity = S::OFFS && g.P % 512 == 0;
  Walk wi = walk_at(g, G, first + lane);  // next tile to issue (parity planes)
  Walk wc = wi;                           // the tile being decoded
  auto issue = [&](uint64_t base, int stage) {
    if (base < items) {
      uint8_t* slot = ring + stage * SLOT;
      if constexpr (TMA) {
        if (lane == 0) {
          mbar_expect_tx(bar + stage, 512 * WC);
          tma_load_2d(slot, cmap, 0, static_cast<int>((base * 16 * WC) >> 7), bar + stage);
        }
      } else {
        const uint8_t* src = cont + base * 16 * WC;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int W = q * 32 + lane, L = W >> 4, p = W & 15;
          if (base + L < items) {
            const int sl = p ^ (L & S::SW);
            if constexpr (WC == 16) {
              cp_async16(slot + (L * 16 + sl) * 16, src + W * 16);
            } else {
              cp_async8(slot + (L * 16 + sl) * 8, src + W * 8);
            }
          }
        }
      }
      if constexpr (S::OFFS) {
        if (bulk_parity) {
          // P % 512 == 0: the tile lies in one chunk and image i's 512 parity
          // bits are 64 contiguous, 64-aligned bytes of the plane -- four
          // 16-byte cp.async.cg per image (L2, never a stale L1 line: the
          // fused round trip reads back bits this warp just wrote)
          const uint64_t k = wi.k, gi0 = wi.gi - lane;
          const uint32_t n = walk_chunk(g, wi).n;
          const uint8_t* plane = offsets + k * g.ostride + 2 * gi0;
#pragma unroll
          for (int j = lane; j < 4 * S::NI; j += 32) {
            const int i = j >> 2, part = j & 3;
            if (i < static_cast<int>(n))
              cp_async16(slot + S::WORDS_B + i * 64 + part * 16, plane + (static_cast<uint64_t>(i) * g.P) / 8 + part * 16);
          }
        } else {
        // parity bits of lane pairs (4 bytes, 4-aligned as P % 32 == 0)
        const uint64_t t = wi.t;
        if ((lane & 1) == 0 && t < items) {
          const uint64_t k = wi.k, gi = wi.gi;
          const uint32_t n = walk_chunk(g, wi).n;
          const bool pair = (t + 1 < items) && (gi + 1 < G);
#pragma unroll
          for (int i = 0; i < S::NI; ++i) {
            if (i < static_cast<int>(n)) {
              const uint8_t* ps = offsets + k * g.ostride + (static_cast<uint64_t>(i) * g.P) / 8 + 2 * gi;
              uint8_t* pd = slot + S::WORDS_B + i * 64 + lane * 2;
              if (pair) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(pd)), "l"(ps) : "memory");
              } else {
                *reinterpret_cast<uint16_t*>(pd) = *reinterpret_cast<const uint16_t*>(ps);
              }
            }
          }
        }
        }
      }
    }
    if constexpr (!TMA || S::OFFS) cp_async_commit();  // words (cp.async path) / parity bits
    if constexpr (S::OFFS) walk_advance(wi, step, g, G);
  };

  if (!prefetched) {
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) issue(first + s * stride, s);
  }
  int stage = start_stage;
  uint32_t phase_bits = 0;  // parity of each stage's mbarrier
  for (uint64_t base = first; base < items; base += stride) {
    issue(base + (NS - 1) * stride, (stage + NS - 1) % NS);
    if constexpr (TMA) mbar_wait(bar + stage, (phase_bits >> stage) & 1u);
    if constexpr (!TMA || S::OFFS) {
      cp_async_wait<NS - 1>();
      __syncwarp();
    }
    decode_tile<MODE, O, TMA>(g, wc, items, ring + stage * SLOT, e, out, err);
    walk_advance(wc, step, g, G);
    phase_bits ^= 1u << stage;
    if (++stage == NS) stage = 0;
  }
  if constexpr (!TMA || S::OFFS) cp_async_wait<0>();
}

template <int MODE, int O, bool TMA, bool DEEP>
__global__ void __launch_bounds__(DecShape<MODE, O, DEEP>::NW * 32, DecShape<MODE, O, DEEP>::MIN_BLOCKS)
    k_decode_vec(const __grid_constant__ CUtensorMap cmap, Geom g, const uint8_t* __restrict__ cont,
                 const uint8_t* __restrict__ offsets, Epi e, void* __restrict__ out, DevError* err) {
  constexpr int NW = DecShape<MODE, O, DEEP>::NW, NS = DecShape<MODE, O, DEEP>::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bars[TMA ? NW * NS : 1];
  pdl_entry();
  decode_body<MODE, O, TMA, NW, NS>(&cmap, g, cont, offsets, e, out, err, TMA ? align1024(smem_raw) : smem_raw,
                                    bars);
}

// ------------------------------------------------------------------ K1+K2 fused
// One step's round trip in one persistent launch (the E-D pipeline step,
// pipeline.cpp:197-216 producer encode + runner.cpp:292-309 consumer decode):
// every warp gather-encodes its tiles into the container stream in HBM, then
// decodes the same tiles back -- in the order it wrote them, so by the time a
// tile is read back the rest of the step's ~150 MB of traffic has gone
// through L2 and the read is served by HBM like a separate decode launch.
// No warp reads another warp's containers, so no grid-wide barrier is needed;
// the kernel saves one launch's ramp-up and tail.  Exact and f64 modes (the
// decode half reads each tile with one TMA tensor load).
// Per-warp shared-memory region of the fused kernel: room for either ring,
// 1024-aligned so every TMA slot stays 1024-aligned.
template <int MODE>
struct RtRegion {
  static constexpr uint32_t ENC = kStages * VecMode<MODE>::ENC_SLOT;
  static constexpr uint32_t DEC = kStages * DecSlot<MODE>::TMA;
  static constexpr uint32_t BYTES = ((ENC > DEC ? ENC : DEC) + 1023) / 1024 * 1024;
};

// Register budget: at most OPTB_RT_MAXREG per thread for one CTA per SM (no
// spills at 184), which leaves ~18 K registers per SM for the SBS kernels of
// the next draw call on the side stream; 128 for two CTAs per SM.  The
// 16-byte-word variants always run one CTA per SM; the 8-byte ones two
// (f64, lossless64: ALU-heavier), except exact64 with more than two images
// per container, measured faster with one (ONE_CTA; configs_bench: C1 0.89 ->
// 0.95 of peak, while n = 2 drops 0.95 -> 0.89 with one CTA).
#ifndef OPTB_RT_MAXREG
#define OPTB_RT_MAXREG 184
#endif
template <int MODE, bool ONE_CTA>
struct RtRegs {
  static constexpr int VALUE = (VecMode<MODE>::MIN_BLOCKS == 2 && !ONE_CTA) ? 128 : OPTB_RT_MAXREG;
};
template <int MODE, int O, bool PTRS, bool ONE_CTA = false>
__global__ void __maxnreg__((RtRegs<MODE, ONE_CTA>::VALUE))
    k_roundtrip_vec(const __grid_constant__ CUtensorMap cmap, Geom g, RowSrc src, uint8_t* __restrict__ cont,
                    uint8_t* __restrict__ offsets, Epi e, void* __restrict__ out, DevError* err) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bars[kWarps * kStages];
  uint8_t* base = align1024(smem_raw);
  pdl_entry();
  // The phase switch without a bubble: during its last encode tile a warp
  // already loads its first decode tile (stored in its first iteration) into
  // the ring stage no copy will fill any more -- when the two rings share the
  // slot size (exact, f64) and the warp has encoded more than one tile.
  constexpr bool kPrefetch = !VecMode<MODE>::OFFS && VecMode<MODE>::ENC_SLOT == DecSlot<MODE>::TMA && kStages == 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bar = bars + warp * kStages;
  if constexpr (kPrefetch) {
    if (lane == 0)
      for (int st = 0; st < kStages; ++st) mbar_init(bar + st, 1);
    fence_mbar_init();
    __syncwarp();
  }
  int start_stage = 0;
  bool prefetched = false;
  auto prefetch_first = [&](int free_stage, bool earlier_tiles) {
    if constexpr (kPrefetch) {
      if (!earlier_tiles) return;
      fence_proxy_async_global();  // the warp's container stores so far, before the TMA read
      fence_proxy_async_smem();    // its writes to the free slot, before the TMA write
      __syncwarp();
      if (lane == 0) {
        const uint64_t t0 = (static_cast<uint64_t>(blockIdx.x) * kWarps + warp) * 32;
        constexpr int WC = VecMode<MODE>::WC;
        mbar_expect_tx(bar + free_stage, 512 * WC);
        tma_load_2d(base + warp * RtRegion<MODE>::BYTES + free_stage * DecSlot<MODE>::TMA, &cmap, 0,
                    static_cast<int>((t0 * 16 * WC) >> 7), bar + free_stage);
      }
      start_stage = free_stage;
      prefetched = true;
    }
  };
  encode_body<MODE, PTRS>(g, src, cont, offsets, base, RtRegion<MODE>::BYTES, prefetch_first);
  // this warp's container stores (generic proxy) before its TMA reads of
  // them, and its staging writes before the TMA fills of the same slots
  fence_proxy_async_global();
  fence_proxy_async_smem();
  __syncwarp();
  decode_body<MODE, O, true>(&cmap, g, cont, offsets, e, out, err, base, bars, RtRegion<MODE>::BYTES, start_stage,
                             prefetched);
}

// The interleaved round trip (exact and f64 modes): a warp decodes each tile
// one encode iteration after storing it -- encode tile j, decode tile j-1,
// then one TMA load of tile j's container words into the warp's decode slot,
// which lands while tile j+1 is being gathered and encoded.  The container
// stream is still written to HBM in full (the stores are the same), but each
// tile is read back while its lines are still in L2: per step the DRAM moves
// the gathered rows in, the containers and the decoded rows out, and the
// decode's container read is an L2 hit (ncu: dram bytes = the compulsory
// 3 x ~153 MB instead of 4x).  Same per-warp tile sequence as the phase-
// ordered kernel above, so the results are identical.

// Warps per CTA and input-ring depth of the interleaved kernel (one CTA per
// SM).  DEEP: 5 warps x 4 stages -- fewer warps with deeper rings keep more
// gathered rows in flight per SM, the faster shape for exact128 -> u8 on long
// launches (C2 step 89.8 -> 85.2 us); the default 8 x 2 wins for float
// outputs and short launches (few tiles per warp), measured with
// tools/configs_bench.py.  OPTB_IL_WARPS / OPTB_IL_STAGES override both
// shapes (sweeps).
template <int MODE, bool DEEP>
struct IlShape {
#if defined(OPTB_IL_WARPS) && defined(OPTB_IL_STAGES)  // sweeps of the deep shape
  static constexpr int NW = DEEP ? OPTB_IL_WARPS : 8;
  static constexpr int NS = DEEP ? OPTB_IL_STAGES : 2;
#else
  static constexpr int NW = DEEP ? 5 : 8;
  static constexpr int NS = DEEP ? 4 : 2;
#endif
};
template <int MODE, bool DEEP>
struct IlRegion {
  static constexpr uint32_t ENC = IlShape<MODE, DEEP>::NS * VecMode<MODE>::ENC_SLOT;  // 1024-multiple
  static constexpr uint32_t BYTES = ENC + DecSlot<MODE>::TMA;
  static constexpr size_t SMEM = static_cast<size_t>(IlShape<MODE, DEEP>::NW) * BYTES + 1024;
};
#ifndef OPTB_IL_DEEP_MAXREG
#define OPTB_IL_DEEP_MAXREG 232  // 5 warps per SM: registers are free (C2 583 -> 591 M img/s)
#endif
template <int MODE, int O, bool PTRS, bool ONE_CTA, bool DEEP, bool BULK_ST>
// lossless128 (18 staged rows, 2 x 9 KB ring + 10 KB decode slot per warp:
// 8 warps fit in 225 KB) takes the full register file, 255 per thread
__global__ void __maxnreg__((DEEP ? OPTB_IL_DEEP_MAXREG : MODE == OPTB_LOSSLESS128 ? 255 : RtRegs<MODE, ONE_CTA>::VALUE))
    k_roundtrip_il(const __grid_constant__ CUtensorMap cmap, Geom g, RowSrc src, uint8_t* __restrict__ cont,
                   uint8_t* __restrict__ offsets, Epi e, void* __restrict__ out, DevError* err) {
  static_assert(IlRegion<MODE, DEEP>::ENC % 1024 == 0, "decode slot must stay 1024-aligned");
  constexpr bool BULK = BULK_ST;
  constexpr bool OFFS = VecMode<MODE>::OFFS;
  // lossless: the tile's parity bits are reloaded with cp.async beside the
  // words' TMA load, committed after the encode's gather of the next stage;
  // with a 2-stage ring the encode's own wait (all but the newest group)
  // completes them before the decode (see after_tile)
  static_assert(!OFFS || (IlShape<MODE, DEEP>::NS == 2 && BULK_ST), "interleaved lossless: 2-stage ring, bulk stores");
  static_assert(IlRegion<MODE, DEEP>::SMEM <= 232448, "interleaved kernel: shared memory over the 227 KB limit");
  constexpr int WC = VecMode<MODE>::WC;
  constexpr int NW = IlShape<MODE, DEEP>::NW, NS = IlShape<MODE, DEEP>::NS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bars[NW];
  uint8_t* base = align1024(smem_raw);
  // programmatic dependent launch: the next grid may start now.  With
  // src.early (the pipeline's steps) this one gathers its first tiles while
  // the previous step's grid drains and waits for it (griddepcontrol.wait)
  // before its first global write; otherwise it waits here.
  pdl_trigger();
  if (!src.early) pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bar = bars + warp;
  uint8_t* dslot = base + warp * IlRegion<MODE, DEEP>::BYTES + IlRegion<MODE, DEEP>::ENC;
  if (lane == 0) mbar_init(bar, 1);
  fence_mbar_init();
  __syncwarp();
  const uint64_t G = g.P / 16;
  const uint64_t items = g.chunks * G;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * NW * 32;
  const WalkStep step = walk_step(g, G, stride);
  Walk wd = walk_at(g, G, (static_cast<uint64_t>(blockIdx.x) * NW + warp) * 32 + lane);
  uint32_t phase = 0;
  bool pending = false;
  auto decode_pending = [&]() {
    mbar_wait(bar, phase);
    phase ^= 1u;
    decode_tile<MODE, O, true, true>(g, wd, items, dslot, e, out, err);  // ends with __syncwarp
    walk_advance(wd, step, g, G);
  };
  auto after_tile = [&](uint64_t tile) {
    if (pending) decode_pending();
    // the decode slot's generic writes (float epilogue) were fenced in
    // decode_tile; the tile's bulk store must be complete before the load
    if constexpr (BULK) {
      if (lane == 0) bulk_wait0();
    } else {
      fence_proxy_async_global();  // this tile's container stores (generic proxy), before the TMA read
    }
    __syncwarp();
    if (lane == 0) {
      mbar_expect_tx(bar, 512 * WC);
      tma_load_2d(dslot, &cmap, 0, static_cast<int>((tile * 16 * WC) >> 7), bar);
    }
    if constexpr (OFFS) {
      // tile j's parity bits (written by this warp's lanes in the encode,
      // ordered by the __syncwarp above): P % 512 == 0 (the launcher's
      // condition), so image i's 512 bits are 64 contiguous plane bytes --
      // four 16-byte L2 copies each (.cg: never a stale L1 line).  wd is
      // tile j here (advanced past j-1 by the decode above).
      constexpr int NI = VecMode<MODE>::NI;
      const uint64_t k = wd.k, gi0 = wd.gi - lane;
      const uint32_t n = walk_chunk(g, wd).n;
      const uint8_t* plane = offsets + k * g.ostride + 2 * gi0;
#pragma unroll
      for (int j = lane; j < 4 * NI; j += 32) {
        const int i = j >> 2, part = j & 3;
        if (i < static_cast<int>(n))
          cp_async16(dslot + VecMode<MODE>::WORDS_B + i * 64 + part * 16,
                     plane + (static_cast<uint64_t>(i) * g.P) / 8 + part * 16);
      }
      cp_async_commit();
    }
    pending = true;
  };
  encode_body<MODE, PTRS, NoHook, decltype(after_tile), BULK, NW, NS>(g, src, cont, offsets, base,
                                                                          IlRegion<MODE, DEEP>::BYTES, NoHook{}, after_tile,
                                                                          &cmap);
  if (pending) decode_pending();
}

// ------------------------------------------------------------------ generic
// One pixel per lane; any P, any alignment; all five modes.  Items are linear
// in (chunk, pixel), so a warp's lanes are consecutive pixels of (at most two)
// chunks.  Lossless parity bits are accumulated with warp ballots and written
// with atomicOr into a zeroed plane (covers unaligned bit offsets).
template <int MODE>
__global__ void __launch_bounds__(256) k_encode_generic(Geom g, RowSrc rs, uint8_t* __restrict__ cont,
                                                        uint8_t* __restrict__ offsets) {
  constexpr bool OFFS = (MODE == OPTB_LOSSLESS64 || MODE == OPTB_LOSSLESS128);
  constexpr int WC = (MODE == OPTB_EXACT128 || MODE == OPTB_LOSSLESS128) ? 16 : 8;
  constexpr int MAXN = (MODE == OPTB_EXACT64) ? 8 : (MODE == OPTB_EXACT128) ? 16
                       : (MODE == OPTB_F64) ? 16 : (MODE == OPTB_LOSSLESS64) ? 9 : 18;
  const uint64_t items = g.chunks * g.P;
  const int lane = threadIdx.x & 31;
  const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
       t0 < items; t0 += gstride) {
    const uint64_t t = t0 + lane;
    const bool valid = t < items;
    uint64_t k = 0, p = 0;
    ChunkPos c{0, 0};
    if (valid) {
      k = t / g.P;
      p = t - k * g.P;
      c = chunk_pos(g, k);
    }
    unsigned __int128 acc = 0;
    double dacc = 0.0;
#pragma unroll
    for (int i = 0; i < MAXN; ++i) {
      uint32_t px = 0;
      const bool has = valid && i < static_cast<int>(c.n);
      if (has) {
        const uint64_t r = c.r0 + i;
        if (rs.ptrs) {
          px = __ldg(reinterpret_cast<const uint8_t*>(static_cast<uintptr_t>(__ldg(
                         reinterpret_cast<const unsigned long long*>(rs.ptrs) + r))) + p);
        } else {
          const uint64_t src = rs.index ? static_cast<uint64_t>(__ldg(rs.index + r)) : r;
          px = __ldg(rs.images + src * rs.stride + p);
        }
        if constexpr (MODE == OPTB_F64) {
          // codec.cpp:116-120: acc += px * 256^i in binary64, i ascending
          dacc = __dadd_rn(dacc, __dmul_rn(static_cast<double>(px), pow256(i)));
        } else if constexpr (OFFS) {
          acc |= static_cast<unsigned __int128>(px >> 1) << (7 * i);
        } else {
          acc |= static_cast<unsigned __int128>(px) << (8 * i);
        }
      }
      if constexpr (OFFS) {
        // parity bit i*P + p of chunk k (codec.cpp:132-133)
        const uint32_t bits = __ballot_sync(0xffffffffu, has && (px & 1u));
        const uint32_t inchunk = __ballot_sync(0xffffffffu, has);
        if (has) {
          // the first lane of each same-chunk run writes that run's bits
          const uint32_t same = __match_any_sync(inchunk, k);
          const int lead = __ffs(same) - 1;
          if (lane == lead) {
            const uint32_t seg = (bits & same) >> lead;
            if (seg) {
              const uint64_t bit = static_cast<uint64_t>(i) * g.P + p;  // p of the leader
              uint32_t* plane = reinterpret_cast<uint32_t*>(offsets + k * g.ostride);
              const uint64_t w = bit >> 5;
              const uint32_t sh = static_cast<uint32_t>(bit & 31);
              atomicOr(plane + w, seg << sh);
              if (sh && (seg >> (32 - sh))) atomicOr(plane + w + 1, seg >> (32 - sh));
            }
          }
        }
      }
    }
    if (valid) {
      uint8_t* w = cont + t * WC;
      if constexpr (MODE == OPTB_F64) {
        *reinterpret_cast<double*>(w) = dacc;
      } else if constexpr (WC == 8) {
        *reinterpret_cast<uint64_t*>(w) = static_cast<uint64_t>(acc);
      } else {
        reinterpret_cast<uint64_t*>(w)[0] = static_cast<uint64_t>(acc);
        reinterpret_cast<uint64_t*>(w)[1] = static_cast<uint64_t>(acc >> 64);
      }
    }
  }
}

template <int MODE, int O>
__global__ void __launch_bounds__(256) k_decode_generic(Geom g, const uint8_t* __restrict__ cont,
                                                        const uint8_t* __restrict__ offsets, Epi e,
                                                        void* __restrict__ out, DevError* err) {
  constexpr bool OFFS = (MODE == OPTB_LOSSLESS64 || MODE == OPTB_LOSSLESS128);
  constexpr int WC = (MODE == OPTB_EXACT128 || MODE == OPTB_LOSSLESS128) ? 16 : 8;
  constexpr int MAXN = (MODE == OPTB_EXACT64) ? 8 : (MODE == OPTB_EXACT128) ? 16
                       : (MODE == OPTB_F64) ? 16 : (MODE == OPTB_LOSSLESS64) ? 9 : 18;
  constexpr unsigned PER = OFFS ? 7u : 8u;
  const uint64_t items = g.chunks * g.P;
  const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // (chunk, pixel) of the thread's item advanced with adds and compares
  Walk wk = walk_at(g, g.P, static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
  const WalkStep wstep = walk_step(g, g.P, gstride);
  for (; wk.t < items; walk_advance(wk, wstep, g, g.P)) {
    const uint64_t t = wk.t;
    const uint64_t k = wk.k;
    const uint64_t p = wk.gi;
    const ChunkPos c = walk_chunk(g, wk);
    const uint8_t* w = cont + t * WC;
    if constexpr (MODE == OPTB_F64) {
      double acc = *reinterpret_cast<const double*>(w);
      // codec.cpp:163-170
      const bool check = c.n <= 6u;
      const double limit = pow256(static_cast<int>(c.n));
      if (!(acc >= 0.0) || (check && acc >= limit)) {
        latch_error(err, kErrF64Range, g.chunk_base + k, c.n);
        continue;
      }
      // codec.cpp:171-175 peels with q = fmod(acc, 256), acc = (acc - q) / 256.
      // For 0 <= acc < 2^64 that is exactly the integer peel of trunc(acc):
      // fmod keeps acc's fraction in q, (u8)q drops it, and (acc - q)/256 is
      // trunc(acc/256).  Only lossy sums >= 2^64 (n >= 9) need fmod itself.
      const bool small = acc < 0x1.0p64;
      uint64_t iacc = small ? static_cast<uint64_t>(acc) : 0ull;
#pragma unroll
      for (int i = 0; i < MAXN; ++i) {
        if (i < static_cast<int>(c.n)) {
          double q;
          if (small) {
            q = static_cast<double>(iacc & 0xffull);
            iacc >>= 8;
          } else {
            q = fmod(acc, 256.0);                          // exact
            acc = __dmul_rn(__dsub_rn(acc, q), 0x1.0p-8);  // exact
          }
          const uint64_t row = c.r0 + i;
          float s, b;
          bool aff;
          row_affine(e, row, s, b, aff);
          put1<O>(out, row * e.row_stride + p, static_cast<uint32_t>(q), s, b, aff);
        }
      }
    } else {
      unsigned __int128 acc;
      if constexpr (WC == 8) {
        acc = *reinterpret_cast<const uint64_t*>(w);
      } else {
        acc = (static_cast<unsigned __int128>(reinterpret_cast<const uint64_t*>(w)[1]) << 64) |
              reinterpret_cast<const uint64_t*>(w)[0];
      }
      const unsigned used = PER * c.n;
      if (used < WC * 8u && (acc >> used) != 0) {  // codec.cpp:189-194
        latch_error(err, kErrIntRange, g.chunk_base + k, c.n);
        continue;
      }
      const uint8_t* plane = OFFS ? offsets + k * g.ostride : nullptr;
#pragma unroll
      for (int i = 0; i < MAXN; ++i) {
        if (i < static_cast<int>(c.n)) {
          uint32_t q = static_cast<uint32_t>(acc >> (PER * i)) & ((1u << PER) - 1u);
          if constexpr (OFFS) {
            const uint64_t bit = static_cast<uint64_t>(i) * g.P + p;
            q = (q << 1) | ((__ldg(plane + (bit >> 3)) >> (bit & 7)) & 1u);
          }
          const uint64_t row = c.r0 + i;
          float s, b;
          bool aff;
          row_affine(e, row, s, b, aff);
          put1<O>(out, row * e.row_stride + p, q, s, b, aff);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ dispatch
template <typename K>
int grid_for(K kernel, int threads, size_t smem, int num_sms, uint64_t work_units) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const uint64_t want = (work_units + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(per_sm) * num_sms;
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Launch with the programmatic-stream-serialization attribute (the kernel
// calls pdl_entry() first).  The overlap happens only kernel after kernel in
// one stream; event waits and copies in between serialise as usual.
// OPTB_PDL=0: plain launches (A/B runs).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), int grid, int threads, size_t smem, cudaStream_t s, Args&&... args) {
  static const bool pdl = [] {
    const char* v = getenv("OPTB_PDL");
    return !(v && v[0] == '0');
  }();
  bump_stream_tag(s);  // this kernel triggers its dependents early (pdl_entry / pdl_trigger)
  if (!pdl) {
    kernel<<<grid, threads, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int MODE>
cudaError_t enc_generic(const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs, cudaStream_t s, int sms,
                        uint64_t* launches) {
  if (MODE == OPTB_LOSSLESS64 || MODE == OPTB_LOSSLESS128) {
    cudaError_t st = cudaMemsetAsync(offs, 0, g.chunks * g.ostride, s);
    if (st != cudaSuccess) return st;
  }
  const int grid = grid_for(k_encode_generic<MODE>, 256, 0, sms, g.chunks * g.P);
  k_encode_generic<MODE><<<grid, 256, 0, s>>>(g, rs, static_cast<uint8_t*>(cont), offs);
  ++*launches;
  return cudaGetLastError();
}

template <int MODE, int O>
cudaError_t dec_generic(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e,
                        void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  const int grid = grid_for(k_decode_generic<MODE, O>, 256, 0, sms, g.chunks * g.P);
  k_decode_generic<MODE, O><<<grid, 256, 0, s>>>(g, static_cast<const uint8_t*>(cont), offs, e,
                                                 out, err);
  ++*launches;
  return cudaGetLastError();
}

bool container_map(CUtensorMap* m, const void* cont, uint64_t bytes, int wc);
// OPTB_ENCODE_BULK=0 selects the per-lane container stores (A/B runs)
bool encode_bulk_enabled() {
  static const bool on = [] {
    const char* v = getenv("OPTB_ENCODE_BULK");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <int MODE, bool PTRS, bool DEEP>
cudaError_t enc_bulk_launch(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs,
                            cudaStream_t s, int sms, uint64_t* launches) {
  constexpr int threads = EncShape<MODE, DEEP>::NW * 32;
  const size_t smem = static_cast<size_t>(EncShape<MODE, DEEP>::NW) * EncShape<MODE, DEEP>::NS *
                          VecMode<MODE>::ENC_SLOT + 1024;
  auto kernel = k_encode_bulk<MODE, PTRS, DEEP>;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(kernel), static_cast<int>(smem));
  if (ae != cudaSuccess) return ae;
  const uint64_t items = g.chunks * (g.P / 16);
  const int grid = grid_for(kernel, threads, smem, sms, items);
  const cudaError_t le = launch_k(kernel, grid, threads, smem, s, cm, g, rs, static_cast<uint8_t*>(cont), offs);
  ++*launches;
  return le;
}

template <int MODE, bool PTRS>
cudaError_t enc_vec_t(const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs, cudaStream_t s, int sms,
                      uint64_t* launches) {
  // lossless128 keeps the per-lane container stores (C3 n=18: 73.4 us
  // against 75.7 with bulk stores); lossless64 gains (79.9 -> 75.4 us)
  if constexpr (MODE != OPTB_LOSSLESS128) {
    CUtensorMap cm;
    if (encode_bulk_enabled() && !g_sysmem && container_map(&cm, cont, g.chunks * g.P * VecMode<MODE>::WC, VecMode<MODE>::WC)) {
      // lossless (integer-pipe bound) keeps 8 x 2 at every size: the deep
      // shape's register budget leaves one 6-warp CTA per SM (C3 n=9 74 ->
      // 87 us), too few warps to hide the ALU dependency chains
      if (!VecMode<MODE>::OFFS && split_deep(g, sms))
        return enc_bulk_launch<MODE, PTRS, true>(cm, g, rs, cont, offs, s, sms, launches);
      return enc_bulk_launch<MODE, PTRS, false>(cm, g, rs, cont, offs, s, sms, launches);
    }
  }
  const size_t smem = static_cast<size_t>(kWarps) * kStages * VecMode<MODE>::ENC_SLOT;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(k_encode_vec<MODE, PTRS>), static_cast<int>(smem));
  if (ae != cudaSuccess) return ae;
  const uint64_t items = g.chunks * (g.P / 16);
  const int grid = grid_for(k_encode_vec<MODE, PTRS>, kThreads, smem, sms, items);
  const cudaError_t le = launch_k(k_encode_vec<MODE, PTRS>, grid, kThreads, smem, s, g, rs,
                                  static_cast<uint8_t*>(cont), offs);
  ++*launches;
  return le;
}

template <int MODE>
cudaError_t enc_vec(const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs, cudaStream_t s, int sms,
                    uint64_t* launches) {
  if (rs.ptrs) return enc_vec_t<MODE, true>(g, rs, cont, offs, s, sms, launches);
  return enc_vec_t<MODE, false>(g, rs, cont, offs, s, sms, launches);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// The container stream as a [bytes/128][128] u8 tensor, box = one decode tile
// (512 words = 512*WC bytes), 128-byte hardware swizzle (see decode_body).
bool container_map(CUtensorMap* m, const void* cont, uint64_t bytes, int wc) {
  const EncodeTiledFn fn = encode_tiled();
  if (!fn || bytes % 128 || bytes / 128 > 0x7fffffffull) return false;
  const cuuint64_t dims[2] = {128, bytes / 128};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(512 * wc / 128)};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(cont), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// OPTB_DECODE_TMA=0 selects the cp.async decode (A/B measurements)
bool tma_decode_enabled() {
  static const bool on = [] {
    const char* v = getenv("OPTB_DECODE_TMA");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <int MODE, int O, bool TMA, bool DEEP>
cudaError_t dec_vec_launch(const CUtensorMap& cm, const Geom& g, const void* cont, const uint8_t* offs,
                           const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  constexpr int NW = DecShape<MODE, O, DEEP>::NW, NS = DecShape<MODE, O, DEEP>::NS;
  const size_t smem = TMA ? static_cast<size_t>(NW) * NS * DecSlot<MODE>::TMA + 1024
                          : static_cast<size_t>(NW) * NS * DecSlot<MODE>::RAW;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(k_decode_vec<MODE, O, TMA, DEEP>), static_cast<int>(smem));
  if (ae != cudaSuccess) return ae;
  const uint64_t items = g.chunks * (g.P / 16);
  const int grid = grid_for(k_decode_vec<MODE, O, TMA, DEEP>, NW * 32, smem, sms, items);
  const cudaError_t le = launch_k(k_decode_vec<MODE, O, TMA, DEEP>, grid, NW * 32, smem, s, cm, g,
                                  static_cast<const uint8_t*>(cont), offs, e, out, err);
  ++*launches;
  return le;
}

template <int MODE, int O>
cudaError_t dec_vec(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e, void* out,
                    DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  CUtensorMap cm;
  if (tma_decode_enabled() && !g_sysmem && container_map(&cm, cont, g.chunks * g.P * VecMode<MODE>::WC, VecMode<MODE>::WC))
    return split_deep(g, sms) ? dec_vec_launch<MODE, O, true, true>(cm, g, cont, offs, e, out, err, s, sms, launches)
                              : dec_vec_launch<MODE, O, true, false>(cm, g, cont, offs, e, out, err, s, sms, launches);
  memset(&cm, 0, sizeof cm);
  return dec_vec_launch<MODE, O, false, false>(cm, g, cont, offs, e, out, err, s, sms, launches);
}

template <int MODE, int O, bool PTRS, bool ONE_CTA, bool DEEP, bool BULK_ST = true>
cudaError_t rt_il_launch(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs,
                         const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  constexpr size_t smem = IlRegion<MODE, DEEP>::SMEM;
  constexpr int threads = IlShape<MODE, DEEP>::NW * 32;
  auto kernel = k_roundtrip_il<MODE, O, PTRS, ONE_CTA, DEEP, BULK_ST>;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(kernel), static_cast<int>(smem));
  if (ae != cudaSuccess) return ae;
  const uint64_t items = g.chunks * (g.P / 16);
  const int grid = grid_for(kernel, threads, smem, sms, items);
  const cudaError_t le =
      launch_k(kernel, grid, threads, smem, s, cm, g, rs, static_cast<uint8_t*>(cont), offs, e, out, err);
  if (le != cudaSuccess) return le;
  ++*launches;
  g_rt_kind = DEEP ? OPTB_RT_INTERLEAVED_DEEP : BULK_ST ? OPTB_RT_INTERLEAVED : OPTB_RT_INTERLEAVED_LANE_ST;
  return cudaGetLastError();
}

bool il_lossless_enabled() {
  const char* v = getenv("OPTB_IL_LOSSLESS");
  return !(v && v[0] == '0');
}

// OPTB_RT_INTERLEAVE=0 selects the phase-ordered fused kernel for every mode
// (A/B runs; the interleaved one is the default where it applies).
bool rt_interleave_enabled() {  // read per call (probes switch it at run time)
  const char* v = getenv("OPTB_RT_INTERLEAVE");
  return !(v && v[0] == '0');
}

template <int MODE, int O, bool PTRS, bool ONE_CTA>
cudaError_t rt_vec_t(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs, const Epi& e,
                     void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  // lossless stays phase-ordered: an interleaved form (the tile's parity
  // bits as 64-byte bulk copies beside the words' TMA load) measured slower
  // for these integer-pipe-bound modes (C3 n=9: 138 -> 174 us, n=18: 148 ->
  // 164 us) and was dropped
  if constexpr (VecMode<MODE>::OFFS) {
    // lossless, P % 512 == 0: interleaved too (2-stage ring, one CTA per SM
    // with 184 registers, parity bits reloaded from L2 beside the words).
    // After the round-2 decode rewrite this beats the phase-ordered kernel
    // (C3 n=9 132.6 -> 104.9 us); OPTB_IL_LOSSLESS=0 selects the latter.
    if (rt_interleave_enabled() && il_lossless_enabled() && g.P % 512 == 0)
      return rt_il_launch<MODE, O, PTRS, true, false>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
  }
  if constexpr (!VecMode<MODE>::OFFS) {
    const uint64_t tiles = (g.chunks * (g.P / 16) + 31) / 32;
    const char* f = getenv("OPTB_IL_SHAPE");  // deep | wide: force a shape (tests, probes)
    const bool forced = f && f[0];
    // float outputs from 3 tiles per warp: per-lane container stores instead
    // of bulk stores (the epilogue's longer decode leaves the per-lane stores
    // time to drain, while a bulk store must complete before the warp
    // reloads its tile: C4 bf16 one batch per launch 32.8 -> 31.9 us, 8 per
    // launch 232 -> 229 us; tools/il_probe.py).  OPTB_IL_BULK=0|1 forces it.
    const double per_warp = static_cast<double>(tiles) / (IlShape<MODE, false>::NW * static_cast<double>(sms));
    const char* fb = getenv("OPTB_IL_BULK");
    const bool lane_st = fb && fb[0] ? fb[0] == '0' : (O != OPTB_OUT_U8 && per_warp >= 3.0);
    if (rt_interleave_enabled()) {
      if (lane_st && !(forced && f[0] == 'd'))
        return rt_il_launch<MODE, O, PTRS, ONE_CTA, false, false>(cm, g, rs, cont, offs, e, out, err, s, sms,
                                                                  launches);
      if constexpr (MODE == OPTB_EXACT128 && O == OPTB_OUT_U8) {
        // deep shape from 12 tiles per warp (il_probe: the shapes tie at ~12)
        const bool deep = forced ? f[0] == 'd' : tiles >= static_cast<uint64_t>(12 * IlShape<MODE, true>::NW) * sms;
        if (deep)
          return rt_il_launch<MODE, O, PTRS, ONE_CTA, true>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
      }
      return rt_il_launch<MODE, O, PTRS, ONE_CTA, false>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
    }
  }
  constexpr size_t smem = static_cast<size_t>(kWarps) * RtRegion<MODE>::BYTES + 1024;
  auto kernel = k_roundtrip_vec<MODE, O, PTRS, ONE_CTA>;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(kernel), static_cast<int>(smem));
  if (ae != cudaSuccess) return ae;
  const uint64_t items = g.chunks * (g.P / 16);
  const int grid = grid_for(kernel, kThreads, smem, sms, items);
  const cudaError_t le = launch_k(kernel, grid, kThreads, smem, s, cm, g, rs, static_cast<uint8_t*>(cont), offs, e,
                                  out, err);
  if (le != cudaSuccess) return le;
  ++*launches;
  g_rt_kind = OPTB_RT_PHASE_ORDERED;
  return cudaGetLastError();
}

template <int MODE, int O, bool PTRS>
cudaError_t rt_vec(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs, const Epi& e,
                   void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches) {
  if constexpr (MODE == OPTB_EXACT64) {
    if (g.per_chunk > 2) return rt_vec_t<MODE, O, PTRS, true>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
  }
  return rt_vec_t<MODE, O, PTRS, false>(cm, g, rs, cont, offs, e, out, err, s, sms, launches);
}

template <int MODE, bool PTRS>
cudaError_t rt_vec_out(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs,
                       const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, uint64_t* l) {
  switch (e.dtype) {
    case OPTB_OUT_U8: return rt_vec<MODE, OPTB_OUT_U8, PTRS>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F32: return rt_vec<MODE, OPTB_OUT_F32, PTRS>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F16: return rt_vec<MODE, OPTB_OUT_F16, PTRS>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
    default: return rt_vec<MODE, OPTB_OUT_BF16, PTRS>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
  }
}

template <int MODE>
cudaError_t rt_vec_any(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont, uint8_t* offs,
                       const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, uint64_t* l) {
  if (rs.ptrs) return rt_vec_out<MODE, true>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
  return rt_vec_out<MODE, false>(cm, g, rs, cont, offs, e, out, err, s, sms, l);
}

template <int MODE>
cudaError_t dec_generic_any(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e,
                            void* out, DevError* err, cudaStream_t s, int sms, uint64_t* l) {
  switch (e.dtype) {
    case OPTB_OUT_U8: return dec_generic<MODE, OPTB_OUT_U8>(g, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F32: return dec_generic<MODE, OPTB_OUT_F32>(g, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F16: return dec_generic<MODE, OPTB_OUT_F16>(g, cont, offs, e, out, err, s, sms, l);
    default: return dec_generic<MODE, OPTB_OUT_BF16>(g, cont, offs, e, out, err, s, sms, l);
  }
}

template <int MODE>
cudaError_t dec_vec_any(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e, void* out,
                        DevError* err, cudaStream_t s, int sms, uint64_t* l) {
  switch (e.dtype) {
    case OPTB_OUT_U8: return dec_vec<MODE, OPTB_OUT_U8>(g, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F32: return dec_vec<MODE, OPTB_OUT_F32>(g, cont, offs, e, out, err, s, sms, l);
    case OPTB_OUT_F16: return dec_vec<MODE, OPTB_OUT_F16>(g, cont, offs, e, out, err, s, sms, l);
    default: return dec_vec<MODE, OPTB_OUT_BF16>(g, cont, offs, e, out, err, s, sms, l);
  }
}

// The vector kernels need 16-pixel groups (P % 16), 16-byte aligned rows and
// planes; the lossless ones also 32-pixel aligned parity words (P % 32).
bool vec_ok(const Geom& g) {
  const bool lossless = g.mode == OPTB_LOSSLESS64 || g.mode == OPTB_LOSSLESS128;
  return lossless ? g.P % 32 == 0 : g.P % 16 == 0;
}

}  // namespace
}  // namespace optb_b200

namespace optb_b200 {
// Per-variant entry points, one translation unit each (codec_v<V>.cu).
// V = the container mode (OPTB_EXACT64 .. OPTB_LOSSLESS128), or 5 for the
// f64 variant with at most 8 images per container.  vec: the vector kernels
// apply (else the generic ones; only for V < 5).
#define OPTB_DECLARE_VARIANT(V)                                                                              \
  cudaError_t encode_v##V(const Geom& g, const RowSrc& rs, bool vec, void* cont, uint8_t* offs, cudaStream_t s, \
                          int sms, uint64_t* launches);                                                      \
  cudaError_t decode_v##V(const Geom& g, const void* cont, const uint8_t* offs, const Epi& e, bool vec,      \
                          void* out, DevError* err, cudaStream_t s, int sms, uint64_t* launches);            \
  cudaError_t roundtrip_v##V(const CUtensorMap& cm, const Geom& g, const RowSrc& rs, void* cont,            \
                             uint8_t* offs, const Epi& e, void* out, DevError* err, cudaStream_t s, int sms, \
                             uint64_t* launches);
OPTB_DECLARE_VARIANT(0)
OPTB_DECLARE_VARIANT(1)
OPTB_DECLARE_VARIANT(2)
OPTB_DECLARE_VARIANT(3)
OPTB_DECLARE_VARIANT(4)
OPTB_DECLARE_VARIANT(5)
#undef OPTB_DECLARE_VARIANT
}  // namespace optb_b200
