/*
 * optb_oracle.h -- CPU restatement of the OpTorch (optb) image data-flow path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2105_00619_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never
 * links, calls or falls back to it.
 *
 * Every function restates a reference function, cited as file:line relative
 * to /root/reference/proj.  Parity of this restatement is pinned against
 *   (1) the reference's own golden vectors (tests/test_codec.cpp,
 *       tests/test_sampler.cpp, tests/test_tensor.cpp), and
 *   (2) fixtures produced by the reference itself compiled from its sources
 *       (oracle/_ref, see oracle/Makefile and tests/golden/make_golden.py).
 *
 * Memory layouts are the device layouts of the new framework:
 *   container plane  [P][Wc] bytes, one little-endian Wc-byte word per pixel
 *                    (Wc = 8 for exact64/lossless64/f64, 16 otherwise);
 *                    f64 words are IEEE binary64 bit patterns;
 *   offsets plane    ceil(n*P/8) bytes, bit (i*P + p) LSB-first
 *                    (codec.cpp:101-104, 128-134);
 *   images           [n][P] u8, row-major HWC per image (codec.hpp:56-62).
 */
#ifndef OPTB_ORACLE_H
#define OPTB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR = 1, ORC_ERR_SHAPE = 2, ORC_ERR_CAPACITY = 3, ORC_ERR_FORMAT = 4 };
enum { ORC_EXACT64 = 0, ORC_EXACT128 = 1, ORC_F64 = 2, ORC_LOSSLESS64 = 3, ORC_LOSSLESS128 = 4 };
enum { ORC_U8 = 0, ORC_F32 = 1, ORC_F16 = 2, ORC_BF16 = 3 };

/* mode metadata -- codec.cpp:13-62 */
uint32_t orc_capacity(int mode);
uint32_t orc_accept_limit(int mode);
uint32_t orc_container_value_bytes(int mode);
int orc_has_offsets(int mode);
const char* orc_mode_name(int mode);
uint64_t orc_offsets_plane_bytes(uint32_t n, uint64_t pixels);

/* one chunk -- codec.cpp:79-146 (encode), 148-208 (decode) */
int orc_encode(int mode, const uint8_t* images, uint32_t n, uint64_t pixels,
               uint8_t* plane, uint8_t* offsets, char* msg, size_t msg_cap);
int orc_decode(int mode, const uint8_t* plane, const uint8_t* offsets, uint32_t n,
               uint64_t pixels, uint8_t* images, char* msg, size_t msg_cap);
/* codec.cpp:210-224 */
int orc_roundtrip_error(int mode, const uint8_t* images, uint32_t n, uint64_t pixels,
                        int32_t* errs, char* msg, size_t msg_cap);

/* Batch stream: n_batches batches of B rows; batch b is split into
 * consecutive chunks of per_chunk rows (runner.cpp:77-90).  Row r of the
 * stream reads dataset row row_index[r] (or r when row_index is NULL) --
 * dataset.cpp:16-22 + runner.cpp:278-290.  Chunk k's plane is at
 * containers + k*P*Wc, its offsets at offsets + k*offsets_stride. */
uint64_t orc_stream_chunks(uint64_t batch, uint64_t n_batches, uint32_t per_chunk);
int orc_encode_stream(int mode, uint32_t per_chunk, uint64_t pixels, uint64_t batch,
                      uint64_t n_batches, const uint8_t* dataset, uint64_t row_stride,
                      const int64_t* row_index, uint8_t* containers, uint8_t* offsets,
                      uint64_t offsets_stride, char* msg, size_t msg_cap);
/* nn.cpp:153-192 (decode_input) + nn.cpp:141-146/235 (fp16 tape store).
 * out_dtype U8 gives codec::decode's pixels; F32 gives float(q)*scale
 * (nn.cpp:186); F16 gives float_to_half of that (tensor.cpp:12-51); BF16
 * gives the RNE bf16 of that (no reference counterpart).
 * Optional per-class epilogue: y = RN(RN(q*class_scale[c]) + class_bias[c])
 * with c = row_class[row]; NULL tables mean scale/0. */
int orc_decode_stream(int mode, uint32_t per_chunk, uint64_t pixels, uint64_t batch,
                      uint64_t n_batches, const uint8_t* containers, const uint8_t* offsets,
                      uint64_t offsets_stride, int out_dtype, float scale,
                      const float* class_scale, const float* class_bias,
                      const int32_t* row_class, void* out, uint64_t out_row_stride,
                      char* msg, size_t msg_cap);

uint16_t orc_float_to_half(float value);  /* tensor.cpp:12-51 */
uint16_t orc_float_to_bf16(float value);  /* RNE, finite inputs */

/* SplitMix64 -- rng.hpp:16-35 */
uint64_t orc_mix(uint64_t z);
uint64_t orc_next_u64(uint64_t* state);
uint64_t orc_next_below(uint64_t* state, uint64_t n);

/* SBS -- sampler.cpp:11-104 */
int orc_sbs_plan(const double* weights, uint64_t n_classes, uint64_t batch, uint64_t* counts,
                 char* msg, size_t msg_cap);
int orc_class_index(const int32_t* labels, uint64_t n, uint64_t n_classes,
                    uint64_t* class_offsets, int64_t* members, char* msg, size_t msg_cap);
typedef struct orc_cursor orc_cursor;
orc_cursor* orc_cursor_create(const uint64_t* counts, uint64_t n_classes, uint64_t batch,
                              uint64_t seed, const uint64_t* class_offsets,
                              const int64_t* members, int* status, char* msg, size_t msg_cap);
void orc_cursor_next(orc_cursor* cur, uint64_t n_batches, int64_t* examples, int32_t* classes);
uint64_t orc_cursor_rng_state(const orc_cursor* cur);
void orc_cursor_destroy(orc_cursor* cur);

/* Synthetic counter-based pixels:
 * w = mix(seed + (e*ceil(P/8) + p/8 + 1)*gamma), pixel = (w >> 8*(p%8)) & 0xff */
void orc_synth_pixels(uint64_t seed, uint64_t first_row, uint64_t n_rows, uint64_t pixels,
                      uint8_t* out);

/* FNV-1a-64 (SURVEY §8(a)/(c) probe goldens) */
uint64_t orc_fnv1a64(const void* data, size_t n);

#ifdef __cplusplus
}
#endif
#endif
