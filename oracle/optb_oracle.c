/*
 * optb_oracle.c -- CPU restatement of the optb image data-flow path.
 * TEST INFRASTRUCTURE ONLY (see optb_oracle.h).  Plain C11, scalar, one
 * thread.  Citations are file:line in /root/reference/proj.
 */
#include "optb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static int fail(int code, char* msg, size_t cap, const char* fmt, ...) {
  if (msg && cap) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(msg, cap, fmt, ap);
    va_end(ap);
  }
  return code;
}

/* ---------------------------------------------------------------- metadata */

uint32_t orc_capacity(int mode) { /* codec.cpp:13-27 */
  switch (mode) {
    case ORC_EXACT64: return 8;
    case ORC_EXACT128: return 16;
    case ORC_F64: return 6;
    case ORC_LOSSLESS64: return 9;
    case ORC_LOSSLESS128: return 18;
  }
  return 0;
}

uint32_t orc_accept_limit(int mode) { /* codec.hpp:36, codec.cpp:95-96 */
  return mode == ORC_F64 ? 16u : orc_capacity(mode);
}

uint32_t orc_container_value_bytes(int mode) { /* codec.cpp:51-62 */
  return (mode == ORC_EXACT128 || mode == ORC_LOSSLESS128) ? 16u : 8u;
}

int orc_has_offsets(int mode) { return mode == ORC_LOSSLESS64 || mode == ORC_LOSSLESS128; }

const char* orc_mode_name(int mode) { /* codec.cpp:31-45 */
  switch (mode) {
    case ORC_EXACT64: return "exact64";
    case ORC_EXACT128: return "exact128";
    case ORC_F64: return "f64";
    case ORC_LOSSLESS64: return "lossless64";
    case ORC_LOSSLESS128: return "lossless128";
  }
  return "?";
}

uint64_t orc_offsets_plane_bytes(uint32_t n, uint64_t pixels) { /* codec.cpp:75-77 */
  return ((uint64_t)n * pixels + 7) / 8;
}

/* codec.cpp:68-73 */
static unsigned value_bit_limit(int mode, uint32_t n) {
  unsigned per = orc_has_offsets(mode) ? 7u : 8u;
  unsigned used = per * n;
  unsigned total = orc_container_value_bytes(mode) * 8u;
  return used >= total ? 0u : used;
}

static u128 load_word(const uint8_t* plane, uint32_t wc, uint64_t p) {
  u128 v = 0;
  const uint8_t* w = plane + p * wc;
  for (int b = (int)wc - 1; b >= 0; --b) v = (v << 8) | w[b];
  return v;
}

static void store_word(uint8_t* plane, uint32_t wc, uint64_t p, u128 v) {
  uint8_t* w = plane + p * wc;
  for (uint32_t b = 0; b < wc; ++b) {
    w[b] = (uint8_t)v;
    v >>= 8;
  }
}

/* ---------------------------------------------------------------- codec */

/* codec.cpp:79-97 (the shape checks are structural in this flat layout) */
static int validate(int mode, uint32_t n, uint64_t pixels, char* msg, size_t cap) {
  if (mode < 0 || mode > 4) return fail(ORC_ERR, msg, cap, "unknown codec mode");
  if (n == 0) return fail(ORC_ERR, msg, cap, "encode: batch must contain at least one image");
  if (pixels == 0) return fail(ORC_ERR_SHAPE, msg, cap, "encode: image extents must be positive");
  uint32_t limit = orc_accept_limit(mode);
  if (n > limit)
    return fail(ORC_ERR_CAPACITY, msg, cap, "encode: %u images exceed %s capacity of %u", n,
                orc_mode_name(mode), limit);
  return ORC_OK;
}

int orc_encode(int mode, const uint8_t* images, uint32_t n, uint64_t pixels, uint8_t* plane,
               uint8_t* offsets, char* msg, size_t cap) {
  int st = validate(mode, n, pixels, msg, cap);
  if (st) return st;
  if (mode == ORC_F64) { /* codec.cpp:114-122: binary64, images ascending */
    double* acc = (double*)calloc(pixels, sizeof(double));
    for (uint32_t i = 0; i < n; ++i) {
      const double scale = ldexp(1.0, (int)(8 * i));
      const uint8_t* px = images + (uint64_t)i * pixels;
      for (uint64_t p = 0; p < pixels; ++p) acc[p] += px[p] * scale;
    }
    memcpy(plane, acc, pixels * sizeof(double));
    free(acc);
    return ORC_OK;
  }
  const uint32_t wc = orc_container_value_bytes(mode);
  memset(plane, 0, pixels * wc);
  if (orc_has_offsets(mode)) { /* codec.cpp:125-135 */
    memset(offsets, 0, orc_offsets_plane_bytes(n, pixels));
    for (uint64_t p = 0; p < pixels; ++p) {
      u128 acc = 0;
      for (uint32_t i = 0; i < n; ++i) {
        const uint8_t px = images[(uint64_t)i * pixels + p];
        acc += (u128)(px >> 1) << (7 * i);
        const uint64_t bit = (uint64_t)i * pixels + p;
        offsets[bit / 8] |= (uint8_t)((px & 1u) << (bit % 8));
      }
      store_word(plane, wc, p, acc);
    }
  } else { /* codec.cpp:136-145 */
    for (uint64_t p = 0; p < pixels; ++p) {
      u128 acc = 0;
      for (uint32_t i = 0; i < n; ++i) acc += (u128)images[(uint64_t)i * pixels + p] << (8 * i);
      store_word(plane, wc, p, acc);
    }
  }
  return ORC_OK;
}

int orc_decode(int mode, const uint8_t* plane, const uint8_t* offsets, uint32_t n,
               uint64_t pixels, uint8_t* images, char* msg, size_t cap) {
  if (mode < 0 || mode > 4) return fail(ORC_ERR, msg, cap, "unknown codec mode");
  if (n == 0 || pixels == 0) return fail(ORC_ERR_FORMAT, msg, cap, "decode: empty encoded batch");
  if (mode == ORC_F64) { /* codec.cpp:159-178 */
    const int check_range = n <= orc_capacity(mode);
    const double limit = ldexp(1.0, (int)(8 * n));
    for (uint64_t p = 0; p < pixels; ++p) {
      double acc;
      memcpy(&acc, plane + p * 8, 8);
      if (!(acc >= 0.0) || (check_range && acc >= limit))
        return fail(ORC_ERR_FORMAT, msg, cap, "decode: container value out of range for %u images",
                    n);
      for (uint32_t i = 0; i < n; ++i) {
        const double q = fmod(acc, 256.0);
        acc = (acc - q) * 0x1.0p-8;
        images[(uint64_t)i * pixels + p] = (uint8_t)q;
      }
    }
    return ORC_OK;
  }
  const uint32_t wc = orc_container_value_bytes(mode);
  const int offs = orc_has_offsets(mode);
  const unsigned bit_limit = value_bit_limit(mode, n);
  const unsigned per = offs ? 7u : 8u;
  const u128 mask = ((u128)1 << per) - 1;
  for (uint64_t p = 0; p < pixels; ++p) { /* codec.cpp:189-207 */
    u128 acc = load_word(plane, wc, p);
    if (bit_limit != 0 && (acc >> bit_limit) != 0)
      return fail(ORC_ERR_FORMAT, msg, cap,
                  "decode: container value exceeds range of %u packed images", n);
    for (uint32_t i = 0; i < n; ++i) {
      const uint8_t q = (uint8_t)(acc & mask);
      acc >>= per;
      if (offs) {
        const uint64_t bit = (uint64_t)i * pixels + p;
        const uint8_t parity = (offsets[bit / 8] >> (bit % 8)) & 1u;
        images[(uint64_t)i * pixels + p] = (uint8_t)((q << 1) | parity);
      } else {
        images[(uint64_t)i * pixels + p] = q;
      }
    }
  }
  return ORC_OK;
}

int orc_roundtrip_error(int mode, const uint8_t* images, uint32_t n, uint64_t pixels,
                        int32_t* errs, char* msg, size_t cap) {
  int st = validate(mode, n, pixels, msg, cap);
  if (st) return st;
  uint8_t* plane = (uint8_t*)malloc(pixels * 16);
  uint8_t* offs = (uint8_t*)malloc(orc_offsets_plane_bytes(n, pixels) + 1);
  uint8_t* back = (uint8_t*)malloc((uint64_t)n * pixels);
  st = orc_encode(mode, images, n, pixels, plane, offs, msg, cap);
  if (!st) st = orc_decode(mode, plane, offs, n, pixels, back, msg, cap);
  if (!st) {
    for (uint32_t i = 0; i < n; ++i) { /* codec.cpp:210-224 */
      int worst = 0;
      for (uint64_t p = 0; p < pixels; ++p) {
        int d = abs((int)images[(uint64_t)i * pixels + p] - (int)back[(uint64_t)i * pixels + p]);
        if (d > worst) worst = d;
      }
      errs[i] = worst;
    }
  }
  free(plane);
  free(offs);
  free(back);
  return st;
}

/* ---------------------------------------------------------------- streams */

uint64_t orc_stream_chunks(uint64_t batch, uint64_t n_batches, uint32_t per_chunk) {
  return n_batches * ((batch + per_chunk - 1) / per_chunk);
}

int orc_encode_stream(int mode, uint32_t per_chunk, uint64_t pixels, uint64_t batch,
                      uint64_t n_batches, const uint8_t* dataset, uint64_t row_stride,
                      const int64_t* row_index, uint8_t* containers, uint8_t* offsets,
                      uint64_t offsets_stride, char* msg, size_t cap) {
  const uint64_t cpb = (batch + per_chunk - 1) / per_chunk;
  const uint32_t wc = orc_container_value_bytes(mode);
  uint8_t* gathered = (uint8_t*)malloc((uint64_t)per_chunk * pixels);
  int st = ORC_OK;
  for (uint64_t b = 0; b < n_batches && !st; ++b) {
    for (uint64_t j = 0; j < cpb && !st; ++j) {
      const uint64_t base = j * per_chunk;
      const uint32_t n = (uint32_t)((batch - base) < per_chunk ? (batch - base) : per_chunk);
      for (uint32_t i = 0; i < n; ++i) { /* dataset.cpp:16-22 image_of */
        const uint64_t r = b * batch + base + i;
        const uint64_t src = row_index ? (uint64_t)row_index[r] : r;
        memcpy(gathered + (uint64_t)i * pixels, dataset + src * row_stride, pixels);
      }
      const uint64_t k = b * cpb + j;
      st = orc_encode(mode, gathered, n, pixels, containers + k * pixels * wc,
                      offsets ? offsets + k * offsets_stride : NULL, msg, cap);
    }
  }
  free(gathered);
  return st;
}

uint16_t orc_float_to_half(float value) { /* tensor.cpp:12-51 */
  uint32_t bits;
  memcpy(&bits, &value, 4);
  const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  const uint32_t exp8 = (bits >> 23) & 0xffu;
  const uint32_t frac = bits & 0x7fffffu;
  if (exp8 == 0xffu) return frac ? (uint16_t)(sign | 0x7e00u) : (uint16_t)(sign | 0x7c00u);
  if (exp8 == 0) return sign;
  const int unbiased = (int)exp8 - 127;
  if (unbiased >= 16) return (uint16_t)(sign | 0x7c00u);
  const uint32_t sig = frac | 0x800000u;
  if (unbiased >= -14) {
    uint32_t rounded = (sig + 0xfffu + ((sig >> 13) & 1u)) >> 13;
    int he = unbiased + 15;
    if (rounded & 0x800u) {
      rounded >>= 1;
      ++he;
    }
    if (he >= 31) return (uint16_t)(sign | 0x7c00u);
    return (uint16_t)(sign | (uint32_t)(he << 10) | (rounded & 0x3ffu));
  }
  const int shift = -unbiased - 1;
  if (shift >= 25) return sign;
  const uint64_t halfway = (uint64_t)1 << (shift - 1);
  const uint64_t rounded = ((uint64_t)sig + halfway - 1 + ((sig >> shift) & 1u)) >> shift;
  return (uint16_t)(sign | rounded);
}

uint16_t orc_float_to_bf16(float value) {
  uint32_t bits;
  memcpy(&bits, &value, 4);
  return (uint16_t)((bits + 0x7fffu + ((bits >> 16) & 1u)) >> 16);
}

int orc_decode_stream(int mode, uint32_t per_chunk, uint64_t pixels, uint64_t batch,
                      uint64_t n_batches, const uint8_t* containers, const uint8_t* offsets,
                      uint64_t offsets_stride, int out_dtype, float scale,
                      const float* class_scale, const float* class_bias,
                      const int32_t* row_class, void* out, uint64_t out_row_stride, char* msg,
                      size_t cap) {
  const uint64_t cpb = (batch + per_chunk - 1) / per_chunk;
  const uint32_t wc = orc_container_value_bytes(mode);
  if (out_row_stride == 0) out_row_stride = pixels;
  uint8_t* imgs = (uint8_t*)malloc((uint64_t)per_chunk * pixels);
  int st = ORC_OK;
  for (uint64_t b = 0; b < n_batches && !st; ++b) {
    for (uint64_t j = 0; j < cpb && !st; ++j) {
      const uint64_t base = j * per_chunk;
      const uint32_t n = (uint32_t)((batch - base) < per_chunk ? (batch - base) : per_chunk);
      const uint64_t k = b * cpb + j;
      st = orc_decode(mode, containers + k * pixels * wc,
                      offsets ? offsets + k * offsets_stride : NULL, n, pixels, imgs, msg, cap);
      if (st) break;
      for (uint32_t i = 0; i < n; ++i) { /* nn.cpp:177-191 */
        const uint64_t row = b * batch + base + i;
        float s = scale, bias = 0.0f;
        int affine = 0;
        if (class_scale && row_class) {
          s = class_scale[row_class[row]];
          bias = class_bias ? class_bias[row_class[row]] : 0.0f;
          affine = class_bias != NULL;
        }
        for (uint64_t p = 0; p < pixels; ++p) {
          const uint8_t q = imgs[(uint64_t)i * pixels + p];
          const uint64_t o = row * out_row_stride + p;
          if (out_dtype == ORC_U8) {
            ((uint8_t*)out)[o] = q;
            continue;
          }
          volatile float v = (float)q * s; /* one binary32 RN multiply, nn.cpp:186 */
          float y = v;
          if (affine) y = y + bias;
          if (out_dtype == ORC_F32)
            ((float*)out)[o] = y;
          else if (out_dtype == ORC_F16)
            ((uint16_t*)out)[o] = orc_float_to_half(y);
          else
            ((uint16_t*)out)[o] = orc_float_to_bf16(y);
        }
      }
    }
  }
  free(imgs);
  return st;
}

/* ---------------------------------------------------------------- rng */

uint64_t orc_mix(uint64_t z) { /* rng.hpp:17-20 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t orc_next_u64(uint64_t* state) { /* rng.hpp:16-21 */
  *state += 0x9e3779b97f4a7c15ull;
  return orc_mix(*state);
}

uint64_t orc_next_below(uint64_t* state, uint64_t n) { /* rng.hpp:29-35 */
  if (n <= 1) return 0;
  const uint64_t limit = ~(uint64_t)0 - (~(uint64_t)0 % n + 1) % n;
  uint64_t x = orc_next_u64(state);
  while (x > limit) x = orc_next_u64(state);
  return x % n;
}

/* ---------------------------------------------------------------- sampler */

int orc_sbs_plan(const double* w, uint64_t C, uint64_t B, uint64_t* counts, char* msg,
                 size_t cap) { /* sampler.cpp:11-51 */
  if (C == 0) return fail(ORC_ERR, msg, cap, "sampler: at least one class weight required");
  if (B == 0) return fail(ORC_ERR, msg, cap, "sampler: batch size must be positive");
  double sum = 0.0;
  for (uint64_t c = 0; c < C; ++c) {
    if (w[c] < 0.0) return fail(ORC_ERR, msg, cap, "sampler: negative weight for class %llu",
                                (unsigned long long)c);
    sum += w[c];
  }
  if (fabs(sum - 1.0) > 1e-9)
    return fail(ORC_ERR, msg, cap, "sampler: class weights sum to %f, expected 1", sum);
  double* rem = (double*)malloc(C * sizeof(double));
  uint64_t* order = (uint64_t*)malloc(C * sizeof(uint64_t));
  uint64_t assigned = 0;
  for (uint64_t c = 0; c < C; ++c) {
    const double exact = w[c] * (double)B;
    counts[c] = (uint64_t)floor(exact);
    rem[c] = exact - floor(exact);
    assigned += counts[c];
    order[c] = c;
  }
  /* stable sort by remainder, descending (insertion sort is stable) */
  for (uint64_t i = 1; i < C; ++i) {
    uint64_t v = order[i];
    uint64_t j = i;
    while (j > 0 && rem[order[j - 1]] < rem[v]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = v;
  }
  for (uint64_t k = 0; assigned < B; ++k) {
    counts[order[k % C]] += 1;
    ++assigned;
  }
  free(rem);
  free(order);
  return ORC_OK;
}

int orc_class_index(const int32_t* labels, uint64_t n, uint64_t C, uint64_t* off,
                    int64_t* members, char* msg, size_t cap) { /* sampler.cpp:53-65 */
  uint64_t* fill = (uint64_t*)calloc(C + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    const int32_t l = labels[i];
    if (l < 0 || (uint64_t)l >= C) {
      free(fill);
      return fail(ORC_ERR, msg, cap, "sampler: label %d outside %llu classes", l,
                  (unsigned long long)C);
    }
    fill[l + 1]++;
  }
  off[0] = 0;
  for (uint64_t c = 0; c < C; ++c) off[c + 1] = off[c] + fill[c + 1];
  for (uint64_t c = 0; c < C; ++c) fill[c] = off[c];
  for (uint64_t i = 0; i < n; ++i) members[fill[labels[i]]++] = (int64_t)i;
  free(fill);
  return ORC_OK;
}

struct orc_cursor {
  uint64_t C, B;
  uint64_t* counts;
  uint64_t* off;    /* C+1 */
  int64_t* order;   /* concatenated per-class orders */
  uint64_t* pos;
  uint64_t rng_state;
};

static void reshuffle(orc_cursor* cur, uint64_t c) { /* sampler.cpp:84-89, rng.hpp:57-64 */
  uint64_t st = cur->rng_state;
  int64_t* a = cur->order + cur->off[c];
  const uint64_t m = cur->off[c + 1] - cur->off[c];
  for (uint64_t i = m; i > 1; --i) {
    const uint64_t j = orc_next_below(&st, i);
    int64_t t = a[i - 1];
    a[i - 1] = a[j];
    a[j] = t;
  }
  cur->rng_state = orc_next_u64(&st);
  cur->pos[c] = 0;
}

orc_cursor* orc_cursor_create(const uint64_t* counts, uint64_t C, uint64_t B, uint64_t seed,
                              const uint64_t* off, const int64_t* members, int* status,
                              char* msg, size_t cap) { /* sampler.cpp:67-82 */
  *status = ORC_OK;
  for (uint64_t c = 0; c < C; ++c) {
    if (counts[c] > 0 && off[c + 1] == off[c]) {
      *status = fail(ORC_ERR, msg, cap,
                     "sampler: class %llu has no examples but a positive batch count",
                     (unsigned long long)c);
      return NULL;
    }
  }
  orc_cursor* cur = (orc_cursor*)calloc(1, sizeof(orc_cursor));
  cur->C = C;
  cur->B = B;
  cur->counts = (uint64_t*)malloc(C * sizeof(uint64_t));
  memcpy(cur->counts, counts, C * sizeof(uint64_t));
  cur->off = (uint64_t*)malloc((C + 1) * sizeof(uint64_t));
  memcpy(cur->off, off, (C + 1) * sizeof(uint64_t));
  cur->order = (int64_t*)malloc((off[C] + 1) * sizeof(int64_t));
  memcpy(cur->order, members, off[C] * sizeof(int64_t));
  cur->pos = (uint64_t*)calloc(C, sizeof(uint64_t));
  cur->rng_state = seed;
  for (uint64_t c = 0; c < C; ++c) reshuffle(cur, c);
  return cur;
}

void orc_cursor_next(orc_cursor* cur, uint64_t n_batches, int64_t* examples, int32_t* classes) {
  uint64_t r = 0;
  for (uint64_t b = 0; b < n_batches; ++b) { /* sampler.cpp:91-104 */
    for (uint64_t c = 0; c < cur->C; ++c) {
      const uint64_t m = cur->off[c + 1] - cur->off[c];
      for (uint64_t k = 0; k < cur->counts[c]; ++k) {
        if (cur->pos[c] == m) reshuffle(cur, c);
        examples[r] = cur->order[cur->off[c] + cur->pos[c]++];
        if (classes) classes[r] = (int32_t)c;
        ++r;
      }
    }
  }
}

uint64_t orc_cursor_rng_state(const orc_cursor* cur) { return cur->rng_state; }

void orc_cursor_destroy(orc_cursor* cur) {
  if (!cur) return;
  free(cur->counts);
  free(cur->off);
  free(cur->order);
  free(cur->pos);
  free(cur);
}

/* ---------------------------------------------------------------- misc */

void orc_synth_pixels(uint64_t seed, uint64_t first_row, uint64_t n_rows, uint64_t pixels,
                      uint8_t* out) {
  const uint64_t words = (pixels + 7) / 8;
  for (uint64_t r = 0; r < n_rows; ++r) {
    const uint64_t e = first_row + r;
    for (uint64_t q = 0; q < words; ++q) {
      const uint64_t w = orc_mix(seed + (e * words + q + 1) * 0x9e3779b97f4a7c15ull);
      for (uint64_t b = 0; b < 8 && q * 8 + b < pixels; ++b)
        out[r * pixels + q * 8 + b] = (uint8_t)(w >> (8 * b));
    }
  }
}

uint64_t orc_fnv1a64(const void* data, size_t n) {
  const uint8_t* p = (const uint8_t*)data;
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
