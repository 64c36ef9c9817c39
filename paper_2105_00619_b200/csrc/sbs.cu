// sbs.cu -- selective batch sampling on sm_100a.
//
// Reference semantics (file:line under /root/reference/proj):
//   ClassIndex::from_labels   sampler.cpp:53-65   (K7 below)
//   BatchCursor ctor/reshuffle sampler.cpp:67-89, Rng rng.hpp:16-64 (K8, K9)
//   BatchCursor::next         sampler.cpp:91-104  (K10)
//
// The reference stream is one sequential SplitMix64 chain threaded through
// every reshuffle.  SplitMix64 is counter based (draw k from state s is
// mix(s + k*gamma)), so a reshuffle of a class of m examples started at chain
// state s consumes K = m-1 draws plus any rejections of next_below and leaves
// the chain at mix(s + (K+1)*gamma) (rng.hpp:16-21, sampler.cpp:84-89).  The
// chain therefore depends only on the event sequence (class sizes) and on
// rejections, never on permutation contents:
//   K9   k_shuffle, one CTA per reshuffling class: walks the event list
//        assuming no rejection (one mix per event) to find its events' start
//        states, then applies its Fisher-Yates passes in generation order in
//        shared memory -- lanes compute every draw, check it for rejection
//        and turn it into a swap target, one lane swaps;
//   K8   k_chain_finish: advances the chain; on any rejection (probability
//        <= m/2^64 per draw) or when forced (optb_sbs_set_force_serial) it
//        redoes the whole call exactly, serially -- correct, never hot;
//   K10  k_gather: the class-major draws of any subset of batches (sharding).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"

namespace optb_b200 {
namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// next_below's acceptance bound (rng.hpp:31): x is rejected iff x > limit.
__device__ __forceinline__ uint64_t below_limit(uint64_t n) {
  const uint64_t all = ~0ull;
  return all - (all % n + 1) % n;
}

// Rejection is possible only when x >= 2^64 - (2^64 mod n); for n <= 2^32
// that needs the top 32 bits set, so the 64-bit modulus is rarely evaluated.
__device__ __forceinline__ bool rejected(uint64_t x, uint64_t n) {
  if (n <= (1ull << 32) && (x >> 32) != 0xffffffffull) return false;
  return x > below_limit(n);
}

// x % i (next_below's reduction, rng.hpp:29-35) for 2 <= i < 2^32: with
// M = floor((2^64-1)/i), q = mulhi(x, M) is floor(x/i) or one less, so the
// remainder needs one conditional subtraction (exhaustively edge-checked
// against %; the sampler's parity tests cover it on the device).
__device__ __forceinline__ uint32_t mod_below(uint64_t x, uint32_t i, const uint64_t* __restrict__ recip) {
  if (!recip) return static_cast<uint32_t>(x % i);
  const uint64_t q = __umul64hi(x, __ldg(recip + i));
  uint64_t r = x - q * i;
  if (r >= i) r -= i;
  return static_cast<uint32_t>(r);
}

__global__ void k_recip(uint64_t* __restrict__ t, uint32_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    t[i] = i >= 2 ? ~0ull / i : 0ull;
}

// ------------------------------------------------------------------ K7
// Stable partition of [0,n) by label.  One warp per tile of kTile labels.
constexpr int kTile = 1024;

__global__ void k_ci_hist(const int32_t* __restrict__ labels, uint64_t n, uint32_t C,
                          uint32_t tiles, uint32_t* __restrict__ hist, DevError* err) {
  extern __shared__ uint32_t h[];
  const uint32_t tile = blockIdx.x;
  for (uint32_t c = threadIdx.x; c < C; c += 32) h[c] = 0;
  __syncwarp();
  const uint64_t begin = static_cast<uint64_t>(tile) * kTile;
  for (uint32_t o = threadIdx.x; o < kTile; o += 32) {
    const uint64_t i = begin + o;
    if (i >= n) break;
    const int32_t l = __ldg(labels + i);
    if (l < 0 || static_cast<uint32_t>(l) >= C) {
      atomicCAS(&err->kind, 0u, kErrLabel);
      atomicMin(&err->key, static_cast<unsigned long long>(i));
      continue;
    }
    atomicAdd(&h[l], 1u);
  }
  __syncwarp();
  for (uint32_t c = threadIdx.x; c < C; c += 32) hist[static_cast<uint64_t>(c) * tiles + tile] = h[c];
}

// Exclusive scan of hist (class-major, tile-minor) in place; class_offsets[c]
// = scan at (c, 0); class_offsets[C] = total.  Single CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_ci_scan(uint32_t* __restrict__ hist, uint64_t total,
                                                  uint32_t C, uint32_t tiles,
                                                  uint64_t* __restrict__ class_offsets) {
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < total; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < total ? hist[i] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive
    }
    __syncthreads();
    const uint64_t excl = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
    if (i < total) {
      hist[i] = static_cast<uint32_t>(excl);
      if (i % tiles == 0) class_offsets[i / tiles] = excl;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) class_offsets[C] = carry;
}

__global__ void k_ci_scatter(const int32_t* __restrict__ labels, uint64_t n, uint32_t C,
                             uint32_t tiles, const uint32_t* __restrict__ offs,
                             int64_t* __restrict__ members) {
  extern __shared__ uint32_t run[];  // running position per class for this tile
  const uint32_t tile = blockIdx.x;
  const int lane = threadIdx.x;
  for (uint32_t c = lane; c < C; c += 32) run[c] = offs[static_cast<uint64_t>(c) * tiles + tile];
  __syncwarp();
  const uint64_t begin = static_cast<uint64_t>(tile) * kTile;
  for (uint32_t o = 0; o < kTile; o += 32) {
    const uint64_t i = begin + o + lane;
    const bool in = i < n;
    int32_t l = in ? __ldg(labels + i) : -1;
    const bool ok = in && l >= 0 && static_cast<uint32_t>(l) < C;
    if (!ok) l = -1 - lane;  // unique, never matches a real class
    const uint32_t peers = __match_any_sync(0xffffffffu, l);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    uint32_t pos = 0;
    if (ok) pos = run[l] + rank;
    __syncwarp();
    if (ok) {
      members[pos] = static_cast<int64_t>(i);
      if (31 - __clz(peers) == lane) run[l] = pos + 1;  // highest peer advances the run
    }
    __syncwarp();
    if (__all_sync(0xffffffffu, !in)) break;
  }
}

__global__ void k_ci_label_value(const int32_t* labels, uint64_t C, DevError* err) {
  if (err->kind == kErrLabel) {
    err->label = labels[err->key];
    err->aux = C;
  }
}

// ------------------------------------------------------------------ K9
// One CTA per class that reshuffles in this call (m >= 2).  The start state
// of every event comes from the host's walk of the chain (ChainArgs::seeds,
// valid when the device chain equals expect_start -- checked first); then,
// per event in generation order, the lanes compute every draw
// x_k = mix(s + k*gamma), check it against
// next_below's bound (rng.hpp:29-35) and turn it into the swap target
// j = x mod i; thread 0 applies the swaps in shared memory.  A rejected draw
// sets calls->flag and the class stops; k_chain_finish then redoes the whole
// call exactly (serially).  The permutation lives in shared memory as u32 when
// it fits (host guarantees ids < 2^32 then), else in the generation pool.
constexpr int kJWin = 2048;

__global__ void __launch_bounds__(64) k_shuffle(ChainArgs a, int use_smem) {
  extern __shared__ uint32_t sh[];
  uint32_t* js = sh;            // kJWin swap targets
  uint32_t* perm = sh + kJWin;  // m entries (smem path)
  const uint32_t b = a.cls_begin[blockIdx.x], end = a.cls_begin[blockIdx.x + 1];
  const SbsEvent first = a.ev[a.cls_list[b]];
  const uint32_t m = first.m;
  const uint64_t copy_to = a.cls_copy[blockIdx.x];
  if (use_smem) {
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) {
      const int64_t v = a.pool[first.src + x];
      perm[x] = static_cast<uint32_t>(v);
      a.pool[copy_to + x] = v;
    }
  } else {
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) a.pool[copy_to + x] = a.pool[first.src + x];
  }
  __syncthreads();
  // the host's seeds hold only if the device chain is where the host assumed;
  // otherwise k_chain_finish redoes the call from the pre-call copies above
  if (*a.chain != a.expect_start) {
    if (threadIdx.x == 0) atomicExch(a.flag, 1u);
    return;
  }
  uint64_t cur_src = copy_to;
  for (uint32_t q = b; q < end; ++q) {
    const uint32_t e = a.cls_list[q];
    const SbsEvent E = a.ev[e];
    const uint64_t s = a.seeds[e];
    int64_t* gperm = a.pool + E.slot;
    if (!use_smem) {
      for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) gperm[x] = a.pool[cur_src + x];
      __syncthreads();
    }
    // step i = m..2 uses draw k = m - i + 1 when nothing is rejected
    for (uint32_t w0 = m; w0 > 1; w0 = (w0 > kJWin + 1) ? w0 - kJWin : 1) {
      const uint32_t cnt = (w0 - 1 < kJWin) ? w0 - 1 : kJWin;  // steps i = w0 .. w0-cnt+1
      bool rej = false;
      for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
        const uint32_t i = w0 - t;
        const uint64_t k = static_cast<uint64_t>(m) - i + 1;
        const uint64_t x = mix64(s + k * kGamma);
        rej |= rejected(x, i);
        js[t] = static_cast<uint32_t>(x % i);
      }
      if (__syncthreads_or(rej)) {
        if (threadIdx.x == 0) atomicExch(a.flag, 1u);
        return;  // k_chain_finish recomputes this call serially
      }
      if (threadIdx.x == 0) {
        if (use_smem) {
#pragma unroll 4
          for (uint32_t t = 0; t < cnt; ++t) {
            const uint32_t i = w0 - t, j = js[t];
            const uint32_t v = perm[j];
            perm[j] = perm[i - 1];
            perm[i - 1] = v;
          }
        } else {
          for (uint32_t t = 0; t < cnt; ++t) {
            const uint32_t i = w0 - t, j = js[t];
            const int64_t v = gperm[j];
            gperm[j] = gperm[i - 1];
            gperm[i - 1] = v;
          }
        }
      }
      __syncthreads();
    }
    if (use_smem)
      for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) gperm[x] = perm[x];
    cur_src = E.slot;
    __syncthreads();
  }
  const uint64_t final_to = a.cls_final[blockIdx.x];
  if (use_smem)
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) a.pool[final_to + x] = perm[x];
  else
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) a.pool[final_to + x] = a.pool[cur_src + x];
}

// ------------------------------------------------------------------ K9 (parallel)
// Fisher-Yates with known swap targets, evaluated for all output positions at
// once.  Let A_k be the array after steps m..k (step i swaps [i-1] and [j_i],
// rng.hpp:57-64; A_{m+1} = input).  For x < k-1, A_k[x] is A_{k+1}[k-1] if
// j_k == x and A_{k+1}[x] otherwise, so
//   A_k[x] = input[x]                       if no step s >= k has j_s == x,
//          = A_{s+1}[s-1]  (s = the smallest such step)   otherwise,
// and the output is out[p] = A_{p+2}[j_{p+1}] for p >= 1, out[0] = A_2[0].
// Each position follows its own short chain through the steps bucketed by
// j, so the pass is one histogram + scan + scatter + chain-follow in shared
// memory -- no serial swap loop (tests/test_chain_model.py and the GPU parity
// tests pin it against the reference sequence).
constexpr int kParThreads = 256;
// Threads per CTA of K9a / K9b when a call carries many generations per
// class (a rank drawing the stream of N ranks): each CTA's chain of
// dependent shared-memory passes is latency bound, so 4x the threads cut
// the per-CTA time, and these CTAs only run in the gaps the persistent codec
// kernel leaves.
constexpr int kParThreadsWide = 1024;
constexpr uint32_t kParMaxM = 11776;  // <= 65535: K9a's indices are 16-bit

// K9a's shared memory: four u16 arrays (js, off, bk, cnt) of m + 1 entries,
// each rounded to an even count so every array is 4-byte aligned for the
// packed 16-bit-pair atomics -- 8 bytes per element, so two 1024-thread CTAs
// fit per SM at C5's class size (m ~ 10 486; 14 bytes per element and one
// CTA per SM with 32-bit indices)
__host__ __device__ inline uint32_t even_up(uint32_t n) { return (n + 1u) & ~1u; }
size_t par_smem_bytes(uint32_t m) { return 2ull * 4ull * even_up(m + 1); }

// ++a[x] on a u16 array through the packed u32 word holding it; returns the
// old value (every entry stays below 2^16, so no carry crosses the halves)
__device__ __forceinline__ uint32_t inc_u16(uint16_t* a, uint32_t x) {
  const uint32_t sh = 16u * (x & 1u);
  const uint32_t old = atomicAdd(reinterpret_cast<uint32_t*>(a) + (x >> 1), 1u << sh);
  return (old >> sh) & 0xffffu;
}

template <int T>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < T / 32 ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < T / 32) warp_tot[lane] = w;
  }
  __syncthreads();
  const uint32_t before = warp ? warp_tot[warp - 1] : 0u;
  __syncthreads();
  return before + x - v;
}

// ------------------------------------------------------------------ K9a / K9b
// The generations of a class in one call are a chain perm_j = FY_j(perm_j-1),
// but FY's swap targets depend only on the draws, so FY_j(A)[p] = A[pi_j[p]]
// with pi_j = FY_j(identity).  K9a computes every pi_j of the call at once --
// one CTA per reshuffle event, the parallel Fisher-Yates above on the
// identity -- and K9b composes them per class, perm_j[p] = perm_j-1[pi_j[p]],
// a shared-memory gather per generation.  The call's critical path is one
// parallel Fisher-Yates plus one gather per generation, instead of one
// Fisher-Yates per generation: it stays flat when a rank draws the batches
// of all N ranks per step (N-GPU runs).
template <int T>
__global__ void __launch_bounds__(T) k_fy_gen(ChainArgs a) {
  extern __shared__ uint32_t sh[];
  __shared__ uint32_t warp_tot[T / 32];
  if (*a.chain != a.expect_start) return;  // stale host seeds: K9b flags, K8 redoes serially
  const uint32_t e = a.cls_list[blockIdx.x];
  const SbsEvent E = a.ev[e];
  const uint32_t m = E.m;
  const uint32_t span = even_up(m + 1);
  uint16_t* js = reinterpret_cast<uint16_t*>(sh);  // [m + 1]  swap target of step i (i = 2..m)
  uint16_t* off = js + span;                       // [m + 1]  bucket starts, then ends
  uint16_t* bk = off + span;                       // [m]      steps bucketed by target
  uint16_t* cnt = bk + span;                       // [m]      bucket sizes
  const uint64_t s = a.seeds[e];
  const uint32_t per = (m + T - 1) / T;
  const uint32_t lo = min(m, threadIdx.x * per), hi = min(m, lo + per);
  bool rej = false;
  for (uint32_t x = threadIdx.x; x < span / 2; x += blockDim.x) reinterpret_cast<uint32_t*>(cnt)[x] = 0u;
  __syncthreads();
  for (uint32_t i = 2 + threadIdx.x; i <= m; i += blockDim.x) {
    const uint64_t x = mix64(s + (static_cast<uint64_t>(m) - i + 1) * kGamma);
    rej |= rejected(x, i);
    const uint32_t j = mod_below(x, i, a.recip);
    js[i] = static_cast<uint16_t>(j);
    inc_u16(cnt, j);
  }
  if (__syncthreads_or(rej)) {
    if (threadIdx.x == 0) atomicExch(a.flag, 1u);
    return;  // k_chain_finish redoes this call serially
  }
  uint32_t local = 0;
  for (uint32_t x = lo; x < hi; ++x) local += cnt[x];
  uint32_t run = block_exclusive_scan<T>(local, warp_tot);
  for (uint32_t x = lo; x < hi; ++x) {
    off[x] = static_cast<uint16_t>(run);
    run += cnt[x];
  }
  __syncthreads();
  for (uint32_t i = 2 + threadIdx.x; i <= m; i += blockDim.x) bk[inc_u16(off, js[i])] = static_cast<uint16_t>(i);
  __syncthreads();  // off[x] now holds the end of bucket x
  int64_t* gout = a.pool + E.slot;
  for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
    uint32_t x = p >= 1 ? js[p + 1] : 0u;
    uint32_t k = p >= 1 ? p + 2 : 2u;
    for (;;) {
      const uint32_t hi_b = off[x], lo_b = hi_b - cnt[x];
      uint32_t best = 0xffffffffu;
      for (uint32_t t = lo_b; t < hi_b; ++t) {
        const uint32_t st = bk[t];
        if (st >= k && st < best) best = st;
      }
      if (best == 0xffffffffu) break;
      x = best - 1;
      k = best + 1;
    }
    gout[p] = x;  // pi[p]: the input position that lands at p
  }
}

// K9a for small classes: one WARP per reshuffle event (kFyWarps events per
// CTA), warp-synchronous -- many more events in flight next to the
// persistent codec kernel than with a CTA each.  Same algorithm as k_fy_gen.
constexpr int kFyWarps = 2;
constexpr uint32_t kFyWarpMaxM = 1536;
__host__ __device__ inline size_t fy_warp_smem_bytes(uint32_t m) { return kFyWarps * (4ull * (3ull * m + 2) + 2ull * (m + 2) + 16); }

__global__ void __launch_bounds__(kFyWarps * 32) k_fy_gen_warp(ChainArgs a, uint32_t n_gen, uint32_t max_m) {
  extern __shared__ uint32_t sh[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t q = blockIdx.x * kFyWarps + w;
  if (q >= n_gen || *a.chain != a.expect_start) return;
  const uint32_t e = a.cls_list[q];
  const SbsEvent E = a.ev[e];
  const uint32_t m = E.m;
  const size_t words = (fy_warp_smem_bytes(max_m) / kFyWarps) / 4;
  uint32_t* js = sh + w * words;   // [m + 1]
  uint32_t* off = js + (m + 1);    // [m + 1]
  uint32_t* bk = off + (m + 1);    // [m]
  uint16_t* cnt = reinterpret_cast<uint16_t*>(bk + m);  // [m]
  const uint64_t s = a.seeds[e];
  for (uint32_t x = lane; x < (m + 1) / 2; x += 32) reinterpret_cast<uint32_t*>(cnt)[x] = 0;
  __syncwarp();
  bool rej = false;
  for (uint32_t i = 2 + lane; i <= m; i += 32) {
    const uint64_t x = mix64(s + (static_cast<uint64_t>(m) - i + 1) * kGamma);
    rej |= rejected(x, i);
    const uint32_t j = mod_below(x, i, a.recip);
    js[i] = j;
    atomicAdd(reinterpret_cast<uint32_t*>(cnt) + (j >> 1), 1u << (16 * (j & 1)));
  }
  if (__any_sync(0xffffffffu, rej)) {
    if (lane == 0) atomicExch(a.flag, 1u);
    return;  // k_chain_finish redoes this call serially
  }
  __syncwarp();
  // exclusive scan of the bucket sizes: contiguous ranges per lane
  const uint32_t per = (m + 31) / 32;
  const uint32_t lo = min(m, lane * per), hi = min(m, lo + per);
  uint32_t local = 0;
  for (uint32_t x = lo; x < hi; ++x) local += cnt[x];
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  uint32_t run = incl - local;
  for (uint32_t x = lo; x < hi; ++x) {
    off[x] = run;
    run += cnt[x];
  }
  __syncwarp();
  for (uint32_t i = 2 + lane; i <= m; i += 32) bk[atomicAdd(&off[js[i]], 1u)] = i;
  __syncwarp();  // off[x] now holds the end of bucket x
  int64_t* gout = a.pool + E.slot;
  for (uint32_t p = lane; p < m; p += 32) {
    uint32_t x = p >= 1 ? js[p + 1] : 0u;
    uint32_t k = p >= 1 ? p + 2 : 2u;
    for (;;) {
      const uint32_t hi_b = off[x], lo_b = hi_b - cnt[x];
      uint32_t best = 0xffffffffu;
      for (uint32_t t = lo_b; t < hi_b; ++t) {
        const uint32_t st = bk[t];
        if (st >= k && st < best) best = st;
      }
      if (best == 0xffffffffu) break;
      x = best - 1;
      k = best + 1;
    }
    gout[p] = x;
  }
}

// prefetch != 0: the class's generations fit in shared memory after the two
// permutation buffers, and are all loaded in one sweep (every load in flight
// at once) before the composition, which then runs from shared memory only.
template <int T>
__global__ void __launch_bounds__(T) k_compose(ChainArgs a, int prefetch) {
  extern __shared__ uint32_t sh[];
  const uint32_t b = a.cls_begin[blockIdx.x], end = a.cls_begin[blockIdx.x + 1];
  const SbsEvent first = a.ev[a.cls_list[b]];
  const uint32_t m = first.m;
  uint32_t* prev = sh;
  uint32_t* next = sh + m;
  uint32_t* pis = sh + 2 * m;  // [gens][m] when prefetching
  const uint64_t copy_to = a.cls_copy[blockIdx.x];
  for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) {
    const int64_t v = a.pool[first.src + x];
    prev[x] = static_cast<uint32_t>(v);
    a.pool[copy_to + x] = v;  // pre-call copy: the input of a serial redo
  }
  __syncthreads();
  if (*a.chain != a.expect_start) {
    if (threadIdx.x == 0) atomicExch(a.flag, 1u);
    return;
  }
  if (*reinterpret_cast<volatile uint32_t*>(a.flag)) return;  // a rejection: K8 redoes the call
  if (prefetch) {
    const uint32_t gens = end - b;
    for (uint32_t x = threadIdx.x; x < gens * m; x += blockDim.x) {
      const uint32_t q = x / m, p = x - q * m;
      pis[x] = static_cast<uint32_t>(a.pool[a.ev[a.cls_list[b + q]].slot + p]);
    }
    __syncthreads();
    for (uint32_t q = 0; q < gens; ++q) {
      int64_t* g = a.pool + a.ev[a.cls_list[b + q]].slot;
      for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
        const uint32_t v = prev[pis[q * m + p]];
        next[p] = v;
        g[p] = v;
      }
      __syncthreads();
      uint32_t* t = prev;
      prev = next;
      next = t;
    }
  } else {
    for (uint32_t q = b; q < end; ++q) {
      int64_t* g = a.pool + a.ev[a.cls_list[q]].slot;
      for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
        const uint32_t v = prev[static_cast<uint32_t>(g[p])];
        next[p] = v;
        g[p] = v;
      }
      __syncthreads();
      uint32_t* t = prev;
      prev = next;
      next = t;
    }
  }
  const uint64_t final_to = a.cls_final[blockIdx.x];
  for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) a.pool[final_to + x] = prev[x];
}

// ------------------------------------------------------------------ K8
// Runs after k_shuffle.  Common case: advance the chain past this call's
// events (one mix each).  If a draw was rejected (or the cursor forces the
// serial path), redo the call exactly as the reference does: events in chain
// order, Fisher-Yates with rejection sampling (rng.hpp:29-64) on the
// generation pool starting from each class's pre-call copy, then write back
// the newest generations.
__global__ void k_chain_finish(ChainArgs a, uint32_t n_cls, int force) {
  if (!force && *a.flag == 0u && *a.chain == a.expect_start) {
    if (threadIdx.x == 0) *a.chain = a.expect_final;  // the host's walk held
    return;
  }
  if (threadIdx.x != 0) return;
  uint64_t s = *a.chain;
  for (uint64_t e = 0; e < a.E; ++e) {
    const SbsEvent ev = a.ev[e];
    uint64_t st = s;
    int64_t* out = nullptr;
    if (ev.m >= 2) {
      // input: the class's previous generation in this call, else its pre-call copy
      uint32_t q = 0;
      while (a.ev[a.cls_list[a.cls_begin[q]]].cls != ev.cls) ++q;
      uint64_t src = a.cls_copy[q];
      for (uint32_t r = a.cls_begin[q]; r < a.cls_begin[q + 1] && a.cls_list[r] != e; ++r)
        src = a.ev[a.cls_list[r]].slot;
      out = a.pool + ev.slot;
      for (uint32_t x = 0; x < ev.m; ++x) out[x] = a.pool[src + x];
    }
    for (uint64_t i = ev.m; i > 1; --i) {
      const uint64_t lim = below_limit(i);
      st += kGamma;
      uint64_t x = mix64(st);
      while (x > lim) {
        st += kGamma;
        x = mix64(st);
      }
      const uint64_t j = x % i;
      const int64_t v = out[j];
      out[j] = out[i - 1];
      out[i - 1] = v;
    }
    st += kGamma;  // rng_state_ = rng.next_u64() (sampler.cpp:87)
    s = mix64(st);
  }
  for (uint32_t q = 0; q < n_cls; ++q) {
    const uint32_t last = a.cls_list[a.cls_begin[q + 1] - 1];
    const SbsEvent ev = a.ev[last];
    for (uint32_t x = 0; x < ev.m; ++x) a.pool[a.cls_final[q] + x] = a.pool[ev.slot + x];
  }
  if (s != a.expect_final && a.diverged) {  // the host must resync its chain mirror
    *reinterpret_cast<volatile unsigned int*>(a.diverged) += 1u;
    __threadfence_system();
  }
  *a.chain = s;
  *a.flag = 0u;
}

// ------------------------------------------------------------------ K10
__global__ void __maxnreg__(32) k_gather(SbsGatherArgs a, int64_t* __restrict__ examples, int32_t* __restrict__ classes,
                         uint64_t out_batches) {
  const uint64_t total = out_batches * a.B;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t lb = t / a.B;
    const uint64_t r = t - lb * a.B;
    const uint32_t c = a.row_cls[r];
    const uint64_t k = r - a.prefix[c];
    const uint64_t beta = a.shard + lb * a.n_shards;  // batch within this call
    const uint64_t D = a.drawn_before[c] + beta * a.counts[c] + k;
    const uint64_t m = a.class_size[c];
    const uint64_t gen = D / m;
    const uint64_t off = a.gen_base_off[c] + (gen - a.gen_base_gen[c]) * a.gen_stride[c] + (D - gen * m);
    examples[t] = a.pool[off];
    if (classes) classes[t] = static_cast<int32_t>(c);
  }
}

}  // namespace

uint64_t class_index_scratch_words(uint64_t n, uint64_t C) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  return tiles * C;
}

cudaError_t launch_class_index(const int32_t* labels, uint64_t n, uint64_t C,
                               uint64_t* class_offsets, int64_t* members, uint32_t* scratch,
                               uint64_t scratch_words, DevError* err, cudaStream_t s,
                               uint64_t* launches) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  if (tiles * C > scratch_words) return cudaErrorInvalidValue;
  const size_t smem = C * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_ci_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_ci_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (tiles > 0) {
    k_ci_hist<<<static_cast<unsigned>(tiles), 32, smem, s>>>(labels, n, (uint32_t)C,
                                                             (uint32_t)tiles, scratch, err);
    ++*launches;
  }
  k_ci_scan<<<1, 1024, 0, s>>>(scratch, tiles * C, (uint32_t)C, (uint32_t)(tiles ? tiles : 1),
                               class_offsets);
  ++*launches;
  if (tiles > 0) {
    k_ci_scatter<<<static_cast<unsigned>(tiles), 32, smem, s>>>(labels, n, (uint32_t)C,
                                                                (uint32_t)tiles, scratch, members);
    ++*launches;
  }
  k_ci_label_value<<<1, 1, 0, s>>>(labels, C, err);
  ++*launches;
  return cudaGetLastError();
}


cudaError_t launch_sbs_events(const ChainArgs& a, uint32_t n_cls, uint32_t n_gen, uint32_t max_m,
                              uint64_t max_gen_words, int force, cudaStream_t s, uint64_t* launches) {
  if (n_cls > 0 && max_m != 0xffffffffu && max_m <= kParMaxM) {
    // wide CTAs from 4 generations per class (OPTB_SBS_WIDE=0|1 forces)
    static const int wide_env = [] {
      const char* v = getenv("OPTB_SBS_WIDE");
      return v && v[0] ? (v[0] == '1' ? 1 : 0) : -1;
    }();
    const bool wide = wide_env >= 0 ? wide_env == 1 : true;
    auto fy = wide ? k_fy_gen<kParThreadsWide> : k_fy_gen<kParThreads>;
    auto comp = wide ? k_compose<kParThreadsWide> : k_compose<kParThreads>;
    cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(fy), static_cast<int>(par_smem_bytes(kParMaxM)));
    if (ae != cudaSuccess) return ae;
    // prefetch the generations into shared memory when the largest class's
    // (gens x m) words fit in 64 KB beside the two permutation buffers
    const size_t pref = static_cast<size_t>(max_gen_words) * 4 <= 64 * 1024 ? static_cast<size_t>(max_gen_words) * 4 : 0;
    const size_t csmem = 8 * static_cast<size_t>(max_m) + pref;
    ae = ensure_smem_attr(reinterpret_cast<const void*>(comp), static_cast<int>(8 * kParMaxM + 64 * 1024));
    if (ae != cudaSuccess) return ae;
    if (max_m <= kFyWarpMaxM) {
      ae = ensure_smem_attr(reinterpret_cast<const void*>(k_fy_gen_warp),
                            static_cast<int>(fy_warp_smem_bytes(kFyWarpMaxM)));
      if (ae != cudaSuccess) return ae;
      k_fy_gen_warp<<<(n_gen + kFyWarps - 1) / kFyWarps, kFyWarps * 32, fy_warp_smem_bytes(max_m), s>>>(a, n_gen,
                                                                                                      max_m);
    } else {
      fy<<<n_gen, wide ? kParThreadsWide : kParThreads, par_smem_bytes(max_m), s>>>(a);
    }
    comp<<<n_cls, wide ? kParThreadsWide : kParThreads, csmem, s>>>(a, pref ? 1 : 0);
    *launches += 2;
  } else if (n_cls > 0) {
    size_t smem = (kJWin + static_cast<size_t>(max_m)) * sizeof(uint32_t);
    int use_smem = 1;
    if (max_m == 0xffffffffu || smem > 200 * 1024) {
      use_smem = 0;
      smem = kJWin * sizeof(uint32_t);
    }
    const cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(k_shuffle), 200 * 1024 + 8192);
    if (ae != cudaSuccess) return ae;
    k_shuffle<<<n_cls, 64, smem, s>>>(a, use_smem);
    ++*launches;
  }
  k_chain_finish<<<1, 128, 0, s>>>(a, n_cls, force);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_recip_table(uint64_t* recip, uint32_t n, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((static_cast<uint64_t>(n) + 256) / 256, 1184));
  k_recip<<<grid, 256, 0, s>>>(recip, n);
  return cudaGetLastError();
}

cudaError_t launch_sbs_gather(const SbsGatherArgs& a, int64_t* examples, int32_t* classes,
                              cudaStream_t s, uint64_t* launches) {
  const uint64_t out_batches =
      a.n_batches > a.shard ? (a.n_batches - a.shard + a.n_shards - 1) / a.n_shards : 0;
  const uint64_t total = out_batches * a.B;
  if (total == 0) return cudaSuccess;
  // Small CTAs (64 threads x <= 32 registers) so the gather co-resides with
  // the encode/decode CTAs of the previous step when it runs on a side stream.
  const uint64_t want = (total + 63) / 64;
  const unsigned grid = static_cast<unsigned>(want < 148 * 2 ? want : 148 * 2);
  k_gather<<<grid, 64, 0, s>>>(a, examples, classes, out_batches);
  ++*launches;
  return cudaGetLastError();
}

namespace {
__global__ void k_copy_in(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n16) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

cudaError_t launch_copy_in(const void* src, void* dst, size_t bytes, cudaStream_t s, uint64_t* launches) {
  const uint64_t n16 = (bytes + 15) / 16;
  const uint64_t blocks = (n16 + 255) / 256;
  k_copy_in<<<static_cast<unsigned>(blocks < 64 ? blocks : 64), 256, 0, s>>>(static_cast<const uint4*>(src),
                                                                             static_cast<uint4*>(dst), n16);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace optb_b200
