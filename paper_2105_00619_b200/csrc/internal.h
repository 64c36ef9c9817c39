// internal.h -- declarations shared between the C-ABI layer (capi.cu) and the
// kernel translation units (codec.cu, sbs.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "optb_cuda.h"

namespace optb_b200 {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size): attributes are per device context, and several contexts on
// different devices may share one process.
cudaError_t ensure_smem_attr(const void* kernel, int bytes);

// Set by the caller around a launch whose buffers are mapped pinned host
// memory (the small host calls run zero-copy): the vector kernels then move
// data with cp.async / per-lane loads and stores only, no tensor-map (TMA)
// transfers.
extern thread_local bool g_sysmem;

// Which kernel the most recent fused round trip of this thread ran
// (OPTB_RT_* in optb_cuda.h); set by launch_roundtrip's launchers.
extern thread_local int g_rt_kind;

// Sets the calling thread's optb_last_error() text; returns `code`.
int set_error_text(int code, const std::string& message);

// Device-side error latch owned by a context (see optb_ctx_sync).
struct DevError {
  uint32_t kind;         // 0 none, 1 int range, 2 f64 range, 3 label
  uint32_t pad;
  unsigned long long key;  // int/f64 range: (chunk << 8) | n ; label: example index
  long long label;         // offending label value (kind 3)
  unsigned long long aux;  // label: number of classes
};
enum : uint32_t { kErrNone = 0, kErrIntRange = 1, kErrF64Range = 2, kErrLabel = 3 };

// Geometry of a batch stream (optb_layout + derived values).
struct Geom {
  int32_t mode;
  uint32_t per_chunk;
  uint32_t wc;          // container bytes per pixel
  uint32_t cpb;         // chunks per batch
  uint64_t P;
  uint64_t B;
  uint64_t chunks;
  uint64_t ostride;     // offsets bytes per chunk (0 without offsets)
  uint64_t chunk_base;  // global index of chunk 0 (error reporting across slices)
};

struct Epi {
  int32_t dtype;
  float scale;
  const float* class_scale;
  const float* class_bias;
  const int32_t* row_class;
  uint64_t row_stride;  // elements
};

// Where the gather-encode reads stream row r: images + index[r] * stride
// (index NULL = identity), or the absolute address ptrs[r] when ptrs is set
// (peer-GPU HBM over NVLink, mapped host memory, ...).
struct RowSrc {
  const uint8_t* images;
  uint64_t stride;
  const int64_t* index;
  const uint64_t* ptrs;
  int32_t ptrs_aligned16;  // every ptrs[r] is 16-byte aligned (vector path)
  // the rows and row ids may be read before the previous kernel in the stream
  // has completed (it cannot have written them): the interleaved round trip
  // then gathers its first tiles while that kernel drains (programmatic
  // dependent launch) and waits for it before its first global write
  int32_t early;
};

// A tag per stream that changes with every kernel the library launches with
// programmatic dependent launch (launch_k).  The pipeline compares it with
// the tag after its previous step: equal means no library kernel that can
// trigger its dependents early was launched on that stream in between.
uint64_t stream_tag(cudaStream_t s);
void bump_stream_tag(cudaStream_t s);
// Examples in a cursor's class index (row ids drawn are < this).
uint64_t sbs_examples(const optb_sbs* s);
// Grow the cursor's generation pool for calls of up to n batches now.
int sbs_reserve(optb_sbs* s, uint64_t n_batches);
// optb_encode_dev with RowSrc::early set as given (the split pipeline step).
int encode_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
               const int64_t* row_index, void* containers, uint8_t* offsets, void* stream, bool early);
// optb_roundtrip_dev with RowSrc::early set as given (the pipeline step).
int roundtrip_dev(optb_ctx* c, const optb_layout* L, const uint8_t* images, uint64_t row_stride,
                  const int64_t* row_index, void* containers, uint8_t* offsets, const optb_epilogue* E, void* out,
                  void* stream, bool early);

// Kernel launchers (codec.cu).  Return cudaError_t of the launch; `launches`
// is incremented by the number of kernels enqueued.
cudaError_t launch_encode(const Geom& g, const RowSrc& rows, void* containers, uint8_t* offsets,
                          cudaStream_t s, int num_sms, uint64_t* launches);
cudaError_t launch_decode(const Geom& g, const void* containers, const uint8_t* offsets,
                          const Epi& e, void* out, DevError* err, cudaStream_t s, int num_sms,
                          uint64_t* launches);
// The generic (any alignment, plain loads / stores) kernels only.
cudaError_t launch_encode_generic(const Geom& g, const RowSrc& rows, void* containers, uint8_t* offsets,
                                  cudaStream_t s, int num_sms, uint64_t* launches);
cudaError_t launch_decode_generic(const Geom& g, const void* containers, const uint8_t* offsets, const Epi& e,
                                  void* out, DevError* err, cudaStream_t s, int num_sms, uint64_t* launches);
// Encode + decode of the same stream in one launch (vector path; lossless
// modes need P % 512 == 0);
// cudaErrorNotSupported when the geometry needs the separate launches.
cudaError_t launch_roundtrip(const Geom& g, const RowSrc& rows, void* containers, uint8_t* offsets, const Epi& e,
                             void* out, DevError* err, cudaStream_t s, int num_sms, uint64_t* launches);
cudaError_t launch_synth(uint64_t seed, uint64_t first_row, uint64_t n_rows, uint64_t P,
                         uint8_t* out, uint64_t row_stride, cudaStream_t s, int num_sms,
                         uint64_t* launches);

// dst[0, bytes) = src[0, bytes) by a kernel (src: mapped pinned host memory;
// both 16-byte aligned, readable / writable up to bytes rounded up to 16).
cudaError_t launch_copy_in(const void* src, void* dst, size_t bytes, cudaStream_t s, uint64_t* launches);

// SBS launchers (sbs.cu).
cudaError_t launch_class_index(const int32_t* labels, uint64_t n, uint64_t C,
                               uint64_t* class_offsets, int64_t* members, uint32_t* scratch,
                               uint64_t scratch_words, DevError* err, cudaStream_t s,
                               uint64_t* launches);
uint64_t class_index_scratch_words(uint64_t n, uint64_t C);

// One reshuffle event of the SplitMix64 chain.
struct SbsEvent {
  uint32_t cls;     // class
  uint32_t m;       // class size
  uint64_t slot;    // element offset of the output permutation in the generation pool
  uint64_t src;     // element offset of the input permutation (previous generation)
};

// Device view of one call's reshuffle events (uploaded as one block).
struct ChainArgs {
  const SbsEvent* ev;         // [E] in chain order
  uint64_t E;
  const uint32_t* cls_begin;  // [n_cls+1] into cls_list
  const uint32_t* cls_list;   // event ids of each reshuffling class, generation order
  const uint64_t* cls_copy;   // pool offset receiving the class's pre-call permutation
  const uint64_t* cls_final;  // pool offset of the class's current permutation
  uint64_t* seeds;            // [E] chain state at the start of each event (host-computed)
  uint32_t* flag;             // [1] rejection seen (forces the exact serial redo)
  unsigned long long* chain;  // chain state before the first event; advanced in place
  int64_t* pool;
  // The host walks the chain (one mix per event, no rejection assumed) from
  // its mirror of the chain state; the kernels use its seeds only if the
  // device state equals expect_start and no draw is rejected, otherwise the
  // call is redone serially from the device state (the authority).
  uint64_t expect_start, expect_final;
  unsigned int* diverged;     // mapped host counter: serial redos that moved the chain off the host's walk
  // [max_m + 1] floor((2^64 - 1) / i): next_below's x % i as a multiply-high
  // and one correction in the parallel Fisher-Yates (nullptr: plain %)
  const uint64_t* recip;
};
// fills recip[i] = floor((2^64 - 1) / i) for 2 <= i <= n (the sampler's table)
cudaError_t launch_recip_table(uint64_t* recip, uint32_t n, cudaStream_t s);

// k_fy_gen (one CTA per reshuffle event) + k_compose (one CTA per reshuffling
// class), or k_shuffle (one CTA per class, large classes), then k_chain_finish
// (chain advance, or the exact serial redo after a rejection / when forced).
// n_gen = reshuffle events with m >= 2 (the length of cls_list);
// max_gen_words = max over reshuffling classes of (its events) x m.
cudaError_t launch_sbs_events(const ChainArgs& a, uint32_t n_cls, uint32_t n_gen, uint32_t max_m,
                              uint64_t max_gen_words, int force, cudaStream_t s, uint64_t* launches);

struct SbsGatherArgs {
  const uint32_t* row_cls;       // [B] class of each batch row (class-major)
  const uint64_t* counts;        // [C]
  const uint64_t* prefix;        // [C+1] exclusive scan of counts (row offset in batch)
  const uint64_t* class_size;    // [C]
  const uint64_t* drawn_before;  // [C] draws from class c before this call
  const uint64_t* gen_base_gen;  // [C] generation held in pool slot 0 of class c
  const uint64_t* gen_base_off;  // [C] pool offset of that generation
  const uint64_t* gen_stride;    // [C] pool elements per generation (= m_c)
  const int64_t* pool;
  uint64_t C, B;
  uint64_t n_batches;  // batches in this call
  uint32_t shard, n_shards;
};
cudaError_t launch_sbs_gather(const SbsGatherArgs& a, int64_t* examples, int32_t* classes,
                              cudaStream_t s, uint64_t* launches);

}  // namespace optb_b200
