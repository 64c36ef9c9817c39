/*
 * optb_cuda.h -- C ABI of the B200-native OpTorch data-flow path
 * (encode / decode / selective batch sampling) for sm_100a.
 *
 * This is the drop-in boundary.  The reference (/root/reference/proj) has no
 * FFI; its boundary is the C++ header API in include/optb/{codec,sampler}.hpp
 * and nn.hpp.  Each entry point below names the reference function it
 * replaces (file:line under /root/reference/proj).  The C++ headers with the
 * reference's exact declarations are re-implemented over this ABI in
 * paper_2105_00619_b200/csrc/shim (liboptb_shim.so), and bound from Python
 * with ctypes in paper_2105_00619_b200/_lib.py; INTEGRATION.md shows both.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory;
 *    "host" pointers are ordinary (pageable or pinned) host memory.
 *  - Every function returns an optb_status.  On failure the message of the
 *    calling thread is available from optb_last_error(); the text equals the
 *    reference exception's what() (errors.hpp:9-42) wherever the reference
 *    has one, so the shim rethrows the same class with the same message.
 *  - *_dev entry points are asynchronous and stream-ordered (stream = a
 *    cudaStream_t passed as void*, NULL = legacy default stream); they never
 *    allocate.  Device-side format errors (decode range checks, bad labels)
 *    are latched in the context and reported by optb_ctx_sync().  *_host
 *    entry points are synchronous and report everything themselves.
 *  - A context is bound to one device and is used by one host thread at a
 *    time (the reference functions are reentrant: use one
 *    context per thread).
 *
 * Device data layout
 *  - images      rows of P = H*W*C u8 pixels, HWC (codec.hpp:56-62), rows
 *                `row_stride` bytes apart.
 *  - stream      n_batches batches of `batch` rows; batch b is split into
 *                ceil(batch/per_chunk) chunks of per_chunk consecutive rows,
 *                the last one partial (runner.cpp:77-90).
 *  - containers  chunk k's plane is P words of Wc bytes at
 *                containers + k*P*Wc, words little-endian (u64 / u128 lo,hi;
 *                binary64 bits for f64) -- the OPTB payload order
 *                (codec.cpp:298-312).  Wc = optb_container_value_bytes().
 *  - offsets     (lossless modes) chunk k's parity plane, ceil(n_k*P/8)
 *                bytes, bit i*P+p LSB-first (codec.cpp:101-104), at
 *                offsets + k*optb_offsets_stride(mode, P, per_chunk).
 *  - decoded     row r = b*batch + j*per_chunk + i at out + r*out_row_stride
 *                elements (nn.cpp:177-191 row order).
 */
#ifndef OPTB_CUDA_H
#define OPTB_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPTB_ABI_VERSION 1

/* status codes <-> errors.hpp:9-42 */
typedef enum optb_status {
  OPTB_OK = 0,
  OPTB_ERR = 1,          /* optb::Error (sampler and generic)      */
  OPTB_ERR_SHAPE = 2,    /* optb::ShapeError                       */
  OPTB_ERR_CAPACITY = 3, /* optb::CapacityError                    */
  OPTB_ERR_FORMAT = 4,   /* optb::FormatError                      */
  OPTB_ERR_CUDA = 5,     /* CUDA runtime failure (no reference twin) */
  OPTB_ERR_ARG = 6       /* invalid argument to the C ABI itself   */
} optb_status;

/* codec modes -- CodecMode, codec.hpp:22-28 (same tags, also the OPTB tag) */
enum { OPTB_EXACT64 = 0, OPTB_EXACT128 = 1, OPTB_F64 = 2, OPTB_LOSSLESS64 = 3, OPTB_LOSSLESS128 = 4 };
/* decoded element types */
enum { OPTB_OUT_U8 = 0, OPTB_OUT_F32 = 1, OPTB_OUT_F16 = 2, OPTB_OUT_BF16 = 3 };

typedef struct optb_ctx optb_ctx;
typedef struct optb_sbs optb_sbs;

/* A batch stream (see "stream" above). */
typedef struct optb_layout {
  int32_t mode;        /* OPTB_EXACT64 ...                                  */
  uint32_t per_chunk;  /* images per container, 1..optb_accept_limit(mode)  */
  uint64_t pixels;     /* P = H*W*C                                         */
  uint64_t batch;      /* rows per batch                                    */
  uint64_t n_batches;  /* batches in the stream                             */
} optb_layout;

/* Decode epilogue (nn.cpp:183-189, 235).  For float outputs every element is
 * RN(float(q) * scale) -- one binary32 multiply, never contracted -- then
 * converted RNE to f16 (tensor.cpp:12-51) or bf16.  With per-class tables
 * (the GPU form of the per-class preprocessing seam, sampler.hpp:39-40) row r
 * uses c = row_class[r]: y = RN(RN(q*class_scale[c]) + class_bias[c]); a
 * table of (scale, 0) reproduces the plain epilogue bit for bit. */
typedef struct optb_epilogue {
  int32_t out_dtype;          /* OPTB_OUT_*                                */
  float scale;                /* e.g. 1/255 = 0x3b808081 (runner.hpp:22)  */
  const float* class_scale;   /* dev, nullable                             */
  const float* class_bias;    /* dev, nullable (requires class_scale)      */
  const int32_t* row_class;   /* dev, required with class tables           */
  uint64_t out_row_stride;    /* elements between output rows; 0 = P       */
} optb_epilogue;

/* ---------------------------------------------------------------- metadata
 * codec.hpp:33-43, codec.cpp:13-62.  Unknown modes return 0 / "?". */
uint32_t optb_abi_version(void);
uint32_t optb_capacity(int32_t mode);
uint32_t optb_accept_limit(int32_t mode);     /* capacity, or 16 for f64 (codec.hpp:36) */
int32_t optb_capacity_is_hard(int32_t mode);
const char* optb_mode_name(int32_t mode);
int32_t optb_mode_has_offsets(int32_t mode);
uint32_t optb_container_value_bytes(int32_t mode);
uint64_t optb_offsets_plane_bytes(uint32_t n_images, uint64_t pixels); /* codec.cpp:75-77 */
uint64_t optb_offsets_stride(int32_t mode, uint64_t pixels, uint32_t per_chunk);
uint64_t optb_layout_chunks(const optb_layout* L);
uint64_t optb_layout_rows(const optb_layout* L);
uint64_t optb_layout_container_bytes(const optb_layout* L);
uint64_t optb_layout_offsets_bytes(const optb_layout* L);
/* Validates a layout like codec.cpp:79-97 (capacity message included). */
int optb_layout_check(const optb_layout* L);

/* ---------------------------------------------------------------- errors */
const char* optb_last_error(void);  /* calling thread's last message ("" if none) */

/* ---------------------------------------------------------------- context */
int optb_ctx_create(int device, optb_ctx** out);
void optb_ctx_destroy(optb_ctx* ctx);
/* Synchronise `stream`, then report (and clear) any device-side error
 * latched by earlier *_dev calls: decode range violations give
 * OPTB_ERR_FORMAT with the reference message (codec.cpp:165-170, 191-194),
 * bad labels give OPTB_ERR (sampler.cpp:58-61). */
int optb_ctx_sync(optb_ctx* ctx, void* stream);
/* Number of device kernels this context has launched (bench evidence). */
uint64_t optb_ctx_launches(const optb_ctx* ctx);

/* ---------------------------------------------------------------- codec, device
 * Replaces codec::encode (codec.cpp:106-146) applied to every chunk of a
 * stream, fused with the gather of Dataset::image_of (dataset.cpp:16-22) as
 * driven by runner.cpp:77-90 / 278-290: stream row r reads image row
 * row_index[r] (dev int64, nullable = identity) of `images`. */
int optb_encode_dev(optb_ctx* ctx, const optb_layout* L, const uint8_t* images,
                    uint64_t row_stride, const int64_t* row_index, void* containers,
                    uint8_t* offsets, void* stream);

/* Replaces codec::decode (codec.cpp:148-208) for every chunk, and with a
 * float epilogue nn::decode_input (nn.cpp:153-192) + the MixedPrecision
 * binary16 store (nn.cpp:141-146, 235): the layer input is written directly. */
int optb_decode_dev(optb_ctx* ctx, const optb_layout* L, const void* containers,
                    const uint8_t* offsets, const optb_epilogue* E, void* out, void* stream);

/* optb_encode_dev followed by optb_decode_dev of the same stream (same
 * results, containers and offsets materialised as by the two calls): one
 * persistent launch on the vector path (lossless modes: pixels % 512 == 0),
 * otherwise the two launches.  Exact / f64 modes: each warp decodes a tile one
 * iteration after storing it, so the container re-read is served from L2
 * (interleaved kernel); lossless: each warp encodes all its tiles, then decodes
 * them back (phase-ordered kernel).  The E-D pipeline step
 * (pipeline.cpp:197-216 encode + runner.cpp:292-309 decode) uses it. */
int optb_roundtrip_dev(optb_ctx* ctx, const optb_layout* L, const uint8_t* images,
                       uint64_t row_stride, const int64_t* row_index, void* containers,
                       uint8_t* offsets, const optb_epilogue* E, void* out, void* stream);

/* ---------------------------------------------------------------- codec, host
 * Same operations on host buffers (images [rows][P] contiguous; containers /
 * offsets / decoded in the layouts above).  H2D and D2H run on side streams
 * through pinned staging, overlapped slice by slice with the kernels.
 * Synchronous; all errors reported on return. */
int optb_encode_host(optb_ctx* ctx, const optb_layout* L, const uint8_t* images,
                     void* containers, uint8_t* offsets);
int optb_decode_host(optb_ctx* ctx, const optb_layout* L, const void* containers,
                     const uint8_t* offsets, const optb_epilogue* E, void* out);

/* ---------------------------------------------------------------- SBS
 * sampler::plan (sampler.cpp:11-51): largest-remainder counts; host
 * arithmetic (binary64), errors and messages as the reference. */
int optb_sbs_plan(const double* weights, uint64_t n_classes, uint64_t batch, uint64_t* counts);

/* ClassIndex::from_labels (sampler.cpp:53-65) on the GPU: a stable
 * partition of [0,n) by label (warp match/ballot ranks + tile x class scan).
 * class_offsets[C+1] and members[n] are dev outputs.  A label outside
 * [0,C) latches OPTB_ERR "sampler: label L outside C classes" (first such
 * example), reported by optb_ctx_sync. */
int optb_class_index_dev(optb_ctx* ctx, const int32_t* labels, uint64_t n, uint64_t n_classes,
                         uint64_t* class_offsets, int64_t* members, void* stream);

/* Same partition with host labels in and host outputs back (synchronous;
 * errors reported on return) -- the form ClassIndex::from_labels returns. */
int optb_class_index_host(optb_ctx* ctx, const int32_t* labels, uint64_t n, uint64_t n_classes,
                          uint64_t* class_offsets, int64_t* members);

/* BatchCursor(plan, index) (sampler.cpp:67-82): per-class permutations and
 * the SplitMix64 chain live on the device.  counts[C] and class_offsets[C+1]
 * are host arrays; members[class_offsets[C]] is dev (members_on_device=1) or
 * host.  Runs the constructor's C reshuffles before returning. */
int optb_sbs_create(optb_ctx* ctx, const uint64_t* counts, uint64_t n_classes, uint64_t batch,
                    uint64_t seed, const uint64_t* class_offsets, const int64_t* members,
                    int32_t members_on_device, optb_sbs** out);
void optb_sbs_destroy(optb_sbs* sbs);
/* A copy of a BatchCursor (the reference class is copyable,
 * sampler.hpp:45-68; a copy continues the identical stream independently):
 * waits for the calls enqueued on `sbs`, then duplicates its permutations,
 * chain state and position. */
int optb_sbs_clone(const optb_sbs* sbs, optb_sbs** out);

/* BatchCursor::next (sampler.cpp:91-104) n_batches times.  Writes the
 * class-major draws of the batches beta0 + t (t < n_batches) with
 * t % n_shards == shard, in order, batch after batch: examples (dev int64)
 * and classes (dev int32, nullable).  Every shard advances the cursor by
 * n_batches, so n_shards processes calling with shard = 0..n_shards-1
 * together reproduce the single-process stream with no communication. */
int optb_sbs_next_dev(optb_sbs* sbs, uint64_t n_batches, uint32_t shard, uint32_t n_shards,
                      int64_t* examples, int32_t* classes, void* stream);
/* Same, all batches, host outputs (synchronous). */
int optb_sbs_next_host(optb_sbs* sbs, uint64_t n_batches, int64_t* examples, int32_t* classes);
uint64_t optb_sbs_batches_drawn(const optb_sbs* sbs);
/* Testing aid (pure host, no device work): the host planner's view of one
 * sampler call -- the reshuffle events of the next n batches after
 * batches_before, in chain order (class and generation of each), given the
 * per-class draw counts, class sizes and generations so far, and the chain
 * state each event starts from when no draw is rejected (the seeds the host
 * hands to the kernels; chain = the state before the call).  n_events gets
 * the event count; more than max_events is OPTB_ERR_ARG. */
int optb_sbs_plan_call(uint64_t n_classes, const uint64_t* counts, const uint64_t* class_sizes,
                       const uint64_t* gen, uint64_t batches_before, uint64_t n, uint64_t chain,
                       uint64_t max_events, uint64_t* ev_class, uint64_t* ev_gen, uint64_t* ev_seed,
                       uint64_t* n_events, uint64_t* chain_after);
/* Testing aid: force the exact serial rejection-sampling path for every
 * reshuffle (results are identical; only speed changes). */
int optb_sbs_set_force_serial(optb_sbs* sbs, int32_t on);
/* Tuning aid: time each next call's phases with CUDA events; report the last
 * call's upload, reshuffle (K9+K8) and gather (K10) durations in ms. */
int optb_sbs_set_profiling(optb_sbs* sbs, int32_t on);
int optb_sbs_profile(optb_sbs* sbs, float* upload_ms, float* reshuffle_ms, float* gather_ms);

/* ---------------------------------------------------------------- sharded dataset
 * Building blocks of the optional dataset-sharded global gather (SURVEY
 * §8(e)): when every rank holds only rows [begin, end) of the dataset, the
 * rows a step draws are exchanged with one all-to-all (NCCL over NVLink;
 * paper_2105_00619_b200/sharded.py).  The exchange plan is a stable
 * partition of each rank's draws by owner rank (optb_class_index_dev with
 * labels = owner); these two kernels pack the outgoing rows and turn the
 * incoming order into a row index for optb_encode_dev.
 *
 * dst row i = src row (index[i] - bias) (16-byte vector copies when aligned). */
int optb_gather_rows_dev(optb_ctx* ctx, const uint8_t* src, uint64_t src_stride, const int64_t* index,
                         uint64_t n, int64_t bias, uint64_t pixels, uint8_t* dst, uint64_t dst_stride,
                         void* stream);
/* inv[perm[j]] = j for j < n (perm a permutation of [0, n)). */
int optb_inverse_perm_dev(optb_ctx* ctx, const int64_t* perm, uint64_t n, int64_t* inv, void* stream);
/* owner[i] = (int32)((examples[i] - 0) / rows_per_shard), clamped to n_shards - 1. */
int optb_owner_labels_dev(optb_ctx* ctx, const int64_t* examples, uint64_t n, uint64_t rows_per_shard,
                          uint32_t n_shards, int32_t* owner, void* stream);

/* Peer-memory variant (no all-to-all, no staging, no host synchronisation) of
 * the sharded gather -- the reference's Dataset::image_of (dataset.cpp:16-22)
 * when the dataset's rows live on several GPUs:
 * every rank maps its peers' dataset shards into its address space with CUDA
 * IPC (NVLink / NVSwitch peer access) and the gather-encode kernel loads each
 * drawn row from the GPU that holds it, tile by tile.
 *
 * row_ptrs[i] = bases[o] + (examples[i] - o*rows_per_shard) * row_stride with
 * o = examples[i] / rows_per_shard clamped to n_shards - 1 (bases: device
 * array of the shards' base addresses as seen by this process). */
int optb_shard_row_ptrs_dev(optb_ctx* ctx, const int64_t* examples, uint64_t n, const uint64_t* bases,
                            uint32_t n_shards, uint64_t rows_per_shard, uint64_t row_stride,
                            uint64_t* row_ptrs, void* stream);
/* Which kernel the calling thread's most recent optb_roundtrip_dev /
 * optb_roundtrip_rows_dev / pipeline step ran (no reference counterpart: for
 * the caller's byte accounting -- the interleaved kernels read the containers
 * back from L2, not HBM). */
#define OPTB_RT_NONE 0
#define OPTB_RT_SPLIT 1            /* optb_encode_dev + optb_decode_dev launches */
#define OPTB_RT_PHASE_ORDERED 2    /* k_roundtrip_vec */
#define OPTB_RT_INTERLEAVED 3      /* k_roundtrip_il, 8 warps x 2 stages */
#define OPTB_RT_INTERLEAVED_DEEP 4 /* k_roundtrip_il, 5 warps x 4 stages */
#define OPTB_RT_INTERLEAVED_LANE_ST 5 /* k_roundtrip_il, 8 x 2, per-lane container stores */
int optb_last_roundtrip_kind(void);

/* optb_encode_dev / optb_roundtrip_dev reading stream row r from the absolute
 * device-accessible address row_ptrs[r] (device array): this GPU's HBM, a
 * peer GPU's HBM opened with optb_ipc_open, or mapped pinned host memory.
 * rows_aligned16 != 0 asserts every address is 16-byte aligned, which (with
 * pixels % 16 == 0) selects the vector kernels. */
int optb_encode_rows_dev(optb_ctx* ctx, const optb_layout* L, const uint64_t* row_ptrs,
                         int32_t rows_aligned16, void* containers, uint8_t* offsets, void* stream);
int optb_roundtrip_rows_dev(optb_ctx* ctx, const optb_layout* L, const uint64_t* row_ptrs,
                            int32_t rows_aligned16, void* containers, uint8_t* offsets,
                            const optb_epilogue* E, void* out, void* stream);
/* CUDA IPC of the device allocation holding dev_ptr: the 64-byte handle and
 * dev_ptr's offset inside the allocation; open maps it on `device` in another
 * process (peer access enabled lazily); close unmaps (pass the same offset). */
#define OPTB_IPC_HANDLE_BYTES 64
int optb_ipc_export(const void* dev_ptr, uint8_t* handle, uint64_t* offset);
int optb_ipc_open(int device, const uint8_t* handle, uint64_t offset, void** dev_ptr);
int optb_ipc_close(void* dev_ptr, uint64_t offset);

/* ---------------------------------------------------------------- OPTB files
 * pipeline::dump / load (pipeline.cpp:246-271) for device streams: chunk k of
 * a stream is the file <dir>/batch_<epoch>_<k>.optb holding write_optb's
 * bytes (codec.cpp:283-317).  The device container planes already are the
 * OPTB payload (little-endian words, binary64 bits for f64) followed by the
 * parity plane, so a file is the 20-byte header plus one D2H copy per plane
 * (staged through pinned memory).  (h, w, c) is the image shape, h*w*c must
 * equal layout.pixels.  Load validates every header like read_optb
 * (codec.cpp:319-367: magic, version, mode tag, capacity) and against the
 * expected layout; a missing file or any mismatch is OPTB_ERR_FORMAT. */
int optb_dump_dev(optb_ctx* ctx, const optb_layout* L, const void* containers,
                  const uint8_t* offsets, uint32_t h, uint32_t w, uint32_t c, const char* dir,
                  uint64_t epoch);
int optb_load_dev(optb_ctx* ctx, const optb_layout* L, uint32_t h, uint32_t w, uint32_t c,
                  const char* dir, uint64_t epoch, void* containers, uint8_t* offsets);

/* data::load_records (dataset.cpp:65-99) onto the device: a file of
 * CIFAR-style records (1 label byte + C planes of H*W bytes) is read into
 * pinned memory, copied up, and one kernel de-interleaves planar CHW into the
 * HWC rows the codec packs (pixels[r][hw*C + c] = plane c byte hw) and
 * extracts the labels (int32).  Errors and messages are the reference's
 * ("records: cannot open ...", "... label L outside K classes in ...",
 * "... trailing partial record in ...", "... no records in ...").
 * *n_records gets the count; at most max_records are accepted. */
int optb_load_records_dev(optb_ctx* ctx, const char* path, uint32_t h, uint32_t w, uint32_t c,
                          uint32_t n_classes, uint8_t* pixels, int32_t* labels,
                          uint64_t max_records, uint64_t* n_records);

/* ---------------------------------------------------------------- E-D pipeline
 * The encode-while-train data path (replaces pipeline.cpp:37-97 HandoffSlot,
 * :116-129 prepare_epoch, :181-244 run): each step gathers the SBS-drawn rows
 * of `dataset` (device memory, or pinned host memory read zero-copy), encodes
 * them into the pipeline's containers and decodes them with `epilogue` into
 * the caller's layer-input buffer, all on the caller's stream; the draws of
 * the next step run meanwhile on a side stream (two draw buffers, event
 * hand-off, no host synchronisation).  `layout` describes one step of this
 * shard: layout.n_batches of the global stream's layout.n_batches*n_shards
 * batches per step (those with index % n_shards == shard).  With class
 * tables in the epilogue and row_class NULL, the step's own draw classes are
 * used (per-class preprocessing). */
typedef struct optb_pipeline optb_pipeline;
typedef struct optb_pipeline_desc {
  optb_layout layout;
  const uint8_t* dataset;
  uint64_t row_stride;
  optb_sbs* sbs;
  uint32_t shard, n_shards;
  optb_epilogue epilogue;
  int32_t record_timings;  /* keep per-step CUDA events for optb_pipeline_timings */
  uint32_t steps_per_draw; /* SBS calls cover this many steps (0 = 1): amortises the
                              per-call reshuffle work when steps are short */
  uint32_t split_kernels;  /* 1: separate encode and decode launches per step;
                              0: optb_roundtrip_dev (one launch where it applies) */
  uint32_t timing_stride;  /* with record_timings: time every timing_stride-th step
                              only (0 = 1); events between launches stop consecutive
                              round trips from overlapping their launch ramps */
} optb_pipeline_desc;

int optb_pipeline_create(optb_ctx* ctx, const optb_pipeline_desc* desc, optb_pipeline** out);
/* Warm start (pipeline.cpp:154-177, PipelineConfig::warm_start): the epoch
 * dumped as <dir>/batch_<epoch>_<k>.optb is loaded and validated once
 * (optb_load_dev) into the pipeline's device planes; every step then only
 * decodes it with `epilogue` into the caller's buffer -- no sampler, no
 * encode.  Class tables need epilogue->row_class (there are no draws). */
int optb_pipeline_create_warm(optb_ctx* ctx, const optb_layout* layout, uint32_t h, uint32_t w, uint32_t c,
                              const char* dir, uint64_t epoch, const optb_epilogue* epilogue,
                              int32_t record_timings, optb_pipeline** out);
/* Enqueue the next step; `out` receives optb_layout_rows(layout) decoded rows. */
int optb_pipeline_step(optb_pipeline* p, void* out, void* stream);
/* Rows for subsequent steps come from `dataset` (e.g. a double-buffered
 * device copy of a host dataset refreshed by the caller every step). */
int optb_pipeline_set_dataset(optb_pipeline* p, const uint8_t* dataset, uint64_t row_stride);
/* Device draws (examples, classes) of a step still buffered (the last two
 * sampler calls; three when n_shards >= 4, where the sampler runs two calls
 * ahead). */
int optb_pipeline_draws(const optb_pipeline* p, uint64_t step, const int64_t** examples,
                        const int32_t** classes);
/* The pipeline's container planes (valid for the last enqueued step). */
const void* optb_pipeline_containers(const optb_pipeline* p);
/* The same step on host buffers (the E-D path for a dataset in host memory,
 * as the reference's pipeline::run consumes an in-memory Dataset and hands
 * decoded batches to the trainer, pipeline.cpp:181-244 / runner.cpp:264-311):
 * uploads dataset_host ([n_rows][row_stride] u8, pinned for overlap) into one
 * of two internal device buffers on a copy stream, runs optb_pipeline_step
 * on `stream` into an internal device buffer, and copies the decoded rows to
 * out_host (layout as optb_pipeline_step's `out`) on a second copy stream.
 * Asynchronous: consecutive calls overlap the upload of step k+1, the kernels
 * and the download of step k.  out_host is complete after
 * optb_pipeline_host_wait. */
int optb_pipeline_step_host(optb_pipeline* p, const uint8_t* dataset_host, uint64_t n_rows,
                            uint64_t row_stride, void* out_host, void* stream);
/* Wait for every download enqueued by optb_pipeline_step_host: on the host
 * (stream NULL), or by making `stream` wait for the last one. */
int optb_pipeline_host_wait(optb_pipeline* p, void* stream);
/* Device-timed durations (ms) of a completed, timed step (a multiple of
 * timing_stride, among the last 64 * timing_stride steps): its SBS draws
 * (side stream; the call that produced them, per step), its gather-encode
 * and its decode (for a fused round-trip step: the whole launch in enc_ms
 * and 0 in dec_ms). */
int optb_pipeline_timings(const optb_pipeline* p, uint64_t step, float* sbs_ms, float* enc_ms,
                          float* dec_ms);
void optb_pipeline_destroy(optb_pipeline* p);

/* ---------------------------------------------------------------- synthetic data
 * Counter-based u8 rows (bench / tests): w = mix(seed + (e*ceil(P/8) + p/8 + 1)*gamma),
 * pixel = (w >> 8*(p%8)) & 0xff for dataset row e = first_row + r. */
int optb_synth_pixels_dev(optb_ctx* ctx, uint64_t seed, uint64_t first_row, uint64_t n_rows,
                          uint64_t pixels, uint8_t* out, uint64_t row_stride, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OPTB_CUDA_H */
