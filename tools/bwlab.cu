// bwlab.cu -- design-space probe for the exact128 codec kernels on B200.
//
// Times, back to back in the bench's two-kernel pattern (dataset -> containers
// -> rows, C2 shapes: 3104 chunks x 16 images x 3072 pixels), a set of
// memory-movement designs so the codec kernels can be built on the fastest:
//   copy_v4      grid-stride 128-bit copy (ceiling of a plain LSU kernel)
//   copy_bulk    per-warp 1D cp.async.bulk load + bulk store through smem
//   enc_tma      exact128 gather-encode: 16 bulk row loads per tile, register
//                transpose, SWIZZLE_128B smem tile, 2D tensor TMA store
//   dec_tma      exact128 decode -> u8: 2D tensor TMA load (SWIZZLE_128B),
//                register transpose, direct coalesced row stores (or a 2D
//                TMA store of the rows with -DDEC_TMA_STORE)
// and checks enc_tma/dec_tma against the definition (round trip + packed bytes).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bwlab.cu -o build/bwlab
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void t4x4(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
  a0 = __byte_perm(t0, t2, 0x5410);
  a1 = __byte_perm(t0, t2, 0x7632);
  a2 = __byte_perm(t1, t3, 0x5410);
  a3 = __byte_perm(t1, t3, 0x7632);
}
__device__ __forceinline__ void transpose16(uint32_t (&m)[16][4]) {
  uint32_t t[16][4];
#pragma unroll
  for (int R = 0; R < 4; ++R)
#pragma unroll
    for (int Q = 0; Q < 4; ++Q) {
      uint32_t a0 = m[4 * R][Q], a1 = m[4 * R + 1][Q], a2 = m[4 * R + 2][Q], a3 = m[4 * R + 3][Q];
      t4x4(a0, a1, a2, a3);
      t[4 * Q][R] = a0;
      t[4 * Q + 1][R] = a1;
      t[4 * Q + 2][R] = a2;
      t[4 * Q + 3][R] = a3;
    }
#pragma unroll
  for (int r = 0; r < 16; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) m[r][q] = t[r][q];
}

// ------------------------------------------------------------------ copies
template <int U>
__global__ void __launch_bounds__(256) copy_v4(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(b + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) b[i] = a[i];
}


// two phases in one launch: every warp copies its tiles a->b, then the same
// tiles b->c (no cross-warp dependency: a warp only reads back what it wrote)
template <int U>
__global__ void __launch_bounds__(256) copy2_v4(const uint4* __restrict__ a, uint4* __restrict__ b,
                                                uint4* __restrict__ c, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t i = i0;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) b[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) b[i] = a[i];
  i = i0;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = b[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(c + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) c[i] = b[i];
}

// per-warp ring of S slots of T bytes: bulk load -> bulk store
template <int W, int S, int T>
__global__ void __launch_bounds__(W * 32, 1) copy_bulk(const uint8_t* a, uint8_t* b, uint64_t tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[W][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + warp * S * T;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t stride = (uint64_t)gridDim.x * W;
  const uint64_t first = (uint64_t)blockIdx.x * W + warp;
  if (lane == 0) {
    for (int s = 0; s < S - 1; ++s) {
      const uint64_t t = first + s * stride;
      if (t < tiles) {
        mbar_expect_tx(&bars[warp][s], T);
        bulk_g2s(ring + s * T, a + t * T, T, &bars[warp][s]);
      }
    }
    uint32_t phase = 0;
    int st = 0;
    for (uint64_t t = first, it = 0; t < tiles; t += stride, ++it) {
      const uint64_t tn = t + (S - 1) * stride;
      const int sn = (st + S - 1) % S;
      if (tn < tiles) {
        bulk_wait_read<S - 2>();  // the store that last used slot sn has read it
        mbar_expect_tx(&bars[warp][sn], T);
        bulk_g2s(ring + sn * T, a + tn * T, T, &bars[warp][sn]);
      }
      mbar_wait(&bars[warp][st], phase);
      bulk_s2g(b + t * T, ring + st * T, T);
      bulk_commit();
      if (++st == S) {
        st = 0;
        phase ^= 1;
      }
    }
    bulk_wait_all();
  }
}

// ------------------------------------------------------------------ exact128 TMA codec
// Geometry: chunks of 16 images x P pixels (P % 512 == 0); tile = 512 pixels
// of one chunk; container tile = 8 KB contiguous at byte (k*P + pb)*16.
struct G {
  uint64_t chunks, P, tpc;  // tiles per chunk = P / 512
};

// conflict-free order for the SWIZZLE_128B container tile: lane L's word p
// (r = 2L + p/8, c = p%8) sits at r*128 + ((c ^ (r & 7)) * 16); at step s lane
// L touches p = s ^ (((L >> 2) & 1) << 3), so the 8 lanes of a quarter-warp
// hit 8 distinct 16-byte bank groups.
__device__ __forceinline__ uint32_t swz_off(int L, int p) {
  const int r = 2 * L + (p >> 3), c = p & 7;
  return r * 128 + ((c ^ (r & 7)) << 4);
}

template <int W, int S>
__global__ void __launch_bounds__(W * 32, 1)
    enc_tma(const __grid_constant__ CUtensorMap cmap, G g, const uint8_t* __restrict__ images, uint64_t stride_b,
            const int64_t* __restrict__ row_index) {
  constexpr int T = 8192;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[W][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + warp * (S + 2) * T;  // S input slots + 2 output slots
  uint8_t* outs = ring + S * T;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t tiles = g.chunks * g.tpc;
  const uint64_t stride = (uint64_t)gridDim.x * W;
  const uint64_t first = (uint64_t)blockIdx.x * W + warp;
  auto issue = [&](uint64_t t, int s) {
    if (t >= tiles) return;
    const uint64_t k = t / g.tpc, pb = (t - k * g.tpc) * 512;
    if (lane == 0) mbar_expect_tx(&bars[warp][s], 16 * 512);
    __syncwarp();
    if (lane < 16) {
      const int64_t r = __ldg(row_index + k * 16 + lane);
      bulk_g2s(ring + s * T + lane * 512, images + (uint64_t)r * stride_b + pb, 512, &bars[warp][s]);
    }
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(first + s * stride, s);
  uint32_t phase = 0;
  int st = 0, ob = 0;
  for (uint64_t t = first; t < tiles; t += stride) {
    issue(t + (S - 1) * stride, (st + S - 1) % S);
    mbar_wait(&bars[warp][st], phase);
    const uint8_t* slot = ring + st * T;
    uint32_t m[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint4 v = *reinterpret_cast<const uint4*>(slot + i * 512 + lane * 16);
      m[i][0] = v.x;
      m[i][1] = v.y;
      m[i][2] = v.z;
      m[i][3] = v.w;
    }
    transpose16(m);  // m[p] = word of pixel 16*lane + p
    // output slot ob: the store issued two tiles ago from it must have read it
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    uint8_t* o = outs + ob * T;
    const bool hi = (lane >> 2) & 1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int pa = hi ? j + 8 : j, pb2 = hi ? j : j + 8;
      uint4 a, b;
      a.x = hi ? m[j + 8][0] : m[j][0];
      a.y = hi ? m[j + 8][1] : m[j][1];
      a.z = hi ? m[j + 8][2] : m[j][2];
      a.w = hi ? m[j + 8][3] : m[j][3];
      b.x = hi ? m[j][0] : m[j + 8][0];
      b.y = hi ? m[j][1] : m[j + 8][1];
      b.z = hi ? m[j][2] : m[j + 8][2];
      b.w = hi ? m[j][3] : m[j + 8][3];
      *reinterpret_cast<uint4*>(o + swz_off(lane, pa)) = a;
      *reinterpret_cast<uint4*>(o + swz_off(lane, pb2)) = b;
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      const uint64_t k = t / g.tpc, pb = (t - k * g.tpc) * 512;
      tma_store2d(&cmap, o, 0, (int)((k * g.P + pb) * 16 / 128));
      bulk_commit();
    }
    ob ^= 1;
    if (++st == S) {
      st = 0;
      phase ^= 1;
    }
  }
  if (lane == 0) bulk_wait_all();
}

template <int W, int S, bool TSTORE>
__global__ void __launch_bounds__(W * 32, 1)
    dec_tma(const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap omap, G g,
            uint8_t* __restrict__ out, uint64_t stride_b) {
  constexpr int T = 8192;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[W][S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + warp * (S + (TSTORE ? 2 : 0)) * T;
  uint8_t* outs = ring + S * T;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t tiles = g.chunks * g.tpc;
  const uint64_t stride = (uint64_t)gridDim.x * W;
  const uint64_t first = (uint64_t)blockIdx.x * W + warp;
  auto issue = [&](uint64_t t, int s) {
    if (t < tiles && lane == 0) {
      const uint64_t k = t / g.tpc, pb = (t - k * g.tpc) * 512;
      mbar_expect_tx(&bars[warp][s], T);
      tma_load2d(ring + s * T, &cmap, 0, (int)((k * g.P + pb) * 16 / 128), &bars[warp][s]);
    }
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(first + s * stride, s);
  uint32_t phase = 0;
  int st = 0, ob = 0;
  for (uint64_t t = first; t < tiles; t += stride) {
    issue(t + (S - 1) * stride, (st + S - 1) % S);
    mbar_wait(&bars[warp][st], phase);
    const uint8_t* slot = ring + st * T;
    uint32_t m[16][4];
    const bool hi = (lane >> 2) & 1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int pa = hi ? j + 8 : j, pb2 = hi ? j : j + 8;
      const uint4 a = *reinterpret_cast<const uint4*>(slot + swz_off(lane, pa));
      const uint4 b = *reinterpret_cast<const uint4*>(slot + swz_off(lane, pb2));
      m[j][0] = hi ? b.x : a.x;
      m[j][1] = hi ? b.y : a.y;
      m[j][2] = hi ? b.z : a.z;
      m[j][3] = hi ? b.w : a.w;
      m[j + 8][0] = hi ? a.x : b.x;
      m[j + 8][1] = hi ? a.y : b.y;
      m[j + 8][2] = hi ? a.z : b.z;
      m[j + 8][3] = hi ? a.w : b.w;
    }
    transpose16(m);  // m[i] = 16 pixels of image i
    const uint64_t k = t / g.tpc, pb = (t - k * g.tpc) * 512;
    if constexpr (TSTORE) {
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      uint8_t* o = outs + ob * T;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        *reinterpret_cast<uint4*>(o + i * 512 + lane * 16) = make_uint4(m[i][0], m[i][1], m[i][2], m[i][3]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store2d(&omap, o, (int)(pb / 4), (int)(k * 16));
        bulk_commit();
      }
      ob ^= 1;
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint4 v = make_uint4(m[i][0], m[i][1], m[i][2], m[i][3]);
        asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + (k * 16 + i) * stride_b + pb + lane * 16),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
    }
    __syncwarp();
    if (++st == S) {
      st = 0;
      phase ^= 1;
    }
  }
  if (TSTORE && lane == 0) bulk_wait_all();
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encodeTiled() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap map_cont(void* base, uint64_t bytes) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, bytes / 128};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, 64};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encodeTiled()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "map_cont %d\n", (int)r);
    exit(1);
  }
  return m;
}
static CUtensorMap map_rows(void* base, uint64_t rows, uint64_t P) {
  CUtensorMap m;
  cuuint64_t dims[2] = {P / 4, rows};
  cuuint64_t strides[1] = {P};
  cuuint32_t box[2] = {128, 16};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encodeTiled()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "map_rows %d\n", (int)r);
    exit(1);
  }
  return m;
}

struct Timer {
  std::vector<cudaEvent_t> ev;
  Timer(int n) : ev(n) {
    for (auto& e : ev) cudaEventCreate(&e);
  }
};

// Run `A` then `B` alternately `reps` times; report per-kernel average us.
template <typename FA, typename FB>
static void pair(const char* name, FA A, FB B, double bytesA, double bytesB, int reps = 40) {
  for (int i = 0; i < 5; ++i) {
    A();
    B();
  }
  CK(cudaDeviceSynchronize());
  std::vector<cudaEvent_t> ev(2 * reps + 1);
  for (auto& e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[0]);
  for (int i = 0; i < reps; ++i) {
    A();
    cudaEventRecord(ev[2 * i + 1]);
    B();
    cudaEventRecord(ev[2 * i + 2]);
  }
  CK(cudaEventSynchronize(ev.back()));
  CK(cudaGetLastError());
  double ta = 0, tb = 0;
  for (int i = 0; i < reps; ++i) {
    float x, y;
    cudaEventElapsedTime(&x, ev[2 * i], ev[2 * i + 1]);
    cudaEventElapsedTime(&y, ev[2 * i + 1], ev[2 * i + 2]);
    ta += x;
    tb += y;
  }
  ta = ta / reps * 1e3;
  tb = tb / reps * 1e3;
  printf("{\"name\": \"%s\", \"a_us\": %.2f, \"b_us\": %.2f, \"a_gbs\": %.1f, \"b_gbs\": %.1f, \"step_gbs\": %.1f}\n",
         name, ta, tb, bytesA / ta / 1e3, bytesB / tb / 1e3, (bytesA + bytesB) / (ta + tb) / 1e3);
  fflush(stdout);
  for (auto& e : ev) cudaEventDestroy(e);
}

int main(int argc, char** argv) {
  const uint64_t N = 50000, P = 3072, B = 512, NB = 97;
  const uint64_t rows = B * NB, chunks = rows / 16;
  const uint64_t cbytes = chunks * P * 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *ds, *cont, *out;
  int64_t* idx;
  CK(cudaMalloc(&ds, N * P));
  CK(cudaMalloc(&cont, cbytes));
  CK(cudaMalloc(&out, rows * P));
  CK(cudaMalloc(&idx, rows * 8));
  {
    std::vector<uint8_t> h(N * P);
    uint64_t s = 12345;
    for (auto& x : h) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      x = (uint8_t)(s >> 33);
    }
    CK(cudaMemcpy(ds, h.data(), h.size(), cudaMemcpyHostToDevice));
    std::vector<int64_t> hi(rows);
    for (uint64_t r = 0; r < rows; ++r) hi[r] = (int64_t)((r * 7919 + 13) % N);
    CK(cudaMemcpy(idx, hi.data(), rows * 8, cudaMemcpyHostToDevice));
  }
  const double bytes = (double)rows * P * 2;  // read + write of one side

  {  // copy size sweep (one buffer pair, back to back) and the two-phase fused copy
    uint8_t *x, *y, *z;
    const uint64_t big = 2400ull << 20;
    CK(cudaMalloc(&x, big));
    CK(cudaMalloc(&y, big));
    CK(cudaMalloc(&z, big));
    CK(cudaMemset(x, 1, big));
    for (uint64_t mb : {38ull, 152ull, 610ull, 2400ull}) {
      const uint64_t n = (mb << 20) / 16;
      char nm[64];
      snprintf(nm, sizeof nm, "copy_v4 %lluMB grid=148*16", (unsigned long long)mb);
      pair(nm, [&] { copy_v4<4><<<sms * 16, 256>>>((const uint4*)x, (uint4*)y, n); },
           [&] { copy_v4<4><<<sms * 16, 256>>>((const uint4*)y, (uint4*)z, n); }, 2.0 * (mb << 20), 2.0 * (mb << 20),
           mb > 1000 ? 6 : 30);
    }
    for (int k : {4, 8, 16}) {
      const uint64_t n = rows * P / 16;
      char nm[64];
      snprintf(nm, sizeof nm, "copy2_v4 fused two-phase 152MB grid=148*%d", k);
      pair(nm, [&] { copy2_v4<4><<<sms * k, 256>>>((const uint4*)ds, (uint4*)cont, (uint4*)out, n); },
           [&] {}, 4.0 * rows * P, 1.0);
    }
    CK(cudaFree(x));
    CK(cudaFree(y));
    CK(cudaFree(z));
  }
  // plain copies (dataset rows -> cont buffer -> out)
  for (int k : {1, 2, 4, 8, 16}) {
    const int grid = sms * k;
    char nm[64];
    snprintf(nm, sizeof nm, "copy_v4x4 grid=%d*%d", sms, k);
    pair(nm, [&] { copy_v4<4><<<grid, 256>>>((const uint4*)ds, (uint4*)cont, rows * P / 16); },
         [&] { copy_v4<4><<<grid, 256>>>((const uint4*)cont, (uint4*)out, rows * P / 16); }, bytes, bytes);
  }
  {
    constexpr int W = 4, S = 6, T = 8192;
    const size_t sm = (size_t)W * S * T;
    CK(cudaFuncSetAttribute(copy_bulk<W, S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const uint64_t tiles = rows * P / T;
    pair("copy_bulk W4 S6 8K", [&] { copy_bulk<W, S, T><<<sms, W * 32, sm>>>(ds, cont, tiles); },
         [&] { copy_bulk<W, S, T><<<sms, W * 32, sm>>>(cont, out, tiles); }, bytes, bytes);
  }
  {
    constexpr int W = 8, S = 3, T = 8192;
    const size_t sm = (size_t)W * S * T;
    CK(cudaFuncSetAttribute(copy_bulk<W, S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const uint64_t tiles = rows * P / T;
    pair("copy_bulk W8 S3 8K", [&] { copy_bulk<W, S, T><<<sms, W * 32, sm>>>(ds, cont, tiles); },
         [&] { copy_bulk<W, S, T><<<sms, W * 32, sm>>>(cont, out, tiles); }, bytes, bytes);
  }
  G g{chunks, P, P / 512};
  CUtensorMap cm = map_cont(cont, cbytes);
  CUtensorMap om = map_rows(out, rows, P);
  const double eb = (double)rows * P * 2 + rows * 8, db = (double)rows * P * 2;
#define RUN_CODEC(W, S, TS)                                                                                  \
  {                                                                                                          \
    const size_t se = (size_t)W * (S + 2) * 8192, sd = (size_t)W * (S + (TS ? 2 : 0)) * 8192;              \
    CK(cudaFuncSetAttribute(enc_tma<W, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)se));          \
    CK(cudaFuncSetAttribute(dec_tma<W, S, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd));      \
    int be = 0, bd = 0;                                                                                      \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&be, enc_tma<W, S>, W * 32, se);                          \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bd, dec_tma<W, S, TS>, W * 32, sd);                      \
    char nm[96];                                                                                             \
    snprintf(nm, sizeof nm, "tma_codec W%d S%d tstore=%d blocks/SM enc %d dec %d", W, S, TS, be, bd);      \
    pair(nm, [&] { enc_tma<W, S><<<sms * be, W * 32, se>>>(cm, g, ds, P, idx); },                           \
         [&] { dec_tma<W, S, TS><<<sms * bd, W * 32, sd>>>(cm, om, g, out, P); }, eb, db);                \
  }
  RUN_CODEC(4, 4, false)
  RUN_CODEC(4, 4, true)
  RUN_CODEC(2, 6, false)
  RUN_CODEC(4, 3, false)
  RUN_CODEC(2, 4, false)
  RUN_CODEC(1, 8, false)
  RUN_CODEC(6, 3, false)
  // correctness of the last configuration: rows round trip, container bytes
  {
    CK(cudaMemset(out, 0, rows * P));
    constexpr int W = 4, S = 4;
    const size_t se = (size_t)W * (S + 2) * 8192, sd = (size_t)W * S * 8192;
    enc_tma<W, S><<<sms, W * 32, se>>>(cm, g, ds, P, idx);
    dec_tma<W, S, false><<<sms, W * 32, sd>>>(cm, om, g, out, P);
    CK(cudaDeviceSynchronize());
    std::vector<uint8_t> hd(N * P), hc(cbytes), ho(rows * P);
    std::vector<int64_t> hi(rows);
    CK(cudaMemcpy(hd.data(), ds, N * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hc.data(), cont, cbytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho.data(), out, rows * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hi.data(), idx, rows * 8, cudaMemcpyDeviceToHost));
    uint64_t bad_rows = 0, bad_cont = 0;
    for (uint64_t r = 0; r < rows; ++r)
      if (memcmp(ho.data() + r * P, hd.data() + hi[r] * P, P)) ++bad_rows;
    for (uint64_t k = 0; k < chunks; k += 7)
      for (uint64_t p = 0; p < P; ++p)
        for (int i = 0; i < 16; ++i)
          if (hc[(k * P + p) * 16 + i] != hd[hi[k * 16 + i] * P + p]) ++bad_cont;
    printf("{\"check\": \"tma_codec\", \"bad_rows\": %llu, \"bad_container_bytes\": %llu}\n",
           (unsigned long long)bad_rows, (unsigned long long)bad_cont);
  }
  {  // 2D TMA store variant check
    CK(cudaMemset(out, 0, rows * P));
    constexpr int W = 4, S = 4;
    const size_t sd = (size_t)W * (S + 2) * 8192;
    dec_tma<W, S, true><<<sms, W * 32, sd>>>(cm, om, g, out, P);
    CK(cudaDeviceSynchronize());
    std::vector<uint8_t> hd(N * P), ho(rows * P);
    std::vector<int64_t> hi(rows);
    CK(cudaMemcpy(hd.data(), ds, N * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho.data(), out, rows * P, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hi.data(), idx, rows * 8, cudaMemcpyDeviceToHost));
    uint64_t bad_rows = 0;
    for (uint64_t r = 0; r < rows; ++r)
      if (memcmp(ho.data() + r * P, hd.data() + hi[r] * P, P)) ++bad_rows;
    printf("{\"check\": \"dec_tma_tstore\", \"bad_rows\": %llu}\n", (unsigned long long)bad_rows);
  }
  return 0;
}
