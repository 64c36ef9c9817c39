// mixlab.cu -- HBM bandwidth of plain streaming kernels by read:write mix, the
// ceiling for a kernel whose compulsory DRAM traffic has that mix.
//
// The interleaved fused round trip (k_roundtrip_il) moves, per step, the
// gathered rows in and the containers + decoded rows out: one byte read for
// every two written.  This probe times, on buffers far larger than L2 (so
// every byte is a DRAM byte), grid-stride 16-byte kernels that
//   read     read R bytes (sum, one word written per CTA)
//   write    write W bytes
//   copy     read N, write N           (1:1, the MEASURED_PEAKS copy shape)
//   r1w2     read N, write 2N          (the round trip's compulsory mix)
//   r1w3     read N, write 3N
//   bulk_*   the copy / r1w2 mixes moved by the bulk-copy (TMA) engine
//   bulkld_* bulk loads into shared memory, 16-byte LSU stores out
// each back to back over 3 rotating buffer sets (the next launch never finds
// its inputs in L2), CUDA events, median of 20.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mixlab.cu -o build/mixlab
//   build/mixlab [MB]       # one JSON line per kernel and grid; MB = input
//                           # bytes per launch (default one C2 step, 152.6;
//                           # 3221 = one C5 epoch), plus cudaMemcpyAsync D2D
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

__device__ __forceinline__ uint4 ld(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st(uint4* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

constexpr int U = 4;  // 16-byte accesses in flight per thread per stream

// NW output streams per input stream (NR = 0: write-only; NW = 0: read-only)
template <int NR, int NW>
__global__ void __launch_bounds__(256) k_mix(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n16,
                                             uint32_t* sink) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t b = tid; b < n16; b += nt * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * nt;
      v[u] = make_uint4(static_cast<uint32_t>(i), 1u, 2u, 3u);
      if (NR && i < n16) v[u] = ld(in + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * nt;
      if (i < n16) {
#pragma unroll
        for (int w = 0; w < NW; ++w) st(out + w * n16 + i, v[u]);
        acc ^= v[u].x ^ v[u].w;
      }
    }
  }
  if (NW == 0 && acc == 0x9e3779b9u) sink[0] = acc;  // keeps the loads
}

// The same mixes moved by the bulk-copy (TMA) engine instead of LSU
// instructions: one thread per CTA streams contiguous CH-byte chunks through
// an S-stage shared-memory ring -- a 1D bulk load on the stage's mbarrier,
// then NW bulk stores of the stage; a stage is refilled once the stores of
// the iteration before have read it (cp.async.bulk.wait_group.read 1).
constexpr uint32_t kCh = 16384;
constexpr int kS = 4;
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int NW>
__global__ void __launch_bounds__(32) k_bulk(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                             uint64_t nbytes) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bar[kS];
  if (threadIdx.x != 0) return;
  const uint64_t nch = nbytes / kCh;
  for (int s = 0; s < kS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto load = [&](uint64_t c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(kCh) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(ring + s * kCh)), "l"(in + c * kCh), "r"(kCh), "r"(su32(bar + s)) : "memory");
  };
  uint64_t c0 = blockIdx.x;
  for (int s = 0; s < kS && c0 + s * gridDim.x < nch; ++s) load(c0 + s * gridDim.x, s);
  uint32_t phase = 0;
  int it = 0;
  for (uint64_t c = c0; c < nch; c += gridDim.x, ++it) {
    const int s = it % kS;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                 ::"r"(su32(bar + s)), "r"((phase >> s) & 1u) : "memory");
    phase ^= 1u << s;
#pragma unroll
    for (int w = 0; w < NW; ++w)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(out + w * nbytes + c * kCh), "r"(su32(ring + s * kCh)), "r"(kCh) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (it >= 1) {  // refill the previous iteration's stage once its stores have read it
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint64_t cn = c - gridDim.x + kS * static_cast<uint64_t>(gridDim.x);
      if (cn < nch) load(cn, (it - 1) % kS);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Bulk (TMA) loads, LSU stores: 128 threads; thread 0 streams CH-byte chunks
// into the ring, every thread then stores its 128 bytes of the stage to the
// NW outputs with 16-byte st.global.
template <int NW>
__global__ void __launch_bounds__(128) k_bulkld(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                                uint64_t nbytes) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bar[kS];
  const uint64_t nch = nbytes / kCh;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto load = [&](uint64_t c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(kCh) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(ring + s * kCh)), "l"(in + c * kCh), "r"(kCh), "r"(su32(bar + s)) : "memory");
  };
  const uint64_t c0 = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < kS && c0 + s * gridDim.x < nch; ++s) load(c0 + s * gridDim.x, s);
  uint32_t phase = 0;
  int it = 0;
  for (uint64_t c = c0; c < nch; c += gridDim.x, ++it) {
    const int s = it % kS;
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                 ::"r"(su32(bar + s)), "r"((phase >> s) & 1u) : "memory");
    phase ^= 1u << s;
#pragma unroll
    for (int u = 0; u < static_cast<int>(kCh / (128 * 16)); ++u) {
      const uint32_t off = (u * 128 + threadIdx.x) * 16;
      const uint4 v = *reinterpret_cast<const uint4*>(ring + s * kCh + off);
#pragma unroll
      for (int w = 0; w < NW; ++w) st(reinterpret_cast<uint4*>(out + w * nbytes + c * kCh + off), v);
    }
    __syncthreads();  // every thread has read the stage
    const uint64_t cn = c + kS * static_cast<uint64_t>(gridDim.x);
    if (threadIdx.x == 0 && cn < nch) load(cn, s);
  }
}

template <int NW>
void run_bulkld(const char* name, int sms, int per_sm, uint64_t n16, std::vector<uint4*>& ins,
                std::vector<uint4*>& outs) {
  const int grid = sms * per_sm;
  const size_t smem = kS * kCh;
  CK(cudaFuncSetAttribute(k_bulkld<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t ev[21];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  const int sets = static_cast<int>(ins.size());
  const uint64_t nb = n16 * 16 / kCh * kCh;
  auto go = [&](int i) {
    k_bulkld<NW><<<grid, 128, smem>>>(reinterpret_cast<const uint8_t*>(ins[i % sets]),
                                      reinterpret_cast<uint8_t*>(outs[i % sets]), nb);
  };
  for (int i = 0; i < 3; ++i) go(i);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(ev[0]));
  for (int i = 0; i < 20; ++i) {
    go(i);
    CK(cudaEventRecord(ev[i + 1]));
  }
  CK(cudaEventSynchronize(ev[20]));
  CK(cudaGetLastError());
  std::vector<float> t;
  for (int i = 0; i < 20; ++i) {
    float ms;
    CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  const double us = t[10] * 1e3;
  const double rb = static_cast<double>(nb), wb = static_cast<double>(NW) * nb;
  printf("{\"kernel\": \"%s\", \"grid\": \"%dx%d\", \"read_mb\": %.1f, \"write_mb\": %.1f, \"us\": %.2f, \"gbs\": %.1f}\n",
         name, sms, per_sm, rb / 1e6, wb / 1e6, us, (rb + wb) / us / 1e3);
  for (auto& e : ev) CK(cudaEventDestroy(e));
}

template <int NW>
void run_bulk(const char* name, int sms, int per_sm, uint64_t n16, std::vector<uint4*>& ins, std::vector<uint4*>& outs) {
  const int grid = sms * per_sm;
  const size_t smem = kS * kCh;
  CK(cudaFuncSetAttribute(k_bulk<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t ev[21];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  const int sets = static_cast<int>(ins.size());
  const uint64_t nb = n16 * 16 / kCh * kCh;
  auto go = [&](int i) {
    k_bulk<NW><<<grid, 32, smem>>>(reinterpret_cast<const uint8_t*>(ins[i % sets]),
                                   reinterpret_cast<uint8_t*>(outs[i % sets]), nb);
  };
  for (int i = 0; i < 3; ++i) go(i);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(ev[0]));
  for (int i = 0; i < 20; ++i) {
    go(i);
    CK(cudaEventRecord(ev[i + 1]));
  }
  CK(cudaEventSynchronize(ev[20]));
  CK(cudaGetLastError());
  std::vector<float> t;
  for (int i = 0; i < 20; ++i) {
    float ms;
    CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  const double us = t[10] * 1e3;
  const double rb = static_cast<double>(nb), wb = static_cast<double>(NW) * nb;
  printf("{\"kernel\": \"%s\", \"grid\": \"%dx%d\", \"read_mb\": %.1f, \"write_mb\": %.1f, \"us\": %.2f, \"gbs\": %.1f}\n",
         name, sms, per_sm, rb / 1e6, wb / 1e6, us, (rb + wb) / us / 1e3);
  for (auto& e : ev) CK(cudaEventDestroy(e));
}

template <int NR, int NW>
void run(const char* name, int sms, int per_sm, uint64_t n16, std::vector<uint4*>& ins, std::vector<uint4*>& outs,
         uint32_t* sink) {
  const int grid = sms * per_sm;
  cudaEvent_t ev[21];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  const int sets = static_cast<int>(ins.size());
  for (int i = 0; i < 3; ++i) k_mix<NR, NW><<<grid, 256>>>(ins[i % sets], outs[i % sets], n16, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(ev[0]));
  for (int i = 0; i < 20; ++i) {
    k_mix<NR, NW><<<grid, 256>>>(ins[i % sets], outs[i % sets], n16, sink);
    CK(cudaEventRecord(ev[i + 1]));
  }
  CK(cudaEventSynchronize(ev[20]));
  std::vector<float> t;
  for (int i = 0; i < 20; ++i) {
    float ms;
    CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  const double us = t[10] * 1e3;
  const double rb = static_cast<double>(NR) * n16 * 16, wb = static_cast<double>(NW) * n16 * 16;
  printf("{\"kernel\": \"%s\", \"grid\": \"%dx%d\", \"read_mb\": %.1f, \"write_mb\": %.1f, \"us\": %.2f, \"gbs\": %.1f}\n",
         name, sms, per_sm, rb / 1e6, wb / 1e6, us, (rb + wb) / us / 1e3);
  for (auto& e : ev) CK(cudaEventDestroy(e));
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  uint64_t n16 = 152567808ull / 16;  // one C2 step's rows (49664 x 3072 B)
  if (argc > 1) n16 = static_cast<uint64_t>(atof(argv[1]) * 1e6) / 16;
  // rotate over enough buffer sets that a launch never finds its inputs in L2
  const int sets = n16 * 16 > (1ull << 30) ? 2 : 3;
  std::vector<uint4*> ins(sets), outs(sets);
  for (int s = 0; s < sets; ++s) {
    CK(cudaMalloc(&ins[s], n16 * 16));
    CK(cudaMalloc(&outs[s], 3 * n16 * 16));
    CK(cudaMemset(ins[s], s + 1, n16 * 16));
    CK(cudaMemset(outs[s], 0, 3 * n16 * 16));
  }
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4));
  {  // the driver's copy: cudaMemcpyAsync device to device
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) CK(cudaMemcpyAsync(outs[i % sets], ins[i % sets], n16 * 16, cudaMemcpyDeviceToDevice));
    std::vector<float> t;
    for (int i = 0; i < 10; ++i) {
      CK(cudaEventRecord(a));
      CK(cudaMemcpyAsync(outs[i % sets], ins[i % sets], n16 * 16, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    printf("{\"kernel\": \"memcpy_d2d\", \"read_mb\": %.1f, \"write_mb\": %.1f, \"us\": %.2f, \"gbs\": %.1f}\n",
           n16 * 16 / 1e6, n16 * 16 / 1e6, t[0] * 1e3, 2.0 * n16 * 16 / (t[0] * 1e3) / 1e3);
  }
  for (int per_sm : {2, 3}) {  // 64 KB rings: at most 3 CTAs per SM
    run_bulk<1>("bulk_copy", sms, per_sm, n16, ins, outs);
    run_bulk<2>("bulk_r1w2", sms, per_sm, n16, ins, outs);
    run_bulkld<1>("bulkld_copy", sms, per_sm, n16, ins, outs);
    run_bulkld<2>("bulkld_r1w2", sms, per_sm, n16, ins, outs);
  }
  for (int per_sm : {4, 8, 16}) {
    run<1, 0>("read", sms, per_sm, n16, ins, outs, sink);
    run<0, 1>("write", sms, per_sm, n16, ins, outs, sink);
    run<1, 1>("copy", sms, per_sm, n16, ins, outs, sink);
    run<1, 2>("r1w2", sms, per_sm, n16, ins, outs, sink);
    run<1, 3>("r1w3", sms, per_sm, n16, ins, outs, sink);
  }
  return 0;
}
