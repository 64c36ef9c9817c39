// peer.cu -- dataset-sharded gather over peer memory.
//
// When every rank holds only rows [r*per, (r+1)*per) of the dataset, the
// reference's gather (Dataset::image_of, dataset.cpp:16-22, driven by
// runner.cpp:77-90) needs rows that live on other GPUs.  Instead of an
// all-to-all of rows into a staging buffer followed by the gather-encode,
// every rank maps its peers' shards into its own address space (CUDA IPC;
// NVLink / NVSwitch peer access) and the gather-encode kernel itself loads
// each drawn row from wherever it lives: one kernel moves the bytes across
// NVLink and packs them, tile by tile, with no host synchronisation and no
// extra HBM round trip.
//   optb_shard_row_ptrs_dev  drawn example ids -> absolute row addresses
//                            (owner = id / per, clamped to the last shard)
//   optb_ipc_export / open / close   CUDA IPC of a shard's allocation
// The encode itself is optb_encode_rows_dev / optb_roundtrip_rows_dev (codec.cu
// PTRS kernels).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>

#include "internal.h"
#include "optb_cuda.h"

namespace {

int peer_fail(int code, const std::string& msg) { return optb_b200::set_error_text(code, msg); }

__global__ void k_shard_row_ptrs(const int64_t* __restrict__ ex, uint64_t n, const uint64_t* __restrict__ bases,
                                 uint32_t shards, uint64_t per, uint64_t stride, uint64_t* __restrict__ out) {
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t e = static_cast<uint64_t>(ex[j]);
    uint64_t o = e / per;
    if (o >= shards) o = shards - 1;
    out[j] = bases[o] + (e - o * per) * stride;
  }
}

using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddressRangeFn address_range() {
  static const AddressRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<AddressRangeFn>(nullptr);
    return reinterpret_cast<AddressRangeFn>(f);
  }();
  return fn;
}

}  // namespace

extern "C" {

int optb_shard_row_ptrs_dev(optb_ctx* ctx, const int64_t* examples, uint64_t n, const uint64_t* bases,
                            uint32_t n_shards, uint64_t rows_per_shard, uint64_t row_stride, uint64_t* row_ptrs,
                            void* stream) {
  if (!ctx || !n_shards || !rows_per_shard || (n && (!examples || !bases || !row_ptrs)))
    return peer_fail(OPTB_ERR_ARG, "shard_row_ptrs: bad argument");
  if (!n) return OPTB_OK;
  const uint64_t blocks = (n + 255) / 256;
  k_shard_row_ptrs<<<static_cast<unsigned>(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0,
                     static_cast<cudaStream_t>(stream)>>>(examples, n, bases, n_shards, rows_per_shard, row_stride,
                                                          row_ptrs);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? OPTB_OK : peer_fail(OPTB_ERR_CUDA, cudaGetErrorString(e));
}

int optb_ipc_export(const void* dev_ptr, uint8_t* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return peer_fail(OPTB_ERR_ARG, "ipc_export: null argument");
  const AddressRangeFn fn = address_range();
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!fn || fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return peer_fail(OPTB_ERR_CUDA, "ipc_export: pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return peer_fail(OPTB_ERR_CUDA, std::string("ipc_export: ") + cudaGetErrorString(e));
  static_assert(sizeof(h) == OPTB_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  memcpy(handle, &h, sizeof h);
  *offset = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  return OPTB_OK;
}

int optb_ipc_open(int device, const uint8_t* handle, uint64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr) return peer_fail(OPTB_ERR_ARG, "ipc_open: null argument");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return peer_fail(OPTB_ERR_CUDA, std::string("ipc_open: ") + cudaGetErrorString(e));
  *dev_ptr = static_cast<uint8_t*>(base) + offset;
  return OPTB_OK;
}

int optb_ipc_close(void* dev_ptr, uint64_t offset) {
  if (!dev_ptr) return peer_fail(OPTB_ERR_ARG, "ipc_close: null argument");
  const cudaError_t e = cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset);
  return e == cudaSuccess ? OPTB_OK : peer_fail(OPTB_ERR_CUDA, std::string("ipc_close: ") + cudaGetErrorString(e));
}

}  // extern "C"
