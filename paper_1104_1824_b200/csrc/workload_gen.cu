// workload_gen.cu — device-side level-0 input generator (libsnpgen.so).
//
// INPUT GENERATION ONLY: no arithmetic of the method lives here.  It writes
// the same counter-based level-0 frontier as workloads.level0_counts() —
//     count(p, s) = (splitmix64(key ^ (p·m + s)) >> 32) mod range[s]
// — directly into device memory, so multi-GB frontiers (config 4: 2^22 ×
// 16384) need no host round trip.  Output layout: neuron-major (s rows of
// `ld` elements) or row-major (p rows of `ld` elements); elem_bytes 1/2/4.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void k_level0(T* dst, int32_t m, int64_t F, int64_t ld, int32_t layout, uint64_t key,
                         const int32_t* range, int64_t row_begin) {
  // neuron-major: x = p (fast), y = s; row-major: x = s (fast), y = p
  const int64_t fast = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t slow = blockIdx.y; slow < (layout == 1 ? (int64_t)m : F); slow += gridDim.y) {
    const int64_t p = layout == 1 ? fast : slow;
    const int64_t s = layout == 1 ? slow : fast;
    if (p >= F || s >= m) continue;
    const uint64_t v = splitmix64(key ^ ((uint64_t)(p + row_begin) * (uint64_t)m + (uint64_t)s));
    const T c = (T)((v >> 32) % (uint64_t)range[s]);
    if (layout == 1) dst[s * ld + p] = c;
    else dst[p * ld + s] = c;
  }
}

}  // namespace

extern "C" int snpgen_level0(void* dst, int32_t elem_bytes, int32_t layout, int64_t ld, int32_t m, int64_t F,
                             uint64_t key, const int32_t* range_host, int64_t row_begin, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  {  // this library's CUDA runtime on the GPU that holds dst (one process per GPU)
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeDevice) cudaSetDevice(pa.device);
    cudaGetLastError();
  }
  int32_t* range = nullptr;
  if (cudaMalloc(&range, sizeof(int32_t) * m) != cudaSuccess) return -5;
  cudaMemcpyAsync(range, range_host, sizeof(int32_t) * m, cudaMemcpyHostToDevice, st);
  const int64_t nfast = layout == 1 ? F : m;
  const int64_t nslow = layout == 1 ? m : F;
  dim3 block(256), grid((unsigned)((nfast + 255) / 256), (unsigned)(nslow < 65535 ? nslow : 65535));
  if (elem_bytes == 1) k_level0<uint8_t><<<grid, block, 0, st>>>((uint8_t*)dst, m, F, ld, layout, key, range, row_begin);
  else if (elem_bytes == 2) k_level0<uint16_t><<<grid, block, 0, st>>>((uint16_t*)dst, m, F, ld, layout, key, range, row_begin);
  else k_level0<int32_t><<<grid, block, 0, st>>>((int32_t*)dst, m, F, ld, layout, key, range, row_begin);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(range);
  return e == cudaSuccess ? 0 : -6;
}
