// Probe: does a TMA tensor store (cp.async.bulk.tensor.2d.global.shared::cta)
// with a box that starts at a negative / in-row column write only the
// in-bounds elements?  Global tensor: R rows × 64 bytes (uint8).  Box 64 × 8.
// Store 1 at column 20 (cols 20..63 in bounds), store 2 at column -30 (cols
// 0..33 in bounds), store 3 at column 0 (full rows).  nvcc -arch=sm_100a.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>

__global__ void k(const __grid_constant__ CUtensorMap tm) {
  __shared__ __align__(128) uint8_t tile[8 * 64];
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) tile[i] = (uint8_t)(100 + (i & 63));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(tile);
    int cs[3] = {20, -30, 0}, rs[3] = {0, 8, 16};
    for (int q = 0; q < 3; ++q)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   :: "l"(&tm), "r"(cs[q]), "r"(rs[q]), "r"(s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int R = 32;
  uint8_t* d;
  cudaMalloc(&d, R * 64);
  cudaMemset(d, 0, R * 64);
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  Enc enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)R}, strides[1] = {64};
  cuuint32_t box[2] = {64, 8}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(tm);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  uint8_t h[R * 64];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int ok = 1;
  for (int row = 0; row < 24; ++row)
    for (int c = 0; c < 64; ++c) {
      int want;
      if (row < 8) want = c >= 20 ? 100 + (c - 20) : 0;          // box col i -> global col 20 + i
      else if (row < 16) want = c < 34 ? 100 + (c + 30) : 0;     // box col i -> global col i - 30
      else want = 100 + c;
      if (h[row * 64 + c] != want) { if (ok) printf("mismatch row %d col %d got %d want %d\n", row, c, h[row * 64 + c], want); ok = 0; }
    }
  for (int row = 24; row < R; ++row)
    for (int c = 0; c < 64; ++c)
      if (h[row * 64 + c]) ok = 0;
  printf("TMA clip probe: %s\n", ok ? "OK (negative and in-row starts clip to the tensor)" : "FAILED");
  return ok ? 0 : 2;
}
