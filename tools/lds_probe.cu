// Shared-memory wavefronts of the K-c store-phase access pattern: a half-warp
// reads one 64-byte x row (16 lanes, each a 4-child window), the other half
// the next row.  Compares two LDS.32 per lane (current) with one LDS.128 of
// an aligned 16-byte window (candidate).  Run under ncu:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum ./lds_probe
#include <cstdio>
#include <cstdint>
__global__ void k32(const int* idx, uint32_t* out, int iters) {
  __shared__ __align__(16) uint32_t row[64 * 20];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) row[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, r = (threadIdx.x >> 4) & 1;
  const int a = idx[lane & 15];  // word index of this lane's window (0..14)
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t* w = row + (r + 2 * (it & 15)) * 17 + a;
    acc += w[0] ^ w[1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k128(const int* idx, uint32_t* out, int iters) {
  __shared__ __align__(16) uint32_t row[64 * 20];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) row[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, r = (threadIdx.x >> 4) & 1;
  const int a = idx[lane & 15] & ~3;  // aligned 16-byte window
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + (r + 2 * (it & 15)) * 20 + a);
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k64(const int* idx, uint32_t* out, int iters) {
  __shared__ __align__(16) uint32_t row[64 * 20];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) row[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, r = (threadIdx.x >> 4) & 1;
  const int a = idx[lane & 15] & ~1;  // aligned 8-byte window
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint2 v = *reinterpret_cast<const uint2*>(row + (r + 2 * (it & 15)) * 18 + a);
    acc += v.x ^ v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  // quad windows of a typical CTA: 16 quads over a 64-byte row, word index rising ~1 per quad
  int h[16] = {0, 1, 2, 3, 3, 4, 5, 6, 7, 8, 8, 9, 10, 11, 12, 13};
  int* d; uint32_t* o;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 148 * 1024 * 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms[3];
    void (*ks[3])(const int*, uint32_t*, int) = {k32, k64, k128};
    for (int k = 0; k < 3; ++k) {
      cudaEventRecord(e0);
      ks[k]<<<148 * 2, 1024>>>(d, o, 4096);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[k], e0, e1);
    }
    printf("lds32x2 %.3f ms  lds64 %.3f ms  lds128 %.3f ms\n", ms[0], ms[1], ms[2]);
  }
  return 0;
}
