// tc_probe.cu — standalone check of the tcgen05 kind::i8 operand layouts used
// by K-a (snp_tc.cuh): D[128×32] = A[128×64] · B[64×32], A MN-major, B K-major,
// u8 × u8 → s32, against a CPU product.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_1104_1824_b200/csrc tools/tc_probe.cu -o /tmp/tc_probe && /tmp/tc_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "snp_tc.cuh"

using namespace snp;

constexpr int M = 128, N = 32, K = 64;
constexpr uint32_t A_LBO = 1024, B_LBO = 512;

__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, int swap) {
  __shared__ __align__(1024) uint8_t sA[M * K];
  __shared__ __align__(1024) uint8_t sB[K * N];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int mn = i / K, k = i % K;
    sA[(k / 8) * A_LBO + (mn / 16) * 128 + (k % 8) * 16 + mn % 16] = A[i];
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    sB[(k / 16) * B_LBO + (n / 8) * 128 + (n % 8) * 16 + k % 16] = B[i];
  }
  if (warp == 0) tc::tmem_alloc(&tslot, 32);
  if (tid == 0) tc::bar_init(&bar, 1);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_u8(M, N, true, false);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint32_t a = tc::smem_u32(sA + ks * 4 * A_LBO), b = tc::smem_u32(sB + ks * 2 * B_LBO);
      const uint64_t da = swap ? tc::sdesc(a, 128, A_LBO) : tc::sdesc(a, A_LBO, 128);
      const uint64_t db = swap ? tc::sdesc(b, 128, B_LBO) : tc::sdesc(b, B_LBO, 128);
      tc::mma_u8(tmem, da, db, idesc, ks > 0);
    }
    tc::commit(&bar);
  }
  tc::bar_wait(&bar, 0);
  tc::fence_after();
  uint32_t r[32];
  tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), r);
  for (int n = 0; n < N; ++n) D[(32 * warp + lane) * N + n] = (int32_t)r[n];
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

int main() {
  std::vector<uint8_t> A(M * K), B(K * N);
  srand(7);
  for (auto& x : A) x = rand() & 15;
  for (auto& x : B) x = rand() & 255;
  std::vector<int64_t> ref(M * N, 0);
  for (int i = 0; i < M; ++i)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) ref[i * N + n] += (int64_t)A[i * K + k] * B[k * N + n];
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  int rc = 1;
  for (int swap = 0; swap < 1; ++swap) {
    cudaMemset(dD, 0xFF, M * N * 4);
    probe<<<1, 128>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> D(M * N);
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += (int64_t)D[i] != ref[i];
    printf("variant swap=%d: cuda=%s mismatches=%d / %d  (D[0]=%d ref %lld, D[last]=%d ref %lld)\n", swap,
           cudaGetErrorString(e), bad, M * N, D[0], (long long)ref[0], D[M * N - 1], (long long)ref[M * N - 1]);
    if (e != cudaSuccess) return 2;
    if (swap == 0 && bad == 0) rc = 0;
  }
  printf(rc == 0 ? "PROBE PASS\n" : "PROBE FAIL\n");
  return rc;
}
