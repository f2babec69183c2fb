// Probes the arithmetic of one tcgen05.mma.kind::tf32 (M=128, N=16, K=8, A and
// B from shared memory, FP32 accumulator in TMEM): how many bits survive inside
// the K=8 product sum and across accumulating MMAs, and the rounding direction.
// Row r of A carries a test vector, B is all ones in column 0 (so D[r][0] is
// the plain sum of row r), and a second MMA optionally adds row r of A2.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2405_18457_b200/csrc
//        tools/tc_precision.cu -o tools/tc_precision
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "tc_util.cuh"

using namespace gpk::tc;

__device__ __forceinline__ void tc_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  tc_mma_tf32_ss(d, a, b, idesc, acc);
}

// canonical no-swizzle K-major: element (r, k) of a rows x 8 operand
__host__ __device__ inline int off8(int r, int k) { return ((r / 8) * 2 + k / 4) * 32 + (r % 8) * 4 + (k % 4); }

__global__ void probe(const float* A1, const float* A2, const float* B, float* D, int second) {
  __shared__ __align__(1024) float sA1[128 * 8];
  __shared__ __align__(1024) float sA2[128 * 8];
  __shared__ __align__(1024) float sB[16 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    sA1[off8(e / 8, e % 8)] = A1[e];
    sA2[off8(e / 8, e % 8)] = A2[e];
  }
  for (int e = tid; e < 16 * 8; e += blockDim.x) sB[off8(e / 8, e % 8)] = B[e];
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    constexpr uint32_t idesc = tf32_idesc(16, 128);
    const uint64_t da1 = umma_desc(smem_u32(sA1), 128, 256);
    const uint64_t da2 = umma_desc(smem_u32(sA2), 128, 256);
    const uint64_t db = umma_desc(smem_u32(sB), 128, 256);
    tc_mma_ss(tmem, da1, db, idesc, 0u);
    if (second) tc_mma_ss(tmem, da2, db, idesc, 1u);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[8];
  tc_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
  tc_wait_ld();
  const int row = warp * 32 + lane;
  for (int e = 0; e < 8; ++e) D[row * 8 + e] = __uint_as_float(v[e]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
  }
}

static void run(const char* name, const std::vector<float>& A1, const std::vector<float>& A2, int second,
                const std::vector<double>& expect) {
  std::vector<float> B(16 * 8, 0.f);
  for (int k = 0; k < 8; ++k) B[0 * 8 + k] = 1.f;  // column 0 sums the row
  float *dA1, *dA2, *dB, *dD;
  cudaMalloc(&dA1, 4 * 128 * 8);
  cudaMalloc(&dA2, 4 * 128 * 8);
  cudaMalloc(&dB, 4 * 16 * 8);
  cudaMalloc(&dD, 4 * 128 * 8);
  cudaMemcpy(dA1, A1.data(), 4 * 128 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dA2, A2.data(), 4 * 128 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * 16 * 8, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA1, dA2, dB, dD, second);
  std::vector<float> D(128 * 8);
  const cudaError_t e = cudaMemcpy(D.data(), dD, 4 * 128 * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    std::printf("%s: CUDA error %s\n", name, cudaGetErrorString(e));
    return;
  }
  std::printf("== %s\n", name);
  for (int r = 0; r < 128; r += 4) {
    const double got = D[r * 8 + 0], ex = expect[r];
    const float exf = static_cast<float>(ex);
    std::printf("row %3d expect %.10e (fp32 RN %.10e) got %.10e  err/ulp(1)=%.3g\n", r, ex, exf, got,
                (got - ex) / std::ldexp(1.0, -23));
  }
  cudaFree(dA1);
  cudaFree(dA2);
  cudaFree(dB);
  cudaFree(dD);
}

int main() {
  std::vector<float> A1(128 * 8, 0.f), A2(128 * 8, 0.f);
  std::vector<double> ex(128);
  // 1) inside one MMA: 1 + 2^-e (row r: e = 8 + r/4), all TF32-exact inputs
  for (int r = 0; r < 128; ++r) {
    const int e = 8 + r / 4;
    A1[r * 8 + 0] = 1.f;
    A1[r * 8 + 1] = std::ldexp(1.f, -e);
    ex[r] = 1.0 + std::ldexp(1.0, -e);
  }
  run("one MMA: 1 + 2^-e, e = 8 + row/4", A1, A2, 0, ex);
  // 2) inside one MMA with cancellation: 1 - 1 + 2^-e
  std::fill(A1.begin(), A1.end(), 0.f);
  for (int r = 0; r < 128; ++r) {
    const int e = 8 + r / 4;
    A1[r * 8 + 0] = 1.f;
    A1[r * 8 + 1] = -1.f;
    A1[r * 8 + 2] = std::ldexp(1.f, -e);
    ex[r] = std::ldexp(1.0, -e);
  }
  run("one MMA: 1 - 1 + 2^-e", A1, A2, 0, ex);
  // 3) across MMAs: D = 1, then D += 2^-e
  std::fill(A1.begin(), A1.end(), 0.f);
  for (int r = 0; r < 128; ++r) {
    const int e = 8 + r / 4;
    A1[r * 8 + 0] = 1.f;
    A2[r * 8 + 0] = std::ldexp(1.f, -e);
    ex[r] = 1.0 + std::ldexp(1.0, -e);
  }
  run("two MMAs: (1) + (2^-e)", A1, A2, 1, ex);
  // 4) rounding direction inside one MMA: 1 + 3 * 2^-25 (FP32 RN -> 1 + 2^-23)
  std::fill(A1.begin(), A1.end(), 0.f);
  std::fill(A2.begin(), A2.end(), 0.f);
  for (int r = 0; r < 128; ++r) {
    const int k = r / 4;  // 1 + k * 2^-25 with k small pieces of 2^-25
    A1[r * 8 + 0] = 1.f;
    for (int q = 0; q < 7; ++q) A1[r * 8 + 1 + q] = (q < (k % 8)) ? std::ldexp(1.f, -25) : 0.f;
    ex[r] = 1.0 + (k % 8) * std::ldexp(1.0, -25);
  }
  run("one MMA: 1 + j*2^-25 (j = (row/4) % 8)", A1, A2, 0, ex);
  // 5) negative: -(1 + j 2^-25)
  for (int r = 0; r < 128; ++r)
    for (int q = 0; q < 8; ++q) A1[r * 8 + q] = -A1[r * 8 + q];
  for (int r = 0; r < 128; ++r) ex[r] = -ex[r];
  run("one MMA: -(1 + j*2^-25)", A1, A2, 0, ex);
  return 0;
}
