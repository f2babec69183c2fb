// Probes the operand split of one CTA-pair tcgen05.mma.cta_group::2.kind::tf32
// (M = 256, N = 80, K = 8, A from TMEM, B from shared memory), the layout the
// paired SGD slab kernel relies on: each CTA holds its own 128 rows of A in
// its TMEM and N/2 = 40 rows of B in its shared memory at the same offset,
// and receives its 128 rows x 80 columns of D in its TMEM. Values are small
// multiples of 1/8, so every product and sum is exact: the check is bitwise.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//          -Ipaper_2405_18457_b200/csrc tools/probe_2sm.cu -o tools/probe_2sm
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "tc_util.cuh"

using namespace gpk::tc;

constexpr int N = 80, NH = 40, K = 8;

// canonical no-swizzle K-major: element (r, k) of a rows x 8 operand
__host__ __device__ inline int off8(int r, int k) { return ((r / 8) * 2 + k / 4) * 32 + (r % 8) * 4 + (k % 4); }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) float sB[NH * K];
  __shared__ uint64_t ready, done;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  for (int e = tid; e < NH * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    sB[off8(n, k)] = B[(rank * NH + n) * K + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    mbar_init(&ready, 2);
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A: this CTA's 128 rows, TMEM columns 64..71
  {
    const int row = warp * 32 + lane;
    uint32_t v[8];
    for (int k = 0; k < K; ++k) v[k] = __float_as_uint(A[(rank * 128 + row) * K + k]);
    tc_st8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 64, v);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) arrive_leader(&ready);
  if (rank == 0 && tid == 0) {
    wait_cluster(&ready, 0);
    tc_fence_after();
    constexpr uint32_t idesc = tf32_idesc(N, 256);
    const uint64_t db = umma_desc(smem_u32(sB), 128, 256);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
        "r"(tmem + 64), "l"(db), "r"(idesc)
        : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&done)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  wait_cluster(&done, 0);
  tc_fence_after();
  {
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      tc_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
      tc_wait_ld();
      for (int e = 0; e < 8; ++e) D[(rank * 128 + row) * N + c + e] = __uint_as_float(v[e]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
  }
}

// occupancy probe: how many CTA pairs of a one-CTA-per-SM kernel are co-resident
__global__ void pair_occupancy_dummy(float* out) {
  extern __shared__ float big[];
  big[threadIdx.x] = 0.f;
  if (out) out[threadIdx.x] = big[threadIdx.x];
}

int main() {
  {
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(pair_occupancy_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(pair_occupancy_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs = 1; cs <= 4; cs *= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148, 1, 1);
      cfg.blockDim = dim3(704, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nc = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, pair_occupancy_dummy, &cfg);
      std::printf("probe_2sm: cluster size %d, one CTA per SM: %d co-resident clusters (%s)\n", cs, nc,
                  cudaGetErrorString(e));
    }
  }
  std::vector<float> A(256 * K), B(N * K), D(256 * N, -1.f);
  unsigned s = 12345;
  auto rnd = [&]() {
    s = s * 1103515245u + 12345u;
    return static_cast<float>(static_cast<int>((s >> 16) % 33) - 16) / 8.f;
  };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, D.size() * 4);
  probe<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("probe_2sm: CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0;
  for (int r = 0; r < 256; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += static_cast<double>(A[r * K + k]) * B[n * K + k];
      const double err = std::fabs(ref - D[r * N + n]);
      maxerr = std::fmax(maxerr, err);
      if (err != 0 && bad++ < 8) std::printf("  D[%d][%d] = %g, expected %g\n", r, n, D[r * N + n], ref);
    }
  std::printf("probe_2sm: M=256 N=%d K=%d cta_group::2 TS tf32: %d mismatches, max err %g -> %s\n", N, K, bad,
              maxerr, bad ? "FAIL" : "OK (A row-split, B N-split across the pair)");
  return bad ? 1 : 0;
}
