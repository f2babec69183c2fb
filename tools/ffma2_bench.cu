// Microbenchmark: FP32 FMA throughput of scalar fma.rn.f32 vs packed
// fma.rn.f32x2 / sub.rn.f32x2 (sm_100a) on B200, independent chains.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float a, float b) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) {
    float lo = threadIdx.x * 0.001f + i, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(lo), "f"(hi));
  }
  unsigned long long A, B;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a), "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b), "f"(b));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd_ffma(float* out, int iters, float a, float b) {
  float r[8], c[8], xx[8];
  for (int i = 0; i < 8; ++i) {
    r[i] = 0.f;
    c[i] = threadIdx.x * 0.001f + i;
    xx[i] = b + i * a;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float d = c[i] - xx[i];
      r[i] = fmaf(d, d, r[i]);
      c[i] += 1e-7f;
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_sub2_ffma2(float* out, int iters, float a, float b) {
  unsigned long long r[4], c[4], xx[4], inc;
  for (int i = 0; i < 4; ++i) {
    float v = threadIdx.x * 0.001f + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r[i]) : "f"(0.f), "f"(0.f));
    asm("mov.b64 %0, {%1, %2};" : "=l"(c[i]) : "f"(v), "f"(v + a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(xx[i]) : "f"(b), "f"(b * 0.5f));
  }
  asm("mov.b64 %0, {%1, %2};" : "=l"(inc) : "f"(1e-7f), "f"(1e-7f));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned long long d;
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(c[i]), "l"(xx[i]));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r[i]) : "l"(d));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(c[i]) : "l"(inc));
    }
  }
  float s = 0;
  for (int i = 0; i < 4; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r[i]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  const int blocks = 148 * 8, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(float*, int, float, float), double lane_ops_per_iter) {
    k<<<blocks, threads>>>(out, 100, 1.0001f, 0.5f);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, 1.0001f, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = lane_ops_per_iter * iters * double(blocks) * threads;
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"G_lane_ops_per_s\": %.1f}\n", name, ms, ops / ms / 1e6);
  };
  run("ffma x8 (8 fma)", k_ffma, 8);
  run("ffma2 x8 (16 fma)", k_ffma2, 16);
  run("fadd+ffma+fadd x8 (24 ops)", k_fadd_ffma, 24);
  run("sub2+ffma2+add2 x4 (24 ops)", k_sub2_ffma2, 24);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
