// K4: fused hyperparameter-gradient quadratic forms.
//
// Replaces KernelOperator::derivative_quadratic_forms_many
// (/root/reference/proj/core/src/kernel.cpp:238-272). For every pair (U, W)
// and every kernel entry (i, c):
//   g_ic     = sum_j U[i,j] W[c,j]                         (row i of U W^T)
//   signal  += k_ic g_ic                 -> (2/s) * sum     (kernel.cpp:264)
//   l_k     += e_ic g_ic (xs_ck - xs_ik)^2 -> 3 s^2 / l_k * sum (kernel.cpp:265-268)
// with k_ic = s^2 (1 + sqrt3 r) e_ic, e_ic = exp(-sqrt3 r). One pass over the
// n x n entries serves every pair and every parameter; the noise term
// (2 sigma sum u.w) is a plain column reduction done elsewhere.
//
// Tiles are 64 x 64 entries. Phase 1 forms G = U_rows W_cols^T for each pair
// with m > 1 by a 4x4 register-tiled SIMT GEMM into shared memory; phase 2
// evaluates the kernel once per entry (thread = one row x 16 columns) and
// accumulates all d+1 sums of all pairs. When every pair has U == W the
// summand is symmetric in (i, c), so only tiles with tc >= ti are visited and
// off-diagonal tiles count twice (half the work of the reference's full pass).
// Per-tile FP32 sums are warp-reduced and added into FP64 per-warp
// accumulators in a fixed order: deterministic, no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "gpk_internal.cuh"

namespace gpk {

namespace {

constexpr int TB = 64;  // tile edge
constexpr int NT = 256;
constexpr int GS = 68;  // Gs row stride (floats): conflict-free phase-2 reads

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kNegSqrt3Log2e = -2.4988211106473432f;  // -sqrt(3) * log2(e)
constexpr float kSqrt3f = 1.7320508075688772f;

__device__ __forceinline__ void tile_coords(long long L, int T, int symmetric, int& ti, int& tc) {
  if (!symmetric) {
    ti = static_cast<int>(L / T);
    tc = static_cast<int>(L % T);
    return;
  }
  // offset(r) = r*T - r*(r-1)/2 ; find largest r with offset(r) <= L
  const double b = 2.0 * T + 1.0;
  int r = static_cast<int>((b - sqrt(b * b - 8.0 * static_cast<double>(L))) / 2.0);
  r = max(0, min(r, T - 1));
  auto off = [&](long long rr) { return rr * T - rr * (rr - 1) / 2; };
  while (r > 0 && off(r) > L) --r;
  while (r + 1 < T && off(r + 1) <= L) ++r;
  ti = r;
  tc = r + static_cast<int>(L - off(r));
}

template <int DP4, int NP>
__global__ void __launch_bounds__(NT, 2) grad_kernel(const GradArgs a) {
  constexpr int DP = 4 * DP4;
  constexpr int DMAX = DP;
  __shared__ __align__(16) float Gs[NP][TB * GS];
  __shared__ __align__(16) float Xc[TB * DP];
  __shared__ float W1[NP][TB];                 // m == 1 pairs: W column values
  __shared__ double wacc[NT / 32][NP * (DMAX + 1)];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = a.d;
  const int T = (a.n + TB - 1) / TB;
  const long long ntiles = a.symmetric ? static_cast<long long>(T) * (T + 1) / 2
                                       : static_cast<long long>(T) * T;
  const long long tb = a.tile_end >= 0 ? a.tile_begin : 0;   // this rank's share of the tile list
  const long long te = a.tile_end >= 0 ? min(a.tile_end, ntiles) : ntiles;
  const long long per = (te - tb + gridDim.x - 1) / gridDim.x;
  const long long L0 = tb + blockIdx.x * per;
  const long long L1 = min(te, L0 + per);

  for (int e = tid; e < (NT / 32) * NP * (DMAX + 1); e += NT) (&wacc[0][0])[e] = 0.0;

  // phase-2 mapping
  const int pr = tid >> 2;        // row within tile
  const int pc = tid & 3;         // column offset; columns pc + 4t
  // phase-1 mapping
  const int ty = tid >> 4, tx = tid & 15;

  for (long long L = L0; L < L1; ++L) {
    int ti, tc;
    tile_coords(L, T, a.symmetric, ti, tc);
    const int row0 = ti * TB, col0 = tc * TB;
    const float weight = (a.symmetric && tc != ti) ? 2.f : 1.f;

    __syncthreads();  // previous tile's smem reads done
    // ---- stage X columns and m==1 W values ----
    for (int e = tid; e < TB * DP4; e += NT) {
      const int c = e / DP4, u = e % DP4;
      const int gc = min(col0 + c, a.n - 1);
      reinterpret_cast<float4*>(Xc)[e] = __ldg(reinterpret_cast<const float4*>(a.xs + static_cast<size_t>(gc) * a.dp) + u);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (a.mcols[p] == 1 && tid < TB) {
        const int gc = col0 + tid;
        W1[p][tid] = gc < a.n ? __ldg(a.w[p] + static_cast<size_t>(gc) * a.ldu[p]) : 0.f;
      }
    }
    // ---- phase 1: G_p = U[rows] W[cols]^T for m > 1 pairs ----
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (a.mcols[p] == 1) continue;
      float g[4][4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) g[x][y] = 0.f;
      const float* U = a.u[p];
      const float* W = a.w[p];
      const int ld = a.ldu[p];
      int ur[4], wr[4];
      bool uv[4], wv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        ur[x] = row0 + ty * 4 + x;
        uv[x] = ur[x] < a.n;
        ur[x] = uv[x] ? ur[x] : 0;
        wr[x] = col0 + tx * 4 + x;
        wv[x] = wr[x] < a.n;
        wr[x] = wv[x] ? wr[x] : 0;
      }
      for (int j = 0; j < a.mcols[p]; j += 4) {
        float4 uu[4], ww[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          uu[x] = __ldg(reinterpret_cast<const float4*>(U + static_cast<size_t>(ur[x]) * ld + j));
          ww[x] = __ldg(reinterpret_cast<const float4*>(W + static_cast<size_t>(wr[x]) * ld + j));
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            g[x][y] = fmaf(uu[x].x, ww[y].x, g[x][y]);
            g[x][y] = fmaf(uu[x].y, ww[y].y, g[x][y]);
            g[x][y] = fmaf(uu[x].z, ww[y].z, g[x][y]);
            g[x][y] = fmaf(uu[x].w, ww[y].w, g[x][y]);
          }
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        float4 o;
        o.x = (uv[x] && wv[0]) ? g[x][0] : 0.f;
        o.y = (uv[x] && wv[1]) ? g[x][1] : 0.f;
        o.z = (uv[x] && wv[2]) ? g[x][2] : 0.f;
        o.w = (uv[x] && wv[3]) ? g[x][3] : 0.f;
        *reinterpret_cast<float4*>(&Gs[p][(ty * 4 + x) * GS + tx * 4]) = o;
      }
    }
    __syncthreads();

    // ---- phase 2: kernel evaluation + accumulation ----
    const int gi = row0 + pr;
    const bool row_ok = gi < a.n;
    const int gic = row_ok ? gi : a.n - 1;
    // x_row as FP32x2 pairs; distance, squares and the d lengthscale sums run
    // on packed FADD2/FMUL2/FFMA2 (two dimensions per instruction)
    uint64_t xi2[2 * DP4];
#pragma unroll
    for (int u = 0; u < DP4; ++u) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(a.xs + static_cast<size_t>(gic) * a.dp) + u);
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(v.x), "f"(v.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(v.z), "f"(v.w));
    }
    float u1[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p)
      u1[p] = (a.mcols[p] == 1 && row_ok) ? __ldg(a.u[p] + static_cast<size_t>(gic) * a.ldu[p]) : 0.f;

    float accs[NP];
    uint64_t accl2[NP][DP / 2];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      accs[p] = 0.f;
#pragma unroll
      for (int k = 0; k < DP / 2; ++k) accl2[p][k] = 0ull;
    }
    const uint32_t xbase = static_cast<uint32_t>(__cvta_generic_to_shared(Xc));
#pragma unroll 2
    for (int t = 0; t < 16; ++t) {
      const int c = pc + 4 * t;
      uint64_t sq2[DP / 2];
      uint64_t r2a = 0ull, r2b = 0ull;
#pragma unroll
      for (int u = 0; u < DP4; ++u) {
        uint64_t c01, c23, d01, d23;
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xbase + (c * DP + 4 * u) * 4));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(c01), "l"(xi2[2 * u]));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(c23), "l"(xi2[2 * u + 1]));
        asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq2[2 * u]) : "l"(d01));
        asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq2[2 * u + 1]) : "l"(d23));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(r2a) : "l"(sq2[2 * u]));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(r2b) : "l"(sq2[2 * u + 1]));
      }
      uint64_t r2s;
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r2s) : "l"(r2a), "l"(r2b));
      float q0, q1;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(q0), "=f"(q1) : "l"(r2s));
      const float r = sqrt_approx(q0 + q1);
      const float e0 = ex2_approx(r * kNegSqrt3Log2e);           // exp(-sqrt3 r)
      const float kv = fmaf(r, kSqrt3f, 1.f) * e0;               // k / s^2
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float g = (a.mcols[p] == 1) ? u1[p] * W1[p][c] : Gs[p][pr * GS + c];
        accs[p] = fmaf(kv, g, accs[p]);
        const float coeff = e0 * g;
        uint64_t coeff2;
        asm("mov.b64 %0, {%1, %1};" : "=l"(coeff2) : "f"(coeff));
#pragma unroll
        for (int k = 0; k < DP / 2; ++k)
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(accl2[p][k]) : "l"(sq2[k]), "l"(coeff2));
      }
    }
    float accl[NP][DMAX];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int k = 0; k < DP / 2; ++k)
        asm("mov.b64 {%0, %1}, %2;" : "=f"(accl[p][2 * k]), "=f"(accl[p][2 * k + 1]) : "l"(accl2[p][k]));
    // ---- per-tile flush: warp reduce, then FP64 per-warp accumulators ----
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int k = 0; k <= DMAX; ++k) {
        if (k < DMAX && k >= d) continue;
        float v = (k == DMAX) ? accs[p] : accl[p][k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) wacc[warp][p * (DMAX + 1) + k] += static_cast<double>(v * weight);
      }
    }
  }
  __syncthreads();
  // block result: fixed-order sum over warps
  for (int e = tid; e < NP * (d + 1); e += NT) {
    const int p = e / (d + 1), k = e % (d + 1);
    const int slot = p * (DMAX + 1) + (k == d ? DMAX : k);
    double acc = 0.0;
    for (int w = 0; w < NT / 32; ++w) acc += wacc[w][slot];
    a.part[static_cast<size_t>(blockIdx.x) * NP * (d + 1) + e] = acc;
  }
}

template <int DP4>
void launch_dp(const GradArgs& a, cudaStream_t s) {
  if (a.npairs == 1)
    grad_kernel<DP4, 1><<<a.blocks, NT, 0, s>>>(a);
  else
    grad_kernel<DP4, 2><<<a.blocks, NT, 0, s>>>(a);
  check_launch("grad_kernel");
}

}  // namespace

void grad_launch(const GradArgs& a, cudaStream_t s) {
  if (a.npairs < 1 || a.npairs > 2) throw std::invalid_argument("gpk: grad pass supports 1 or 2 pairs");
  switch (a.dp / 4) {
    case 1: return launch_dp<1>(a, s);
    case 2: return launch_dp<2>(a, s);
    case 3: return launch_dp<3>(a, s);
    case 4: return launch_dp<4>(a, s);
    case 5: return launch_dp<5>(a, s);
    case 6: return launch_dp<6>(a, s);
    case 7: return launch_dp<7>(a, s);
    case 8: return launch_dp<8>(a, s);
    default: throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  }
}

}  // namespace gpk
