// Solver-state kernels: CG recurrences (K6), pivoted-Cholesky preconditioner
// (K7), alternating-projection block steps (K8), SGD minibatch sampling and
// momentum updates (K2 epilogue + K9), RFF pathwise targets (K5).
//
// All solver vectors are FP64 row-major [n][m] (m = s+1 RHS). Every
// reduction is deterministic: a fixed grid of row groups writes partials and
// a single block sums them in ascending group order — no float atomics.
// Kernels that run inside a solver iteration take a `skip` flag (device int)
// so the host can enqueue iterations ahead of the termination test: once the
// device sets the flag, the remaining enqueued kernels are no-ops.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "gpk_internal.cuh"
#include "tc_util.cuh"
#include "philox.cuh"

namespace gpk {

namespace {
inline int blocks_for(long long n, int threads, int cap = 148 * 16) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}
#define SKIP_IF(flag) \
  if ((flag) && *(flag)) return;
}  // namespace

// ---------------------------------------------------------------- layout
__global__ void prescale_kernel(const double* x64, int n, int d, int dp, const double* inv_ls,
                                float* xs32, double* xs64) {
  const long long total = static_cast<long long>(n) * dp;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / dp), k = static_cast<int>(e % dp);
    if (k < d) {
      const double v = x64[static_cast<size_t>(i) * d + k] * inv_ls[k];  // kernel.cpp:94
      xs32[e] = static_cast<float>(v);
      xs64[static_cast<size_t>(i) * d + k] = v;
    } else {
      xs32[e] = 0.f;
    }
  }
}
void prescale_launch(const double* x64, int n, int d, int dp, const double* inv_ls, float* xs32,
                     double* xs64, cudaStream_t s) {
  prescale_kernel<<<blocks_for(static_cast<long long>(n) * dp, 256), 256, 0, s>>>(x64, n, d, dp, inv_ls, xs32, xs64);
  check_launch("prescale");
}

// Distance-by-Gram image for the tensor-core operator kernels (d >= 21): row i
// = (x_i, |x_i|^2, 0...) with |x_i|^2 summed in FP64 from the FP32 coordinates
// and rounded once, so r^2 = |x_i|^2 + |x_c|^2 - 2 x_i.x_c is one FFMA chain
// over the padded row (kv_tc_kernel.cu, ap_persistent.cu).
__global__ void gram_image_kernel(const float* xs32, int n, int d, int dp, int dpg, float* xg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float* src = xs32 + static_cast<size_t>(i) * dp;
    float* dst = xg + static_cast<size_t>(i) * dpg;
    double nn = 0.0;
    for (int k = 0; k < d; ++k) {
      const float v = src[k];
      nn += static_cast<double>(v) * v;
      dst[k] = v;
    }
    dst[d] = static_cast<float>(nn);
    for (int k = d + 1; k < dpg; ++k) dst[k] = 0.f;
  }
}
void gram_image_launch(const float* xs32, int n, int d, int dp, int dpg, float* xg, cudaStream_t s) {
  gram_image_kernel<<<blocks_for(n, 256), 256, 0, s>>>(xs32, n, d, dp, dpg, xg);
  check_launch("gram_image");
}

// Column images of the tensor-core Gram distances (kv_tc_kernel TG): chunk q
// of 32 points holds B hi | B lo, the TF32 pieces of -2 x'_c in the canonical
// K-major no-swizzle layout (element (j, k) at ((j/8) (KG/4) + k/4) 32 +
// (j%8) 4 + k%4, K = KG), then |x'_c|^2 for the 32 points. Covers the 128
// zero rows of padding of xs32 as well (zero images and norms).
int tg_kg(int d) { return ((d + 3) / 4 + 1) / 2 * 8; }
size_t tg_image_floats(int n, int d) {
  const int kg = tg_kg(d);
  return static_cast<size_t>((n + 128) / 32) * (64 * kg + 32);
}
__global__ void tg_image_kernel(const float* xs32, int nchunks, int dp, int kg, float* xtg) {
  const int total = nchunks * 32;
  const int chunk = 64 * kg + 32;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    const float* src = xs32 + static_cast<size_t>(c) * dp;
    float* base = xtg + static_cast<size_t>(c / 32) * chunk;
    const int j = c % 32;
    float nn = 0.f;
    for (int k = 0; k < kg; ++k) {
      float hi = 0.f, lo = 0.f;
      if (k < dp) tc::tg_split(src[k], hi, lo);
      if (k < dp) nn = tc::tg_norm_step(nn, hi, lo);
      const int off = ((j / 8) * (kg / 4) + k / 4) * 32 + (j % 8) * 4 + k % 4;
      base[off] = -2.f * hi;
      base[32 * kg + off] = -2.f * lo;
    }
    base[64 * kg + j] = nn;
  }
}
void tg_image_launch(const float* xs32, int n, int d, int dp, float* xtg, cudaStream_t s) {
  const int nchunks = (n + 128) / 32;
  tg_image_kernel<<<blocks_for(static_cast<long long>(nchunks) * 32, 256), 256, 0, s>>>(xs32, nchunks, dp, tg_kg(d),
                                                                                      xtg);
  check_launch("tg_image");
}

__global__ void to_f32_kernel(const double* src, int n, int m, int lds, float* dst, int ldd, const int* skip) {
  SKIP_IF(skip);
  const long long total = static_cast<long long>(n) * ldd;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / ldd), j = static_cast<int>(e % ldd);
    dst[e] = j < m ? static_cast<float>(src[static_cast<size_t>(i) * lds + j]) : 0.f;
  }
}
void to_f32_launch(const double* src, int n, int m, int lds, float* dst, int ldd, const int* skip, cudaStream_t s) {
  to_f32_kernel<<<blocks_for(static_cast<long long>(n) * ldd, 256), 256, 0, s>>>(src, n, m, lds, dst, ldd, skip);
  check_launch("to_f32");
}

__global__ void transpose_kernel(const double* src, int rows, int cols, int lds, double* dst, int ldd) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / cols), c = static_cast<int>(e % cols);
    dst[static_cast<size_t>(c) * ldd + r] = src[static_cast<size_t>(r) * lds + c];
  }
}
void transpose_launch(const double* src, int rows, int cols, int lds, double* dst, int ldd, cudaStream_t s) {
  transpose_kernel<<<blocks_for(static_cast<long long>(rows) * cols, 256), 256, 0, s>>>(src, rows, cols, lds, dst, ldd);
  check_launch("transpose");
}

// ---------------------------------------------------------- reductions
// part[g][k*m + j]: per-column sums over rows [g*n/G, (g+1)*n/G).
__global__ void col_reduce_kernel(const double* a, const double* b, int n, int m, int lda, int mode,
                                  double* part, const int* skip) {
  SKIP_IF(skip);
  __shared__ double s1[8][33], s2[8][33];
  const int g = blockIdx.x, G = gridDim.x;
  const long long rb = static_cast<long long>(n) * g / G, re = static_cast<long long>(n) * (g + 1) / G;
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  const int nout = mode == 1 ? 2 : 1;
  for (int j0 = 0; j0 < m; j0 += 32) {
    const int j = j0 + tx;
    double acc1 = 0.0, acc2 = 0.0;
    if (j < m) {
      for (long long i = rb + ty; i < re; i += 8) {
        const double x = a[i * lda + j];
        if (mode == 2) {
          acc1 = fma(x, x, acc1);
        } else {
          acc1 = fma(x, b[i * lda + j], acc1);
          if (mode == 1) acc2 = fma(x, x, acc2);
        }
      }
    }
    s1[ty][tx] = acc1;
    s2[ty][tx] = acc2;
    __syncthreads();
    if (ty == 0 && j < m) {
      double t1 = 0.0, t2 = 0.0;
      for (int q = 0; q < 8; ++q) {
        t1 += s1[q][tx];
        t2 += s2[q][tx];
      }
      part[static_cast<size_t>(g) * nout * m + j] = t1;
      if (mode == 1) part[static_cast<size_t>(g) * nout * m + m + j] = t2;
    }
    __syncthreads();
  }
}
void col_reduce_launch(const double* a, const double* b, int n, int m, int lda, int mode, double* part,
                       int groups, const int* skip, cudaStream_t s) {
  col_reduce_kernel<<<groups, 256, 0, s>>>(a, b, n, m, lda, mode, part, skip);
  check_launch("col_reduce");
}

namespace {
// Sum of partial `off` over groups, fixed order (single thread; small counts only).
__device__ double gsum(const double* part, int groups, int stride, int off) {
  double acc = 0.0;
  for (int g = 0; g < groups; ++g) acc += part[static_cast<size_t>(g) * stride + off];
  return acc;
}
// Same sum by one warp: lane l adds groups l, l+32, ... then a fixed xor tree.
// Deterministic (the summation shape depends only on `groups`); every lane
// returns the total.
__device__ __forceinline__ double warp_gsum(const double* part, int groups, int stride, int off) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int g = lane; g < groups; g += 32) acc += part[static_cast<size_t>(g) * stride + off];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}
// Termination norms (linear_system.cpp:38-53) from per-column sums of squares
// in shared memory (overwritten). Called by every thread of the block: the
// per-column terms sqrt(ss_j) / scale_j are formed in parallel, then one thread
// adds them in column order (the reference's order). The results are valid in
// every thread on return.
__device__ void termination_block(double* ss, int m, const double* scales, double tol, double& mean, double& probe,
                                  int& done) {
  __shared__ double res[3];
  for (int j = threadIdx.x; j < m; j += blockDim.x) ss[j] = sqrt(ss[j]) / scales[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int j = 1; j < m; ++j) sum += ss[j];
    res[0] = ss[0];
    res[1] = m > 1 ? sum / (m - 1) : 0.0;
    res[2] = (res[0] <= tol && res[1] <= tol) ? 1.0 : 0.0;
  }
  __syncthreads();
  mean = res[0];
  probe = res[1];
  done = res[2] != 0.0;
}
}  // namespace

// gamma = r.p ; termination from r.r
__global__ void cg_init_scalars_kernel(const double* part, int groups, int m, const double* scales,
                                       double tol, double* gamma, CgCtl* ctl) {
  __shared__ double ss[512];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < m; j += nw) {
    const double g = warp_gsum(part, groups, 2 * m, j);
    const double q = warp_gsum(part, groups, 2 * m, m + j);
    if (lane == 0) {
      gamma[j] = g;
      ss[j] = q;
    }
  }
  __syncthreads();
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    ctl->mean_norm = mean;
    ctl->probe_norm = probe;
    ctl->done = done;
    ctl->aborted = 0;
    ctl->iters = 0;
    ctl->stop = (done || ctl->iters >= ctl->budget) ? 1 : 0;
  }
}
void cg_init_scalars_launch(const double* part, int groups, int m, const double* scales, double tol,
                            double* gamma, CgCtl* ctl, cudaStream_t s) {
  cg_init_scalars_kernel<<<1, 1024, 0, s>>>(part, groups, m, scales, tol, gamma, ctl);
  check_launch("cg_init");
}

// alpha_j = gamma_j / d_j.Hd_j with the reference's breakdown rules (solvers.cpp:55-71).
__global__ void cg_alpha_kernel(const double* part, int groups, int m, const double* gamma, double* alpha,
                                CgCtl* ctl) {
  if (ctl->stop) return;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < m; j += nw) {
    const double denom = warp_gsum(part, groups, m, j);
    if (lane == 0) {
      double a;
      if (denom > 0.0) a = gamma[j] / denom;
      else if (gamma[j] == 0.0 && denom == 0.0) a = 0.0;
      else a = __longlong_as_double(0x7ff8000000000000ULL);
      alpha[j] = a;
      if (!isfinite(a)) atomicOr(&bad, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad) {
    ctl->aborted = 1;
    ctl->stop = 1;
  }
}
void cg_alpha_launch(const double* part, int groups, int m, const double* gamma, double* alpha, CgCtl* ctl,
                     cudaStream_t s) {
  cg_alpha_kernel<<<1, 1024, 0, s>>>(part, groups, m, gamma, alpha, ctl);
  check_launch("cg_alpha");
}

// v += d*alpha ; r -= hd*alpha (solvers.cpp:72-73); products rounded before the add.
__global__ void cg_update_kernel(double* v, double* r, const double* d, const double* hd, const double* alpha,
                                 int n, int m, const int* skip) {
  SKIP_IF(skip);
  const long long total = static_cast<long long>(n) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double a = alpha[e % m];
    v[e] = __dadd_rn(v[e], __dmul_rn(d[e], a));
    r[e] = __dsub_rn(r[e], __dmul_rn(hd[e], a));
  }
}
void cg_update_launch(double* v, double* r, const double* d, const double* hd, const double* alpha, int n, int m,
                      const int* skip, cudaStream_t s) {
  cg_update_kernel<<<blocks_for(static_cast<long long>(n) * m, 256), 256, 0, s>>>(v, r, d, hd, alpha, n, m, skip);
  check_launch("cg_update");
}

// gamma' = r.p, beta = gamma'/gamma (0 if gamma == 0), iteration++, termination.
__global__ void cg_beta_kernel(const double* part, int groups, int m, const double* scales, double tol,
                               double* gamma, double* beta, CgCtl* ctl) {
  if (ctl->stop) return;
  __shared__ double ss[512];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < m; j += nw) {
    const double gn = warp_gsum(part, groups, 2 * m, j);
    const double q = warp_gsum(part, groups, 2 * m, m + j);
    if (lane == 0) {
      beta[j] = gamma[j] != 0.0 ? gn / gamma[j] : 0.0;
      gamma[j] = gn;
      ss[j] = q;
    }
  }
  __syncthreads();
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    ctl->iters += 1;
    ctl->mean_norm = mean;
    ctl->probe_norm = probe;
    ctl->done = done;
    ctl->stop = (done || ctl->iters >= ctl->budget) ? 1 : 0;
  }
}
void cg_beta_launch(const double* part, int groups, int m, const double* scales, double tol, double* gamma,
                    double* beta, CgCtl* ctl, cudaStream_t s) {
  cg_beta_kernel<<<1, 1024, 0, s>>>(part, groups, m, scales, tol, gamma, beta, ctl);
  check_launch("cg_beta");
}

// d = p + d*beta (solvers.cpp:80) and its FP32 copy for the next operator product.
__global__ void cg_direction_kernel(double* d, const double* p, const double* beta, int n, int m, float* d32,
                                    int ldv, const int* skip) {
  SKIP_IF(skip);
  if (!d32) {  // tcgen05 path: the operator packs d itself
    const long long tot = static_cast<long long>(n) * m;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x)
      d[e] = __dadd_rn(p[e], __dmul_rn(d[e], beta[e % m]));
    return;
  }
  const long long total = static_cast<long long>(n) * ldv;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / ldv), j = static_cast<int>(e % ldv);
    if (j < m) {
      const size_t o = static_cast<size_t>(i) * m + j;
      const double nd = __dadd_rn(p[o], __dmul_rn(d[o], beta[j]));
      d[o] = nd;
      d32[e] = static_cast<float>(nd);
    } else {
      d32[e] = 0.f;
    }
  }
}
void cg_direction_launch(double* d, const double* p, const double* beta, int n, int m, float* d32, int ldv,
                         const int* skip, cudaStream_t s) {
  cg_direction_kernel<<<blocks_for(static_cast<long long>(n) * (d32 ? ldv : m), 256), 256, 0, s>>>(d, p, beta, n, m,
                                                                                                 d32, ldv, skip);
  check_launch("cg_direction");
}

__global__ void norms_kernel(const double* part, int groups, int m, const double* scales, double tol, double* out3) {
  __shared__ double ss[512];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < m; j += nw) {
    const double q = warp_gsum(part, groups, m, j);
    if (lane == 0) ss[j] = q;
  }
  __syncthreads();
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    out3[0] = mean;
    out3[1] = probe;
    out3[2] = done;
  }
}
void norms_launch(const double* part, int groups, int m, const double* scales, double tol, double* out3,
                  cudaStream_t s) {
  norms_kernel<<<1, 1024, 0, s>>>(part, groups, m, scales, tol, out3);
  check_launch("norms");
}

// ------------------------------------------------------ preconditioner K7
// Per-group (max, lowest index) of diag; strict '>' scan semantics
// (pivoted_cholesky.cpp:22-27).
__global__ void argmax_partials_kernel(const double* diag, int n, double* pval, int* pidx) {
  __shared__ double sv[256];
  __shared__ int si[256];
  const int g = blockIdx.x, G = gridDim.x;
  const int rb = static_cast<int>(static_cast<long long>(n) * g / G);
  const int re = static_cast<int>(static_cast<long long>(n) * (g + 1) / G);
  double best = -DBL_MAX;
  int bi = 0x7fffffff;
  for (int i = rb + threadIdx.x; i < re; i += blockDim.x) {
    const double v = diag[i];
    if (v > best) { best = v; bi = i; }  // ascending i per thread: first max kept
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double v2 = sv[threadIdx.x + off];
      const int i2 = si[threadIdx.x + off];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pval[g] = sv[0];
    pidx[g] = si[0];
  }
}
void argmax_partials_launch(const double* diag, int n, double* pval, int* pidx, int groups, cudaStream_t s) {
  argmax_partials_kernel<<<groups, 256, 0, s>>>(diag, n, pval, pidx);
  check_launch("argmax_partials");
}

__device__ __forceinline__ double matern64(const double* xs64, int d, int i, int c, double s2) {
  const double* a = xs64 + static_cast<size_t>(i) * d;
  const double* b = xs64 + static_cast<size_t>(c) * d;
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = b[k] - a[k];
    r2 += t * t;
  }
  const double r = sqrt(r2);
  return s2 * (1.0 + kSqrt3 * r) * exp(-kSqrt3 * r);  // kernel.cpp:35-39
}

// One greedy step (pivoted_cholesky.cpp:19-39): pivot = argmax diag; column
// = (k(:, pivot) - L[:, :m] L[pivot, :m]^T) / sqrt(best); diag -= column^2.
__global__ void __launch_bounds__(256) pchol_step_kernel(const double* xs64, int n, int d, double s2,
                                                         const double* pval, const int* pidx, int groups, double* L,
                                                         int ldl, int mcol, double* diag, int* pivots, int* stop_flag) {
  if (*stop_flag) return;
  __shared__ double s_best;
  __shared__ int s_piv;
  __shared__ double lp[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {  // argmax over the group partials: larger value, then lower index (strict '>' scan order)
    double best = -DBL_MAX;
    int bi = 0x7fffffff;
    for (int g = lane; g < groups; g += 32)
      if (pval[g] > best || (pval[g] == best && pidx[g] < bi)) {
        best = pval[g];
        bi = pidx[g];
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_best = best;
      s_piv = bi;
    }
  }
  __syncthreads();
  const double best = s_best;
  const int piv = s_piv;
  if (!(best > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *stop_flag = 1;
    return;
  }
  for (int k = threadIdx.x; k < mcol; k += blockDim.x) lp[k] = L[static_cast<size_t>(piv) * ldl + k];
  __syncthreads();
  const double sb = sqrt(best);
  // A warp takes PR <= 16 rows at a time: the lanes split each row's rank-mcol dot
  // product with the pivot row (butterfly sum: every lane ends with the same
  // bits), lane r keeps row r's, and then the PR lanes evaluate their rows'
  // kernel entries side by side. (With lane 0 evaluating one row at a time
  // the FP64 distance / sqrt / exp chain ran serially for every row: 45.7 us
  // per step at n = 43008, 100 steps per preconditioner build.)
  // PR = rows per warp at one iteration each (1 while there is a warp per row)
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  const int PR = min(16, (n + nw - 1) / nw);
  for (int i0 = gw * PR; i0 < n; i0 += nw * PR) {
    const int nrows = min(PR, n - i0);
    double mine = 0.0;
#pragma unroll 4
    for (int r = 0; r < nrows; ++r) {
      const double* li = L + static_cast<size_t>(i0 + r) * ldl;
      double acc = 0.0;
      for (int k = lane; k < mcol; k += 32) acc += li[k] * lp[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == r) mine = acc;
    }
    if (lane < nrows) {
      const int i = i0 + lane;
      const double col = (matern64(xs64, d, piv, i, s2) - mine) / sb;
      L[static_cast<size_t>(i) * ldl + mcol] = col;
      diag[i] = (i == piv) ? 0.0 : diag[i] - col * col;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) pivots[mcol] = piv;
}
void pchol_step_launch(const double* xs64, int n, int d, double s2, const double* pval, const int* pidx, int groups,
                       double* L, int ldl, int mcol, double* diag, int* pivots, int* stop_flag, cudaStream_t s) {
  if (mcol > 1024) throw std::invalid_argument("gpk: preconditioner rank > 1024 is not supported");
  pchol_step_kernel<<<std::min((n + 7) / 8, 148 * 4), 256, 0, s>>>(xs64, n, d, s2, pval, pidx, groups, L, ldl, mcol,
                                                                  diag, pivots, stop_flag);
  check_launch("pchol_step");
}

// part[g][a*r + b] = sum_{i in group} L[i][a] L[i][b]
__global__ void gram_partials_kernel(const double* L, int n, int r, int ldl, double* part) {
  const int g = blockIdx.x, G = gridDim.x;
  const int rb = static_cast<int>(static_cast<long long>(n) * g / G);
  const int re = static_cast<int>(static_cast<long long>(n) * (g + 1) / G);
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int a = e / r, b = e % r;
    double acc = 0.0;
    for (int i = rb; i < re; ++i) acc += L[static_cast<size_t>(i) * ldl + a] * L[static_cast<size_t>(i) * ldl + b];
    part[static_cast<size_t>(g) * r * r + e] = acc;
  }
}
void gram_partials_launch(const double* L, int n, int r, int ldl, double* part, int groups, cudaStream_t s) {
  gram_partials_kernel<<<groups, 256, 0, s>>>(L, n, r, ldl, part);
  check_launch("gram_partials");
}

// part[g][k*m + j] = sum_{i in group} L[i][k] R[i][j]
__global__ void lt_times_kernel(const double* L, int n, int r, int ldl, const double* R, int m, double* part,
                                const int* skip) {
  SKIP_IF(skip);
  const int g = blockIdx.x, G = gridDim.x;
  const int rb = static_cast<int>(static_cast<long long>(n) * g / G);
  const int re = static_cast<int>(static_cast<long long>(n) * (g + 1) / G);
  for (int e = threadIdx.x; e < r * m; e += blockDim.x) {
    const int k = e / m, j = e % m;
    double acc = 0.0;
    for (int i = rb; i < re; ++i) acc += L[static_cast<size_t>(i) * ldl + k] * R[static_cast<size_t>(i) * m + j];
    part[static_cast<size_t>(g) * r * m + e] = acc;
  }
}
void lt_times_launch(const double* L, int n, int r, int ldl, const double* R, int m, double* part, int groups,
                     const int* skip, cudaStream_t s) {
  lt_times_kernel<<<groups, 256, 0, s>>>(L, n, r, ldl, R, m, part, skip);
  check_launch("lt_times");
}

__global__ void sum_partials_kernel(const double* part, int groups, int count, double* out, const int* skip) {
  SKIP_IF(skip);
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int e = gw; e < count; e += nw) {
    const double v = warp_gsum(part, groups, count, e);
    if ((threadIdx.x & 31) == 0) out[e] = v;
  }
}
// scales_j = sqrt(ss_j) + 1e-12 (linear_system.cpp:21), inv_j = 1 / scales_j
// (IEEE sqrt and division: the host formulas' results).
__global__ void scales_kernel(const double* ss, int m, double* scales, double* inv) {
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double sc = sqrt(ss[j]) + 1e-12;
    if (scales) scales[j] = sc;
    if (inv) inv[j] = 1.0 / sc;
  }
}
void scales_launch(const double* ss, int m, double* scales, double* inv, cudaStream_t s) {
  scales_kernel<<<1, 128, 0, s>>>(ss, m, scales, inv);
  check_launch("scales");
}
__global__ void inv_scales_kernel(const double* scales, int m, double* inv) {
  for (int j = threadIdx.x; j < m; j += blockDim.x) inv[j] = 1.0 / scales[j];
}
void inv_scales_launch(const double* scales, int m, double* inv, cudaStream_t s) {
  inv_scales_kernel<<<1, 128, 0, s>>>(scales, m, inv);
  check_launch("inv_scales");
}

void sum_partials_launch(const double* part, int groups, int count, double* out, const int* skip, cudaStream_t s) {
  sum_partials_kernel<<<blocks_for(static_cast<long long>(count) * 32, 256, 1024), 256, 0, s>>>(part, groups, count,
                                                                                               out, skip);
  check_launch("sum_partials");
}

// C[ra x cb] = A[ra x ca] B[ca x cb], all row-major.
__global__ void small_gemm_kernel(const double* A, int ra, int ca, const double* B, int cb, double* Cm,
                                  const int* skip) {
  SKIP_IF(skip);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ra * cb; e += gridDim.x * blockDim.x) {
    const int i = e / cb, j = e % cb;
    double acc = 0.0;
    for (int k = 0; k < ca; ++k) acc += A[static_cast<size_t>(i) * ca + k] * B[static_cast<size_t>(k) * cb + j];
    Cm[e] = acc;
  }
}
void small_gemm_launch(const double* A, int ra, int ca, const double* B, int cb, double* Cm, const int* skip,
                       cudaStream_t s) {
  small_gemm_kernel<<<blocks_for(static_cast<long long>(ra) * cb, 128, 512), 128, 0, s>>>(A, ra, ca, B, cb, Cm, skip);
  check_launch("small_gemm");
}

// out = (R - L inner) / sigma^2 (pivoted_cholesky.cpp:56-57).
__global__ void woodbury_kernel(const double* R, const double* L, int n, int r, int ldl, const double* inner, int m,
                                double sigma2, double* out, const int* skip) {
  SKIP_IF(skip);
  const long long total = static_cast<long long>(n) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / m), j = static_cast<int>(e % m);
    const double* li = L + static_cast<size_t>(i) * ldl;
    double acc = 0.0;
    for (int k = 0; k < r; ++k) acc += li[k] * inner[static_cast<size_t>(k) * m + j];
    out[e] = (R[e] - acc) / sigma2;
  }
}
void woodbury_launch(const double* R, const double* L, int n, int r, int ldl, const double* inner, int m,
                     double sigma2, double* out, const int* skip, cudaStream_t s) {
  woodbury_kernel<<<blocks_for(static_cast<long long>(n) * m, 256), 256, 0, s>>>(R, L, n, r, ldl, inner, m, sigma2,
                                                                               out, skip);
  check_launch("woodbury");
}

__global__ void scale_kernel(const double* src, long long count, double factor, double* dst, const int* skip) {
  SKIP_IF(skip);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[e] = src[e] / factor;
}
void scale_launch(const double* src, int count, double factor, double* dst, const int* skip, cudaStream_t s) {
  scale_kernel<<<blocks_for(count, 256), 256, 0, s>>>(src, count, factor, dst, skip);
  check_launch("scale");
}

// FP64 dense block of H (kernel.cpp:179-184), row-major [rows][ldo].
__global__ void dense_block64_kernel(const double* xs64, int n, int d, double s2, double sigma2, int r0, int rows,
                                     int c0, int cols, double* out, int ldo, int add_noise) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / cols), c = static_cast<int>(e % cols);
    double v = matern64(xs64, d, r0 + r, c0 + c, s2);
    if (add_noise && r0 + r == c0 + c) v += sigma2;
    out[static_cast<size_t>(r) * ldo + c] = v;
  }
}
void dense_block64_launch(const double* xs64, int n, int d, double s2, double sigma2, int r0, int rows, int c0,
                          int cols, double* out, int ldo, int add_noise, cudaStream_t s) {
  dense_block64_kernel<<<blocks_for(static_cast<long long>(rows) * cols, 256), 256, 0, s>>>(
      xs64, n, d, s2, sigma2, r0, rows, c0, cols, out, ldo, add_noise);
  check_launch("dense_block64");
}

// All AP diagonal blocks H[blk_k, blk_k] (block x block, FP64) in one launch;
// the last block's rows/columns beyond n are identity padding. CTA = one 32 x 32
// tile of one block (grid.z = block index): its 32 row and 32 column points are
// staged in shared memory, each thread forms 4 entries (same arithmetic as
// matern64, kernel.cpp:35-39).
__global__ void ap_blocks_kernel(const double* xs64, int n, int d, const double* hyp, int block, double* mats) {
  __shared__ double xr[32][33], xc[32][33];
  const double s2 = hyp[0], sigma2 = hyp[1];  // device copy: the launch is graph-replayable
  const int k = blockIdx.z, r0 = k * block, len = min(block, n - r0);
  const int tr = blockIdx.y * 32, tcl = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int a = e / 32, q = e % 32;
    xr[a][q] = (q < d && tr + a < len) ? xs64[static_cast<size_t>(r0 + tr + a) * d + q] : 0.0;
    xc[a][q] = (q < d && tcl + a < len) ? xs64[static_cast<size_t>(r0 + tcl + a) * d + q] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x & 31;
  double* out = mats + static_cast<size_t>(k) * block * block;
  for (int rr = threadIdx.x >> 5; rr < 32; rr += blockDim.x >> 5) {
    const int r = tr + rr, cc = tcl + c;
    if (r >= block || cc >= block) continue;
    double v;
    if (r < len && cc < len) {
      double r2 = 0.0;
      for (int q = 0; q < d; ++q) {
        const double t = xc[c][q] - xr[rr][q];
        r2 += t * t;
      }
      const double rad = sqrt(r2);
      v = s2 * (1.0 + kSqrt3 * rad) * exp(-kSqrt3 * rad);
      if (r == cc) v += sigma2;
    } else {
      v = r == cc ? 1.0 : 0.0;
    }
    out[static_cast<size_t>(r) * block + cc] = v;
  }
}
void ap_blocks_launch(const double* xs64, int n, int d, const double* hyp, int block, int nblocks, double* mats,
                      cudaStream_t s) {
  if (d > 32) throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  dim3 grid((block + 31) / 32, (block + 31) / 32, nblocks);
  ap_blocks_kernel<<<grid, 256, 0, s>>>(xs64, n, d, hyp, block, mats);
  check_launch("ap_blocks");
}

// Leaf of the recursive SPD inversion: the nn x nn (nn <= 64) diagonal
// sub-block at (off, off) of every matrix (column-major, leading dimension ld,
// matrix stride `stride`) is inverted by in-place Gauss-Jordan elimination
// without pivoting (stable for SPD; the pivots are the Schur-complement
// diagonal, a non-positive one flags the matrix) and written to the same
// sub-block of `out`. One CTA per matrix; the 64 x 64 working matrix lives in
// registers (thread (ty, tx) of 16 x 16 owns rows 4ty.., columns 4tx..; rows
// and columns beyond nn are identity padding); pivot row and column are
// exchanged through double-buffered shared memory, one barrier per step.
__global__ void __launch_bounds__(256) spd_leaf_inverse_kernel(const double* a, double* out, int off, int nn, int ld,
                                                               long long stride, int* info) {
  __shared__ double colb[2][64], rowb[2][64];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const double* A = a + blockIdx.x * stride + off + static_cast<size_t>(off) * ld;
  double* B = out + blockIdx.x * stride + off + static_cast<size_t>(off) * ld;
  double M[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * ty + p, j = 4 * tx + q;
      M[p][q] = (i < nn && j < nn) ? A[i + static_cast<size_t>(j) * ld] : (i == j ? 1.0 : 0.0);
    }
  bool bad = false;
  for (int k = 0; k < 64; ++k) {
    const int buf = k & 1;
    const int kq = k & 3;  // register selects with static indices keep M out of local memory
    if (tx == (k >> 2)) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
        colb[buf][4 * ty + p] = kq == 0 ? M[p][0] : kq == 1 ? M[p][1] : kq == 2 ? M[p][2] : M[p][3];
    }
    if (ty == (k >> 2)) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        rowb[buf][4 * tx + q] = kq == 0 ? M[0][q] : kq == 1 ? M[1][q] : kq == 2 ? M[2][q] : M[3][q];
    }
    __syncthreads();
    const double pk = rowb[buf][k];
    bad |= !(pk > 0.0);
    const double piv = 1.0 / pk;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int i = 4 * ty + p;
      const double ci = colb[buf][i] * piv;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * tx + q;
        const double m = M[p][q];
        double v = fma(-ci, rowb[buf][j], m);
        if (j == k) v = -m * piv;
        if (i == k) v = (j == k) ? piv : m * piv;
        M[p][q] = v;
      }
    }
  }
  if (bad && threadIdx.x == 0) info[blockIdx.x] = 1;
  // symmetrise the rounding: the recursion's Schur updates assume symmetric
  // leaf inverses (the antisymmetric GJ rounding otherwise propagates)
  __shared__ double S[64][65];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) S[4 * ty + p][4 * tx + q] = M[p][q];
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 4 * ty + p, j = 4 * tx + q;
      if (i < nn && j < nn) B[i + static_cast<size_t>(j) * ld] = 0.5 * (S[i][j] + S[j][i]);
    }
}
void spd_leaf_inverse_launch(const double* a, double* out, int off, int nn, int ld, long long stride, int batch,
                             int* info, cudaStream_t s) {
  if (nn > 64) throw std::invalid_argument("spd_leaf_inverse: block > 64");
  spd_leaf_inverse_kernel<<<batch, 256, 0, s>>>(a, out, off, nn, ld, stride, info);
  check_launch("spd_leaf_inverse");
}

// dst (rows x cols block) = src^T (cols x rows block), per matrix.
__global__ void block_transpose_kernel(const double* src, double* dst, int rows, int cols, int ld, long long stride) {
  const long long per = static_cast<long long>(rows) * cols;
  const long long total = per * gridDim.y;
  (void)total;
  const double* S = src + blockIdx.y * stride;
  double* D = dst + blockIdx.y * stride;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < per;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % rows), j = static_cast<int>(e / rows);  // dst(i, j) = src(j, i)
    D[i + static_cast<size_t>(j) * ld] = S[j + static_cast<size_t>(i) * ld];
  }
}
void block_transpose_launch(const double* src, double* dst, int rows, int cols, int ld, long long stride, int batch,
                            cudaStream_t s) {
  const long long per = static_cast<long long>(rows) * cols;
  dim3 grid(static_cast<unsigned>(std::min<long long>((per + 255) / 256, 64)), batch);
  block_transpose_kernel<<<grid, 256, 0, s>>>(src, dst, rows, cols, ld, stride);
  check_launch("block_transpose");
}

// Exact marginal-likelihood gradient forms (exact.cpp:33-50): with
// W = (alpha alpha^T - H^-1) / 2, the constrained gradient is
// sum_ij W_ij dH_ij/dtheta; dH is evaluated on the fly (FP64, kernel.cpp:200-232
// in scaled differences), W from alpha and the lower triangle of H^-1
// (column-major, cuSOLVER potri). CTA = one 32 x 32 tile (ti >= tj, weight 2
// off the diagonal tile and for i > j inside it); per-CTA partials
// [d lengthscale sums | signal sum | diagonal sum] in a fixed order.
__global__ void exact_forms_kernel(const double* xs64, int n, int d, const double* hinv, const double* alpha,
                                   double* part) {
  __shared__ double xr[32][33], xc[32][33];
  __shared__ double red[8][34];
  const int T = (n + 31) / 32;
  const long long L = blockIdx.x;
  // tile (ti, tj), ti >= tj: row-major lower-triangle enumeration
  int ti = static_cast<int>((sqrt(8.0 * static_cast<double>(L) + 1.0) - 1.0) / 2.0);
  while (static_cast<long long>(ti) * (ti + 1) / 2 > L) --ti;
  while (static_cast<long long>(ti + 1) * (ti + 2) / 2 <= L) ++ti;
  const int tj = static_cast<int>(L - static_cast<long long>(ti) * (ti + 1) / 2);
  (void)T;
  for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
    const int a = e / 32, q = e % 32;
    const int ri = ti * 32 + a, rj = tj * 32 + a;
    xr[a][q] = (q < d && ri < n) ? xs64[static_cast<size_t>(ri) * d + q] : 0.0;
    xc[a][q] = (q < d && rj < n) ? xs64[static_cast<size_t>(rj) * d + q] : 0.0;
  }
  __syncthreads();
  double al[32], as = 0.0, an = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) al[k] = 0.0;
  const int c = threadIdx.x & 31;
  const int j = tj * 32 + c;
  for (int rr = threadIdx.x >> 5; rr < 32; rr += blockDim.x >> 5) {
    const int i = ti * 32 + rr;
    if (i >= n || j >= n || i < j) continue;
    const double Wij = 0.5 * (alpha[i] * alpha[j] - hinv[static_cast<size_t>(i) + static_cast<size_t>(j) * n]);
    const double w = (i == j) ? Wij : 2.0 * Wij;
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = xc[c][k] - xr[rr][k];
      r2 += t * t;
    }
    const double r = sqrt(r2);
    const double e0 = exp(-1.7320508075688772 * r);
    as += w * (1.0 + 1.7320508075688772 * r) * e0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < d) {
        const double t = xc[c][k] - xr[rr][k];
        al[k] += w * e0 * (t * t);
      }
    if (i == j) an += Wij;
  }
  // fixed-order block reduction: warp xor trees, then warps in order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < d + 2; ++k) {
    double v = k < d ? al[k < 32 ? k : 0] : (k == d ? as : an);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < d + 2; k += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += red[w][k];
    part[static_cast<size_t>(blockIdx.x) * (d + 2) + k] = v;
  }
}
void exact_forms_launch(const double* xs64, int n, int d, const double* hinv, const double* alpha, double* part,
                        cudaStream_t s) {
  if (d > 32) throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  const long long T = (n + 31) / 32;
  exact_forms_kernel<<<static_cast<unsigned>(T * (T + 1) / 2), 256, 0, s>>>(xs64, n, d, hinv, alpha, part);
  check_launch("exact_forms");
}
long long exact_forms_blocks(int n) {
  const long long T = (n + 31) / 32;
  return T * (T + 1) / 2;
}

__global__ void set_identity_kernel(double* mats, int dim, long long total) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long w = e % (static_cast<long long>(dim) * dim);
    mats[e] = (w / dim == w % dim) ? 1.0 : 0.0;
  }
}
void set_identity_launch(double* mats, int dim, int batch, cudaStream_t s) {
  const long long total = static_cast<long long>(dim) * dim * batch;
  set_identity_kernel<<<blocks_for(total, 256), 256, 0, s>>>(mats, dim, total);
  check_launch("set_identity");
}

// ------------------------------------------------------------------ AP K8
// score_k = || R[blk_k] * inv_scales || (solvers.cpp:123-132); one CTA per block.
__global__ void ap_scores_kernel(const double* R, int n, int m, const double* inv_scales, int block, double* scores,
                                 const int* skip) {
  SKIP_IF(skip);
  __shared__ double red[256];
  const int k = blockIdx.x;
  const int r0 = k * block, r1 = min(n, r0 + block);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int i = r0 + warp; i < r1; i += nw) {  // warp per row: coalesced
    double w = 0.0;
    const double* row = R + static_cast<size_t>(i) * m;
    for (int j = lane; j < m; j += 32) w += row[j] * inv_scales[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    acc += w * w;  // identical on every lane
  }
  red[threadIdx.x] = lane == 0 ? acc : 0.0;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) scores[k] = sqrt(red[0]);
}
void ap_scores_launch(const double* R, int n, int m, const double* inv_scales, int block, int nblocks, double* scores,
                      const int* skip, cudaStream_t s) {
  ap_scores_kernel<<<nblocks, 256, 0, s>>>(R, n, m, inv_scales, block, scores, skip);
  check_launch("ap_scores");
}

__global__ void ap_select_kernel(const double* scores, int nblocks, int* sel, const int* skip) {
  SKIP_IF(skip);
  int best_k = 0;
  double best = -1.0;
  for (int k = 0; k < nblocks; ++k)
    if (scores[k] > best) { best = scores[k]; best_k = k; }
  *sel = best_k;
}
void ap_select_launch(const double* scores, int nblocks, int* sel, const int* skip, cudaStream_t s) {
  ap_select_kernel<<<1, 1, 0, s>>>(scores, nblocks, sel, skip);
  check_launch("ap_select");
}

// upd = Hinv[sel] R[blk]; V[blk] += upd; FP32 copy for the slab kernel.
__global__ void ap_block_update_kernel(const double* inv_blocks, int block, int n, const int* sel, const double* R,
                                       int m, double* V, double* upd64, float* upd32, int ldv32, const int* skip) {
  SKIP_IF(skip);
  // upd[i][j] = sum_c Hinv[i][c] R[r0 + c][j]; CTA = 8 rows x all m columns,
  // thread (ty = row, tx) owns columns tx, tx+32, tx+64; R staged by 64-row chunks.
  constexpr int RPC = 8, KC = 32, MAXM = 96;
  __shared__ double rs[KC][MAXM];
  __shared__ double hs[RPC][KC];
  const int k = *sel;
  const int r0 = k * block, len = min(block, n - r0);
  const double* Hi = inv_blocks + static_cast<size_t>(k) * block * block;
  const int i0 = blockIdx.x * RPC;
  if (i0 >= len) return;
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int c0 = 0; c0 < len; c0 += KC) {
    const int kc = min(KC, len - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < kc * m; e += blockDim.x) {
      const int c = e / m, j = e % m;
      rs[c][j] = R[static_cast<size_t>(r0 + c0 + c) * m + j];
    }
    for (int e = threadIdx.x; e < RPC * KC; e += blockDim.x) {
      const int rr = e / KC, c = e % KC;
      hs[rr][c] = (i0 + rr < len && c < kc) ? Hi[static_cast<size_t>(i0 + rr) * block + c0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < kc; ++c) {
      const double h = hs[ty][c];
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (tx + 32 * q < m) acc[q] += h * rs[c][tx + 32 * q];
    }
  }
  const int i = i0 + ty;
  if (i < len) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = tx + 32 * q;
      if (j < m) {
        upd64[static_cast<size_t>(i) * m + j] = acc[q];
        upd32[static_cast<size_t>(i) * ldv32 + j] = static_cast<float>(acc[q]);
        V[static_cast<size_t>(r0 + i) * m + j] += acc[q];
      }
    }
    for (int j = m + tx; j < ldv32; j += 32) upd32[static_cast<size_t>(i) * ldv32 + j] = 0.f;
  }
}
void ap_block_update_launch(const double* inv_blocks, int block, int n, const int* sel, const double* R, int m,
                            double* V, double* upd64, float* upd32, int ldv32, const int* skip, cudaStream_t s) {
  if (m > 96) throw std::invalid_argument("gpk: AP supports at most 96 right-hand sides");
  ap_block_update_kernel<<<(block + 7) / 8, 256, 0, s>>>(inv_blocks, block, n, sel, R, m, V, upd64, upd32, ldv32, skip);
  check_launch("ap_block_update");
}

__global__ void ap_select_groups_kernel(const double* spart, int nblocks, int gpb, int* sel, const int* skip) {
  SKIP_IF(skip);
  __shared__ double sc[4096];
  for (int k = threadIdx.x; k < nblocks; k += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < gpb; ++q) t += spart[static_cast<size_t>(k) * gpb + q];
    sc[k] = sqrt(t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best_k = 0;
    double best = -1.0;
    for (int k = 0; k < nblocks; ++k)
      if (sc[k] > best) { best = sc[k]; best_k = k; }  // strict '>' as solvers.cpp:129
    *sel = best_k;
  }
}
void ap_select_groups_launch(const double* spart, int nblocks, int gpb, int* sel, const int* skip, cudaStream_t s) {
  if (nblocks > 4096) throw std::invalid_argument("gpk: at most 4096 AP blocks");
  ap_select_groups_kernel<<<1, 256, 0, s>>>(spart, nblocks, gpb, sel, skip);
  check_launch("ap_select_groups");
}

__global__ void ap_gather_kernel(const double* R, int n, int m, int block, const int* sel, double* Rs,
                                 const double* inv_blocks, double* upd, double** ptrs, const int* skip) {
  SKIP_IF(skip);
  const int k = *sel;
  const int r0 = k * block, len = min(block, n - r0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ptrs[0] = Rs;
    ptrs[1] = const_cast<double*>(inv_blocks) + static_cast<size_t>(k) * block * block;
    ptrs[2] = upd;
  }
  const long long total = static_cast<long long>(block) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = e / m;
    Rs[e] = c < len ? R[static_cast<size_t>(r0) * m + e] : 0.0;
  }
}
void ap_gather_launch(const double* R, int n, int m, int block, const int* sel, double* Rs, const double* inv_blocks,
                      double* upd, double** ptrs, const int* skip, cudaStream_t s) {
  ap_gather_kernel<<<blocks_for(static_cast<long long>(block) * m, 256, 148), 256, 0, s>>>(R, n, m, block, sel, Rs,
                                                                                         inv_blocks, upd, ptrs, skip);
  check_launch("ap_gather");
}

__global__ void ap_apply_update_kernel(const double* upd, int n, int m, int block, const int* sel, double* V,
                                       float* upd32, int ldv32, const int* skip) {
  SKIP_IF(skip);
  const int k = *sel;
  const int r0 = k * block, len = min(block, n - r0);
  const long long total = static_cast<long long>(len) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / m;
    const int j = static_cast<int>(e % m);
    V[static_cast<size_t>(r0) * m + e] += upd[e];  // solutions[blk] += update (solvers.cpp:136)
    if (upd32) upd32[i * ldv32 + j] = static_cast<float>(upd[e]);
  }
}
void ap_apply_update_launch(const double* upd, int n, int m, int block, const int* sel, double* V, float* upd32,
                            int ldv32, const int* skip, cudaStream_t s) {
  ap_apply_update_kernel<<<blocks_for(static_cast<long long>(block) * m, 256, 148), 256, 0, s>>>(
      upd, n, m, block, sel, V, upd32, ldv32, skip);
  check_launch("ap_apply_update");
}

// One warp per update row i (8 rows per CTA); lane owns columns lane + 32 q.
__global__ void ap_update_pack_kernel(const double* R, int n, int m, int block, const int* sel,
                                      const double* inv_blocks, double* V, double* upd64, float* vpk, int npad,
                                      int rows_pad, const int* skip) {
  SKIP_IF(skip);
  const int k = *sel;
  const int r0 = k * block, len = min(block, n - r0);
  const double* Hi = inv_blocks + static_cast<size_t>(k) * block * block;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + warp;
  if (i >= rows_pad) return;  // rows in [len, rows_pad) pack as zeros
  double acc[3] = {0.0, 0.0, 0.0};
  if (i < len) {
    const double* hrow = Hi + static_cast<size_t>(i) * block;  // Hinv symmetric: row i == column i
    const double* rb = R + static_cast<size_t>(r0) * m;
#pragma unroll 4
    for (int c = 0; c < len; ++c) {
      const double h = hrow[c];
      const double* rr = rb + static_cast<size_t>(c) * m;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (lane + 32 * q < m) acc[q] = fma(h, rr[lane + 32 * q], acc[q]);
    }
  }
  const int img = npad * 32;
  const int chunk = i / 32, kk = i % 32;
  float* base = vpk + static_cast<size_t>(chunk) * 2 * img;
  for (int j = lane; j < npad; j += 32) {
    const int q = j / 32;
    double x = 0.0;
    if (i < len && j < m) {
      x = acc[q];
      upd64[static_cast<size_t>(i) * m + j] = x;
      V[static_cast<size_t>(r0 + i) * m + j] += x;  // solutions[blk] += update (solvers.cpp:136)
    }
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(static_cast<float>(x)));
    const float h = __uint_as_float(hb);
    uint32_t lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(static_cast<float>(x - static_cast<double>(h))));
    const int off = ((j / 8) * 8 + kk / 4) * 32 + (j % 8) * 4 + (kk % 4);
    base[off] = h;
    base[img + off] = __uint_as_float(lb);
  }
}
void ap_update_pack_launch(const double* R, int n, int m, int block, const int* sel, const double* inv_blocks,
                           double* V, double* upd64, float* vpk, int npad, const int* skip, cudaStream_t s) {
  if (m > 96) throw std::invalid_argument("gpk: AP supports at most 96 right-hand sides");
  const int rows = (block + 31) / 32 * 32;  // whole 32-row chunks (zero rows beyond the block)
  ap_update_pack_kernel<<<(rows + 7) / 8, 256, 0, s>>>(R, n, m, block, sel, inv_blocks, V, upd64, vpk, npad, rows,
                                                       skip);
  check_launch("ap_update_pack");
}

__global__ void ap_apply_pack_kernel(const double* upd64, int n, int m, int block, const int* sel, double* V,
                                     float* vpk, int npad, int rows_pad, const int* skip) {
  SKIP_IF(skip);
  const int k = *sel;
  const int r0 = k * block, len = min(block, n - r0);
  const int img = npad * 32;
  const long long total = static_cast<long long>(rows_pad) * npad;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    // e walks the 32-row TF32 images linearly (coalesced stores), see kv_pack_kernel
    const int q32 = static_cast<int>(e / img), w = static_cast<int>(e % img);
    const int core = w >> 5, ln = w & 31;
    const int j = (core >> 3) * 8 + (ln >> 2);
    const int i = q32 * 32 + (core & 7) * 4 + (ln & 3);
    double x = 0.0;
    if (i < len && j < m) {
      x = upd64[static_cast<size_t>(i) * m + j];
      V[static_cast<size_t>(r0 + i) * m + j] += x;  // solutions[blk] += update (solvers.cpp:136)
    }
    uint32_t hb, lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(static_cast<float>(x)));
    const float h = __uint_as_float(hb);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(static_cast<float>(x - static_cast<double>(h))));
    float* base = vpk + static_cast<size_t>(q32) * 2 * img;
    base[w] = h;
    base[img + w] = __uint_as_float(lb);
  }
}
void ap_apply_pack_launch(const double* upd64, int n, int m, int block, const int* sel, double* V, float* vpk,
                          int npad, const int* skip, cudaStream_t s) {
  const int rows = (block + 31) / 32 * 32;
  ap_apply_pack_kernel<<<blocks_for(static_cast<long long>(rows) * npad, 256), 256, 0, s>>>(upd64, n, m, block, sel,
                                                                                          V, vpk, npad, rows, skip);
  check_launch("ap_apply_pack");
}

// iteration++ ; termination from sum of squares partials.
__global__ void ap_check_kernel(const double* part, int groups, int m, const double* scales, double tol, CgCtl* ctl) {
  if (ctl->stop) return;
  __shared__ double ss[512];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < m; j += nw) {
    const double q = warp_gsum(part, groups, m, j);
    if (lane == 0) ss[j] = q;
  }
  __syncthreads();
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    ctl->iters += 1;
    ctl->mean_norm = mean;
    ctl->probe_norm = probe;
    ctl->done = done;
    ctl->stop = (done || ctl->iters >= ctl->budget) ? 1 : 0;
  }
}
void ap_check_launch(const double* part, int groups, int m, const double* scales, double tol, CgCtl* ctl,
                     cudaStream_t s) {
  ap_check_kernel<<<1, 1024, 0, s>>>(part, groups, m, scales, tol, ctl);
  check_launch("ap_check");
}

// ----------------------------------------------------------------- SGD
// Floyd sampling (rng.cpp:108-126) for iterations first..first+count-1 of a
// solve: iteration t consumes u64 draws [t*b, (t+1)*b) of stream
// (seed, kSolver = 6, substream). The modulo reductions are independent and
// run in parallel; the sequential collision pass touches only a bitmap; the
// sorted output is the bitmap's set bits in ascending order.
__global__ void sgd_batches_kernel(uint64_t seed, uint64_t substream, int n, int b, int first, int* out,
                                   const int* first_dev = nullptr, const int* skip = nullptr) {
  extern __shared__ unsigned bitmap[];
  __shared__ int tvals[1024];
  __shared__ int wcount[1025];
  if (skip && *skip) return;
  const int t = (first_dev ? *first_dev : first) + blockIdx.x;
  const int words = (n + 31) / 32;
  for (int w = threadIdx.x; w < words; w += blockDim.x) bitmap[w] = 0u;
  for (int q = threadIdx.x; q < b; q += blockDim.x) {
    const uint64_t k = static_cast<uint64_t>(t) * b + q;
    const uint64_t u = stream_u64(seed, 6, substream, k);
    const uint64_t bound = static_cast<uint64_t>(n - b + q) + 1;
    tvals[q] = static_cast<int>(u % bound);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < b; ++q) {
      const int j = n - b + q;
      const int tv = tvals[q];
      const int pick = ((bitmap[tv >> 5] >> (tv & 31)) & 1u) ? j : tv;
      bitmap[pick >> 5] |= 1u << (pick & 31);
    }
  }
  __syncthreads();
  // ascending set-bit positions: per-thread word ranges + exclusive scan
  const int per = (words + blockDim.x - 1) / blockDim.x;
  const int w0 = threadIdx.x * per, w1 = min(words, w0 + per);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
  wcount[threadIdx.x + 1] = cnt;
  if (threadIdx.x == 0) wcount[0] = 0;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 1; i <= blockDim.x; ++i) wcount[i] += wcount[i - 1];
  __syncthreads();
  int pos = wcount[threadIdx.x];
  int* o = out + static_cast<size_t>(blockIdx.x) * b;
  for (int w = w0; w < w1; ++w) {
    unsigned bits = bitmap[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      o[pos++] = w * 32 + bit;
      bits &= bits - 1;
    }
  }
}
size_t sgd_batches_smem(int n, int b) {
  if (b > 1024) throw std::invalid_argument("gpk: SGD batch_size > 1024 is not supported");
  const size_t smem = sizeof(unsigned) * ((n + 31) / 32);
  if (smem > 200 * 1024) throw std::invalid_argument("gpk: SGD sampling supports n <= 1.6M");
  static size_t configured = 0;
  // dynamic bitmap + ~8 KB static scratch must fit; raise the opt-in limit whenever it grows
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(sgd_batches_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  return smem;
}
void sgd_batches_launch(uint64_t seed, uint64_t substream, int n, int b, int first, int count, int* out,
                        cudaStream_t s) {
  const size_t smem = sgd_batches_smem(n, b);
  sgd_batches_kernel<<<count, 256, smem, s>>>(seed, substream, n, b, first, out);
  check_launch("sgd_batches");
}
void sgd_batches_dev_launch(uint64_t seed, uint64_t substream, int n, int b, const int* first, int count, int* out,
                            const int* skip, cudaStream_t s) {
  const size_t smem = sgd_batches_smem(n, b);
  sgd_batches_kernel<<<count, 256, smem, s>>>(seed, substream, n, b, 0, out, first, skip);
  check_launch("sgd_batches");
}

// grad[q][j] = hv[q][j] - targets[idx[q]][j]
__global__ void sgd_step_kernel(const double* hv, const int* idx, int b, const double* targets, double* grad, int m,
                                const int* skip) {
  SKIP_IF(skip);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < b * m; e += gridDim.x * blockDim.x) {
    const int q = e / m, j = e % m;
    grad[e] = hv[e] - targets[static_cast<size_t>(idx[q]) * m + j];
  }
}
void sgd_step_launch(const double* hv, const int* idx, int b, const double* targets, double* grad, int m,
                     const int* skip, cudaStream_t s) {
  sgd_step_kernel<<<blocks_for(static_cast<long long>(b) * m, 256), 256, 0, s>>>(hv, idx, b, targets, grad, m, skip);
  check_launch("sgd_step");
}

__global__ void sgd_scatter_kernel(const int* idx, int b, int* pos, int value_is_q, const int* skip) {
  SKIP_IF(skip);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < b; q += gridDim.x * blockDim.x)
    pos[idx[q]] = value_is_q ? q : -1;
}
void sgd_scatter_launch(const int* idx, int b, int* pos, int value_is_q, const int* skip, cudaStream_t s) {
  sgd_scatter_kernel<<<blocks_for(b, 256), 256, 0, s>>>(idx, b, pos, value_is_q, skip);
  check_launch("sgd_scatter");
}

// momentum *= rho; momentum[idx] -= step*g; V += momentum (solvers.cpp:168-170).
__global__ void sgd_update_kernel(double* M, double* V, float* V32, int ldv, const int* pos, const double* grad,
                                  double rho, double step, int n, int m, int* nonfinite, const int* skip) {
  SKIP_IF(skip);
  const long long total = static_cast<long long>(n) * m;
  int bad = 0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / m), j = static_cast<int>(e % m);
    double mo = __dmul_rn(M[e], rho);
    const int q = pos[i];
    if (q >= 0) mo = __dsub_rn(mo, __dmul_rn(step, grad[static_cast<size_t>(q) * m + j]));
    M[e] = mo;
    const double v = __dadd_rn(V[e], mo);
    V[e] = v;
    V32[static_cast<size_t>(i) * ldv + j] = static_cast<float>(v);
    if (!isfinite(v)) bad = 1;
  }
  if (bad) atomicOr(nonfinite, 1);
}
void sgd_update_launch(double* M, double* V, float* V32, int ldv, const int* pos, const double* grad, double rho,
                       double step, int n, int m, int* nonfinite, const int* skip, cudaStream_t s) {
  sgd_update_kernel<<<blocks_for(static_cast<long long>(n) * m, 256), 256, 0, s>>>(M, V, V32, ldv, pos, grad, rho,
                                                                                 step, n, m, nonfinite, skip);
  check_launch("sgd_update");
}

// R[idx] = -g, with the per-column sum of squares updated incrementally.
__global__ void sgd_residual_kernel(double* R, const int* idx, int b, const double* grad, int m, double* sumsq,
                                    const int* skip) {
  SKIP_IF(skip);
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    double delta = 0.0;
    for (int q = 0; q < b; ++q) {
      double* rp = R + static_cast<size_t>(idx[q]) * m + j;
      const double old = *rp;
      const double nw = -grad[static_cast<size_t>(q) * m + j];
      delta += nw * nw - old * old;
      *rp = nw;
    }
    sumsq[j] += delta;
  }
}
void sgd_residual_launch(double* R, const int* idx, int b, const double* grad, int m, double* sumsq, const int* skip,
                         cudaStream_t s) {
  sgd_residual_kernel<<<1, 128, 0, s>>>(R, idx, b, grad, m, sumsq, skip);
  check_launch("sgd_residual");
}

__global__ void sgd_check_kernel(const double* sumsq, int m, const double* scales, double tol, const int* nonfinite,
                                 CgCtl* ctl) {
  if (ctl->stop) return;
  if (*nonfinite) {
    if (threadIdx.x == 0) {
      ctl->iters += 1;
      ctl->aborted = 1;
      ctl->stop = 1;
    }
    return;
  }
  __shared__ double ss[512];
  for (int j = threadIdx.x; j < m; j += blockDim.x) ss[j] = fmax(sumsq[j], 0.0);
  __syncthreads();
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    ctl->iters += 1;
    ctl->mean_norm = mean;
    ctl->probe_norm = probe;
    ctl->done = done;
    ctl->stop = (done || ctl->iters >= ctl->budget) ? 1 : 0;
  }
}
void sgd_check_launch(const double* sumsq, int m, const double* scales, double tol, const int* nonfinite, CgCtl* ctl,
                      cudaStream_t s) {
  sgd_check_kernel<<<1, 128, 0, s>>>(sumsq, m, scales, tol, nonfinite, ctl);
  check_launch("sgd_check");
}

// ------------------------------------------------- SGD, row-sharded form
// H[idx] V = sum over ranks of K[idx, own rows] V_own (+ s2 V[idx] on the
// owning rank). Each rank contributes hv_part - B[idx] on its own rows, so the
// rank-ordered sum of slices is g = H[idx] V - B[idx] (solvers.cpp:166-167).
// The residual-estimate update R[idx] = -g changes the squared norms by
// sum_q g^2 - sum_{own q} R_old[idx_q]^2; the old squares travel with the
// slice so every rank updates an identical replicated copy.
__global__ void sgd_prep_kernel(const double* hv_part, const int* idx, int b, const double* targets,
                                const double* R, int row0, int nloc, int m, int* pos, const int* nonfinite,
                                double* slice, int grad_blocks, const int* skip) {
  SKIP_IF(skip);
  const int bm = b * m;
  if (static_cast<int>(blockIdx.x) >= grad_blocks) {
    // one block per column j: sum over the batch rows owned by this rank of
    // R_old[row][j]^2 (fixed order: strided lanes, xor trees, warps in order)
    const int j = blockIdx.x - grad_blocks;
    __shared__ double wsum[32];
    double acc = 0.0;
    for (int q = threadIdx.x; q < b; q += blockDim.x) {
      const int li = idx[q] - row0;
      if (li >= 0 && li < nloc) {
        const double r = R[static_cast<size_t>(li) * m + j];
        acc += r * r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += wsum[w];
      slice[bm + j] = t;
      if (j == 0) slice[bm + m] = *nonfinite ? 1.0 : 0.0;
    }
    if (j == 0)
      for (int q = threadIdx.x; q < b; q += blockDim.x) {
        const int li = idx[q] - row0;
        if (li >= 0 && li < nloc) pos[li] = q;
      }
    return;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bm; e += grad_blocks * blockDim.x) {
    const int q = e / m, jj = e - q * m;
    const int li = idx[q] - row0;
    double g = hv_part[e];
    if (li >= 0 && li < nloc) g -= targets[static_cast<size_t>(li) * m + jj];
    slice[e] = g;
  }
}
void sgd_prep_launch(const double* hv_part, const int* idx, int b, const double* targets, const double* R,
                     int row0, int nloc, int m, int* pos, const int* nonfinite, double* slice, const int* skip,
                     cudaStream_t s) {
  const int gb = blocks_for(static_cast<long long>(b) * m, 256, 64);
  sgd_prep_kernel<<<gb + m, 256, 0, s>>>(hv_part, idx, b, targets, R, row0, nloc, m, pos, nonfinite, slice, gb,
                                         skip);
  check_launch("sgd_prep");
}

__global__ void sgd_gsum_kernel(const double* gbuf, int nr, long long stride, int bm, double* grad,
                                const int* skip) {
  SKIP_IF(skip);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bm; e += gridDim.x * blockDim.x) {
    double g = gbuf[e];
    for (int r = 1; r < nr; ++r) g += gbuf[r * stride + e];  // rank order
    grad[e] = g;
  }
}
void sgd_gsum_launch(const double* gbuf, int nr, long long stride, int b, int m, double* grad, const int* skip,
                     cudaStream_t s) {
  sgd_gsum_kernel<<<blocks_for(static_cast<long long>(b) * m, 256, 64), 256, 0, s>>>(gbuf, nr, stride, b * m, grad,
                                                                                    skip);
  check_launch("sgd_gsum");
}

// Replicated termination test (solvers.cpp:172-177): one warp per column.
__global__ void sgd_check_sharded_kernel(const double* gbuf, int nr, long long stride, const double* grad, int b,
                                         int m, double* sumsq, const double* scales, double tol, CgCtl* ctl) {
  // pad = stop as it was before this test: this iteration's update still runs
  // when the test below terminates (solvers.cpp updates, then tests)
  const int stopped = ctl->stop;
  __syncthreads();
  if (threadIdx.x == 0) ctl->pad = stopped;
  if (stopped) return;
  __shared__ double ss[512];
  __shared__ int bad;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int bm = b * m;
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int r = 0; r < nr; ++r) f += gbuf[r * stride + bm + m];
    bad = f != 0.0;
  }
  __syncthreads();
  for (int j = warp; j < m; j += nw) {
    double acc = 0.0;
    for (int q = lane; q < b; q += 32) {
      const double g = grad[static_cast<size_t>(q) * m + j];
      acc += g * g;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      // a non-finite gradient makes this iteration's update non-finite
      // (solvers.cpp:168-171 tests the iterate right after it)
      if (!isfinite(acc)) bad = 1;
      double old = 0.0;
      for (int r = 0; r < nr; ++r) old += gbuf[r * stride + bm + j];
      const double v = sumsq[j] + (acc - old);
      sumsq[j] = v;
      ss[j] = fmax(v, 0.0);
    }
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) {
      ctl->iters += 1;
      ctl->aborted = 1;
      ctl->stop = 1;
    }
    return;
  }
  double mean, probe;
  int done;
  termination_block(ss, m, scales, tol, mean, probe, done);
  if (threadIdx.x == 0) {
    ctl->iters += 1;
    ctl->mean_norm = mean;
    ctl->probe_norm = probe;
    ctl->done = done;
    ctl->stop = (done || ctl->iters >= ctl->budget) ? 1 : 0;
  }
}
void sgd_check_sharded_launch(const double* gbuf, int nr, long long stride, const double* grad, int b, int m,
                              double* sumsq, const double* scales, double tol, CgCtl* ctl, cudaStream_t s) {
  sgd_check_sharded_kernel<<<1, 1024, 0, s>>>(gbuf, nr, stride, grad, b, m, sumsq, scales, tol, ctl);
  check_launch("sgd_check_sharded");
}

// momentum *= rho; momentum[idx] -= step g; V += momentum; R[idx] = -g, over
// this rank's rows, writing V's TF32 hi/lo operator images in the same pass
// (the kv_tc B-operand layout, see kv_pack_kernel).
__global__ void sgd_update_pack_kernel(double* M, double* V, double* R, float* vpk, int npad, int rows_pad,
                                       const int* pos, const double* grad, double rho, double step, int nloc, int m,
                                       int* nonfinite, const int* skip) {
  SKIP_IF(skip);
  const int img = npad * 32;
  const long long total = static_cast<long long>(rows_pad) * npad;
  int bad = 0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    // e walks the 32-row TF32 images linearly (coalesced stores), see kv_pack_kernel
    const int q32 = static_cast<int>(e / img), w = static_cast<int>(e % img);
    const int core = w >> 5, ln = w & 31;
    const int j = (core >> 3) * 8 + (ln >> 2);
    const int i = q32 * 32 + (core & 7) * 4 + (ln & 3);
    double v = 0.0;
    if (i < nloc && j < m) {
      const size_t o = static_cast<size_t>(i) * m + j;
      double mo = __dmul_rn(M[o], rho);
      const int q = pos[i];
      if (q >= 0) {
        const double g = grad[static_cast<size_t>(q) * m + j];
        mo = __dsub_rn(mo, __dmul_rn(step, g));
        R[o] = -g;
      }
      M[o] = mo;
      v = __dadd_rn(V[o], mo);
      V[o] = v;
      if (!isfinite(v)) bad = 1;
    }
    uint32_t hb, lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(static_cast<float>(v)));
    const float h = __uint_as_float(hb);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(static_cast<float>(v - static_cast<double>(h))));
    float* base = vpk + static_cast<size_t>(q32) * 2 * img;
    base[w] = h;
    base[img + w] = __uint_as_float(lb);
  }
  if (bad) atomicOr(nonfinite, 1);
}
void sgd_update_pack_launch(double* M, double* V, double* R, float* vpk, int npad, const int* pos,
                            const double* grad, double rho, double step, int nloc, int m, int* nonfinite,
                            const int* skip, cudaStream_t s) {
  const int rows_pad = (nloc + 31) / 32 * 32;
  sgd_update_pack_kernel<<<blocks_for(static_cast<long long>(rows_pad) * npad, 256), 256, 0, s>>>(
      M, V, R, vpk, npad, rows_pad, pos, grad, rho, step, nloc, m, nonfinite, skip);
  check_launch("sgd_update_pack");
}

// AP: a block inverse whose factorisation failed stops the solve before its
// first update (the solutions are never touched), solvers.cpp:104-113 throws
// from factor_for; the host raises after the solve from the info copy.
__global__ void ap_info_gate_kernel(const int* info, int nblocks, CgCtl* ctl) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nblocks; k += blockDim.x)
    if (info[k] != 0) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && bad) {
    ctl->aborted = 1;
    ctl->stop = 1;
  }
}
void ap_info_gate_launch(const int* info, int nblocks, CgCtl* ctl, cudaStream_t s) {
  ap_info_gate_kernel<<<1, 256, 0, s>>>(info, nblocks, ctl);
  check_launch("ap_info_gate");
}

// Single-rank divergence test right after the update (solvers.cpp:172-176:
// the reference tests the iterate it just formed and reports t + 1 updates).
// pad = stop before this iteration's check, i.e. the update ran.
__global__ void sgd_diverge_now_kernel(const int* nonfinite, CgCtl* ctl) {
  if (ctl->pad == 0 && *nonfinite && !ctl->aborted) {
    ctl->aborted = 1;
    ctl->stop = 1;
  }
}
void sgd_diverge_now_launch(const int* nonfinite, CgCtl* ctl, cudaStream_t s) {
  sgd_diverge_now_kernel<<<1, 1, 0, s>>>(nonfinite, ctl);
  check_launch("sgd_diverge_now");
}

__global__ void sgd_unscatter_kernel(const int* idx, int b, int row0, int nloc, int* pos, const int* skip) {
  SKIP_IF(skip);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < b; q += gridDim.x * blockDim.x) {
    const int li = idx[q] - row0;
    if (li >= 0 && li < nloc) pos[li] = -1;
  }
}
void sgd_unscatter_launch(const int* idx, int b, int row0, int nloc, int* pos, const int* skip, cudaStream_t s) {
  sgd_unscatter_kernel<<<blocks_for(b, 256), 256, 0, s>>>(idx, b, row0, nloc, pos, skip);
  check_launch("sgd_unscatter");
}

// sin and cos of an FP64 angle to ~1 ulp for |t| < 2^30: Cody-Waite
// reduction by pi/2 in three parts (fma, exact products), then the Taylor
// series on |r| <= pi/4 through r^17 / r^18 (truncation < 1e-19). CUDA's
// sincos(double) takes a slow table path (local memory) for the heavy-tailed
// Matern frequencies; this one is branch-free (~30 DFMA).
__device__ __forceinline__ void sincos_rr(double t, double* sn, double* cs) {
  const double q = rint(t * 0.63661977236758134308);                    // 2 / pi
  double r = fma(-q, 1.5707963267948965579989817342720925807952880859375, t);  // pi/2 in 3 parts
  r = fma(-q, 6.123233995736766035868820147291818e-17, r);
  r = fma(-q, -1.4973849048591698329435778716705e-33, r);
  const double z = r * r;
  // sin r = r (1 - z/3! + z^2/5! - ... - z^8/17!)
  double ps = 2.8114572543455207632e-15;      //  1/17!
  ps = fma(ps, z, -7.6471637318198164759e-13);  // -1/15!
  ps = fma(ps, z, 1.6059043836821614599e-10);   //  1/13!
  ps = fma(ps, z, -2.5052108385441718775e-08);  // -1/11!
  ps = fma(ps, z, 2.7557319223985890653e-06);   //  1/9!
  ps = fma(ps, z, -1.9841269841269841270e-04);  // -1/7!
  ps = fma(ps, z, 8.3333333333333333333e-03);   //  1/5!
  ps = fma(ps, z, -1.6666666666666666667e-01);  // -1/3!
  const double sr = fma(ps * z, r, r);
  // cos r = 1 - z/2! + z^2/4! - ... + z^9/18!
  double pc = -1.5619206968586225796e-16;      // -1/18!
  pc = fma(pc, z, 4.7794773323873852974e-14);   //  1/16!
  pc = fma(pc, z, -1.1470745597729724714e-11);  // -1/14!
  pc = fma(pc, z, 2.0876756987868098979e-09);   //  1/12!
  pc = fma(pc, z, -2.7557319223985890653e-07);  // -1/10!
  pc = fma(pc, z, 2.4801587301587301587e-05);   //  1/8!
  pc = fma(pc, z, -1.3888888888888888889e-03);  // -1/6!
  pc = fma(pc, z, 4.1666666666666666667e-02);   //  1/4!
  pc = fma(pc, z, -0.5);
  const double cr = fma(pc, z, 1.0);
  const int n = static_cast<int>(static_cast<long long>(q) & 3);
  const double s0 = (n & 1) ? cr : sr, c0 = (n & 1) ? sr : cr;
  *sn = (n & 2) ? -s0 : s0;
  *cs = ((n + 1) & 2) ? -c0 : c0;
}

// F[i][2p] = amp cos(theta_ip), F[i][2p+1] = amp sin(theta_ip),
// theta_ip = x_i . (Omega_p / l) in FP64 (rff.cpp:36-54). Block = 128
// consecutive features p (one per thread, Omega_p in registers) x 64 rows
// (x tile in shared memory, read as warp broadcasts); lanes write consecutive
// (cos, sin) pairs of a row. freq is [d][pairs] (already divided by the
// lengthscales).
constexpr int RFF_TP = 128, RFF_TR = 64;
__global__ void __launch_bounds__(RFF_TP) rff_features_kernel(const double* x64, int n, int d, const double* freq,
                                                              int pairs, double amplitude, double* F) {
  __shared__ double xt[RFF_TR][32];
  const int p = blockIdx.x * RFF_TP + threadIdx.x;
  const int i0 = blockIdx.y * RFF_TR;
  const int rows = min(RFF_TR, n - i0);
  for (int e = threadIdx.x; e < rows * d; e += RFF_TP) xt[e / d][e % d] = x64[static_cast<size_t>(i0) * d + e];
  double w[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) w[k] = (k < d && p < pairs) ? freq[static_cast<size_t>(k) * pairs + p] : 0.0;
  __syncthreads();
  if (p >= pairs) return;
  double2* out = reinterpret_cast<double2*>(F);
  for (int r = 0; r < rows; ++r) {
    double a0 = 0.0, a1 = 0.0;  // two chains, summed in a fixed order
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      if (k < d) a0 = fma(xt[r][k], w[k], a0);
      if (k + 1 < d) a1 = fma(xt[r][k + 1], w[k + 1], a1);
    }
    const double ang = a0 + a1;
    double sn, c;
    if (fabs(ang) < 1073741824.0) {
      sincos_rr(ang, &sn, &c);
    } else {
      sincos(ang, &sn, &c);  // huge angles: the library's full-precision reduction
    }
    out[static_cast<size_t>(i0 + r) * pairs + p] = make_double2(amplitude * c, amplitude * sn);
  }
}
// derivative_apply (kernel.cpp:200-236): out[r][j] = sum_c dK_k[r][c] v[c][j]
// in FP64 for parameter k < d (lengthscale: 3 s2 (1/l_k) e^{-sqrt3 r} dxs_k^2)
// or k == d (signal: (2/s) k(r)); the noise case (2 sigma V) never reaches the
// device. CTA = 32 rows; per 32-column chunk the entries go to shared memory
// and each thread accumulates 4 rows x its columns j = lane + 32 u (ascending c).
__global__ void __launch_bounds__(256) deriv_apply_kernel(const double* __restrict__ xs, int n, int d, int k,
                                                          double sv, double coef, const double* __restrict__ v,
                                                          int m, double* __restrict__ out) {
  __shared__ double xr[32][33];
  __shared__ double xc[32][33];
  __shared__ double kt[32][33];
  __shared__ double vt[32][80];
  const int tid = threadIdx.x, lane = tid & 31, rg = tid >> 5;
  const int r0 = blockIdx.x * 32;
  for (int e = tid; e < 32 * d; e += 256) {
    const int r = e / d, q = e % d;
    xr[r][q] = r0 + r < n ? xs[static_cast<size_t>(r0 + r) * d + q] : 0.0;
  }
  double acc[4][3] = {};
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int cn = min(32, n - c0);
    __syncthreads();
    for (int e = tid; e < 32 * d; e += 256) {
      const int c = e / d, q = e % d;
      xc[c][q] = c < cn ? xs[static_cast<size_t>(c0 + c) * d + q] : 0.0;
    }
    for (int e = tid; e < 32 * m; e += 256) {
      const int c = e / m, j = e % m;
      vt[c][j] = c < cn ? v[static_cast<size_t>(c0 + c) * m + j] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int c = e >> 5, r = e & 31;
      double r2 = 0.0;
      for (int q = 0; q < d; ++q) {
        const double t = xc[c][q] - xr[r][q];
        r2 += t * t;
      }
      const double rr = sqrt(r2);
      double val;
      if (k == d) {
        val = coef * (sv * (1.0 + kSqrt3 * rr) * exp(-kSqrt3 * rr));
      } else {
        const double dk = xc[c][k] - xr[r][k];
        val = coef * exp(-kSqrt3 * rr) * (dk * dk);
      }
      kt[c][r] = c < cn ? val : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < cn; ++c)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double kv = kt[c][rg * 4 + a];
#pragma unroll
        for (int u = 0; u < 3; ++u)
          if (lane + 32 * u < m) acc[a][u] = fma(kv, vt[c][lane + 32 * u], acc[a][u]);
      }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = r0 + rg * 4 + a;
    if (r >= n) continue;
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (lane + 32 * u < m) out[static_cast<size_t>(r) * m + lane + 32 * u] = acc[a][u];
  }
}
void deriv_apply_launch(const double* xs64, int n, int d, int k, double sv, double coef, const double* v, int m,
                        double* out, cudaStream_t s) {
  if (d > 32 || m > 80) throw std::invalid_argument("gpk: derivative_apply supports d <= 32 and m <= 80");
  deriv_apply_kernel<<<(n + 31) / 32, 256, 0, s>>>(xs64, n, d, k, sv, coef, v, m, out);
  check_launch("deriv_apply");
}

// FP64 operator product with on-the-fly kernel evaluation (the high-accuracy
// operator for n <= dense_cache_cap, where the reference caches H in FP64):
// part[split][r][j] = sum over the split's columns c of k(x_{r0+r}, x_c) v[c][j]
// (kernel only; kv_reduce adds sigma^2 v on the diagonal). CTA = 32 rows x one
// column split; per 32-column chunk the FP64 entries go to shared memory and
// each thread accumulates 4 rows x its columns j = lane + 32 u (ascending c).
__global__ void __launch_bounds__(256) kv64_kernel(const double* __restrict__ xs, int n, int d, double sv, int r0,
                                                   int R, const double* __restrict__ v, int m, int cols_per_split,
                                                   double* __restrict__ part, const int* skip) {
  if (skip && *skip) return;
  __shared__ double xr[32][33];
  __shared__ double xc[32][33];
  __shared__ double kt[32][33];
  __shared__ double vt[32][80];
  const int tid = threadIdx.x, lane = tid & 31, rg = tid >> 5;
  const int rb = blockIdx.x * 32;
  const int cb = blockIdx.y * cols_per_split, ce = min(n, cb + cols_per_split);
  for (int e = tid; e < 32 * d; e += 256) {
    const int r = e / d, q = e % d;
    xr[r][q] = rb + r < R ? xs[static_cast<size_t>(r0 + rb + r) * d + q] : 0.0;
  }
  double acc[4][3] = {};
  for (int c0 = cb; c0 < ce; c0 += 32) {
    const int cn = min(32, ce - c0);
    __syncthreads();
    for (int e = tid; e < 32 * d; e += 256) {
      const int c = e / d, q = e % d;
      xc[c][q] = c < cn ? xs[static_cast<size_t>(c0 + c) * d + q] : 0.0;
    }
    for (int e = tid; e < 32 * m; e += 256) {
      const int c = e / m, j = e % m;
      vt[c][j] = c < cn ? v[static_cast<size_t>(c0 + c) * m + j] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int c = e >> 5, r = e & 31;
      double r2 = 0.0;
      for (int q = 0; q < d; ++q) {
        const double t = xc[c][q] - xr[r][q];
        r2 += t * t;
      }
      const double rr = sqrt(r2);
      kt[c][r] = c < cn ? sv * (1.0 + kSqrt3 * rr) * exp(-kSqrt3 * rr) : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < cn; ++c)
#pragma unroll
      for (int a4 = 0; a4 < 4; ++a4) {
        const double kv = kt[c][rg * 4 + a4];
#pragma unroll
        for (int u = 0; u < 3; ++u)
          if (lane + 32 * u < m) acc[a4][u] = fma(kv, vt[c][lane + 32 * u], acc[a4][u]);
      }
  }
#pragma unroll
  for (int a4 = 0; a4 < 4; ++a4) {
    const int r = rb + rg * 4 + a4;
    if (r >= R) continue;
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (lane + 32 * u < m) part[(static_cast<size_t>(blockIdx.y) * R + r) * m + lane + 32 * u] = acc[a4][u];
  }
}
// kv64 v2 (m <= 32): CTA = 128 rows x one column split, 256 threads; thread
// (row, half) keeps its row's coordinates and its FP64 accumulators in
// registers and, per 32-column chunk, evaluates the 16 entries of its half
// and contracts each at once into its m accumulators (x_c and V rows are
// shared-memory broadcasts; no entry ever leaves registers). The two halves
// are combined in a fixed order at the end. DP-pipe bound: ~45 FP64 ops per
// entry for the Matern profile + m FMAs.
template <int DM, int MJ>
__global__ void __launch_bounds__(256, 2) kv64v2_kernel(const double* __restrict__ xs, int n, int d, double sv,
                                                         int r0, int R, const double* __restrict__ v, int m,
                                                         int cols_per_split, double* __restrict__ part,
                                                         const int* skip) {
  if (skip && *skip) return;
  constexpr int HJ = MJ / 2;  // the halves are combined in two passes of HJ columns
  constexpr int LOOP = 2 * 32 * (DM + MJ), COMB = 128 * (HJ + 1);
  __shared__ __align__(16) double sm[LOOP > COMB ? LOOP : COMB];
  auto xc = reinterpret_cast<double(*)[32][DM]>(sm);
  auto vt = reinterpret_cast<double(*)[32][MJ]>(sm + 2 * 32 * DM);
  auto comb = reinterpret_cast<double(*)[HJ + 1]>(sm);
  const int tid = threadIdx.x, row = tid & 127, h = tid >> 7;
  const int er = blockIdx.x * 128 + row;
  const int cb = blockIdx.y * cols_per_split, ce = min(n, cb + cols_per_split);
  double xr[DM];
#pragma unroll
  for (int q = 0; q < DM; ++q) xr[q] = (er < R && q < d) ? xs[static_cast<size_t>(r0 + er) * d + q] : 0.0;
  double acc[MJ];
#pragma unroll
  for (int j = 0; j < MJ; ++j) acc[j] = 0.0;
  constexpr int XE = 32 * DM, VE = 32 * MJ;
  constexpr int PER = (XE + VE + 255) / 256;
  auto fetch = [&](int c0, double* pre) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + 256 * u;
      double val = 0.0;
      if (e < XE) {
        const int c = e / DM, q = e % DM;
        if (c0 + c < ce && q < d) val = xs[static_cast<size_t>(c0 + c) * d + q];
      } else if (e < XE + VE) {
        const int c = (e - XE) / MJ, j = (e - XE) % MJ;
        if (c0 + c < ce && j < m) val = v[static_cast<size_t>(c0 + c) * m + j];
      }
      pre[u] = val;
    }
  };
  auto stash = [&](int buf, const double* pre) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + 256 * u;
      if (e < XE)
        (&xc[buf][0][0])[e] = pre[u];
      else if (e < XE + VE)
        (&vt[buf][0][0])[e - XE] = pre[u];
    }
  };
  double pre[PER];
  int buf = 0;
  if (cb < ce) {
    fetch(cb, pre);
    stash(0, pre);
  }
  __syncthreads();
  for (int c0 = cb; c0 < ce; c0 += 32) {
    const bool more = c0 + 32 < ce;
    if (more) fetch(c0 + 32, pre);  // in flight during this chunk
#pragma unroll 2
    for (int cc = 0; cc < 16; ++cc) {
      const int c = h * 16 + cc;
      double r2 = 0.0;
#pragma unroll
      for (int q = 0; q < DM; q += 2) {
        const double2 x2 = *reinterpret_cast<const double2*>(&xc[buf][c][q]);
        const double t0 = x2.x - xr[q], t1 = x2.y - xr[q + 1];
        r2 = fma(t0, t0, r2);
        r2 = fma(t1, t1, r2);
      }
      const double rr = sqrt(r2);
      // zero V rows beyond the split make the padded columns contribute 0
      const double kv = sv * (1.0 + kSqrt3 * rr) * exp(-kSqrt3 * rr);
#pragma unroll
      for (int j = 0; j < MJ; j += 2) {
        const double2 w = *reinterpret_cast<const double2*>(&vt[buf][c][j]);
        acc[j] = fma(kv, w.x, acc[j]);
        acc[j + 1] = fma(kv, w.y, acc[j + 1]);
      }
    }
    if (more) stash(buf ^ 1, pre);
    __syncthreads();
    buf ^= 1;
  }
  double* out = part + (static_cast<size_t>(blockIdx.y) * R + er) * m;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    if (h == 1) {
#pragma unroll
      for (int j = 0; j < HJ; ++j) comb[row][j] = acc[p * HJ + j];
    }
    __syncthreads();
    if (h == 0 && er < R) {
#pragma unroll
      for (int j = 0; j < HJ; ++j)
        if (p * HJ + j < m) out[p * HJ + j] = acc[p * HJ + j] + comb[row][j];
    }
    __syncthreads();
  }
}

int kv64_splits(int R, int n, int sms) {
  const int rb = (R + 31) / 32;
  const int want = std::max(1, (4 * sms + rb - 1) / rb);  // ~4 CTAs per SM
  return std::min(want, std::max(1, (n + 31) / 32));
}
int kv64v2_splits(int R, int n, int sms) {
  const int rb = (R + 127) / 128;
  const int want = std::max(1, (2 * sms + rb - 1) / rb);  // two resident CTAs per SM
  return std::min(want, std::max(1, (n + 31) / 32));
}
int kv64_splits_for(int R, int n, int m, int d, int sms) {
  return (m <= 32 && d <= 16) ? kv64v2_splits(R, n, sms) : kv64_splits(R, n, sms);
}

template <int DM, int MJ>
void kv64v2_launch_t(const double* xs64, int n, int d, double sv, int r0, int R, const double* v, int m,
                     int splits, double* part, const int* skip, cudaStream_t s) {
  int cps = (n + splits - 1) / splits;
  cps = (cps + 31) / 32 * 32;
  kv64v2_kernel<DM, MJ><<<dim3((R + 127) / 128, splits), 256, 0, s>>>(xs64, n, d, sv, r0, R, v, m, cps, part, skip);
  check_launch("kv64v2_kernel");
}
template <int DM>
void kv64v2_launch_d(const double* xs64, int n, int d, double sv, int r0, int R, const double* v, int m,
                     int splits, double* part, const int* skip, cudaStream_t s) {
  if (m <= 8) return kv64v2_launch_t<DM, 8>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
  if (m <= 18) return kv64v2_launch_t<DM, 18>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
  return kv64v2_launch_t<DM, 32>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
}

void kv64_launch(const double* xs64, int n, int d, double sv, int r0, int R, const double* v, int m, int splits,
                 double* part, const int* skip, cudaStream_t s) {
  if (d > 32 || m > 80) throw std::invalid_argument("gpk: the FP64 operator supports d <= 32 and m <= 80");
  if (m <= 32 && d <= 16) {  // splits from kv64_splits_for
    if (d <= 4) return kv64v2_launch_d<4>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
    if (d <= 8) return kv64v2_launch_d<8>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
    return kv64v2_launch_d<16>(xs64, n, d, sv, r0, R, v, m, splits, part, skip, s);
  }
  int cps = (n + splits - 1) / splits;
  cps = (cps + 31) / 32 * 32;
  kv64_kernel<<<dim3((R + 31) / 32, splits), 256, 0, s>>>(xs64, n, d, sv, r0, R, v, m, cps, part, skip);
  check_launch("kv64_kernel");
}

// K5, streaming (rff.cpp:36-54, 64-73): prior[i][j] = sum_q phi_q(x_i) W[q][j]
// without materialising Phi. CTA = 64 rows x 64 samples; per chunk of 16
// pairs the CTA forms phi (FP64 angles, sincos, interleaved cos/sin as
// rff.cpp:48-52) for its rows in shared memory next to the chunk of W, and
// each thread accumulates a 4 x 4 block of the product over features in
// ascending order (FP64 FMA).
constexpr int RP_ROWS = 64, RP_COLS = 64, RP_PAIRS = 16, RP_F = 2 * RP_PAIRS;
__global__ void __launch_bounds__(256) rff_prior_kernel(const double* __restrict__ x64, int n, int d,
                                                        const double* __restrict__ freq, int pairs, double amplitude,
                                                        const double* __restrict__ W, int ldw, int s_count,
                                                        double* __restrict__ prior) {
  extern __shared__ double rp_sm[];
  double* xt = rp_sm;                      // [64][d]
  double* ph = xt + RP_ROWS * d;           // [32 features][64 rows]
  double* wt = ph + RP_F * RP_ROWS;        // [32 features][64 samples]
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * RP_ROWS, j0 = blockIdx.y * RP_COLS;
  const int rows = min(RP_ROWS, n - i0);
  for (int e = tid; e < RP_ROWS * d; e += 256) xt[e] = e < rows * d ? x64[static_cast<size_t>(i0) * d + e] : 0.0;
  const int tr = tid >> 4, tc = tid & 15;  // rows 4 tr .. 4 tr + 3, samples 4 tc .. 4 tc + 3
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int p0 = 0; p0 < pairs; p0 += RP_PAIRS) {
    const int pn = min(RP_PAIRS, pairs - p0);
    __syncthreads();
    for (int e = tid; e < RP_ROWS * RP_PAIRS; e += 256) {
      const int r = e & (RP_ROWS - 1), pp = e / RP_ROWS;
      double cv = 0.0, sv = 0.0;
      if (pp < pn) {
        double a0 = 0.0, a1 = 0.0;  // two chains summed in a fixed order, as rff_features_kernel
        for (int k = 0; k < d; k += 2) {
          a0 = fma(xt[r * d + k], freq[static_cast<size_t>(k) * pairs + p0 + pp], a0);
          if (k + 1 < d) a1 = fma(xt[r * d + k + 1], freq[static_cast<size_t>(k + 1) * pairs + p0 + pp], a1);
        }
        const double ang = a0 + a1;
        if (fabs(ang) < 1073741824.0)
          sincos_rr(ang, &sv, &cv);
        else
          sincos(ang, &sv, &cv);
        cv *= amplitude;
        sv *= amplitude;
      }
      ph[(2 * pp) * RP_ROWS + r] = cv;
      ph[(2 * pp + 1) * RP_ROWS + r] = sv;
    }
    for (int e = tid; e < RP_F * RP_COLS; e += 256) {
      const int q = e & (RP_F - 1), c = e / RP_F;
      wt[q * RP_COLS + c] =
          (q < 2 * pn && j0 + c < s_count) ? W[static_cast<size_t>(j0 + c) * ldw + 2 * p0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < RP_F; ++q) {
      const double2 pa = *reinterpret_cast<const double2*>(ph + q * RP_ROWS + 4 * tr);
      const double2 pb = *reinterpret_cast<const double2*>(ph + q * RP_ROWS + 4 * tr + 2);
      const double2 wa = *reinterpret_cast<const double2*>(wt + q * RP_COLS + 4 * tc);
      const double2 wb = *reinterpret_cast<const double2*>(wt + q * RP_COLS + 4 * tc + 2);
      const double pv[4] = {pa.x, pa.y, pb.x, pb.y}, wv[4] = {wa.x, wa.y, wb.x, wb.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(pv[a], wv[b], acc[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = 4 * tr + a;
    if (r >= rows) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + 4 * tc + b;
      if (j < s_count) prior[static_cast<size_t>(i0 + r) * s_count + j] = acc[a][b];
    }
  }
}
void rff_prior_launch(const double* x64, int n, int d, const double* freq, int pairs, double amplitude,
                      const double* W, int ldw, int s_count, double* prior, cudaStream_t s) {
  if (n <= 0) return;
  if (d > 32) throw std::invalid_argument("gpk: RFF prior supports d <= 32");
  const size_t smem = sizeof(double) * (RP_ROWS * d + RP_F * RP_ROWS + RP_F * RP_COLS);
  static size_t configured = 0;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(rff_prior_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  const dim3 grid((n + RP_ROWS - 1) / RP_ROWS, (s_count + RP_COLS - 1) / RP_COLS);
  rff_prior_kernel<<<grid, 256, smem, s>>>(x64, n, d, freq, pairs, amplitude, W, ldw, s_count, prior);
  check_launch("rff_prior");
}

void rff_features_launch(const double* x64, int n, int d, const double* freq, int pairs, double amplitude, double* F,
                         cudaStream_t s) {
  if (n <= 0) return;
  const dim3 grid((pairs + RFF_TP - 1) / RFF_TP, (n + RFF_TR - 1) / RFF_TR);
  rff_features_kernel<<<grid, RFF_TP, 0, s>>>(x64, n, d, freq, pairs, amplitude, F);
  check_launch("rff_features");
}


// Box-Muller pairs (rng.cpp:64-77), element e of the column-major n x s fill
// (rng.cpp:86-90) -> out[i][j] row-major, i = e % n, j = e / n.
__global__ void gaussian_fill_kernel(uint64_t seed, uint64_t stream, uint64_t substream, long long count, int n, int s,
                                     double* out) {
  const long long pairs = (count + 1) / 2;
  for (long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; p < pairs;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    const U64x4 blk = philox4x64(static_cast<uint64_t>(p) >> 1, substream, 0, 0, seed, stream);
    const int o = static_cast<int>((p & 1) * 2);
    const double u1 = static_cast<double>((blk.v[o] >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(blk.v[o + 1] >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 6.283185307179586 * u2;  // 2.0 * pi, as rng.cpp:73
    double sn, cs;
    sincos(angle, &sn, &cs);
    const long long e0 = 2 * p, e1 = 2 * p + 1;
    out[(e0 % n) * s + e0 / n] = radius * cs;
    if (e1 < count) out[(e1 % n) * s + e1 / n] = radius * sn;
  }
}
void gaussian_fill_launch(uint64_t seed, uint64_t stream, uint64_t substream, int64_t count, int n, int s,
                          double* out_rowmajor, cudaStream_t st) {
  gaussian_fill_kernel<<<blocks_for((count + 1) / 2, 256), 256, 0, st>>>(seed, stream, substream, count, n, s,
                                                                        out_rowmajor);
  check_launch("gaussian_fill");
}

// Element (i, j) of the column-major n x s Gaussian fill for local rows
// i in [row0, row0 + nloc): draw e = j*n + i is the cos (e even) or sin (e odd)
// half of Box-Muller pair e/2, counter-indexed so any row block can be drawn.
__global__ void gaussian_fill_rows_kernel(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s, int row0,
                                          int nloc, double* out) {
  const long long total = static_cast<long long>(nloc) * s;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int il = static_cast<int>(q / s), j = static_cast<int>(q % s);
    const long long e = static_cast<long long>(j) * n + row0 + il;
    const long long p = e >> 1;
    const U64x4 blk = philox4x64(static_cast<uint64_t>(p) >> 1, substream, 0, 0, seed, stream);
    const int o = static_cast<int>((p & 1) * 2);
    const double u1 = static_cast<double>((blk.v[o] >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(blk.v[o + 1] >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 6.283185307179586 * u2;
    double sn, cs;
    sincos(angle, &sn, &cs);
    out[q] = (e & 1) ? radius * sn : radius * cs;
  }
}
void gaussian_fill_rows_launch(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s, int row0, int nloc,
                               double* out_rowmajor, cudaStream_t st) {
  gaussian_fill_rows_kernel<<<blocks_for(static_cast<long long>(nloc) * s, 256), 256, 0, st>>>(
      seed, stream, substream, n, s, row0, nloc, out_rowmajor);
  check_launch("gaussian_fill_rows");
}

__global__ void rademacher_fill_rows_kernel(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s,
                                            int row0, int nloc, double* out) {
  const long long total = static_cast<long long>(nloc) * s;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int il = static_cast<int>(q / s), j = static_cast<int>(q % s);
    const uint64_t e = static_cast<uint64_t>(j) * n + row0 + il;
    out[q] = (stream_u64(seed, stream, substream, e) & 1u) ? 1.0 : -1.0;
  }
}
void rademacher_fill_rows_launch(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s, int row0, int nloc,
                                 double* out_rowmajor, cudaStream_t st) {
  rademacher_fill_rows_kernel<<<blocks_for(static_cast<long long>(nloc) * s, 256), 256, 0, st>>>(
      seed, stream, substream, n, s, row0, nloc, out_rowmajor);
  check_launch("rademacher_fill_rows");
}

// out[i][col0 + j] = prior[i][j] + sigma * noise[i][j] (rff.cpp:77)
__global__ void xi_assemble_kernel(const double* prior, const double* noise, int n, int s, double sigma, double* out,
                                   int ldo, int col0, double* xi_copy) {
  const long long total = static_cast<long long>(n) * s;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / s), j = static_cast<int>(e % s);
    const double v = __dadd_rn(prior[e], __dmul_rn(sigma, noise[e]));
    if (out) out[static_cast<size_t>(i) * ldo + col0 + j] = v;
    if (xi_copy) xi_copy[e] = v;
  }
}
void xi_assemble_launch(const double* prior, const double* noise, int n, int s, double sigma, double* out, int ldo,
                        int col0, double* xi_copy, cudaStream_t st) {
  xi_assemble_kernel<<<blocks_for(static_cast<long long>(n) * s, 256), 256, 0, st>>>(prior, noise, n, s, sigma, out,
                                                                                   ldo, col0, xi_copy);
  check_launch("xi_assemble");
}

}  // namespace gpk
