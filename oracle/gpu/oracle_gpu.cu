// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Oracle-at-scale (hard part 5): naive FP64 CUDA
// restatements of the reference's O(n^2) passes, plugged into the CPU
// restatement (oracle/gpiter_oracle.cpp) through its OracleBackend hook, so the
// unchanged oracle optimise / solve_cg / solve_sgd / estimator code runs the
// BASELINE configurations C4 (SGD, n = 393216) and C5 (CG, n = 1835008) whose
// CPU cost is 1e13 .. 1e15 FP64 flops per epoch. Linked only into
// oracle/build/liboracle_gpu.so; the product library (libgpk.so) never sees it.
//
// What is restated (and from where):
//   apply / apply_rows     kernel.cpp:133-168 (H = K + sigma^2 I, Matern-3/2 on
//                          scaled inputs, kernel.cpp:35-39, 111-131)
//   quad forms             kernel.cpp:238-272 (noise term stays on the host)
//   RFF prior values       rff.cpp:36-54, 64-73 (Phi W, interleaved cos/sin)
//   solve_sgd              solvers.cpp:147-184 (state n x m on the device; the
//                          minibatches come from the host RandomStream, bit-exact)
// Everything is FP64 (exp/sqrt/sincos in double). Sums run in a fixed order
// (ascending column within a 32-column chunk, chunks ascending within a
// split, splits ascending), which is not the CPU oracle's single ascending
// loop: results agree to rounding (~1e-15 relative), not bitwise.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../gpiter_oracle.hpp"

namespace oracle {
namespace gpu {

#define OG_CUDA(x)                                                                                   \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("oracle_gpu: ") + #x + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr double kSqrt3 = 1.7320508075688772935;
constexpr int TR = 32;    // rows per block
constexpr int TC = 32;    // columns per chunk
constexpr int MAXD = 32;  // input dimension bound
constexpr int MAXM = 80;  // RHS columns bound (3 slots of 32 lanes)

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t count) { alloc(count); }
  void alloc(size_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    OG_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

__device__ __forceinline__ double matern(double r2, double sv) {
  const double r = sqrt(r2);
  return sv * (1.0 + kSqrt3 * r) * exp(-kSqrt3 * r);
}

// part[split][R][m] = sum over this split's columns c of H[row(r), c] v[c][j]
// (v row-major [n][m]); rows = row list or null (rows r0 .. r0 + R).
__global__ void __launch_bounds__(256) apply_kernel(const double* __restrict__ xs, int n, int d, double sv, double nv,
                                                    const int* __restrict__ rows, int R, const double* __restrict__ v,
                                                    int m, int cols_per_split, double* __restrict__ part) {
  __shared__ double xr[TR][MAXD];
  __shared__ double xc[TC][MAXD + 1];
  __shared__ double vt[TC][MAXM];
  __shared__ double kt[TC][TR + 1];
  __shared__ int grow[TR];
  const int tid = threadIdx.x, lane = tid & 31, rg = tid >> 5;  // 8 row groups of 4 rows
  const int r0 = blockIdx.x * TR;
  const int cb = blockIdx.y * cols_per_split, ce = min(n, cb + cols_per_split);
  if (tid < TR) {
    const int r = r0 + tid;
    grow[tid] = r < R ? (rows ? rows[r] : r) : -1;
  }
  __syncthreads();
  for (int e = tid; e < TR * d; e += blockDim.x) {
    const int r = e / d, k = e % d;
    xr[r][k] = grow[r] >= 0 ? xs[static_cast<size_t>(grow[r]) * d + k] : 0.0;
  }
  double acc[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[a][q] = 0.0;
  for (int c0 = cb; c0 < ce; c0 += TC) {
    const int cn = min(TC, ce - c0);
    __syncthreads();
    for (int e = tid; e < TC * d; e += blockDim.x) {
      const int c = e / d, k = e % d;
      xc[c][k] = c < cn ? xs[static_cast<size_t>(c0 + c) * d + k] : 0.0;
    }
    for (int e = tid; e < TC * m; e += blockDim.x) {
      const int c = e / m, j = e % m;
      vt[c][j] = c < cn ? v[static_cast<size_t>(c0 + c) * m + j] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < TC * TR; e += blockDim.x) {
      const int c = e / TR, r = e % TR;
      double r2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double t = xc[c][k] - xr[r][k];
        r2 += t * t;
      }
      double kv = c < cn ? matern(r2, sv) : 0.0;
      if (c < cn && grow[r] == c0 + c) kv += nv;
      kt[c][r] = kv;
    }
    __syncthreads();
    for (int c = 0; c < cn; ++c) {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double kv = kt[c][rg * 4 + a];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int j = lane + 32 * q;
          if (j < m) acc[a][q] += kv * vt[c][j];
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = r0 + rg * 4 + a;
    if (r >= R) continue;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = lane + 32 * q;
      if (j < m) part[(static_cast<size_t>(blockIdx.y) * R + r) * m + j] = acc[a][q];
    }
  }
}

__global__ void sum_splits_kernel(const double* part, int splits, long long count, double* out) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += part[static_cast<size_t>(k) * count + e];
    out[e] = s;
  }
}

struct Ctx {
  Dev<double> xs, v, part, out;
  Dev<int> rows;
};
Ctx& ctx() {
  static Ctx c;
  return c;
}

int grid_blocks(long long count) { return static_cast<int>(std::min<long long>((count + 255) / 256, 148 * 8)); }

// out (device, row-major [R][m]) = H[rows, :] v for v device row-major.
void apply_dev(const double* xs, int n, int d, double sv, double nv, const int* rows_dev, int R, const double* v,
               int m, double* out) {
  if (d > MAXD || m > MAXM) throw std::invalid_argument("oracle_gpu: d <= 32 and m <= 80");
  const int rb = (R + TR - 1) / TR;
  int splits = std::max(1, std::min(512, 1184 / rb));
  int cps = (n + splits - 1) / splits;
  cps = (cps + TC - 1) / TC * TC;
  splits = (n + cps - 1) / cps;
  Ctx& c = ctx();
  c.part.alloc(static_cast<size_t>(splits) * R * m);
  apply_kernel<<<dim3(rb, splits), 256>>>(xs, n, d, sv, nv, rows_dev, R, v, m, cps, c.part.p);
  OG_CUDA(cudaGetLastError());
  const long long count = static_cast<long long>(R) * m;
  sum_splits_kernel<<<grid_blocks(count), 256>>>(c.part.p, splits, count, out);
  OG_CUDA(cudaGetLastError());
}

void upload_rowmajor(const Mat& a, Dev<double>& d) {  // col-major host -> row-major device
  std::vector<double> h(a.size());
  for (int i = 0; i < a.rows; ++i)
    for (int j = 0; j < a.cols; ++j) h[static_cast<size_t>(i) * a.cols + j] = a(i, j);
  d.alloc(h.size());
  OG_CUDA(cudaMemcpy(d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
}
Mat download_rowmajor(const double* p, int rows, int cols) {
  std::vector<double> h(static_cast<size_t>(rows) * cols);
  OG_CUDA(cudaMemcpy(h.data(), p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
  Mat out(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out(i, j) = h[static_cast<size_t>(i) * cols + j];
  return out;
}
void upload_xs(const KernelOperator& op, Dev<double>& d) {
  const size_t cnt = static_cast<size_t>(op.size()) * op.dim();
  d.alloc(cnt);
  OG_CUDA(cudaMemcpy(d.p, op.scaled_inputs(), sizeof(double) * cnt, cudaMemcpyHostToDevice));
}

bool apply_hook(const KernelOperator& op, const int* rows, int count, const Mat& v, Mat& out) {
  Ctx& c = ctx();
  const int n = op.size(), d = op.dim(), m = v.cols;
  upload_xs(op, c.xs);
  upload_rowmajor(v, c.v);
  if (rows) {
    c.rows.alloc(count);
    OG_CUDA(cudaMemcpy(c.rows.p, rows, sizeof(int) * count, cudaMemcpyHostToDevice));
  }
  c.out.alloc(static_cast<size_t>(count) * m);
  apply_dev(c.xs.p, n, d, op.signal_variance(), op.noise_variance(), rows ? c.rows.p : nullptr, count, c.v.p, m,
            c.out.p);
  out = download_rowmajor(c.out.p, count, m);
  return true;
}

// ---- quadratic forms (kernel.cpp:238-272) --------------------------------
// contrib[i][p][0..d] (row i's terms; the host sums rows ascending, as the CPU
// oracle does). Block: 32 rows; thread (row r = tid / 8, lane group cs = tid % 8)
// walks columns c = cs, cs + 8, ... of every chunk; per-thread sums are
// combined over the 8 threads of a row in a fixed order at the end.
constexpr int QMAXP = 2;
__global__ void __launch_bounds__(256) quad_kernel(const double* __restrict__ xs, int n, int d, double sv,
                                                   const double* const* __restrict__ us,
                                                   const double* const* __restrict__ ws, const int* __restrict__ ms,
                                                   int npairs, double* __restrict__ contrib) {
  extern __shared__ double qsm[];
  double (*xr)[MAXD] = reinterpret_cast<double (*)[MAXD]>(qsm);
  double (*xc)[MAXD + 1] = reinterpret_cast<double (*)[MAXD + 1]>(qsm + TR * MAXD);
  double (*ur)[TR][65] = reinterpret_cast<double (*)[TR][65]>(qsm + TR * MAXD + TC * (MAXD + 1));
  double (*wc)[TC][65] = reinterpret_cast<double (*)[TC][65]>(qsm + TR * MAXD + TC * (MAXD + 1) + QMAXP * TR * 65);
  const int tid = threadIdx.x, r = tid >> 3, cs = tid & 7;
  const int r0 = blockIdx.x * TR;
  for (int e = tid; e < TR * d; e += blockDim.x) {
    const int rr = e / d, k = e % d;
    xr[rr][k] = r0 + rr < n ? xs[static_cast<size_t>(r0 + rr) * d + k] : 0.0;
  }
  for (int p = 0; p < npairs; ++p)
    for (int e = tid; e < TR * ms[p]; e += blockDim.x) {
      const int rr = e / ms[p], j = e % ms[p];
      ur[p][rr][j] = r0 + rr < n ? us[p][static_cast<size_t>(r0 + rr) * ms[p] + j] : 0.0;
    }
  double sig[QMAXP], ls[QMAXP][MAXD];
  for (int p = 0; p < QMAXP; ++p) {
    sig[p] = 0.0;
    for (int q = 0; q < MAXD; ++q) ls[p][q] = 0.0;
  }
  for (int c0 = 0; c0 < n; c0 += TC) {
    const int cn = min(TC, n - c0);
    __syncthreads();
    for (int e = tid; e < TC * d; e += blockDim.x) {
      const int c = e / d, k = e % d;
      xc[c][k] = c < cn ? xs[static_cast<size_t>(c0 + c) * d + k] : 0.0;
    }
    for (int p = 0; p < npairs; ++p)
      for (int e = tid; e < TC * ms[p]; e += blockDim.x) {
        const int c = e / ms[p], j = e % ms[p];
        wc[p][c][j] = c < cn ? ws[p][static_cast<size_t>(c0 + c) * ms[p] + j] : 0.0;
      }
    __syncthreads();
    for (int c = cs; c < cn; c += 8) {
      double r2 = 0.0;
      double d2[MAXD];
      for (int k = 0; k < d; ++k) {
        const double t = xc[c][k] - xr[r][k];
        d2[k] = t * t;
        r2 += t * t;
      }
      const double value = matern(r2, sv);
      const double et = exp(-kSqrt3 * sqrt(r2));
      for (int p = 0; p < npairs; ++p) {
        double g = 0.0;
        for (int j = 0; j < ms[p]; ++j) g += wc[p][c][j] * ur[p][r][j];
        sig[p] += value * g;
        const double w = 3.0 * sv * et * g;
        for (int k = 0; k < d; ++k) ls[p][k] += w * d2[k];
      }
    }
  }
  // fixed-order combine of the 8 column-lane partials of each row
  for (int p = 0; p < npairs; ++p) {
    for (int k = 0; k <= d; ++k) {
      double v = k < d ? ls[p][k] : sig[p];
      for (int o = 1; o < 8; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (cs == 0 && r0 + r < n) contrib[(static_cast<size_t>(r0 + r) * npairs + p) * (d + 1) + k] = v;
    }
  }
}

bool quad_hook(const KernelOperator& op, const std::vector<std::pair<const Mat*, const Mat*>>& pairs,
               std::vector<Vec>& out) {
  const int n = op.size(), d = op.dim(), P = static_cast<int>(pairs.size());
  if (P > QMAXP || d > MAXD) return false;
  for (const auto& pr : pairs)
    if (pr.first->cols > 65) return false;
  Ctx& c = ctx();
  upload_xs(op, c.xs);
  std::vector<Dev<double>> U(P), W(P);
  std::vector<const double*> up(P), wp(P);
  std::vector<int> ms(P);
  for (int p = 0; p < P; ++p) {
    upload_rowmajor(*pairs[p].first, U[p]);
    upload_rowmajor(*pairs[p].second, W[p]);
    up[p] = U[p].p;
    wp[p] = W[p].p;
    ms[p] = pairs[p].first->cols;
  }
  Dev<const double*> upd(P), wpd(P);
  Dev<int> msd(P);
  OG_CUDA(cudaMemcpy(upd.p, up.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
  OG_CUDA(cudaMemcpy(wpd.p, wp.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
  OG_CUDA(cudaMemcpy(msd.p, ms.data(), sizeof(int) * P, cudaMemcpyHostToDevice));
  Dev<double> contrib(static_cast<size_t>(n) * P * (d + 1));
  const size_t qsmem = sizeof(double) * (TR * MAXD + TC * (MAXD + 1) + QMAXP * (TR + TC) * 65);
  OG_CUDA(cudaFuncSetAttribute(quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(qsmem)));
  quad_kernel<<<(n + TR - 1) / TR, 256, qsmem>>>(c.xs.p, n, d, op.signal_variance(), upd.p, wpd.p, msd.p, P, contrib.p);
  OG_CUDA(cudaGetLastError());
  std::vector<double> h(static_cast<size_t>(n) * P * (d + 1));
  OG_CUDA(cudaMemcpy(h.data(), contrib.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
  const double s = std::sqrt(op.signal_variance());
  const Vec& inv_ls = op.inverse_lengthscales();
  out.assign(P, Vec(d + 2, 0.0));
  for (int i = 0; i < n; ++i)  // rows ascending (kernel.cpp:265-271's per-row terms)
    for (int p = 0; p < P; ++p) {
      const double* t = &h[(static_cast<size_t>(i) * P + p) * (d + 1)];
      out[p][d] += (2.0 / s) * t[d];
      for (int q = 0; q < d; ++q) out[p][q] += inv_ls[q] * t[q];
    }
  return true;
}

// ---- RFF prior values (rff.cpp:36-54, 64-73) ------------------------------
// prior[i][j] = sum_q phi_q(x_i) W[q][j], features interleaved (2p cos, 2p+1 sin)
// and summed in ascending q, as the CPU loop does.
__global__ void __launch_bounds__(1024) prior_kernel(const double* __restrict__ x, int n, int d,
                                                     const double* __restrict__ freq, int P, double amp,
                                                     const double* __restrict__ w, int s, double* __restrict__ prior) {
  constexpr int RB = 16, PB = 32;
  __shared__ double xr[RB][MAXD];
  __shared__ double ph[RB][2 * PB];
  __shared__ double wt[2 * PB][64];
  const int tid = threadIdx.x, r = tid / 64, j = tid % 64;
  const int r0 = blockIdx.x * RB;
  for (int e = tid; e < RB * d; e += blockDim.x) {
    const int rr = e / d, k = e % d;
    xr[rr][k] = r0 + rr < n ? x[static_cast<size_t>(r0 + rr) * d + k] : 0.0;
  }
  double acc = 0.0;
  for (int p0 = 0; p0 < P; p0 += PB) {
    const int pn = min(PB, P - p0);
    __syncthreads();
    for (int e = tid; e < RB * PB; e += blockDim.x) {
      const int rr = e / PB, pp = e % PB;
      double cv = 0.0, sv = 0.0;
      if (pp < pn) {
        double angle = 0.0;
        for (int k = 0; k < d; ++k) angle += xr[rr][k] * freq[static_cast<size_t>(p0 + pp) * d + k];
        sincos(angle, &sv, &cv);
        cv *= amp;
        sv *= amp;
      }
      ph[rr][2 * pp] = cv;
      ph[rr][2 * pp + 1] = sv;
    }
    for (int e = tid; e < 2 * PB * 64; e += blockDim.x) {
      const int q = e / 64, jj = e % 64;
      wt[q][jj] = (q < 2 * pn && jj < s) ? w[static_cast<size_t>(2 * p0 + q) * s + jj] : 0.0;
    }
    __syncthreads();
    if (j < s)
      for (int q = 0; q < 2 * pn; ++q) acc += ph[r][q] * wt[q][j];
  }
  if (r0 + r < n && j < s) prior[static_cast<size_t>(r0 + r) * s + j] = acc;
}

bool prior_hook(const RffBasis& basis, const Hyper& hp, const Dataset& data, int s, Mat& prior) {
  const int n = data.n(), d = data.dim(), P = basis.pairs();
  if (s > 64 || d > MAXD) return false;
  const Vec ls = hp.lengthscales();
  std::vector<double> freq(static_cast<size_t>(P) * d), w(static_cast<size_t>(2) * P * s), x(static_cast<size_t>(n) * d);
  for (int p = 0; p < P; ++p)
    for (int k = 0; k < d; ++k) freq[static_cast<size_t>(p) * d + k] = basis.base_frequencies(p, k) * (1.0 / ls[k]);
  for (int q = 0; q < 2 * P; ++q)
    for (int j = 0; j < s; ++j) w[static_cast<size_t>(q) * s + j] = basis.weights(q, j);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) x[static_cast<size_t>(i) * d + k] = data.inputs(i, k);
  const double amp = hp.signal_scale() / std::sqrt(static_cast<double>(P));
  Dev<double> fd(freq.size()), wd(w.size()), xd(x.size()), pd(static_cast<size_t>(n) * s);
  OG_CUDA(cudaMemcpy(fd.p, freq.data(), sizeof(double) * freq.size(), cudaMemcpyHostToDevice));
  OG_CUDA(cudaMemcpy(wd.p, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
  OG_CUDA(cudaMemcpy(xd.p, x.data(), sizeof(double) * x.size(), cudaMemcpyHostToDevice));
  prior_kernel<<<(n + 15) / 16, 1024>>>(xd.p, n, d, fd.p, P, amp, wd.p, s, pd.p);
  OG_CUDA(cudaGetLastError());
  prior = download_rowmajor(pd.p, n, s);
  return true;
}

// ---- solve_sgd (solvers.cpp:147-184) --------------------------------------
// g = H[idx] V - B[idx]; M *= rho; M[idx] -= (lr/b) g; V += M; R[idx] = -g;
// the loop test is termination_check on the tracked R (full column norms, as
// the reference), the abort test V.allFinite() after every iteration.
__global__ void sgd_grad_kernel(double* g, const double* targets, const int* idx, int b, int m) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= b * m) return;
  const int q = e / m, j = e % m;
  g[e] -= targets[static_cast<size_t>(idx[q]) * m + j];
}
__global__ void sgd_mark_kernel(int* pos, const int* idx, int b, int set) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < b) pos[idx[q]] = set ? q : -1;
}
__global__ void sgd_update_kernel(double* M, double* V, double* R, const int* pos, const double* g, int n, int m,
                                  double rho, double step, int* nonfinite) {
  const long long count = static_cast<long long>(n) * m;
  int bad = 0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / m), j = static_cast<int>(e % m);
    double mo = M[e] * rho;
    const int q = pos[i];
    if (q >= 0) {
      const double upd = step * g[static_cast<size_t>(q) * m + j];
      mo -= upd;
      R[e] = -g[static_cast<size_t>(q) * m + j];
    }
    M[e] = mo;
    const double v = V[e] + mo;
    V[e] = v;
    if (!isfinite(v)) bad = 1;
  }
  if (bad) atomicOr(nonfinite, 1);
}
// column sums of squares of R (row-major [n][m]) in a fixed order: block
// partials over row ranges, then summed in block order.
__global__ void colsq_kernel(const double* R, int n, int m, double* part) {
  const int j = threadIdx.x;  // blockDim.x = m
  const int rows = (n + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * rows, i1 = min(n, i0 + rows);
  double s = 0.0;
  for (int i = i0; i < i1; ++i) {
    const double r = R[static_cast<size_t>(i) * m + j];
    s += r * r;
  }
  part[static_cast<size_t>(blockIdx.x) * m + j] = s;
}

bool sgd_hook(LinearSystemBatch& batch, const SolverConfig& config, SolverReport& rep,
              std::vector<std::vector<int>>* batches_out, int record) {
  const KernelOperator& op = *batch.op;
  const int n = op.size(), d = op.dim(), m = batch.columns();
  if (m > MAXM || d > MAXD) return false;
  const int b = std::min(config.batch_size, n);
  Ctx& c = ctx();
  upload_xs(op, c.xs);
  Dev<double> B, V, Mo, R, g, cpart;
  upload_rowmajor(batch.targets, B);
  upload_rowmajor(batch.solutions, V);
  R.alloc(static_cast<size_t>(n) * m);
  OG_CUDA(cudaMemcpy(R.p, B.p, sizeof(double) * n * m, cudaMemcpyDeviceToDevice));  // R := B
  Mo.alloc(static_cast<size_t>(n) * m);
  OG_CUDA(cudaMemset(Mo.p, 0, sizeof(double) * n * m));
  g.alloc(static_cast<size_t>(b) * m);
  Dev<int> idx(b), pos(n), flag(1);
  OG_CUDA(cudaMemset(pos.p, 0xff, sizeof(int) * n));
  OG_CUDA(cudaMemset(flag.p, 0, sizeof(int)));
  const int cblocks = 256;
  cpart.alloc(static_cast<size_t>(cblocks) * m);
  std::vector<double> hp(static_cast<size_t>(cblocks) * m);
  auto done = [&]() {  // termination_check on the tracked residuals (linear_system.cpp:47-53)
    colsq_kernel<<<cblocks, m>>>(R.p, n, m, cpart.p);
    OG_CUDA(cudaGetLastError());
    OG_CUDA(cudaMemcpy(hp.data(), cpart.p, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost));
    std::vector<double> ss(m, 0.0);
    for (int k = 0; k < cblocks; ++k)
      for (int j = 0; j < m; ++j) ss[j] += hp[static_cast<size_t>(k) * m + j];
    const double mean = std::sqrt(ss[0]) / batch.scales[0];
    double probe = 0.0;
    for (int j = 1; j < m; ++j) probe += std::sqrt(ss[j]) / batch.scales[j];
    if (m > 1) probe /= (m - 1);
    return mean <= config.tolerance && probe <= config.tolerance;
  };
  RandomStream rng(config.seed, streams::kSolver, config.substream);
  const double max_iterations = g_sgd_iteration_cap >= 0
                                    ? std::min<double>(g_sgd_iteration_cap, static_cast<double>(config.max_epochs) * n / b)
                                    : static_cast<double>(config.max_epochs) * n / b;
  const double step = config.learning_rate / b;
  const int ublocks = 148 * 8;
  int t = 0;
  while (t < max_iterations && !done()) {
    const std::vector<int> ix = rng.sample_without_replacement(n, b);
    if (batches_out && t < record) batches_out->push_back(ix);
    OG_CUDA(cudaMemcpy(idx.p, ix.data(), sizeof(int) * b, cudaMemcpyHostToDevice));
    apply_dev(c.xs.p, n, d, op.signal_variance(), op.noise_variance(), idx.p, b, V.p, m, g.p);
    sgd_grad_kernel<<<(b * m + 255) / 256, 256>>>(g.p, B.p, idx.p, b, m);
    sgd_mark_kernel<<<(b + 255) / 256, 256>>>(pos.p, idx.p, b, 1);
    sgd_update_kernel<<<ublocks, 256>>>(Mo.p, V.p, R.p, pos.p, g.p, n, m, config.momentum, step, flag.p);
    sgd_mark_kernel<<<(b + 255) / 256, 256>>>(pos.p, idx.p, b, 0);
    OG_CUDA(cudaGetLastError());
    ++t;
    int bad = 0;
    OG_CUDA(cudaMemcpy(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad) {
      rep.aborted = true;
      rep.abort_reason = "sgd divergence: non-finite iterate";
      break;
    }
  }
  batch.solutions = download_rowmajor(V.p, n, m);
  batch.residuals = download_rowmajor(R.p, n, m);
  rep.iterations = t;
  rep.epochs_consumed = static_cast<double>(t) * b / n;
  return true;
}

const OracleBackend kBackend{apply_hook, quad_hook, prior_hook, sgd_hook};

}  // namespace gpu
}  // namespace oracle

extern "C" {
// Routes the oracle's O(n^2) passes to the FP64 CUDA restatements on `device`
// (enable = 0 restores the CPU loops). Returns 0 on success.
int oracle_gpu_enable(int device, int enable) {
  if (!enable) {
    oracle::g_backend = nullptr;
    return 0;
  }
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  oracle::g_backend = &oracle::gpu::kBackend;
  return 0;
}
}
