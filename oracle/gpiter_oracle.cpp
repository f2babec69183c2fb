// TEST INFRASTRUCTURE — NOT PRODUCT CODE. FP64 restatement of the reference
// gpiter library without Eigen; see gpiter_oracle.hpp for the contract.
// Summation orders are fixed (ascending index) so results are deterministic
// and, where the reference pins it, independent of tiling and threading.
#include "gpiter_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <limits>
#include <stdexcept>

#include <atomic>
#include <functional>
#include <thread>

namespace oracle {

const OracleBackend* g_backend = nullptr;
int g_sgd_iteration_cap = -1;
int g_apply_order = 0;
double g_apply_noise = 0.0;
namespace {
unsigned long long g_apply_calls = 0;
// Sensitivity knob: out *= 1 + eps u, u in [-1, 1) from a counter hash
// (splitmix64 of (call, element)), deterministic across runs.
void perturb(std::vector<double>& out) {
  if (g_apply_noise == 0.0) return;
  const unsigned long long call = g_apply_calls++;
  for (size_t e = 0; e < out.size(); ++e) {
    unsigned long long z = call * 0x9E3779B97F4A7C15ull + e + 1;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-52 - 1.0;
    out[e] *= 1.0 + g_apply_noise * u;
  }
}
}  // namespace

namespace {
// Dynamic parallel-for over [0, count) with std::thread (no OpenMP in this
// toolchain). Each index is processed by exactly one worker, so results that
// depend only on per-index work are independent of the thread count.
void parallel_for(int threads, int count, const std::function<void(int, int)>& body) {
  if (threads <= 1 || count <= 1) {
    for (int i = 0; i < count; ++i) body(0, i);
    return;
  }
  const int workers = std::min(threads, count);
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (int i = next.fetch_add(1); i < count; i = next.fetch_add(1)) body(w, i);
    });
  for (auto& t : pool) t.join();
}
}  // namespace

bool Mat::all_finite() const {
  for (double x : a)
    if (!std::isfinite(x)) return false;
  return true;
}

// ===================== rng.cpp:12-126 ====================================
namespace {
constexpr uint64_t kMul0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kMul1 = 0xCA5A826395121157ULL;
constexpr uint64_t kWeyl0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kWeyl1 = 0xBB67AE8584CAA73BULL;
constexpr double kPi = 3.141592653589793;
constexpr double kSqrt3 = 1.7320508075688772;  // kernel.cpp:13
}  // namespace

// rng.cpp:34-47
std::array<uint64_t, 4> philox4x64(const std::array<uint64_t, 4>& counter,
                                   const std::array<uint64_t, 2>& key) {
  std::array<uint64_t, 4> c = counter;
  std::array<uint64_t, 2> k = key;
  for (int round = 0; round < 10; ++round) {
    const unsigned __int128 p0 = static_cast<unsigned __int128>(kMul0) * c[0];
    const unsigned __int128 p1 = static_cast<unsigned __int128>(kMul1) * c[2];
    const uint64_t hi0 = static_cast<uint64_t>(p0 >> 64), lo0 = static_cast<uint64_t>(p0);
    const uint64_t hi1 = static_cast<uint64_t>(p1 >> 64), lo1 = static_cast<uint64_t>(p1);
    c = {hi1 ^ c[1] ^ k[0], lo1, hi0 ^ c[3] ^ k[1], lo0};
    k[0] += kWeyl0;
    k[1] += kWeyl1;
  }
  return c;
}

// rng.cpp:49-53
void RandomStream::refill() {
  buffer_ = philox4x64(counter_, key_);
  buffer_pos_ = 0;
  ++counter_[0];
}

uint64_t RandomStream::next_u64() {  // rng.cpp:55-58
  if (buffer_pos_ >= 4) refill();
  return buffer_[buffer_pos_++];
}

double RandomStream::next_double() {  // rng.cpp:60-62
  return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
}

double RandomStream::next_gaussian() {  // rng.cpp:64-77 (Box-Muller, cos first, sin cached)
  if (has_cached_gaussian_) {
    has_cached_gaussian_ = false;
    return cached_gaussian_;
  }
  const double u1 = static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53;
  const double u2 = next_double();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * kPi * u2;
  cached_gaussian_ = radius * std::sin(angle);
  has_cached_gaussian_ = true;
  return radius * std::cos(angle);
}

uint64_t RandomStream::next_below(uint64_t bound) {  // rng.cpp:79-84
  if (bound == 0) throw std::invalid_argument("next_below: bound must be positive");
  return next_u64() % bound;
}

void RandomStream::fill_gaussian(double* data, size_t count) {  // rng.cpp:86-90
  for (size_t i = 0; i < count; ++i) data[i] = next_gaussian();
}

void RandomStream::fill_rademacher(double* data, size_t count) {  // rng.cpp:92-96
  for (size_t i = 0; i < count; ++i) data[i] = (next_u64() & 1u) ? 1.0 : -1.0;
}

std::vector<int> RandomStream::permutation(int n) {  // rng.cpp:98-106
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int i = n - 1; i > 0; --i) {
    const int j = static_cast<int>(next_below(static_cast<uint64_t>(i) + 1));
    std::swap(perm[i], perm[j]);
  }
  return perm;
}

std::vector<int> RandomStream::sample_without_replacement(int n, int k) {  // rng.cpp:108-126
  if (k > n) throw std::invalid_argument("sample_without_replacement: k > n");
  std::vector<int> chosen;
  chosen.reserve(k);
  std::vector<bool> taken(n, false);
  for (int j = n - k; j < n; ++j) {
    const int t = static_cast<int>(next_below(static_cast<uint64_t>(j) + 1));
    if (taken[t]) {
      chosen.push_back(j);
      taken[j] = true;
    } else {
      chosen.push_back(t);
      taken[t] = true;
    }
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// ===================== hyperparameters.cpp:8-65 ==========================
double softplus(double x) {
  if (x > 0.0) return x + std::log1p(std::exp(-x));
  return std::log1p(std::exp(x));
}

double softplus_inverse(double y) {
  if (y <= 0.0) throw std::invalid_argument("softplus_inverse: argument must be positive");
  return y + std::log(-std::expm1(-y));
}

double sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}

Hyper Hyper::from_raw(Vec raw) {
  if (raw.size() < 3) throw std::invalid_argument("Hyperparameters: need at least d=1 plus scales");
  Hyper h;
  h.raw = std::move(raw);
  return h;
}

Hyper Hyper::from_constrained(const Vec& c) {
  Vec raw(c.size());
  for (size_t i = 0; i < c.size(); ++i) raw[i] = softplus_inverse(c[i]);
  return from_raw(std::move(raw));
}

Hyper Hyper::constant(int d, double v) { return from_constrained(Vec(d + 2, v)); }

Vec Hyper::constrained() const {
  Vec out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) out[i] = softplus(raw[i]);
  return out;
}

Vec Hyper::lengthscales() const {
  Vec out(input_dim());
  for (int i = 0; i < input_dim(); ++i) out[i] = softplus(raw[i]);
  return out;
}

void Hyper::validate() const {
  const Vec c = constrained();
  for (size_t i = 0; i < c.size(); ++i)
    if (!std::isfinite(c[i]) || c[i] <= 0.0)
      throw std::invalid_argument("Hyperparameters: constrained value " + std::to_string(i) +
                                  " is not finite and positive");
}

// ===================== kernel.cpp ========================================
namespace {
// kernel.cpp:35-39
inline double matern_profile(double r2, double signal_variance) {
  const double r = std::sqrt(r2);
  return signal_variance * (1.0 + kSqrt3 * r) * std::exp(-kSqrt3 * r);
}

// kernel.cpp:15-30: out[r*m+j] = sum_c a[r*n+c] v[c*m+j], ascending c.
void accumulate_rows_product(const double* a, int rows, int n, const double* v, int m,
                             double* out) {
  constexpr int kRowBlock = 8;
  for (int r0 = 0; r0 < rows; r0 += kRowBlock) {
    const int rb = std::min(kRowBlock, rows - r0);
    for (int r = r0; r < r0 + rb; ++r) std::fill(out + static_cast<size_t>(r) * m,
                                                 out + static_cast<size_t>(r + 1) * m, 0.0);
    for (int c = 0; c < n; ++c) {
      const double* vrow = v + static_cast<size_t>(c) * m;
      for (int r = r0; r < r0 + rb; ++r) {
        const double coeff = a[static_cast<size_t>(r) * n + c];
        double* acc = out + static_cast<size_t>(r) * m;
        for (int j = 0; j < m; ++j) acc[j] += coeff * vrow[j];
      }
    }
  }
}

// Sensitivity variant (test knob g_apply_order = 1): the same products summed
// in descending column order.
void accumulate_rows_product_reversed(const double* a, int rows, int n, const double* v, int m, double* out) {
  for (int r = 0; r < rows; ++r) {
    double* acc = out + static_cast<size_t>(r) * m;
    std::fill(acc, acc + m, 0.0);
    for (int c = n - 1; c >= 0; --c) {
      const double coeff = a[static_cast<size_t>(r) * n + c];
      const double* vrow = v + static_cast<size_t>(c) * m;
      for (int j = 0; j < m; ++j) acc[j] += coeff * vrow[j];
    }
  }
}

std::vector<double> to_row_major(const Mat& v) {
  std::vector<double> out(v.size());
  for (int i = 0; i < v.rows; ++i)
    for (int j = 0; j < v.cols; ++j) out[static_cast<size_t>(i) * v.cols + j] = v(i, j);
  return out;
}

Mat from_row_major(const std::vector<double>& rm, int rows, int cols) {
  Mat out(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out(i, j) = rm[static_cast<size_t>(i) * cols + j];
  return out;
}
}  // namespace

// kernel.cpp:43-55
double matern32(const double* x, const double* x2, int d, const Hyper& hp) {
  if (d != hp.input_dim())
    throw std::invalid_argument("matern32: point dimension does not match hyperparameters");
  for (int i = 0; i < d; ++i)
    if (!std::isfinite(x[i]) || !std::isfinite(x2[i]))
      throw std::invalid_argument("matern32: non-finite input");
  const Vec ls = hp.lengthscales();
  double sq = 0.0;
  for (int i = 0; i < d; ++i) {
    const double t = (x[i] - x2[i]) / ls[i];
    sq += t * t;
  }
  const double r = std::sqrt(sq);
  const double s = hp.signal_scale();
  return s * s * (1.0 + kSqrt3 * r) * std::exp(-kSqrt3 * r);
}

// kernel.cpp:83-109 (the dense cache is omitted: with the fixed accumulation
// order it produces bitwise the same products, kernel.hpp:32-36).
KernelOperator::KernelOperator(const Dataset* data, Hyper hp, int block_rows, int threads)
    : data_(data), hp_(std::move(hp)), block_rows_(block_rows), threads_(std::max(1, threads)) {
  hp_.validate();
  if (data_->dim() != hp_.input_dim())
    throw std::invalid_argument("KernelOperator: dataset dimension does not match hyperparameters");
  if (block_rows_ < 1) throw std::invalid_argument("KernelOperator: block_rows >= 1");
  n_ = data_->n();
  d_ = data_->dim();
  const Vec ls = hp_.lengthscales();
  inv_ls_.resize(d_);
  for (int k = 0; k < d_; ++k) inv_ls_[k] = 1.0 / ls[k];
  xs_.resize(static_cast<size_t>(n_) * d_);
  for (int i = 0; i < n_; ++i)
    for (int k = 0; k < d_; ++k) xs_[static_cast<size_t>(i) * d_ + k] = data_->inputs(i, k) * inv_ls_[k];
  xst_.resize(xs_.size());  // the same values dimension-major (fill_row's first pass)
  for (int i = 0; i < n_; ++i)
    for (int k = 0; k < d_; ++k) xst_[static_cast<size_t>(k) * n_ + i] = xs_[static_cast<size_t>(i) * d_ + k];
  const double s = hp_.signal_scale();
  signal_variance_ = s * s;
  noise_variance_ = hp_.noise_variance();
}

// kernel.cpp:111-120: row i of H (kernel + noise on the diagonal).
// Two passes over the row (squared distances dimension by dimension, then the
// profile): every r2 is still summed over k = 0..d-1 in ascending order from
// 0.0, so the values are bitwise those of the per-entry loop, and the profile
// loop vectorises (libmvec exp/sqrt) in the timing build (Makefile `native`).
void KernelOperator::fill_row(int i, double* out) const {
  const double* xi = &xs_[static_cast<size_t>(i) * d_];
  std::fill(out, out + n_, 0.0);
  for (int k = 0; k < d_; ++k) {
    const double* xk = &xst_[static_cast<size_t>(k) * n_];
    const double xik = xi[k];
    for (int c = 0; c < n_; ++c) {
      const double t = xk[c] - xik;
      out[c] += t * t;
    }
  }
  const double sv = signal_variance_;
  for (int c = 0; c < n_; ++c) out[c] = matern_profile(out[c], sv);
  out[i] += noise_variance_;
}

void KernelOperator::fill_rows(int row0, int count, double* out) const {
  for (int r = 0; r < count; ++r) fill_row(row0 + r, out + static_cast<size_t>(r) * n_);
}

// kernel.cpp:133-152. Row tiles are independent and each output element is
// accumulated in ascending column order by one worker, so threading does not
// change a single bit (SPEC.md concurrency model).
Mat KernelOperator::apply(const Mat& v) const {
  if (v.rows != n_) throw std::invalid_argument("KernelOperator::apply: dimension mismatch");
  if (!v.all_finite()) throw std::invalid_argument("KernelOperator::apply: non-finite input");
  if (g_backend && g_backend->apply) {
    Mat out;
    if (g_backend->apply(*this, nullptr, n_, v, out)) {
      if (g_apply_noise != 0.0) {
        perturb(out.a);  // column-major here; any fixed element order will do
      }
      return out;
    }
  }
  const int m = v.cols;
  const std::vector<double> vr = to_row_major(v);
  std::vector<double> out(static_cast<size_t>(n_) * m);
  const int tiles = (n_ + block_rows_ - 1) / block_rows_;
std::vector<std::vector<double>> tiles_buf(std::max(1, std::min(threads_, tiles)));
  parallel_for(threads_, tiles, [&](int w, int t) {
    std::vector<double>& tile = tiles_buf[w];
    if (tile.empty()) tile.resize(static_cast<size_t>(std::min(block_rows_, n_)) * n_);
    const int r0 = t * block_rows_;
    const int rows = std::min(block_rows_, n_ - r0);
    fill_rows(r0, rows, tile.data());
    if (g_apply_order == 1)
      accumulate_rows_product_reversed(tile.data(), rows, n_, vr.data(), m, out.data() + static_cast<size_t>(r0) * m);
    else
      accumulate_rows_product(tile.data(), rows, n_, vr.data(), m, out.data() + static_cast<size_t>(r0) * m);
  });
  perturb(out);
  return from_row_major(out, n_, m);
}

// kernel.cpp:154-168
Mat KernelOperator::apply_rows(const std::vector<int>& rows, const Mat& v) const {
  const int m = v.cols;
  const int count = static_cast<int>(rows.size());
  if (g_backend && g_backend->apply) {
    Mat out;
    if (g_backend->apply(*this, rows.data(), count, v, out)) return out;
  }
  const std::vector<double> vr = to_row_major(v);
  std::vector<double> out(static_cast<size_t>(count) * m);
  const int chunk = 8;
  const int nchunks = (count + chunk - 1) / chunk;
std::vector<std::vector<double>> tiles_buf(std::max(1, std::min(threads_, nchunks)));
  parallel_for(threads_, nchunks, [&](int w, int q) {
    std::vector<double>& tile = tiles_buf[w];
    if (tile.empty()) tile.resize(static_cast<size_t>(chunk) * n_);
    const int r0 = q * chunk, rc = std::min(chunk, count - r0);
    for (int r = 0; r < rc; ++r) fill_row(rows[r0 + r], tile.data() + static_cast<size_t>(r) * n_);
    accumulate_rows_product(tile.data(), rc, n_, vr.data(), m, out.data() + static_cast<size_t>(r0) * m);
  });
  return from_row_major(out, count, m);
}

// kernel.cpp:170-177: H[:, c0:c0+len] U = tile^T U, ascending c within the block.
Mat KernelOperator::apply_columns(int c0, int len, const Mat& u) const {
  if (u.rows != len) throw std::invalid_argument("KernelOperator::apply_columns: height mismatch");
  const int m = u.cols;
  std::vector<double> tile(static_cast<size_t>(len) * n_);
parallel_for(threads_, len, [&](int, int r) { fill_row(c0 + r, tile.data() + static_cast<size_t>(r) * n_); });
  Mat out(n_, m);
  parallel_for(threads_, n_, [&](int, int i) {
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int c = 0; c < len; ++c) acc += tile[static_cast<size_t>(c) * n_ + i] * u(c, j);
      out(i, j) = acc;
    }
  });
  return out;
}

// kernel.cpp:179-184
Mat KernelOperator::dense_block(int r0, int rows, int c0, int cols) const {
  Mat out(rows, cols);
  std::vector<double> row(n_);
  for (int r = 0; r < rows; ++r) {
    fill_row(r0 + r, row.data());
    for (int c = 0; c < cols; ++c) out(r, c) = row[c0 + c];
  }
  return out;
}

// kernel.cpp:188-194
Vec KernelOperator::kernel_column(int i) const {
  Vec out(n_);
  const double* xi = &xs_[static_cast<size_t>(i) * d_];
  for (int c = 0; c < n_; ++c) {
    const double* xc = &xs_[static_cast<size_t>(c) * d_];
    double r2 = 0.0;
    for (int k = 0; k < d_; ++k) {
      const double t = xc[k] - xi[k];
      r2 += t * t;
    }
    out[c] = matern_profile(r2, signal_variance_);
  }
  return out;
}

// kernel.cpp:200-236
Mat KernelOperator::derivative_apply(int k, const Mat& v) const {
  if (k < 0 || k >= hp_.count()) throw std::out_of_range("KernelOperator::derivative_apply: parameter index");
  if (v.rows != n_) throw std::invalid_argument("KernelOperator::derivative_apply: dimension mismatch");
  const int d = d_;
  Mat out(n_, v.cols);
  if (k == d + 1) {
    const double two_sigma = 2.0 * hp_.noise_scale();
    for (size_t e = 0; e < v.size(); ++e) out.a[e] = two_sigma * v.a[e];
    return out;
  }
  const double s = hp_.signal_scale();
  std::vector<double> row(n_);
  for (int i = 0; i < n_; ++i) {
    const double* xi = &xs_[static_cast<size_t>(i) * d_];
    for (int c = 0; c < n_; ++c) {
      const double* xc = &xs_[static_cast<size_t>(c) * d_];
      double r2 = 0.0;
      for (int q = 0; q < d_; ++q) {
        const double t = xc[q] - xi[q];
        r2 += t * t;
      }
      if (k == d) {
        row[c] = (2.0 / s) * matern_profile(r2, signal_variance_);
      } else {
        const double expterm = std::exp(-kSqrt3 * std::sqrt(r2));
        const double dk = xc[k] - xi[k];
        row[c] = 3.0 * signal_variance_ * inv_ls_[k] * expterm * (dk * dk);
      }
    }
    for (int j = 0; j < v.cols; ++j) {
      double acc = 0.0;
      for (int c = 0; c < n_; ++c) acc += row[c] * v(c, j);
      out(i, j) = acc;
    }
  }
  return out;
}

// kernel.cpp:238-272. Per-row contributions are formed in parallel and summed
// into the gradients in ascending row order, so the result is independent of
// the thread count.
std::vector<Vec> KernelOperator::derivative_quadratic_forms_many(
    const std::vector<std::pair<const Mat*, const Mat*>>& pairs) const {
  const int d = d_;
  const double s = hp_.signal_scale();
  const size_t count = pairs.size();
  const int P = d + 2;
  std::vector<Vec> grads(count, Vec(P, 0.0));
  for (size_t p = 0; p < count; ++p) {
    const Mat* u = pairs[p].first;
    const Mat* w = pairs[p].second;
    if (u->rows != n_ || w->rows != n_ || u->cols != w->cols)
      throw std::invalid_argument("derivative_quadratic_forms: shape mismatch");
    double acc = 0.0;
    for (size_t e = 0; e < u->size(); ++e) acc += u->a[e] * w->a[e];
    grads[p][d + 1] = 2.0 * hp_.noise_scale() * acc;
  }
  if (g_backend && g_backend->quad_forms) {
    std::vector<Vec> dev;
    if (g_backend->quad_forms(*this, pairs, dev)) {
      for (size_t p = 0; p < count; ++p)
        for (int q = 0; q <= d; ++q) grads[p][q] = dev[p][q];
      return grads;
    }
  }
  // Row-major copies of W for contiguous row access.
  std::vector<std::vector<double>> wr(count), ur(count);
  for (size_t p = 0; p < count; ++p) {
    wr[p] = to_row_major(*pairs[p].second);
    ur[p] = to_row_major(*pairs[p].first);
  }
  const int R = 64;  // rows per parallel chunk
  std::vector<double> contrib(static_cast<size_t>(n_) * count * (d + 1));
const int nchunk = (n_ + R - 1) / R;
  parallel_for(threads_, nchunk, [&](int, int ch) {
    std::vector<double> diffs2(static_cast<size_t>(n_) * d), values(n_), expterm(n_), g(n_);
    {
      const int i0 = ch * R;
      for (int i = i0; i < std::min(n_, i0 + R); ++i) {
        const double* xi = &xs_[static_cast<size_t>(i) * d_];
        for (int c = 0; c < n_; ++c) {
          const double* xc = &xs_[static_cast<size_t>(c) * d_];
          double r2 = 0.0;
          for (int q = 0; q < d; ++q) {
            const double t = xc[q] - xi[q];
            diffs2[static_cast<size_t>(c) * d + q] = t * t;
            r2 += t * t;
          }
          values[c] = matern_profile(r2, signal_variance_);
          expterm[c] = std::exp(-kSqrt3 * std::sqrt(r2));
        }
        for (size_t p = 0; p < count; ++p) {
          const int m = pairs[p].first->cols;
          const double* ui = &ur[p][static_cast<size_t>(i) * m];
          for (int c = 0; c < n_; ++c) {
            const double* wc = &wr[p][static_cast<size_t>(c) * m];
            double acc = 0.0;
            for (int j = 0; j < m; ++j) acc += wc[j] * ui[j];
            g[c] = acc;
          }
          double* out = &contrib[(static_cast<size_t>(i) * count + p) * (d + 1)];
          double sig = 0.0;
          for (int c = 0; c < n_; ++c) sig += values[c] * g[c];
          out[d] = (2.0 / s) * sig;
          for (int q = 0; q < d; ++q) {
            double acc = 0.0;
            for (int c = 0; c < n_; ++c)
              acc += (3.0 * signal_variance_ * expterm[c] * g[c]) * diffs2[static_cast<size_t>(c) * d + q];
            out[q] = inv_ls_[q] * acc;
          }
        }
      }
    }
  });
  for (int i = 0; i < n_; ++i)
    for (size_t p = 0; p < count; ++p) {
      const double* out = &contrib[(static_cast<size_t>(i) * count + p) * (d + 1)];
      grads[p][d] += out[d];
      for (int q = 0; q < d; ++q) grads[p][q] += out[q];
    }
  return grads;
}

// ===================== linear_system.cpp:7-53 ============================
void SolverConfig::validate() const {
  if (!(tolerance > 0.0)) throw std::invalid_argument("SolverConfig: tolerance > 0");
  if (max_epochs < 1) throw std::invalid_argument("SolverConfig: max_epochs >= 1");
  if (block_size < 1) throw std::invalid_argument("SolverConfig: block_size >= 1");
  if (batch_size < 1) throw std::invalid_argument("SolverConfig: batch_size >= 1");
  if (momentum < 0.0 || momentum >= 1.0) throw std::invalid_argument("SolverConfig: 0 <= momentum < 1");
  if (preconditioner_rank < 0) throw std::invalid_argument("SolverConfig: preconditioner_rank >= 0");
}

namespace {
double col_norm(const Mat& a, int j) {
  const double* c = a.col(j);
  double acc = 0.0;
  for (int i = 0; i < a.rows; ++i) acc += c[i] * c[i];
  return std::sqrt(acc);
}
double col_dot(const Mat& a, int ja, const Mat& b, int jb) {
  const double* x = a.col(ja);
  const double* y = b.col(jb);
  double acc = 0.0;
  for (int i = 0; i < a.rows; ++i) acc += x[i] * y[i];
  return acc;
}
}  // namespace

LinearSystemBatch::LinearSystemBatch(const KernelOperator& op_in, Mat t)
    : op(&op_in), targets(std::move(t)) {
  if (targets.rows != op->size())
    throw std::invalid_argument("LinearSystemBatch: target height does not match operator");
  scales.resize(targets.cols);
  for (int j = 0; j < targets.cols; ++j) scales[j] = col_norm(targets, j) + kNormEpsilon;
  solutions = Mat(targets.rows, targets.cols);
  residuals = Mat(targets.rows, targets.cols);
}

void LinearSystemBatch::warm_start(const Mat& prev) {
  if (prev.rows != targets.rows || prev.cols != targets.cols)
    throw std::invalid_argument("LinearSystemBatch::warm_start: shape mismatch");
  solutions = prev;
}

void LinearSystemBatch::refresh_residuals() {
  const Mat hv = op->apply(solutions);
  for (size_t e = 0; e < residuals.size(); ++e) residuals.a[e] = targets.a[e] - hv.a[e];
}

double LinearSystemBatch::mean_residual_norm() const { return col_norm(residuals, 0) / scales[0]; }

double LinearSystemBatch::probe_residual_norm() const {
  const int s = probe_count();
  if (s == 0) return 0.0;
  double sum = 0.0;
  for (int j = 1; j < columns(); ++j) sum += col_norm(residuals, j) / scales[j];
  return sum / s;
}

TerminationStatus termination_check(const LinearSystemBatch& b, double tol) {
  TerminationStatus st;
  st.mean_norm = b.mean_residual_norm();
  st.probe_norm = b.probe_residual_norm();
  st.done = st.mean_norm <= tol && st.probe_norm <= tol;
  return st;
}

// ===================== dense LLT (stands in for Eigen::LLT) ===============
void LLT::compute(const Mat& a) {
  n = a.rows;
  L = Mat(n, n);
  ok = true;
  for (int j = 0; j < n; ++j) {
    double s = a(j, j);
    for (int k = 0; k < j; ++k) s -= L(j, k) * L(j, k);
    if (!(s > 0.0) || !std::isfinite(s)) { ok = false; return; }
    const double ljj = std::sqrt(s);
    L(j, j) = ljj;
    for (int i = j + 1; i < n; ++i) {
      double t = a(i, j);
      for (int k = 0; k < j; ++k) t -= L(i, k) * L(j, k);
      L(i, j) = t / ljj;
    }
  }
}

Mat LLT::solve(const Mat& b) const {
  Mat x = b;
  for (int c = 0; c < x.cols; ++c) {
    double* y = x.col(c);
    for (int i = 0; i < n; ++i) {
      double t = y[i];
      for (int k = 0; k < i; ++k) t -= L(i, k) * y[k];
      y[i] = t / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double t = y[i];
      for (int k = i + 1; k < n; ++k) t -= L(k, i) * y[k];
      y[i] = t / L(i, i);
    }
  }
  return x;
}

// ===================== pivoted_cholesky.cpp:10-58 =========================
PivotedCholesky::PivotedCholesky(const KernelOperator& op, int rank) {
  const int n = op.size();
  if (rank < 0 || rank > n) throw std::invalid_argument("PivotedCholeskyPreconditioner: rank must be in [0, n]");
  noise_variance_ = op.noise_variance();
  Vec diag = op.kernel_diagonal();
  std::vector<double> f(static_cast<size_t>(n) * std::max(rank, 1));  // col-major n x rank
  int m = 0;
  for (; m < rank; ++m) {
    int pivot = 0;
    double best = diag[0];
    for (int i = 1; i < n; ++i)
      if (diag[i] > best) { best = diag[i]; pivot = i; }
    if (!(best > 0.0)) { stopped_early_ = true; break; }
    Vec column = op.kernel_column(pivot);
    if (m > 0) {
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < m; ++k) acc += f[static_cast<size_t>(k) * n + i] * f[static_cast<size_t>(k) * n + pivot];
        column[i] -= acc;
      }
    }
    const double sb = std::sqrt(best);
    for (int i = 0; i < n; ++i) column[i] /= sb;
    for (int i = 0; i < n; ++i) f[static_cast<size_t>(m) * n + i] = column[i];
    for (int i = 0; i < n; ++i) diag[i] -= column[i] * column[i];
    diag[pivot] = 0.0;
    pivots_.push_back(pivot);
  }
  achieved_rank_ = m;
  factor_ = Mat(n, m);
  std::copy(f.begin(), f.begin() + static_cast<size_t>(n) * m, factor_.a.begin());
  if (m > 0) {
    Mat small(m, m);
    for (int a = 0; a < m; ++a)
      for (int b = 0; b < m; ++b) small(a, b) = col_dot(factor_, a, factor_, b);
    for (int a = 0; a < m; ++a) small(a, a) += noise_variance_;
    small_.compute(small);
    if (!small_.ok) throw std::runtime_error("PivotedCholeskyPreconditioner: inner factorisation failed");
  }
}

Mat PivotedCholesky::apply(const Mat& v) const {
  Mat out(v.rows, v.cols);
  if (achieved_rank_ == 0) {
    for (size_t e = 0; e < v.size(); ++e) out.a[e] = v.a[e] / noise_variance_;
    return out;
  }
  const int r = achieved_rank_, n = v.rows;
  Mat ltv(r, v.cols);
  for (int j = 0; j < v.cols; ++j)
    for (int k = 0; k < r; ++k) ltv(k, j) = col_dot(factor_, k, v, j);
  const Mat inner = small_.solve(ltv);
  for (int j = 0; j < v.cols; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k < r; ++k) acc += factor_(i, k) * inner(k, j);
      out(i, j) = (v(i, j) - acc) / noise_variance_;
    }
  return out;
}

// ===================== solvers.cpp:34-202 =================================
namespace {
using Clock = std::chrono::steady_clock;
void finalise(SolverReport& rep, const LinearSystemBatch& b, double tol, Clock::time_point start) {
  const TerminationStatus st = termination_check(b, tol);
  rep.mean_residual_norm = st.mean_norm;
  rep.probe_residual_norm = st.probe_norm;
  rep.reached_tolerance = st.done;
  rep.wall_seconds = std::chrono::duration<double>(Clock::now() - start).count();
}
}  // namespace

SolverReport solve_cg(LinearSystemBatch& batch, const SolverConfig& config, const PivotedCholesky* pc) {
  config.validate();
  const auto start = Clock::now();
  const int cols = batch.columns();
  SolverReport report;
  auto precondition = [&](const Mat& r) { return pc ? pc->apply(r) : r; };
  batch.refresh_residuals();
  Mat p = precondition(batch.residuals);
  Mat d = p;
  Vec gamma(cols);
  for (int j = 0; j < cols; ++j) gamma[j] = col_dot(batch.residuals, j, p, j);
  int t = 0;
  while (t < config.max_epochs && !termination_check(batch, config.tolerance).done) {
    const Mat hd = batch.op->apply(d);
    Vec alpha(cols);
    bool finite = true;
    for (int j = 0; j < cols; ++j) {
      const double denom = col_dot(d, j, hd, j);
      if (denom > 0.0) alpha[j] = gamma[j] / denom;
      else if (gamma[j] == 0.0 && denom == 0.0) alpha[j] = 0.0;
      else alpha[j] = std::numeric_limits<double>::quiet_NaN();
      finite = finite && std::isfinite(alpha[j]);
    }
    if (!finite) {
      report.aborted = true;
      report.abort_reason = "cg breakdown: non-finite step size";
      break;
    }
    for (int j = 0; j < cols; ++j) {
      double* v = batch.solutions.col(j);
      double* r = batch.residuals.col(j);
      const double* dj = d.col(j);
      const double* hj = hd.col(j);
      for (int i = 0; i < batch.targets.rows; ++i) {
        v[i] += dj[i] * alpha[j];
        r[i] -= hj[i] * alpha[j];
      }
    }
    p = precondition(batch.residuals);
    Vec gamma_next(cols), beta(cols);
    for (int j = 0; j < cols; ++j) gamma_next[j] = col_dot(batch.residuals, j, p, j);
    for (int j = 0; j < cols; ++j) beta[j] = gamma[j] != 0.0 ? gamma_next[j] / gamma[j] : 0.0;
    gamma = gamma_next;
    for (int j = 0; j < cols; ++j) {
      double* dj = d.col(j);
      const double* pj = p.col(j);
      for (int i = 0; i < batch.targets.rows; ++i) dj[i] = pj[i] + dj[i] * beta[j];
    }
    ++t;
  }
  report.iterations = t;
  report.epochs_consumed = static_cast<double>(t);
  finalise(report, batch, config.tolerance, start);
  return report;
}

SolverReport solve_ap(LinearSystemBatch& batch, const SolverConfig& config) {
  config.validate();
  const auto start = Clock::now();
  const int n = batch.op->size();
  const int block = std::min(config.block_size, n);
  const int num_blocks = (n + block - 1) / block;
  const int cols = batch.columns();
  SolverReport report;
  batch.refresh_residuals();
  Vec inv_scales(cols);
  for (int j = 0; j < cols; ++j) inv_scales[j] = 1.0 / batch.scales[j];
  std::vector<LLT> factors(num_blocks);
  std::vector<bool> have(num_blocks, false);
  auto bstart = [&](int k) { return k * block; };
  auto blen = [&](int k) { return std::min(block, n - k * block); };
  const double max_iterations = static_cast<double>(config.max_epochs) * n / block;
  int t = 0;
  while (t < max_iterations && !termination_check(batch, config.tolerance).done) {
    int selected = 0;
    double best = -1.0;
    for (int k = 0; k < num_blocks; ++k) {
      double acc = 0.0;
      for (int i = bstart(k); i < bstart(k) + blen(k); ++i) {
        double w = 0.0;
        for (int j = 0; j < cols; ++j) w += batch.residuals(i, j) * inv_scales[j];
        acc += w * w;
      }
      const double score = std::sqrt(acc);
      if (score > best) { best = score; selected = k; }
    }
    const int r0 = bstart(selected), len = blen(selected);
    if (!have[selected]) {
      factors[selected].compute(batch.op->dense_block(r0, len, r0, len));
      if (!factors[selected].ok)
        throw std::runtime_error("solve_ap: block Cholesky failed; block is not positive definite (noise scale too small)");
      have[selected] = true;
    }
    Mat rb(len, cols);
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < len; ++i) rb(i, j) = batch.residuals(r0 + i, j);
    const Mat update = factors[selected].solve(rb);
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < len; ++i) batch.solutions(r0 + i, j) += update(i, j);
    const Mat hu = batch.op->apply_columns(r0, len, update);
    for (size_t e = 0; e < hu.size(); ++e) batch.residuals.a[e] -= hu.a[e];
    ++t;
  }
  report.iterations = t;
  report.epochs_consumed = static_cast<double>(t) * block / n;
  finalise(report, batch, config.tolerance, start);
  return report;
}

SolverReport solve_sgd(LinearSystemBatch& batch, const SolverConfig& config,
                       std::vector<std::vector<int>>* batches_out, int record) {
  config.validate();
  const auto start = Clock::now();
  const int n = batch.op->size();
  const int b = std::min(config.batch_size, n);
  const int cols = batch.columns();
  SolverReport report;
  report.residuals_estimated = true;
  if (g_backend && g_backend->solve_sgd && g_backend->solve_sgd(batch, config, report, batches_out, record)) {
    finalise(report, batch, config.tolerance, start);
    return report;
  }
  batch.residuals = batch.targets;
  Mat momentum(n, cols);
  RandomStream rng(config.seed, streams::kSolver, config.substream);
  const double max_iterations = g_sgd_iteration_cap >= 0
                                    ? std::min<double>(g_sgd_iteration_cap, static_cast<double>(config.max_epochs) * n / b)
                                    : static_cast<double>(config.max_epochs) * n / b;
  const double step = config.learning_rate / b;
  int t = 0;
  while (t < max_iterations && !termination_check(batch, config.tolerance).done) {
    const std::vector<int> idx = rng.sample_without_replacement(n, b);
    if (batches_out && t < record) batches_out->push_back(idx);
    Mat g = batch.op->apply_rows(idx, batch.solutions);
    for (int j = 0; j < cols; ++j)
      for (int q = 0; q < b; ++q) g(q, j) -= batch.targets(idx[q], j);
    for (size_t e = 0; e < momentum.size(); ++e) momentum.a[e] *= config.momentum;
    for (int j = 0; j < cols; ++j)
      for (int q = 0; q < b; ++q) {
        const double upd = step * g(q, j);
        momentum(idx[q], j) -= upd;
      }
    for (size_t e = 0; e < momentum.size(); ++e) batch.solutions.a[e] += momentum.a[e];
    for (int j = 0; j < cols; ++j)
      for (int q = 0; q < b; ++q) batch.residuals(idx[q], j) = -g(q, j);
    ++t;
    if (!batch.solutions.all_finite()) {
      report.aborted = true;
      report.abort_reason = "sgd divergence: non-finite iterate";
      break;
    }
  }
  report.iterations = t;
  report.epochs_consumed = static_cast<double>(t) * b / n;
  finalise(report, batch, config.tolerance, start);
  return report;
}

SolverReport solve(LinearSystemBatch& batch, const SolverConfig& config) {
  switch (config.kind) {
    case CG:
      if (config.preconditioner_rank > 0) {
        PivotedCholesky pc(*batch.op, std::min(config.preconditioner_rank, batch.op->size()));
        return solve_cg(batch, config, &pc);
      }
      return solve_cg(batch, config, nullptr);
    case AP: return solve_ap(batch, config);
    case SGD: return solve_sgd(batch, config);
  }
  throw std::logic_error("solve: unknown solver kind");
}

// ===================== gradients.cpp:10-70 ================================
Mat gen_standard_probes(int n, int s, uint64_t seed, int distribution, uint64_t substream) {
  if (s < 1) throw std::invalid_argument("gen_standard_probes: s >= 1");
  Mat out(n, s);
  RandomStream stream(seed, streams::kProbes, substream);
  if (distribution == 1) stream.fill_rademacher(out.a.data(), out.size());
  else stream.fill_gaussian(out.a.data(), out.size());
  return out;
}

namespace {
GradientEstimate assemble(const KernelOperator& op, const Vec& v_y, const Mat& u, const Mat& w) {
  const int s = u.cols;
  Mat vy(static_cast<int>(v_y.size()), 1);
  vy.a = v_y;
  const auto forms = op.derivative_quadratic_forms_many({{&vy, &vy}, {&u, &w}});
  GradientEstimate e;
  e.quadratic_term = forms[0];
  e.trace_term = forms[1];
  for (double& x : e.trace_term) x /= s;
  e.values.resize(e.quadratic_term.size());
  for (size_t k = 0; k < e.values.size(); ++k)
    e.values[k] = 0.5 * e.quadratic_term[k] - 0.5 * e.trace_term[k];
  return e;
}
}  // namespace

GradientEstimate estimate_gradient_standard(const KernelOperator& op, const Vec& v_y,
                                            const Mat& solutions, const Mat& probes) {
  if (solutions.rows != op.size() || probes.rows != op.size() || solutions.cols != probes.cols)
    throw std::invalid_argument("estimate_gradient_standard: shape mismatch");
  return assemble(op, v_y, solutions, probes);
}

GradientEstimate estimate_gradient_pathwise(const KernelOperator& op, const Vec& v_y, const Mat& zhat) {
  if (zhat.rows != op.size()) throw std::invalid_argument("estimate_gradient_pathwise: shape mismatch");
  return assemble(op, v_y, zhat, zhat);
}

// ===================== rff.cpp:10-79 =====================================
RffBasis build_rff_basis(int d, int m_pairs, int sample_count, uint64_t seed, uint64_t substream) {
  if (m_pairs < 1) throw std::invalid_argument("build_rff_basis: m_pairs >= 1");
  if (sample_count < 1) throw std::invalid_argument("build_rff_basis: sample_count >= 1");
  RffBasis basis;
  basis.seed = seed;
  basis.base_frequencies = Mat(m_pairs, d);
  RandomStream fs(seed, streams::kFrequencies, substream);
  for (int p = 0; p < m_pairs; ++p) {
    double chi2 = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double g = fs.next_gaussian();
      chi2 += g * g;
    }
    const double scale = std::sqrt(3.0 / chi2);
    for (int k = 0; k < d; ++k) basis.base_frequencies(p, k) = scale * fs.next_gaussian();
  }
  basis.weights = Mat(2 * m_pairs, sample_count);
  RandomStream ws(seed, streams::kWeights, substream);
  ws.fill_gaussian(basis.weights.a.data(), basis.weights.size());
  return basis;
}

Mat rff_features(const RffBasis& basis, const Hyper& hp, const Mat& points) {
  const int P = basis.pairs(), d = basis.base_frequencies.cols;
  if (points.cols != d) throw std::invalid_argument("rff_features: point dimension does not match basis");
  const Vec ls = hp.lengthscales();
  Mat freq(P, d);
  for (int p = 0; p < P; ++p)
    for (int k = 0; k < d; ++k) freq(p, k) = basis.base_frequencies(p, k) * (1.0 / ls[k]);
  const double amplitude = hp.signal_scale() / std::sqrt(static_cast<double>(P));
  Mat features(points.rows, 2 * P);
  for (int i = 0; i < points.rows; ++i)
    for (int p = 0; p < P; ++p) {
      double angle = 0.0;
      for (int k = 0; k < d; ++k) angle += points(i, k) * freq(p, k);
      features(i, 2 * p) = amplitude * std::cos(angle);
      features(i, 2 * p + 1) = amplitude * std::sin(angle);
    }
  return features;
}

// Streams over row blocks so Phi is never materialised beyond 1024 rows
// (identical values: every element is an ascending-feature dot product).
PathwiseTargets pathwise_targets(const RffBasis& basis, const Hyper& hp, const Dataset& data, int s,
                                 uint64_t seed, uint64_t substream) {
  if (s < 1) throw std::invalid_argument("pathwise_targets: s >= 1");
  if (s > basis.weights.cols) throw std::invalid_argument("pathwise_targets: basis holds fewer samples than requested");
  const int n = data.n(), d = data.dim(), F = 2 * basis.pairs();
  PathwiseTargets t;
  t.prior_values = Mat(n, s);
  const int RB = 1024;
  const bool dev = g_backend && g_backend->prior && g_backend->prior(basis, hp, data, s, t.prior_values);
  for (int r0 = dev ? n : 0; r0 < n; r0 += RB) {
    const int rows = std::min(RB, n - r0);
    Mat pts(rows, d);
    for (int i = 0; i < rows; ++i)
      for (int k = 0; k < d; ++k) pts(i, k) = data.inputs(r0 + i, k);
    const Mat feat = rff_features(basis, hp, pts);
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int q = 0; q < F; ++q) acc += feat(i, q) * basis.weights(q, j);
        t.prior_values(r0 + i, j) = acc;
      }
  }
  t.noise = Mat(n, s);
  RandomStream ns(seed, streams::kNoiseDraws, substream);
  ns.fill_gaussian(t.noise.a.data(), t.noise.size());
  t.xi = Mat(n, s);
  const double sigma = hp.noise_scale();
  for (size_t e = 0; e < t.xi.size(); ++e) t.xi.a[e] = t.prior_values.a[e] + sigma * t.noise.a[e];
  return t;
}

// ===================== posterior =========================================
// kernel.cpp:57-81: ps = P diag(1/l), xs = X diag(1/l); row i of k(P, X) from
// the squared distances; products accumulate in ascending training index.
Mat cross_kernel_apply(const Mat& points, const Mat& inputs, const Hyper& hp, const Mat& v, int block_rows,
                       int threads) {
  const int p = points.rows, n = inputs.rows, d = inputs.cols, m = v.cols;
  if (points.cols != d) throw std::invalid_argument("predict_mean: point dimension mismatch");
  const Vec ls = hp.lengthscales();
  Vec inv(d);
  for (int k = 0; k < d; ++k) inv[k] = 1.0 / ls[k];
  const double s2 = hp.signal_scale() * hp.signal_scale();
  std::vector<double> xs(static_cast<size_t>(n) * d), ps(static_cast<size_t>(p) * d);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) xs[static_cast<size_t>(i) * d + k] = inputs(i, k) * inv[k];
  for (int i = 0; i < p; ++i)
    for (int k = 0; k < d; ++k) ps[static_cast<size_t>(i) * d + k] = points(i, k) * inv[k];
  Mat out(p, m);
  (void)block_rows;  // per-row results do not depend on the tile height
  parallel_for(threads, p, [&](int, int i) {
    std::vector<double> row(n);
    const double* pi = &ps[static_cast<size_t>(i) * d];
    for (int c = 0; c < n; ++c) {
      const double* xc = &xs[static_cast<size_t>(c) * d];
      double r2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double t = xc[k] - pi[k];
        r2 += t * t;
      }
      row[c] = matern_profile(r2, s2);
    }
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int c = 0; c < n; ++c) acc += row[c] * v(c, j);
      out(i, j) = acc;
    }
  });
  return out;
}

Mat evaluate_prior_all(const RffBasis& basis, const Hyper& hp, const Mat& points, int s) {  // rff.cpp:56-62
  const Mat feat = rff_features(basis, hp, points);
  const int F = feat.cols;
  Mat out(points.rows, s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < points.rows; ++i) {
      double acc = 0.0;
      for (int q = 0; q < F; ++q) acc += feat(i, q) * basis.weights(q, j);
      out(i, j) = acc;
    }
  return out;
}

Mat sample_posterior_all(const Mat& prior, const Mat& points, const Mat& inputs, const Hyper& hp, const Vec& v_y,
                         const Mat& zhat, int threads) {  // posterior.cpp:19-27
  const int n = inputs.rows, s = zhat.cols;
  Mat corr(n, s);
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < n; ++i) corr(i, j) = v_y[i] - zhat(i, j);
  Mat out = cross_kernel_apply(points, inputs, hp, corr, 1024, threads);
  if (prior.size())
    for (size_t e = 0; e < out.size(); ++e) out.a[e] = prior.a[e] + out.a[e];
  return out;
}

TestMetrics test_metrics(const Mat& prior, const Mat& points, const Vec& targets, const Mat& inputs, const Hyper& hp,
                         const Vec& v_y, const Mat& zhat, double target_scale, int threads) {  // posterior.cpp:29-59
  const int p = points.rows, n = inputs.rows;
  Mat vy(n, 1);
  vy.a = v_y;
  const Mat mean = cross_kernel_apply(points, inputs, hp, vy, 1024, threads);
  TestMetrics mt;
  double se = 0.0;
  Vec err(p);
  for (int i = 0; i < p; ++i) {
    err[i] = targets[i] - mean.a[i];
    se += err[i] * err[i];
  }
  mt.rmse = std::sqrt(se / p);
  mt.rmse_raw = mt.rmse * target_scale;
  const int s = zhat.cols;
  if (s >= 2 && prior.size()) {
    const Mat samples = sample_posterior_all(prior, points, inputs, hp, v_y, zhat, threads);
    const double noise_var = hp.noise_variance();
    double llh = 0.0;
    for (int i = 0; i < p; ++i) {
      double mu = 0.0;
      for (int j = 0; j < s; ++j) mu += samples(i, j);
      mu /= s;
      double var = 0.0;
      for (int j = 0; j < s; ++j) var += (samples(i, j) - mu) * (samples(i, j) - mu);
      var = var / (s - 1) + noise_var;
      llh += -0.5 * std::log(2.0 * kPi * var) - 0.5 * err[i] * err[i] / var;
    }
    mt.llh = llh / p;
    mt.llh_raw = mt.llh - std::log(target_scale);
    mt.has_llh = true;
  }
  return mt;
}

// ===================== outer_loop.cpp:39-246 ===============================
namespace {
struct Adam {
  Vec m, v;
  int step = 0;
  double lr, b1 = 0.9, b2 = 0.999, eps = 1e-8;
  Adam(int dim, double lr_) : m(dim, 0.0), v(dim, 0.0), lr(lr_) {}
  Vec update(const Vec& g) {  // outer_loop.cpp:42-49
    ++step;
    Vec out(g.size());
    const double ms = 1.0 / (1.0 - std::pow(b1, step));
    const double vs = 1.0 / (1.0 - std::pow(b2, step));
    for (size_t i = 0; i < g.size(); ++i) {
      m[i] = b1 * m[i] + (1.0 - b1) * g[i];
      v[i] = b2 * v[i] + (1.0 - b2) * (g[i] * g[i]);
      out[i] = (-lr) * (ms * m[i] / (std::sqrt(vs * v[i]) + eps));
    }
    return out;
  }
};
}  // namespace

PathwiseTargets pathwise_targets_from_prior(const Mat& prior_values, const Hyper& hp, uint64_t seed,
                                            uint64_t substream) {  // rff.cpp:81-91
  PathwiseTargets t;
  t.prior_values = prior_values;
  t.noise = Mat(prior_values.rows, prior_values.cols);
  RandomStream ns(seed, streams::kNoiseDraws, substream);
  ns.fill_gaussian(t.noise.a.data(), t.noise.size());
  t.xi = Mat(prior_values.rows, prior_values.cols);
  const double sigma = hp.noise_scale();
  for (size_t e = 0; e < t.xi.a.size(); ++e) t.xi.a[e] = t.prior_values.a[e] + sigma * t.noise.a[e];
  return t;
}

Mat jittered_kernel_cholesky(const Mat& kernel_matrix) {  // exact.cpp:52-61
  const int n = kernel_matrix.rows;
  double mean_diag = 0.0;
  for (int i = 0; i < n; ++i) mean_diag += kernel_matrix(i, i);
  mean_diag /= n;
  for (double jitter = 1e-10; jitter <= 1.0000001e-6; jitter *= 10.0) {
    Mat attempt = kernel_matrix;
    for (int i = 0; i < n; ++i) attempt(i, i) += jitter * mean_diag;
    LLT llt;
    llt.compute(attempt);
    if (llt.ok) return llt.L;
  }
  throw std::runtime_error("jittered_kernel_cholesky: factorisation failed beyond 1e-6 jitter");
}

Mat exact_dense_prior(const KernelOperator& op, const Hyper& hp, const Mat& weights) {
  const int n = op.size(), s = weights.cols;
  Mat kernel_matrix = op.dense_block(0, n, 0, n);
  for (int i = 0; i < n; ++i) kernel_matrix(i, i) -= hp.noise_variance();
  const Mat chol = jittered_kernel_cholesky(kernel_matrix);
  Mat prior(n, s);  // chol * weights (lower triangular)
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k <= i; ++k) acc += chol(i, k) * weights(k, j);
      prior(i, j) = acc;
    }
  return prior;
}

OuterResult optimise(const Dataset& train, const OuterConfig& config, int threads, int block_rows) {
  const int n = train.n(), d = train.dim(), s = config.probe_count;
  config.solver.validate();
  if (config.steps < 0) throw std::invalid_argument("optimise: steps >= 0");
  OuterResult result;
  Vec raw = config.init_constrained.empty() ? Hyper::constant(d, config.init_value).raw
                                            : Hyper::from_constrained(config.init_constrained).raw;
  Adam adam(d + 2, config.learning_rate);
  SolverConfig sc = config.solver;
  sc.warm_start = config.warm_start;
  bool sgd_halved = false;
  const bool pathwise = config.estimator == 1;
  bool have_basis = false;
  RffBasis basis;
  Mat probes;
  Mat exact_prior_weights;  // n x s, fixed draws for the ExactDense prior
  Mat previous;
  bool have_previous = false;
  for (int t = 0; t < config.steps; ++t) {
    const Hyper hp = Hyper::from_raw(raw);
    KernelOperator op(&train, hp, block_rows, threads);
    const uint64_t substream = config.warm_start ? 0 : static_cast<uint64_t>(t);
    Mat probe_targets;
    if (pathwise) {
      if (!have_basis || !config.warm_start) {
        basis = build_rff_basis(d, config.rff_pairs, s, config.feature_seed, substream);
        have_basis = true;
      }
      if (config.prior_mode == 0) {
        probe_targets = pathwise_targets(basis, hp, train, s, config.feature_seed, substream).xi;
      } else {  // ExactDense (outer_loop.cpp:140-153)
        if (n > kDefaultDenseCap) throw std::invalid_argument("optimise: exact prior draws need n within the dense cap");
        if (exact_prior_weights.size() == 0 || !config.warm_start) {
          RandomStream stream(config.feature_seed, streams::kPriorSample, substream);
          exact_prior_weights = Mat(n, s);
          stream.fill_gaussian(exact_prior_weights.a.data(), exact_prior_weights.size());
        }
        probe_targets = pathwise_targets_from_prior(exact_dense_prior(op, hp, exact_prior_weights), hp,
                                                    config.feature_seed, substream).xi;
      }
    } else {
      if (probes.size() == 0 || !config.warm_start)
        probes = gen_standard_probes(n, s, config.probe_seed, config.probe_distribution, substream);
      probe_targets = probes;
    }
    Mat bt(n, probe_targets.cols + 1);
    std::copy(train.targets.begin(), train.targets.end(), bt.col(0));
    std::copy(probe_targets.a.begin(), probe_targets.a.end(), bt.col(1));
    LinearSystemBatch batch(op, std::move(bt));
    if (config.warm_start && have_previous) batch.warm_start(previous);
    sc.substream = static_cast<uint64_t>(t);
    sc.seed = config.solver_seed;
    const SolverReport report = solve(batch, sc);
    TraceRow row;
    row.step = t;
    row.constrained = hp.constrained();
    row.mean_residual_norm = report.mean_residual_norm;
    row.probe_residual_norm = report.probe_residual_norm;
    row.epochs = report.epochs_consumed;
    row.iterations = report.iterations;
    row.solver_diverged = report.aborted;
    if (report.aborted) {
      if (config.divergence_policy == 1) {
        result.aborted = true;
        result.abort_reason = report.abort_reason;
        result.trace.push_back(row);
        break;
      }
      if (sc.kind == SGD && !sgd_halved) {
        sc.learning_rate *= 0.5;
        sgd_halved = true;
      }
    } else {
      Vec v_y(batch.solutions.col(0), batch.solutions.col(0) + n);
      Mat zhat(n, batch.columns() - 1);
      std::copy(batch.solutions.col(1), batch.solutions.col(1) + zhat.size(), zhat.a.begin());
      GradientEstimate g;
      if (pathwise) {
        g = estimate_gradient_pathwise(op, v_y, zhat);
      } else {
        Mat pt(n, batch.columns() - 1);
        std::copy(batch.targets.col(1), batch.targets.col(1) + pt.size(), pt.a.begin());
        g = estimate_gradient_standard(op, v_y, zhat, pt);
      }
      double inf = 0.0;
      for (double x : g.values) inf = std::max(inf, std::abs(x));
      row.grad_inf_norm = inf;
      row.gradient = g.values;
      Vec neg_raw_grad(raw.size());
      for (size_t k = 0; k < raw.size(); ++k) neg_raw_grad[k] = -(g.values[k] * sigmoid(raw[k]));
      const Vec upd = adam.update(neg_raw_grad);
      for (size_t k = 0; k < raw.size(); ++k) raw[k] += upd[k];
      previous = batch.solutions;
      have_previous = true;
    }
    result.trace.push_back(row);
  }
  result.hp = Hyper::from_raw(raw);
  return result;
}

// ===================== exact.cpp:11-50 ====================================
DenseProblem build_dense_problem(const Dataset& data, const Hyper& hp) {
  KernelOperator op(&data, hp);
  DenseProblem dp;
  dp.hp = hp;
  const int n = data.n();
  dp.h = op.dense_block(0, n, 0, n);
  dp.chol.compute(dp.h);
  if (!dp.chol.ok) throw std::runtime_error("build_dense_problem: H is not positive definite");
  Mat eye(n, n);
  for (int i = 0; i < n; ++i) eye(i, i) = 1.0;
  for (int k = 0; k < hp.count(); ++k) dp.dh.push_back(op.derivative_apply(k, eye));
  return dp;
}

double exact_mll(const DenseProblem& dp, const Vec& y) {
  const int n = dp.h.rows;
  Mat ym(n, 1);
  ym.a = y;
  const Mat alpha = dp.chol.solve(ym);
  double logdet = 0.0, quad = 0.0;
  for (int i = 0; i < n; ++i) logdet += std::log(dp.chol.L(i, i));
  logdet *= 2.0;
  for (int i = 0; i < n; ++i) quad += y[i] * alpha.a[i];
  return -0.5 * quad - 0.5 * logdet - 0.5 * n * std::log(2.0 * kPi);
}

Vec exact_gradient(const DenseProblem& dp, const Vec& y) {
  const int n = dp.h.rows;
  Mat ym(n, 1);
  ym.a = y;
  const Mat alpha = dp.chol.solve(ym);
  Vec grad(dp.hp.count());
  for (size_t k = 0; k < dp.dh.size(); ++k) {
    const Mat solved = dp.chol.solve(dp.dh[k]);
    double tr = 0.0, q = 0.0;
    for (int i = 0; i < n; ++i) tr += solved(i, i);
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int c = 0; c < n; ++c) acc += dp.dh[k](i, c) * alpha.a[c];
      q += alpha.a[i] * acc;
    }
    grad[k] = 0.5 * q - 0.5 * tr;
  }
  return grad;
}

// ===================== BASELINE sin-sum generator =========================
void make_sinsum_dataset(int n, int d, bool uniform, double noise, uint64_t seed,
                         std::vector<float>& x_rowmajor, std::vector<float>& y) {
  std::vector<double> x(static_cast<size_t>(n) * d);  // col-major fill order
  RandomStream xs(seed, streams::kSynthetic, 0);
  if (uniform) {
    for (size_t e = 0; e < x.size(); ++e) x[e] = 2.0 * xs.next_double() - 1.0;
  } else {
    xs.fill_gaussian(x.data(), x.size());
  }
  std::vector<double> w(static_cast<size_t>(d) * 4);  // d x 4 col-major
  RandomStream ws(seed, streams::kSynthetic, 1);
  ws.fill_gaussian(w.data(), w.size());
  const double wscale = 1.0 / std::sqrt(static_cast<double>(d));
  std::vector<double> eps(n);
  RandomStream es(seed, streams::kSynthetic, 2);
  es.fill_gaussian(eps.data(), eps.size());
  std::vector<double> yy(n);
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int k = 0; k < 4; ++k) {
      double dot = 0.0;
      for (int q = 0; q < d; ++q) dot += x[static_cast<size_t>(q) * n + i] * (w[static_cast<size_t>(k) * d + q] * wscale);
      acc += std::sin(dot);
    }
    yy[i] = acc + noise * eps[i];
  }
  // Standardise features and targets (data_io.cpp:148-168, train = all rows).
  x_rowmajor.resize(static_cast<size_t>(n) * d);
  for (int q = 0; q < d; ++q) {
    double mean = 0.0;
    for (int i = 0; i < n; ++i) mean += x[static_cast<size_t>(q) * n + i];
    mean /= n;
    double var = 0.0;
    for (int i = 0; i < n; ++i) {
      const double t = x[static_cast<size_t>(q) * n + i] - mean;
      var += t * t;
    }
    var /= n;
    double scale = std::sqrt(var);
    if (!(scale > 0.0)) scale = 1.0;
    const double inv = 1.0 / scale;
    for (int i = 0; i < n; ++i)
      x_rowmajor[static_cast<size_t>(i) * d + q] = static_cast<float>((x[static_cast<size_t>(q) * n + i] - mean) * inv);
  }
  double mean = 0.0;
  for (double v : yy) mean += v;
  mean /= n;
  double var = 0.0;
  for (double v : yy) var += (v - mean) * (v - mean);
  var /= n;
  const double scale = var > 0.0 ? std::sqrt(var) : 1.0;
  y.resize(n);
  for (int i = 0; i < n; ++i) y[i] = static_cast<float>((yy[i] - mean) / scale);
}

ExactTrajectory optimise_exact(const Dataset& data, const Hyper& init, int steps, double learning_rate) {
  ExactTrajectory tr;  // outer_loop.cpp:248-262
  Vec raw = init.raw;
  Adam adam(static_cast<int>(raw.size()), learning_rate);
  for (int t = 0; t < steps; ++t) {
    const Hyper hp = Hyper::from_raw(raw);
    tr.constrained_per_step.push_back(hp.constrained());
    const DenseProblem dense = build_dense_problem(data, hp);
    const Vec grad = exact_gradient(dense, data.targets);
    Vec neg(raw.size());
    for (size_t k = 0; k < raw.size(); ++k) neg[k] = -(grad[k] * sigmoid(raw[k]));
    const Vec upd = adam.update(neg);
    for (size_t k = 0; k < raw.size(); ++k) raw[k] += upd[k];
  }
  tr.hp = Hyper::from_raw(raw);
  return tr;
}

Hyper init_heuristic(const Dataset& data, int n_centroids, int subset, uint64_t seed, int adam_steps,
                     double learning_rate) {  // outer_loop.cpp:264-296
  const int n = data.n(), d = data.dim();
  const Hyper init = Hyper::constant(d, 1.0);
  if (subset >= n) return optimise_exact(data, init, adam_steps, learning_rate).hp;
  RandomStream stream(seed, streams::kCentroids, 0);
  Vec acc(d + 2, 0.0);
  for (int c = 0; c < n_centroids; ++c) {
    const int centroid = static_cast<int>(stream.next_below(static_cast<uint64_t>(n)));
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> dist2(n);
    for (int i = 0; i < n; ++i) {
      double s2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double t = data.inputs(i, k) - data.inputs(centroid, k);
        s2 += t * t;
      }
      dist2[i] = s2;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dist2[a] < dist2[b]; });
    Dataset local;
    local.inputs = Mat(subset, d);
    local.targets.assign(subset, 0.0);
    for (int i = 0; i < subset; ++i) {
      for (int k = 0; k < d; ++k) local.inputs(i, k) = data.inputs(order[i], k);
      local.targets[i] = data.targets[order[i]];
    }
    const Vec fitted = optimise_exact(local, init, adam_steps, learning_rate).hp.constrained();
    for (int k = 0; k < d + 2; ++k) acc[k] += fitted[k];
  }
  Vec mean(d + 2);
  for (int k = 0; k < d + 2; ++k) mean[k] = acc[k] / n_centroids;
  return Hyper::from_constrained(mean);
}

}  // namespace oracle
