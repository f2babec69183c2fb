// Host C++ of libgpk: the C-ABI (include/gpk.h) over device-resident solver
// state. Mirrors the reference's KernelOperator / LinearSystemBatch / solvers
// / estimators / optimise (/root/reference/proj/core/src/*.cpp), with all
// n-sized state on the GPU and only d+2-sized scalars (Adam, hyperparameters)
// on the host.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gpk.h"
#include "gpk_internal.cuh"
#include "philox.cuh"

namespace gpk {
thread_local long long* g_launch_counter = nullptr;
}

using namespace gpk;

namespace {

thread_local std::string g_err;

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
  using std::out_of_range::out_of_range;
};

// Device buffers come from the device's default stream-ordered pool with an
// unbounded release threshold: freed blocks stay mapped and are handed to the
// next allocation of the process, so creating / destroying operators, batches
// and optimisers (every gpk_optimise call) costs no cudaMalloc/cudaFree
// page-table work. A free first waits for the device (the old cudaFree's
// implicit synchronisation, without the unmap), an allocation is ordered on
// the legacy stream and waited for, so no stream ever touches a block another
// stream still uses. GPK_DEVICE_POOL=0 restores cudaMalloc/cudaFree.
bool device_pool_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GPK_DEVICE_POOL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// Reference dense_cache_cap (outer_loop.hpp:60): the optimiser's operators
// with n <= 4096 keep the FP64 kernel matrix (operators created through the
// operator API do not, as KernelOperatorOptions::dense_cache defaults to
// false); GPK_DENSE_CAP overrides (0: never).
int dense_cache_cap() {
  static const int cap = [] {
    const char* e = std::getenv("GPK_DENSE_CAP");
    return e ? std::atoi(e) : 4096;
  }();
  return cap;
}

// n <= dense_cache_cap: FP64 products, as the reference computes them there
// (outer_loop.cpp:72 caches H in FP64). Default: the FP64 on-the-fly
// operator kv64v2_kernel, which never materialises H (entries evaluated in
// FP64 and contracted in registers); GPK_DENSE_KV64=0 keeps the reference's
// cached FP64 kernel matrix and applies it by cuBLAS DGEMM instead.
bool dense_dgemm() {
  static const bool on = [] {
    const char* e = std::getenv("GPK_DENSE_KV64");
    return e && std::atoi(e) == 0;
  }();
  return on;
}

// Tensor-core Gram distances for d >= GPK_TGRAM_MIN_D (default 9; measured
// on one B200 with the warp-uniform MMA issue, full products: d = 11 -16%,
// d = 13 -24% (C5's product 145 -> 122 ms at n = 262144), d = 20/26 on by
// then already; round 1 with per-MMA elect issue: d = 11 +2%, d = 3 +16%);
// GPK_TGRAM=0 keeps the FP32 distance loops everywhere.
bool tg_enabled(int d) {
  static const int min_d = [] {
    const char* e = std::getenv("GPK_TGRAM");
    if (e && std::atoi(e) == 0) return 1 << 30;
    const char* m = std::getenv("GPK_TGRAM_MIN_D");
    return m ? std::atoi(m) : 9;
  }();
  return d >= min_d && d <= 32;
}

void* device_alloc(size_t bytes) {
  void* p = nullptr;
  if (!device_pool_enabled()) {
    GPK_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  static std::array<bool, 64> configured{};
  int dev = 0;
  GPK_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !configured[dev]) {
    cudaMemPool_t pool;
    GPK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    GPK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured[dev] = true;
  }
  GPK_CUDA(cudaMallocAsync(&p, bytes, 0));
  GPK_CUDA(cudaStreamSynchronize(0));
  return p;
}

void device_free(void* p) {
  if (!p) return;
  if (!device_pool_enabled()) {
    cudaFree(p);
    return;
  }
  cudaDeviceSynchronize();
  cudaFreeAsync(p, 0);
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { device_free(p); }
  T* ensure(size_t count) {
    if (count > cap) {
      device_free(p);
      p = nullptr;
      p = static_cast<T*>(device_alloc(std::max<size_t>(count, 1) * sizeof(T)));
      cap = count;
    }
    return p;
  }
};

double softplus(double x) {  // hyperparameters.cpp:8-11
  if (x > 0.0) return x + std::log1p(std::exp(-x));
  return std::log1p(std::exp(x));
}
double softplus_inverse(double y) {  // hyperparameters.cpp:13-17
  if (y <= 0.0) throw InvalidArgument("softplus_inverse: argument must be positive");
  return y + std::log(-std::expm1(-y));
}
double sigmoid(double x) {  // hyperparameters.cpp:19-23
  if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}

}  // namespace

constexpr size_t kBlasWorkspace = 32u << 20;

struct gpk_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  long long launches = 0;
  CgCtl* ctl_host = nullptr;  // pinned, 2 slots
  cudaEvent_t ev[2]{};
  double* stats = nullptr;    // device [evals x RHS, flops]
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof;  // K.V launch brackets
  size_t prof_used = 0;
  int kernel = 1;  // operator kernel: 0 SIMT FP32, 1 tcgen05 3xTF32 (default)
  bool fused_ap = true;  // AP slabs: reduce + epilogue fused into the tcgen05 kernel
  int spd_inverse = 1;   // AP block inverses: 1 recursive Schur/DGEMM, 0 cuSOLVER potrf + 2 trsm
  bool ap_persistent = true;  // AP iterations in one cooperative launch (GPK_AP_PERSISTENT=0 disables)
  int kv_deep = -1;  // operator launches one CTA per SM with 16 eval warps: -1 auto (>= 1e8 entries), 0/1 forced
  bool kv_streamk = false;  // deep launches as stream-K (GPK_KV_STREAMK=1); measured 1-7% slower than the 2-D grid
  bool graphs = true;  // CG/AP iteration groups as CUDA graphs (GPK_GRAPHS=0 disables)
  bool sgd_lazy = true;  // SGD: lazily evaluated momentum + sgd_slab_kernel (GPK_SGD_LAZY=0: full-state passes)
  void* blas_ws = nullptr;  // cuBLAS workspace (graph capture)
  DBuf<double*> ptr_a, ptr_b;  // batched-factorisation pointer arrays
  DBuf<int> info;
  DBuf<double> rff_feat;  // RFF feature rows (prior GEMM), reused across calls
  int* info_host = nullptr;    // pinned
  // auxiliary stream: AP block factorisation runs here, overlapped with the
  // pathwise targets and the residual refresh on the main stream
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_m2a = nullptr, ev_aux = nullptr;
  ncclComm_t comm = nullptr;   // multi-GPU (one process per GPU)
  int nranks = 1, rank = 0;
  // ring all-gather of the sharded operator's RHS on its own stream, one event
  // per received slice (apply_local)
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ring_ev;
  cudaEvent_t ring_start = nullptr;
  bool ring_gather = true;  // GPK_RING_GATHER=0: one all-gather, then one operator launch
};

struct gpk_operator {
  gpk_ctx* ctx = nullptr;
  // row shard owned by this rank (nr == 1: the whole problem). Only operators
  // built by the sharded optimiser have nr > 1.
  int nr = 1, rk = 0, row0 = 0, nloc = 0, S = 0;
  bool sharded = false;  // built by the optimiser on a context with a communicator
  uint64_t hyper_version = 0;  // bumped by every set_hyper (AP block inverses are keyed on it)
  DBuf<double> hyp_dev;        // {s2, sigma2} on the device (graph-replayable AP block build)
  // gradient-pass workspace (persistent across steps)
  DBuf<float> gbuf[4];
  DBuf<double> gpart, gtot, gdots;
  DBuf<float> gpk_b, gpk_n;  // tensor-core gradient pass: packed W images, narrow-pair vectors
  int n = 0, d = 0, dp = 0;
  DBuf<double> x64;       // [n][d] unscaled
  DBuf<float> xs32;       // [n][dp]
  DBuf<float> gpk_xsoa;   // gradient pass, d <= 4: SoA image of xs32 per 32-row chunk
  int dpg = 0;            // Gram image width (gram_dp(d)); 0: direct-difference operator
  bool tg = false;        // tensor-core Gram distances in the tcgen05 operator (tg_enabled)
  DBuf<float> xtg;        // their column images (tg_image_launch), rebuilt with the scaled inputs
  // dense FP64 kernel matrix K (no noise) for n <= dense_cache_cap, as the
  // reference caches H for small problems (kernel.cpp:83-109,
  // outer_loop.cpp:72); full unsharded products then run as one DGEMM
  bool dense = false;
  DBuf<double> kdense;
  DBuf<float> xg32;       // [n + 128][dpg] (x, |x|^2, 0...) for the tensor-core operator
  DBuf<double> xs64;      // [n][d]
  DBuf<double> inv_ls_dev;
  std::vector<double> raw, inv_ls;
  double s = 1, s2 = 1, sigma = 1, sigma2 = 1;
  DBuf<double> part;      // kv split partials
  DBuf<float> vpk;        // packed TF32 hi/lo RHS images (tcgen05 path)
  DBuf<float> v32g;       // sharded products: the all-gathered FP32 RHS [S nr][m]
  DBuf<double> pts64, pts64s;  // posterior query points FP64 [p][d] (raw, scaled)
  DBuf<float> pts32;           // and scaled FP32 [p + 32][dp]
  DBuf<float> ptsg32;          // and their Gram image [p + 32][dpg]
  // scratch for host-facing calls
  DBuf<float> v32;
  DBuf<double> v64, out64, tmp64;
  DBuf<int> idx;
};

struct gpk_precond {
  gpk_operator* op = nullptr;
  int n = 0, rank = 0, achieved = 0, stopped = 0;
  DBuf<double> L;      // [n][rank] row-major
  DBuf<double> minv;   // [r][r]
  DBuf<int> pivots;
  double sigma2 = 1;
  DBuf<double> part, T, inner;
  DBuf<double> diag, pval, gpart, gram;
  DBuf<int> pidx, stop;
};

struct gpk_batch {
  gpk_operator* op = nullptr;
  int n = 0, m = 0;
  DBuf<double> targets, solutions, residuals;
  std::vector<double> scales;
  bool scales_stale = false;  // scales_dev newer than the host copy (device-computed in the optimiser)
  DBuf<double> scales_dev;
  // solver workspace
  DBuf<double> w1, w2, w3, w4, w5, red, vec1, vec2, vec3;
  DBuf<float> f32;
  DBuf<CgCtl> ctl;
  DBuf<int> ibuf, ibuf2, flag;
  DBuf<double> blocks;
  std::unique_ptr<gpk_precond> pc;  // dispatch-built preconditioner, reused across solves
  DBuf<unsigned> ticket;             // last-block ticket of fused reductions (kept at 0 between uses)
  DBuf<float> apk;                   // AP block update's TF32 operator images
  DBuf<double> spart_t;              // fused AP slabs: block-score partial per 128-row tile
  // lazy-momentum SGD (sgd_lazy.cu): FP32 records, last-update iterations,
  // S / rho^Delta tables, slab partials, apply-block partials, flags
  DBuf<float> sgd_rec, sgd_s32, sgd_xg, sgd_xsoa;
  DBuf<double> sgd_gpart2;  // fused SGD finish: per-block g^2 and old R^2 partials
  DBuf<int> sgd_tau, sgd_flags;
  DBuf<double> sgd_tab, sgd_part, sgd_gpart;
  DBuf<unsigned> gbar;               // persistent AP: grid-barrier counter
  DBuf<double> ap_cpart;             // persistent AP: block-update partials [8][block][m]
  DBuf<unsigned long long> ap_prof;  // persistent AP development phase clock (GPK_AP_PROF)
  // CUDA graph of the AP block build + inverse (ap_prepare), keyed on its buffers
  cudaGraphExec_t ap_graph = nullptr;
  std::array<const void*, 6> ap_graph_key{};
  std::pair<int, int> ap_graph_dims{0, 0};
  long long ap_graph_launches = 0;
  ~gpk_batch() {
    if (ap_graph) cudaGraphExecDestroy(ap_graph);
  }
  // AP block inverses enqueued on the auxiliary stream (ap_prepare)
  bool ap_ready = false;
  int ap_block = 0;
  uint64_t ap_version = 0;
};

struct gpk_rff_basis {
  gpk_ctx* ctx = nullptr;
  int d = 0, pairs = 0, samples = 0;
  uint64_t seed = 0, substream = 0;
  std::vector<double> freq;     // P x d col-major (host, exact)
  std::vector<double> weights;  // 2P x S col-major
  DBuf<double> w_dev, freq_dev;
};

namespace {

struct LaunchScope {
  explicit LaunchScope(gpk_ctx* c) {
    prev = g_launch_counter;
    g_launch_counter = &c->launches;
    GPK_CUDA(cudaSetDevice(c->device));
  }
  ~LaunchScope() { g_launch_counter = prev; }
  long long* prev;
};

template <class F>
gpk_status guarded(F&& f) {
  try {
    f();
    return GPK_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return GPK_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return GPK_ERANGE;
  } catch (const CudaError& e) {
    g_err = e.what();
    return GPK_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GPK_ENUMERIC;
  }
}

// NCCL is resolved at run time (dlopen) so libgpk carries no link-time NCCL
// dependency: a process that already loaded one (e.g. PyTorch's bundled
// libnccl.so.2) shares it, otherwise the system library is loaded.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error(std::string("gpk: cannot load libnccl.so.2: ") + dlerror());
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_gather || !a.all_reduce || !a.send ||
        !a.recv || !a.group_start || !a.group_end || !a.error_string)
      throw std::runtime_error("gpk: libnccl.so.2 lacks required symbols");
    return a;
  }();
  return api;
}

// In-place all-gather of equal per-rank slices (no-op on one rank).
void gather_inplace(gpk_operator* op, void* buf, size_t bytes_per_rank) {
  if (!op->sharded) return;  // (a 1-rank communicator still issues the in-place all-gather)
  gpk_ctx* ctx = op->ctx;
  char* b = static_cast<char*>(buf);
  const ncclResult_t r = nccl().all_gather(b + static_cast<size_t>(op->rk) * bytes_per_rank, b, bytes_per_rank,
                                           ncclChar, ctx->comm, ctx->stream);
  if (r != ncclSuccess) throw std::runtime_error(std::string("ncclAllGather: ") + nccl().error_string(r));
  count_launch();
}

// In-place FP64 sum over the ranks (no-op on one rank). Every rank receives
// the same values (NCCL's reduction result is broadcast), so decisions taken
// from them agree across ranks.
void allreduce_inplace(gpk_operator* op, double* buf, size_t count) {
  if (!op->sharded) return;
  gpk_ctx* ctx = op->ctx;
  const ncclResult_t r = nccl().all_reduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream);
  if (r != ncclSuccess) throw std::runtime_error(std::string("ncclAllReduce: ") + nccl().error_string(r));
  count_launch();
}

void require(bool ok, const char* msg) {
  if (!ok) throw InvalidArgument(msg);
}

bool all_finite(const double* p, size_t count) {
  for (size_t i = 0; i < count; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// col-major host (rows x cols) -> row-major device [rows][cols]
void upload_colmajor(gpk_operator* op, const double* host, int rows, int cols, double* dev) {
  cudaStream_t s = op->ctx->stream;
  double* tmp = op->tmp64.ensure(static_cast<size_t>(rows) * cols);
  GPK_CUDA(cudaMemcpyAsync(tmp, host, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
  transpose_launch(tmp, cols, rows, rows, dev, cols, s);
}
void download_colmajor(gpk_operator* op, const double* dev, int rows, int cols, double* host) {
  cudaStream_t s = op->ctx->stream;
  double* tmp = op->tmp64.ensure(static_cast<size_t>(rows) * cols);
  transpose_launch(dev, rows, cols, cols, tmp, rows, s);
  GPK_CUDA(cudaMemcpyAsync(host, tmp, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaStreamSynchronize(s));
}

void set_hyper(gpk_operator* op, const double* raw) {
  const int d = op->d;
  std::vector<double> r(raw, raw + d + 2);
  for (int k = 0; k < d + 2; ++k) {
    const double c = softplus(r[k]);
    if (!std::isfinite(c) || c <= 0.0)
      throw InvalidArgument("Hyperparameters: constrained value " + std::to_string(k) + " is not finite and positive");
  }
  if (op->raw == r && op->hyper_version > 0) return;  // unchanged: scaled inputs and AP blocks stay valid
  op->raw = r;
  ++op->hyper_version;
  op->inv_ls.resize(d);
  for (int k = 0; k < d; ++k) op->inv_ls[k] = 1.0 / softplus(r[k]);
  op->s = softplus(r[d]);
  op->s2 = op->s * op->s;
  op->sigma = softplus(r[d + 1]);
  op->sigma2 = op->sigma * op->sigma;
  cudaStream_t s = op->ctx->stream;
  double* il = op->inv_ls_dev.ensure(d);
  GPK_CUDA(cudaMemcpyAsync(il, op->inv_ls.data(), sizeof(double) * d, cudaMemcpyHostToDevice, s));
  const double hv[2] = {op->s2, op->sigma2};
  GPK_CUDA(cudaMemcpyAsync(op->hyp_dev.ensure(2), hv, sizeof(hv), cudaMemcpyHostToDevice, s));
  prescale_launch(op->x64.p, op->n, d, op->dp, il, op->xs32.p, op->xs64.p, s);
  if (op->dpg) gram_image_launch(op->xs32.p, op->n, d, op->dp, op->dpg, op->xg32.p, s);
  if (op->tg) tg_image_launch(op->xs32.p, op->n, d, op->dp, op->xtg.p, s);
  if (op->dense && dense_dgemm())
    dense_block64_launch(op->xs64.p, op->n, d, op->s2, op->sigma2, 0, op->n, 0, op->n,
                         op->kdense.ensure(static_cast<size_t>(op->n) * op->n), op->n, 0, s);
  GPK_CUDA(cudaStreamSynchronize(s));  // inv_ls host buffer lifetime
}

// Core operator product: out = base + alpha * H[rows, cols] v.
struct KvCall {
  const float* v = nullptr;  // FP32 RHS [C][ld]
  int m = 0;
  const int* row_idx = nullptr;
  int r0 = 0, R = 0;
  int c0 = 0, C = 0;
  const int* sel = nullptr;
  int sel_block = 0;
  const double* vdiag = nullptr;  // FP64 RHS for the diagonal, [C][m]
  double* out = nullptr;
  int ldo = 0;
  const double* base = nullptr;
  int ldb = 0;
  double alpha = 1.0;
  const int* skip = nullptr;
  const double* dotw = nullptr;  // fused column dot of the result (see KvReduceArgs)
  double* dpart = nullptr;
  int groups = kReduceGroups;
  const double* inv_scales = nullptr;  // fused AP block scores
  double* spart = nullptr;
  int score_block = 0, gpb = 1;
  const float* vpk = nullptr;  // pre-packed (and, sharded, all-gathered) TF32 RHS images
  int vshift = 0;              // diagonal RHS row offset (row shard start)
  // fused AP epilogue (see KvReduceArgs)
  CgCtl* ctl = nullptr;
  const double* scales = nullptr;
  double tol = 0.0;
  int* sel_out = nullptr;
  int nblocks = 0;
  unsigned* ticket = nullptr;
  double** ap_ptrs = nullptr;
  double* ap_inv = nullptr;
  long long ap_bb = 0;
  double* ap_upd = nullptr;
  const float* xs_rows = nullptr;  // cross kernel: rows from these scaled points, no noise diagonal
  bool fused = false;              // AP slab: reduce + epilogue inside the tcgen05 kernel
};

__global__ void stats_add_kernel(double* st, double entries, int m, int d, const int* skip) {
  if (skip && *skip) return;
  atomicAdd(st, entries * m);
  atomicAdd(st + 1, entries * (2.0 * m + 3.0 * d + 6.0));
  atomicAdd(st + 2, entries * (3.0 * d + 6.0));
}
void stats_add_launch(double* st, double entries, int m, int d, const int* skip, cudaStream_t s) {
  stats_add_kernel<<<1, 1, 0, s>>>(st, entries, m, d, skip);
  check_launch("stats_add");
}

void run_kv_one(gpk_operator* op, const KvCall& c);

// Column panels for products whose packed RHS images exceed the L2: every row
// tile streams all of the images, and once the concurrently running CTAs have
// drifted apart over a stream larger than the cache each of them re-reads it
// from DRAM (measured at n = 524288, m = 65: 390-420 GB of DRAM reads per
// product against 0.37 GB of images, and the entry rate falls from 5.6e11/s
// at n <= 262144 to 5.2e11/s at n = 1048576). Running the product panel by
// panel -- all row tiles over one L2-sized block of columns, accumulating into
// out in FP64 as the sharded ring does per slice -- keeps a panel's images
// resident. GPK_KV_PANEL_MB: image bytes per panel (default 48; 0: off).
int kv_panel_cols(gpk_operator* op, const KvCall& c) {
  static const bool panel_env = std::getenv("GPK_KV_PANEL_MB") != nullptr;  // (set: panels at any size, for tests)
  static const int panel_mb = [] {
    const char* e = std::getenv("GPK_KV_PANEL_MB");
    return e ? std::atoi(e) : 48;
  }();
  const bool tc = op->ctx->kernel == 1 && c.m <= 80;
  if (panel_mb <= 0 || !tc || c.fused || c.sel || c.ctl || c.spart || c.inv_scales || !c.out) return 0;
  const size_t col_bytes = kv_tc_pack_floats(c.m, 32) / 32 * sizeof(float);
  const size_t panel_bytes = static_cast<size_t>(panel_mb) << 20;
  if (static_cast<size_t>(c.C) * col_bytes <= 2 * panel_bytes || (!panel_env && static_cast<double>(c.R) * c.C < 1e9)) return 0;
  const int pc = static_cast<int>(panel_bytes / col_bytes) / 1024 * 1024;
  return pc >= 1024 ? pc : 0;
}

void run_kv(gpk_operator* op, const KvCall& c) {
  const int pc = kv_panel_cols(op, c);
  if (pc == 0) return run_kv_one(op, c);
  cudaStream_t s = op->ctx->stream;
  const float* vpk = c.vpk;
  if (!vpk) {  // the images of the whole column range once (as run_kv_one would)
    float* buf = op->vpk.ensure(kv_tc_pack_floats(c.m, c.C));
    kv_tc_pack_launch(c.vdiag, c.v, c.vdiag ? c.m : kv_ld_for(c.m), c.C, c.m, nullptr, 0, op->n, buf, c.skip, s);
    vpk = buf;
  }
  const size_t cf = kv_tc_pack_floats(c.m, 32);  // floats per 32-column image chunk
  for (int off = 0; off < c.C; off += pc) {
    KvCall p = c;
    p.vpk = vpk + static_cast<size_t>(off / 32) * cf;
    p.c0 = c.c0 + off;
    p.C = std::min(pc, c.C - off);
    p.vshift = c.vshift - off;  // the diagonal rows index vdiag relative to the whole range's first column
    if (off > 0) {
      p.base = c.out;
      p.ldb = c.ldo;
    }
    if (off + pc < c.C) {  // the fused column dot belongs to the complete result
      p.dotw = nullptr;
      p.dpart = nullptr;
    }
    run_kv_one(op, p);
  }
}

void run_kv_one(gpk_operator* op, const KvCall& c) {
  cudaStream_t s = op->ctx->stream;
  const int Cmax = c.sel ? c.sel_block : c.C;
  const bool tc = op->ctx->kernel == 1 && c.m <= 80;
  // AP slab on the tensor cores: one column split, reduce + AP epilogue fused
  // into the operator kernel (every 128-row tile lies inside one AP block)
  const bool fused = c.fused;
  if (fused && !(tc && c.sel && c.ctl && c.spart && c.dotw == c.out && !c.row_idx && c.r0 == 0 &&
                 c.score_block % 128 == 0 && c.groups == (c.R + 127) / 128 && c.gpb == c.score_block / 128))
    throw std::logic_error("run_kv: fused AP slab preconditions");
  // deep variant (1 CTA/SM, 16 eval warps, 4 TMEM A buffers) measured faster
  // on large launches (C2 -4%, d=3 -24%) and slower on small ones (C1 +26%)
  const bool deep = tc && !fused &&
                    (op->ctx->kv_deep >= 0 ? op->ctx->kv_deep != 0 : static_cast<double>(c.R) * Cmax >= 1e8);
  int splits = fused ? 1
               : tc ? kv_tc_choose_splits(c.R, Cmax, op->ctx->sms, deep ? 1 : 2)
                    : kv_choose_splits(c.R, Cmax, op->ctx->sms);
  int cps = (Cmax + splits - 1) / splits;
  cps = (cps + 31) / 32 * 32;
  splits = std::max(1, (Cmax + cps - 1) / cps);
  // deep launches with a host-known column range run stream-K: one persistent
  // CTA per SM over the (row tile, chunk) units; a tile's partials occupy the
  // split slots 0 .. (number of CTAs that touched it) - 1
  const bool streamk = deep && !c.sel && op->ctx->kv_streamk;
  int sk_G = 0, sk_Q = 0;
  long long sk_U = 0;
  if (streamk) {
    const long long T = (c.R + 127) / 128;
    sk_Q = (Cmax + 31) / 32;
    sk_U = T * sk_Q;
    sk_G = static_cast<int>(std::min<long long>(op->ctx->sms, sk_U));
    int maxseg = 1;
    for (long long t = 0; t < T; ++t)
      maxseg = std::max(maxseg, static_cast<int>(sk_last(t, sk_Q, sk_G, sk_U) - sk_first(t, sk_Q, sk_G, sk_U) + 1));
    splits = maxseg;
  }
  double* part = op->part.ensure(static_cast<size_t>(splits) * c.R * c.m);
  KvArgs a{};
  // tensor-core Gram distances (whole 32-column chunks from column c0)
  const bool tgram = tc && op->tg && (deep || fused) && !streamk && (c.sel ? c.sel_block % 32 == 0 : c.c0 % 32 == 0);
  // else FP32 Gram-form distances for d >= 21 (image width >= 24)
  const bool gram = tc && !tgram && op->dpg > 0;
  if (gram && c.xs_rows && c.xs_rows != op->pts32.p) throw std::logic_error("run_kv: cross rows without a Gram image");
  a.xs = gram ? op->xg32.p : op->xs32.p;
  a.n = op->n;
  a.dp = gram ? op->dpg : op->dp;
  a.row_idx = c.row_idx;
  a.r0 = c.r0;
  a.R = c.R;
  a.c0 = c.c0;
  a.C = c.C;
  a.sel = c.sel;
  a.sel_block = c.sel_block;
  a.v = c.v;
  a.ldv = kv_ld_for(c.m);
  a.m = c.m;
  a.log2_s2 = static_cast<float>(std::log2(op->s2));
  a.part = part;
  a.splits = splits;
  a.cols_per_split = cps;
  // FP32 TMEM accumulation spans flush_chunks 32-column chunks before the FP64
  // partial (GPK_FLUSH_CHUNKS: parity experiments; default 16 = 512 columns)
  static const int flush_default = [] {
    const char* e = std::getenv("GPK_FLUSH_CHUNKS");
    return e ? std::max(1, std::atoi(e)) : 16;
  }();
  a.flush_chunks = fused ? std::max(flush_default, (cps + 31) / 32) : flush_default;
  a.skip = c.skip;
  a.stats = op->ctx->stats;
  a.d = op->d;
  a.xs_rows = (gram && c.xs_rows) ? op->ptsg32.p : c.xs_rows;
  a.xtg = tgram ? op->xtg.p : nullptr;
  a.sk_ctas = sk_G;
  gpk_ctx* ctx = op->ctx;
  if (c.vpk && !tc) throw InvalidArgument("gpk: pre-packed operator input needs the tcgen05 kernel");
  const float* vpk = c.vpk;
  // dense cache (n <= dense_cache_cap): a full unsharded product with an FP64
  // RHS is K V by cuBLAS DGEMM in FP64 (the reference's cached path), reduced
  // by kv_reduce as one split
  const bool dense = op->dense && !op->sharded && !fused && !c.sel && !c.row_idx && !c.xs_rows && c.vdiag &&
                     c.r0 == 0 && c.R == op->n && c.c0 == 0 && c.C == op->n;
  if (tc && !vpk && !dense) {
    float* buf = op->vpk.ensure(kv_tc_pack_floats(c.m, Cmax));
    kv_tc_pack_launch(c.vdiag, c.v, c.vdiag ? c.m : a.ldv, Cmax, c.m, c.sel, c.sel_block, op->n, buf, c.skip, s);
    vpk = buf;
  }
  cudaEvent_t* prof_end = nullptr;
  if (ctx->profiling) {
    if (ctx->prof_used == ctx->prof.size()) {
      cudaEvent_t e0, e1;
      GPK_CUDA(cudaEventCreate(&e0));
      GPK_CUDA(cudaEventCreate(&e1));
      ctx->prof.push_back({e0, e1});
    }
    auto& pr = ctx->prof[ctx->prof_used++];
    GPK_CUDA(cudaEventRecord(pr.first, s));
    prof_end = &pr.second;
  }
  KvReduceArgs r{};
  r.part = part;
  r.splits = splits;
  r.R = c.R;
  r.m = c.m;
  r.vdiag = c.vdiag;
  r.ldvd = c.m;
  r.vdiag32 = c.v;
  r.ldv32 = a.ldv;
  r.row_idx = c.row_idx;
  r.r0 = c.r0;
  r.c0 = c.c0;
  r.C = c.C;
  r.sel = c.sel;
  r.sel_block = c.sel_block;
  r.n = op->n;
  r.sigma2 = op->sigma2;
  r.out = c.out;
  r.ldo = c.ldo;
  r.base = c.base;
  r.ldb = c.ldb;
  r.alpha = c.alpha;
  r.skip = c.skip;
  r.dotw = c.dotw;
  r.dpart = c.dpart;
  r.groups = c.groups;
  r.inv_scales = c.inv_scales;
  r.spart = c.spart;
  r.score_block = c.score_block;
  r.gpb = c.gpb;
  r.vshift = c.vshift;
  r.ctl = c.ctl;
  r.scales = c.scales;
  r.tol = c.tol;
  r.sel_out = c.sel_out;
  r.nblocks = c.nblocks;
  r.ticket = c.ticket;
  r.ap_ptrs = c.ap_ptrs;
  r.ap_inv = c.ap_inv;
  r.ap_bb = c.ap_bb;
  r.ap_upd = c.ap_upd;
  r.nodiag = c.xs_rows != nullptr;
  r.sk_G = sk_G;
  r.sk_Q = sk_Q;
  r.sk_U = sk_U;
  if (fused) {
    kv_tc_fused_launch(a, vpk, r, s);
    if (prof_end) GPK_CUDA(cudaEventRecord(*prof_end, s));
    return;
  }
  if (dense && !dense_dgemm()) {
    // FP64 operator with on-the-fly entries (kv64_kernel): the reference's
    // exact FP64 products for n <= dense_cache_cap without materialising H
    const int sp = kv64_splits_for(op->n, op->n, c.m, op->d, op->ctx->sms);
    double* p64 = op->part.ensure(static_cast<size_t>(sp) * op->n * c.m);
    kv64_launch(op->xs64.p, op->n, op->d, op->s2, 0, op->n, c.vdiag, c.m, sp, p64, c.skip, s);
    if (a.stats) stats_add_launch(a.stats, static_cast<double>(op->n) * op->n, c.m, op->d, c.skip, s);
    r.part = p64;
    r.splits = sp;
    r.sk_G = 0;
  } else if (dense) {
    // part (row-major [n][m]) = K V: column-major part^T (m x n) = V^T K (K symmetric)
    gpk_ctx* cx = op->ctx;
    if (cublasSetStream(cx->blas, s) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
    const double one = 1.0, zero = 0.0;
    if (cublasDgemm(cx->blas, CUBLAS_OP_N, CUBLAS_OP_N, c.m, op->n, op->n, &one, c.vdiag, c.m, op->kdense.p, op->n,
                    &zero, part, c.m) != CUBLAS_STATUS_SUCCESS)
      throw CudaError("cublasDgemm (dense operator)");
    count_launch();
    if (a.stats) stats_add_launch(a.stats, static_cast<double>(op->n) * op->n, c.m, op->d, c.skip, s);
    r.splits = 1;
    r.sk_G = 0;
  } else if (tc) {
    kv_tc_launch(a, vpk, s, streamk ? 3 : (deep ? 2 : 0));
  } else {
    kv_slab_launch(a, op->d, s);
  }
  if (prof_end) GPK_CUDA(cudaEventRecord(*prof_end, s));
  kv_reduce_launch(r, s);
}

// Ring all-gather overlapped with the operator: the slices of the
// FP32 RHS travel one hop per step on the communication stream (step j:
// send slice rk - j to rank rk + 1, receive slice rk - j - 1 from rank rk - 1),
// and as each slice lands the compute stream packs its TF32 images and runs
// the operator over that column block, accumulating into out (the own slice,
// which holds the noise diagonal, first; the fused column dot on the last).
// With n/N rows per slice the transfer of a slice hides behind the product
// of the previous one whenever a slice's compute outlasts its transfer.
void apply_local_ring(gpk_operator* op, float* v32, const double* v_local, int m, double* out, const double* base,
                      double alpha, const int* skip, const double* dotw, double* dpart) {
  gpk_ctx* ctx = op->ctx;
  cudaStream_t s = ctx->stream, cs = ctx->comm_stream;
  const int S = op->S, nr = op->nr, rk = op->rk, n = op->n;
  const size_t slice = static_cast<size_t>(S) * m;
  const size_t cf = kv_tc_pack_floats(m, 32);  // floats per 32-row image chunk
  float* vpk = op->vpk.ensure(kv_tc_pack_floats(m, S * nr));
  GPK_CUDA(cudaEventRecord(ctx->ring_start, s));  // own slice converted
  GPK_CUDA(cudaStreamWaitEvent(cs, ctx->ring_start, 0));
  const int next = (rk + 1) % nr, prev = (rk + nr - 1) % nr;
  for (int j = 0; j + 1 < nr; ++j) {
    const int snd = (rk - j + nr) % nr, rcv = (rk - j - 1 + 2 * nr) % nr;
    nccl().group_start();
    ncclResult_t r1 = nccl().send(v32 + snd * slice, slice, ncclFloat, next, ctx->comm, cs);
    ncclResult_t r2 = nccl().recv(v32 + rcv * slice, slice, ncclFloat, prev, ctx->comm, cs);
    const ncclResult_t r3 = nccl().group_end();
    if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
      throw std::runtime_error(std::string("gpk ring all-gather: ") +
                               nccl().error_string(r1 != ncclSuccess ? r1 : r2 != ncclSuccess ? r2 : r3));
    count_launch();
    GPK_CUDA(cudaEventRecord(ctx->ring_ev[rcv], cs));
  }
  for (int j = 0; j < nr; ++j) {
    const int src = (rk - j + nr) % nr;
    if (j > 0) GPK_CUDA(cudaStreamWaitEvent(s, ctx->ring_ev[src], 0));
    const int c0 = src * S, rows = std::max(0, std::min(S, n - c0));
    if (rows == 0) continue;
    float* img = vpk + static_cast<size_t>(src) * (S / 32) * cf;
    kv_tc_pack_launch(nullptr, v32 + src * slice, m, S, m, nullptr, 0, n, img, skip, s, rows);
    KvCall c;
    c.vpk = img;
    c.m = m;
    c.r0 = op->row0;
    c.R = op->nloc;
    c.c0 = c0;
    c.C = rows;
    c.vdiag = src == rk ? v_local : nullptr;
    c.vshift = 0;
    c.out = out;
    c.ldo = m;
    c.base = j == 0 ? base : out;
    c.ldb = m;
    c.alpha = alpha;
    c.skip = skip;
    const bool last = j + 1 == nr;
    c.dotw = last ? dotw : nullptr;
    c.dpart = last ? dpart : nullptr;
    run_kv(op, c);
  }
}

// out_local = base + alpha * H[own rows, :] V, for V given by this rank's rows
// v_local (FP64 [nloc][m]). The local rows are packed into this rank's slice
// of the TF32 image buffer and all-gathered so every rank holds the full RHS.
// Optional fused column dot (dotw/dpart) as in KvCall.
void apply_local(gpk_operator* op, const double* v_local, int m, double* out, const double* base, double alpha,
                 const int* skip, const double* dotw = nullptr, double* dpart = nullptr) {
  cudaStream_t s = op->ctx->stream;
  const int S = op->S, nr = op->nr;
  // the rank's rows in FP32 (4 m bytes a row on the wire, not the 8 NPAD of
  // the TF32 hi/lo images), all-gathered into the full-height RHS (rank
  // slices S rows apart = global row order), then packed into the operator's
  // TF32 images locally
  float* v32 = op->v32g.ensure(static_cast<size_t>(S) * nr * m);
  float* mine = v32 + static_cast<size_t>(op->rk) * S * m;
  to_f32_launch(v_local, op->nloc, m, m, mine, m, skip, s);
  if (op->nloc < S)
    GPK_CUDA(cudaMemsetAsync(mine + static_cast<size_t>(op->nloc) * m, 0, sizeof(float) * (S - op->nloc) * m, s));
  gpk_ctx* ctx = op->ctx;
  if (op->sharded && nr > 1 && ctx->ring_gather && ctx->comm_stream) {
    apply_local_ring(op, v32, v_local, m, out, base, alpha, skip, dotw, dpart);
    return;
  }
  gather_inplace(op, v32, sizeof(float) * S * m);
  float* vpk = op->vpk.ensure(kv_tc_pack_floats(m, S * nr));
  kv_tc_pack_launch(nullptr, v32, m, S * nr, m, nullptr, 0, op->n, vpk, skip, s, op->n);
  KvCall c;
  c.vpk = vpk;
  c.m = m;
  c.r0 = op->row0;
  c.R = op->nloc;
  c.c0 = 0;
  c.C = op->n;
  c.vdiag = v_local;
  c.vshift = op->row0;
  c.out = out;
  c.ldo = m;
  c.base = base;
  c.ldb = m;
  c.alpha = alpha;
  c.skip = skip;
  c.dotw = dotw;
  c.dpart = dpart;
  run_kv(op, c);
}

// H V for V FP64 row-major [n][m] on device -> out row-major (ldo = m).
void apply_dev64(gpk_operator* op, const double* v64, int m, double* out, const double* base, double alpha,
                 float* v32buf, const int* skip) {
  const int ld = kv_ld_for(m);
  to_f32_launch(v64, op->n, m, m, v32buf, ld, skip, op->ctx->stream);
  KvCall c;
  c.v = v32buf;
  c.m = m;
  c.R = op->n;
  c.C = op->n;
  c.vdiag = v64;
  c.out = out;
  c.ldo = m;
  c.base = base;
  c.ldb = m;
  c.alpha = alpha;
  c.skip = skip;
  run_kv(op, c);
}

// RHS groups of at most 65 columns (the kernel's widest tile).
constexpr int kMaxRhs = 65;
// Zero rows after the residual block: AP's batched GEMM reads a whole block of
// rows in place, which may run past row n for the last (partial) block.
constexpr int kResidPad = 1024;

// -------------------------------------------------------------- precond
void build_precond(gpk_precond* pc) {
  gpk_operator* op = pc->op;
  cudaStream_t s = op->ctx->stream;
  const int n = op->n, rank = pc->rank;
  pc->sigma2 = op->sigma2;
  pc->achieved = 0;
  pc->stopped = 0;
  if (rank == 0) return;
  double* L = pc->L.ensure(static_cast<size_t>(n) * rank);
  int* piv = pc->pivots.ensure(rank);
  DBuf<double>& diag = pc->diag;
  DBuf<double>& pval = pc->pval;
  DBuf<int>& pidx = pc->pidx;
  DBuf<int>& stop = pc->stop;
  diag.ensure(n);
  const int G = kReduceGroups;
  pval.ensure(G);
  pidx.ensure(G);
  stop.ensure(2);
  GPK_CUDA(cudaMemsetAsync(stop.p, 0, sizeof(int) * 2, s));
  // diag = s^2 (kernel_diagonal, kernel.cpp:196-198)
  std::vector<double> h(n, op->s2);
  GPK_CUDA(cudaMemcpyAsync(diag.p, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  for (int mcol = 0; mcol < rank; ++mcol) {
    argmax_partials_launch(diag.p, n, pval.p, pidx.p, G, s);
    pchol_step_launch(op->xs64.p, n, op->d, op->s2, pval.p, pidx.p, G, L, rank, mcol, diag.p, piv, stop.p, s);
  }
  // achieved rank = number of pivots before the stop flag: recompute on host
  std::vector<int> pv(rank);
  int stop_h = 0;
  GPK_CUDA(cudaMemcpyAsync(pv.data(), piv, sizeof(int) * rank, cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaMemcpyAsync(&stop_h, stop.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaStreamSynchronize(s));
  // The stop flag is set at the first non-positive pivot; pivots written
  // before it are valid. Recount by replaying: steps that ran wrote pivots
  // in order, so find how many ran via a marker pass.
  int achieved = rank;
  if (stop_h) {
    // Re-run the count cheaply: pivots of skipped steps were never written;
    // mark them by a sentinel pass.
    std::vector<int> marker(rank, -1);
    GPK_CUDA(cudaMemcpyAsync(piv, marker.data(), sizeof(int) * rank, cudaMemcpyHostToDevice, s));
    GPK_CUDA(cudaMemsetAsync(stop.p, 0, sizeof(int), s));
    GPK_CUDA(cudaMemcpyAsync(diag.p, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    for (int mcol = 0; mcol < rank; ++mcol) {
      argmax_partials_launch(diag.p, n, pval.p, pidx.p, G, s);
      pchol_step_launch(op->xs64.p, n, op->d, op->s2, pval.p, pidx.p, G, L, rank, mcol, diag.p, piv, stop.p, s);
    }
    GPK_CUDA(cudaMemcpyAsync(pv.data(), piv, sizeof(int) * rank, cudaMemcpyDeviceToHost, s));
    GPK_CUDA(cudaStreamSynchronize(s));
    achieved = 0;
    while (achieved < rank && pv[achieved] >= 0) ++achieved;
    pc->stopped = 1;
  }
  pc->achieved = achieved;
  if (achieved == 0) return;
  // small = L^T L + sigma^2 I (achieved x achieved), then its inverse
  const int r = achieved;
  DBuf<double>& gpart = pc->gpart;
  DBuf<double>& gram = pc->gram;
  gpart.ensure(static_cast<size_t>(G) * r * r);
  gram.ensure(static_cast<size_t>(r) * r);
  // gram over the first r columns of L (ld = rank)
  gram_partials_launch(L, n, r, rank, gpart.p, G, s);
  sum_partials_launch(gpart.p, G, r * r, gram.p, nullptr, s);
  std::vector<double> gh(static_cast<size_t>(r) * r);
  GPK_CUDA(cudaMemcpyAsync(gh.data(), gram.p, sizeof(double) * r * r, cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaStreamSynchronize(s));
  for (int a = 0; a < r; ++a) gh[static_cast<size_t>(a) * r + a] += pc->sigma2;
  // FP64 Cholesky + inverse on the host (r <= rank ~ 100: microseconds).
  std::vector<double> Lc(static_cast<size_t>(r) * r, 0.0);
  for (int j = 0; j < r; ++j) {
    double sjj = gh[static_cast<size_t>(j) * r + j];
    for (int k = 0; k < j; ++k) sjj -= Lc[static_cast<size_t>(j) * r + k] * Lc[static_cast<size_t>(j) * r + k];
    if (!(sjj > 0.0)) throw NumericError("PivotedCholeskyPreconditioner: inner factorisation failed");
    const double ljj = std::sqrt(sjj);
    Lc[static_cast<size_t>(j) * r + j] = ljj;
    for (int i = j + 1; i < r; ++i) {
      double t = gh[static_cast<size_t>(i) * r + j];
      for (int k = 0; k < j; ++k) t -= Lc[static_cast<size_t>(i) * r + k] * Lc[static_cast<size_t>(j) * r + k];
      Lc[static_cast<size_t>(i) * r + j] = t / ljj;
    }
  }
  std::vector<double> inv(static_cast<size_t>(r) * r, 0.0);
  for (int c = 0; c < r; ++c) {
    std::vector<double> y(r, 0.0);
    y[c] = 1.0;
    for (int i = 0; i < r; ++i) {
      double t = y[i];
      for (int k = 0; k < i; ++k) t -= Lc[static_cast<size_t>(i) * r + k] * y[k];
      y[i] = t / Lc[static_cast<size_t>(i) * r + i];
    }
    for (int i = r - 1; i >= 0; --i) {
      double t = y[i];
      for (int k = i + 1; k < r; ++k) t -= Lc[static_cast<size_t>(k) * r + i] * y[k];
      y[i] = t / Lc[static_cast<size_t>(i) * r + i];
    }
    for (int i = 0; i < r; ++i) inv[static_cast<size_t>(i) * r + c] = y[i];
  }
  pc->minv.ensure(static_cast<size_t>(r) * r);
  GPK_CUDA(cudaMemcpyAsync(pc->minv.p, inv.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, s));
  GPK_CUDA(cudaStreamSynchronize(s));
}

// out = P^-1 R (device, row-major [n][m]); P == nullptr -> identity copy.
void precond_apply_dev(gpk_precond* pc, gpk_operator* op, const double* R, int m, double* out, const int* skip) {
  cudaStream_t s = op->ctx->stream;
  const int n = op->nloc;  // this rank's rows (the whole problem on one GPU)
  if (!pc) {
    scale_launch(R, n * m, 1.0, out, skip, s);
    return;
  }
  if (pc->achieved == 0) {
    scale_launch(R, n * m, pc->sigma2, out, skip, s);
    return;
  }
  // (L L^T + s2 I)^-1 R = (R - L (s2 I + L^T L)^-1 L^T R) / s2 ; L is replicated
  // (identical pivots on every rank), L^T R is a sum over rows -> partials of
  // this rank's rows, all-gathered and summed in rank order.
  const int r = pc->achieved, nr = op->nr;
  const double* Lloc = pc->L.p + static_cast<size_t>(op->row0) * pc->rank;  // column-major view: rank x n
  double* part = pc->part.ensure(static_cast<size_t>(nr) * r * m);
  double* T = nr > 1 ? pc->T.ensure(static_cast<size_t>(r) * m) : part;
  double* inner = pc->inner.ensure(static_cast<size_t>(r) * m);
  cublasHandle_t h = op->ctx->blas;
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  const double one = 1.0, zero = 0.0, neg = -1.0 / pc->sigma2;
  // T (r x m, column-major) = L^T R over this rank's rows; ranks' T summed in rank order
  if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, r, m, n, &one, Lloc, pc->rank, R, m, &zero,
                  part + static_cast<size_t>(op->rk) * r * m, r) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDgemm (L^T R)");
  gather_inplace(op, part, sizeof(double) * r * m);
  if (nr > 1) sum_partials_launch(part, nr, r * m, T, skip, s);
  // inner = (s2 I + L^T L)^-1 T
  if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, r, m, r, &one, pc->minv.p, r, T, r, &zero, inner, r) !=
      CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDgemm (Minv T)");
  // out = R / s2 - L inner / s2  (row-major out == column-major m x n)
  scale_launch(R, n * m, pc->sigma2, out, skip, s);
  if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, m, n, r, &neg, inner, r, Lloc, pc->rank, &one, out, m) !=
      CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDgemm (L inner)");
  count_launch(3);
}

// ----------------------------------------------------------------- batch
void batch_norms(gpk_batch* b, const double* R, double tol, double* mean, double* probe, int* done) {
  gpk_operator* op = b->op;
  cudaStream_t s = op->ctx->stream;
  const int G = kReduceGroups, nr = op->nr;
  double* part = b->red.ensure(static_cast<size_t>(nr) * G * 2 * b->m + 8);
  double* o3 = b->vec3.ensure(std::max(3, b->m));
  col_reduce_launch(R, nullptr, b->n, b->m, b->m, 2, part + static_cast<size_t>(op->rk) * G * b->m, G, nullptr, s);
  gather_inplace(op, part, sizeof(double) * G * b->m);
  norms_launch(part, G * nr, b->m, b->scales_dev.p, tol, o3, s);
  double h[3];
  GPK_CUDA(cudaMemcpyAsync(h, o3, sizeof(h), cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaStreamSynchronize(s));
  *mean = h[0];
  *probe = h[1];
  *done = h[2] != 0.0;
}

void refresh_residuals(gpk_batch* b) {  // linear_system.cpp:33
  gpk_operator* op = b->op;
  if (b->m > kMaxRhs) throw InvalidArgument("gpk: batches wider than 65 columns are not supported by the solvers");
  if (op->ctx->kernel == 1) {
    apply_local(op, b->solutions.p, b->m, b->residuals.p, b->targets.p, -1.0, nullptr);
  } else {
    if (op->nr > 1) throw InvalidArgument("gpk: the sharded operator needs the tcgen05 kernel");
    float* v32 = b->f32.ensure(static_cast<size_t>(b->n) * kv_ld_for(b->m));
    apply_dev64(op, b->solutions.p, b->m, b->residuals.p, b->targets.p, -1.0, v32, nullptr);
  }
}

void validate(const gpk_solver_config* c) {  // linear_system.cpp:7-14
  if (!(c->tolerance > 0.0)) throw InvalidArgument("SolverConfig: tolerance > 0");
  if (c->max_epochs < 1) throw InvalidArgument("SolverConfig: max_epochs >= 1");
  if (c->block_size < 1) throw InvalidArgument("SolverConfig: block_size >= 1");
  if (c->batch_size < 1) throw InvalidArgument("SolverConfig: batch_size >= 1");
  if (c->momentum < 0.0 || c->momentum >= 1.0) throw InvalidArgument("SolverConfig: 0 <= momentum < 1");
  if (c->preconditioner_rank < 0) throw InvalidArgument("SolverConfig: preconditioner_rank >= 0");
}

using Clock = std::chrono::steady_clock;

// GPK_PHASE_TIMING=1: synchronising phase timer for the outer step (stderr,
// one JSON line per step). Diagnostic only; off by default.
struct PhaseTimer {
  bool on = false;
  cudaStream_t stream = nullptr;
  Clock::time_point last;
  std::string line;
  static bool enabled() {
    static const bool e = [] {
      const char* v = std::getenv("GPK_PHASE_TIMING");
      return v && std::atoi(v) != 0;
    }();
    return e;
  }
  void start(cudaStream_t s) {
    on = enabled();
    if (!on) return;
    stream = s;
    cudaStreamSynchronize(s);
    last = Clock::now();
    line = "{";
  }
  void mark(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(stream);
    const auto now = Clock::now();
    char buf[96];
    std::snprintf(buf, sizeof(buf), "%s\"%s\": %.1f", line.size() > 1 ? ", " : "", name,
                  std::chrono::duration<double, std::micro>(now - last).count());
    line += buf;
    last = now;
  }
  void finish() {
    if (!on) return;
    std::fprintf(stderr, "%s}\n", line.c_str());
  }
};
PhaseTimer g_phase;

void finalise(gpk_batch* b, double tol, gpk_solver_report* rep, Clock::time_point start) {
  int done;
  batch_norms(b, b->residuals.p, tol, &rep->mean_residual_norm, &rep->probe_residual_norm, &done);
  rep->reached_tolerance = done;
  rep->wall_seconds = std::chrono::duration<double>(Clock::now() - start).count();
}

// Runs `enqueue_iteration` in groups, keeping one group in flight while the
// previous group's control block is read back; stops once ctl.stop is set.
template <class F>
void drive(gpk_batch* b, CgCtl* ctl, int group, int max_iters, F&& enqueue_iteration, bool capturable = false) {
  gpk_ctx* ctx = b->op->ctx;
  cudaStream_t s = ctx->stream;
  // CUDA graph of one group of iterations (CG, AP): the iteration enqueues the
  // same launches with the same arguments every time (all control flow is on
  // device flags), so the group is captured once per solve and replayed; a
  // replay past the budget is a no-op (every kernel tests ctl->stop).
  const bool use_graph = capturable && ctx->graphs && !ctx->profiling && max_iters > group;
  cudaGraphExec_t exec = nullptr;
  long long per_group = 0;
  auto enqueue_group = [&](int g) {
    if (!use_graph) {
      for (int i = 0; i < g; ++i) enqueue_iteration();
      return;
    }
    if (!exec) {
      const long long before = g_launch_counter ? *g_launch_counter : 0;
      cudaGraph_t graph = nullptr;
      GPK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
      try {
        for (int i = 0; i < group; ++i) enqueue_iteration();
      } catch (...) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      GPK_CUDA(cudaStreamEndCapture(s, &graph));
      const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      GPK_CUDA(e);
      per_group = (g_launch_counter ? *g_launch_counter : 0) - before;  // counted once at capture
    } else {
      count_launch(static_cast<int>(per_group));
    }
    GPK_CUDA(cudaGraphLaunch(exec, s));
  };
  int issued = 0, k = 0;
  bool pending = false;
  try {
    while (true) {
      const int g = use_graph ? (issued < max_iters ? group : 0) : std::min(group, max_iters - issued);
      if (g > 0) {
        enqueue_group(g);
        issued += g;
      }
      GPK_CUDA(cudaMemcpyAsync(&ctx->ctl_host[k & 1], ctl, sizeof(CgCtl), cudaMemcpyDeviceToHost, s));
      GPK_CUDA(cudaEventRecord(ctx->ev[k & 1], s));
      if (pending) {
        GPK_CUDA(cudaEventSynchronize(ctx->ev[(k - 1) & 1]));
        if (ctx->ctl_host[(k - 1) & 1].stop) break;
      }
      if (g <= 0) {
        GPK_CUDA(cudaEventSynchronize(ctx->ev[k & 1]));
        break;
      }
      pending = true;
      ++k;
    }
    GPK_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    if (exec) cudaGraphExecDestroy(exec);
    throw;
  }
  if (exec) GPK_CUDA(cudaGraphExecDestroy(exec));
}

void init_ctl(gpk_batch* b, int budget, int iters) {
  CgCtl h{};
  h.budget = budget;
  h.iters = iters;
  GPK_CUDA(cudaMemcpyAsync(b->ctl.ensure(1), &h, sizeof(CgCtl), cudaMemcpyHostToDevice, b->op->ctx->stream));
  GPK_CUDA(cudaStreamSynchronize(b->op->ctx->stream));
}

CgCtl read_ctl(gpk_batch* b) {
  CgCtl h{};
  GPK_CUDA(cudaMemcpyAsync(&h, b->ctl.p, sizeof(CgCtl), cudaMemcpyDeviceToHost, b->op->ctx->stream));
  GPK_CUDA(cudaStreamSynchronize(b->op->ctx->stream));
  return h;
}

int iteration_group(int n) { return n >= 32768 ? 1 : (n >= 8192 ? 2 : 4); }

// --------------------------------------------------------------- solvers
void solve_cg(gpk_batch* b, const gpk_solver_config* c, gpk_precond* pc, gpk_solver_report* rep) {
  validate(c);
  const auto start = Clock::now();
  gpk_operator* op = b->op;
  cudaStream_t s = op->ctx->stream;
  const int n = b->n, m = b->m, G = kReduceGroups;  // n: this rank's rows
  const int nr = op->nr, rk = op->rk;
  const bool tc = op->ctx->kernel == 1;
  if (!tc && nr > 1) throw InvalidArgument("gpk: the sharded operator needs the tcgen05 kernel");
  if (m > kMaxRhs) throw InvalidArgument("gpk: batches wider than 65 columns are not supported by the solvers");
  std::memset(rep, 0, sizeof(*rep));
  const size_t nm = static_cast<size_t>(n) * m;
  double* d = b->w1.ensure(nm);
  double* p = b->w2.ensure(nm);
  double* hd = b->w3.ensure(nm);
  float* d32 = tc ? nullptr : b->f32.ensure(static_cast<size_t>(n) * kv_ld_for(m));
  // per-rank reduction partials [nr][G][2m]; each rank fills its slice, then all-gather
  double* part = b->red.ensure(static_cast<size_t>(nr) * G * 2 * m + 8);
  double* part2 = part + static_cast<size_t>(rk) * G * 2 * m;  // mode-1 slice ([G][2m])
  double* part1 = part + static_cast<size_t>(rk) * G * m;      // dot slice ([G][m])
  double* gamma = b->vec1.ensure(m);
  double* alpha = b->vec2.ensure(m);
  double* beta = b->vec3.ensure(std::max(m, 3));
  init_ctl(b, c->max_epochs, 0);
  CgCtl* ctl = b->ctl.p;
  const int* stop = &ctl->stop;

  refresh_residuals(b);                                       // solvers.cpp:45
  precond_apply_dev(pc, op, b->residuals.p, m, p, nullptr);   // p = P^-1 r
  GPK_CUDA(cudaMemcpyAsync(d, p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, s));
  if (!tc) to_f32_launch(d, n, m, m, d32, kv_ld_for(m), nullptr, s);
  col_reduce_launch(b->residuals.p, p, n, m, m, 1, part2, G, nullptr, s);
  gather_inplace(op, part, sizeof(double) * G * 2 * m);
  cg_init_scalars_launch(part, G * nr, m, b->scales_dev.p, c->tolerance, gamma, ctl, s);

  auto iteration = [&]() {  // solvers.cpp:52-82
    if (tc) {
      apply_local(op, d, m, hd, nullptr, 1.0, stop, d, part1);  // Hd and the fused d.Hd partials
    } else {
      KvCall kc;
      kc.v = d32;
      kc.m = m;
      kc.R = n;
      kc.C = n;
      kc.vdiag = d;
      kc.out = hd;
      kc.ldo = m;
      kc.skip = stop;
      kc.dotw = d;
      kc.dpart = part1;
      run_kv(op, kc);
    }
    gather_inplace(op, part, sizeof(double) * G * m);
    cg_alpha_launch(part, G * nr, m, gamma, alpha, ctl, s);
    cg_update_launch(b->solutions.p, b->residuals.p, d, hd, alpha, n, m, stop, s);
    precond_apply_dev(pc, op, b->residuals.p, m, p, stop);
    col_reduce_launch(b->residuals.p, p, n, m, m, 1, part2, G, stop, s);
    gather_inplace(op, part, sizeof(double) * G * 2 * m);
    cg_beta_launch(part, G * nr, m, b->scales_dev.p, c->tolerance, gamma, beta, ctl, s);
    cg_direction_launch(d, p, beta, n, m, d32, tc ? 0 : kv_ld_for(m), stop, s);
  };
  drive(b, ctl, iteration_group(op->n), c->max_epochs, iteration, true);
  const CgCtl h = read_ctl(b);
  rep->iterations = h.iters;
  rep->epochs_consumed = h.iters;
  rep->aborted = h.aborted;
  if (h.aborted) std::strncpy(rep->abort_reason, "cg breakdown: non-finite step size", 127);
  finalise(b, c->tolerance, rep, start);
}

// SPD inverses of `batch` dim x dim matrices (in place input destroyed).
__global__ void fill_ptrs_kernel(double** p, double* a, double* b, long long stride, int batch) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < batch; k += gridDim.x * blockDim.x) {
    p[k] = a + k * stride;
    p[batch + k] = b + k * stride;
  }
}

// Batched SPD inverse on stream `st` without host synchronisation: cuSOLVER
// potrfBatched (L L^T), then L^{-1} and L^{-T} L^{-1} by two batched
// triangular solves against the identity. Pointer arrays are filled on the
// device; the per-matrix info goes to pinned host memory and is checked by
// the caller after its next synchronisation (spd_inverse_check).
void spd_inverse_batched(gpk_ctx* ctx, cudaStream_t st, double* mats, int dim, int batch, double* inv) {
  GPK_CUDA(cudaSetDevice(ctx->device));
  if (batch > 4096) throw InvalidArgument("gpk: at most 4096 AP blocks");
  if (cusolverDnSetStream(ctx->solver, st) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnSetStream");
  if (cublasSetStream(ctx->blas, st) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  double** da = ctx->ptr_a.ensure(2 * batch);
  double** db = da + batch;
  int* info = ctx->info.ensure(batch);
  if (!ctx->info_host) GPK_CUDA(cudaMallocHost(&ctx->info_host, sizeof(int) * 4096));
  fill_ptrs_kernel<<<(batch + 255) / 256, 256, 0, st>>>(da, mats, inv, static_cast<long long>(dim) * dim, batch);
  check_launch("fill_ptrs");
  if (cusolverDnDpotrfBatched(ctx->solver, CUBLAS_FILL_MODE_LOWER, dim, da, dim, info, batch) !=
      CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDpotrfBatched");
  count_launch();
  GPK_CUDA(cudaMemcpyAsync(ctx->info_host, info, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
  set_identity_launch(inv, dim, batch, st);
  const double one = 1.0;
  if (cublasDtrsmBatched(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, dim,
                         dim, &one, da, dim, db, dim, batch) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrsmBatched");
  if (cublasDtrsmBatched(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, dim,
                         dim, &one, da, dim, db, dim, batch) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrsmBatched");
  count_launch(2);
  if (cusolverDnSetStream(ctx->solver, ctx->stream) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnSetStream");
  if (cublasSetStream(ctx->blas, ctx->stream) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
}
// Batched SPD inverse by recursive 2 x 2 blocking on the Schur complement
// (no factorisation kernels, all level-3 work in strided-batched DGEMMs):
//   B11 = inv(A11); X = B11 A12; S = A22 - A21 X; B22 = inv(S);
//   B12 = -X B22; B11 -= B12 X^T; B21 = B12^T,
// down to <= 64 x 64 leaves inverted in shared memory. A (column-major,
// ld = dim, stride dim^2) is destroyed; B receives the inverse. Same
// arithmetic class as the reference's Cholesky block solve (FP64, SPD, no
// pivoting); ~dim^3 flops per matrix. The info array stays zero unless a
// leaf pivot is non-positive (checked after the solve by spd_inverse_check).
struct SpdRec {
  gpk_ctx* ctx;
  cudaStream_t st;
  double* A;
  double* B;
  double* X;  // scratch: every recursion level owns its X (n1 x n2) at its own offset
  int* info;  // per matrix: 1 if a leaf pivot was not positive
  int ld, batch;
  long long stride, xstride;
  void gemm(cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, double alpha, const double* a, int lda,
            const double* b, int ldb, double beta, double* c, int ldc, long long sa, long long sb, long long sc) {
    if (cublasDgemmStridedBatched(ctx->blas, ta, tb, m, n, k, &alpha, a, lda, sa, b, ldb, sb, &beta, c, ldc, sc,
                                  batch) != CUBLAS_STATUS_SUCCESS)
      throw CudaError("cublasDgemmStridedBatched (SPD inverse)");
    count_launch();
  }
  void inv(int off, int nn, long long xoff) {
    if (nn <= 64) {
      spd_leaf_inverse_launch(A, B, off, nn, ld, stride, batch, info, st);
      count_launch();
      return;
    }
    const int n1 = ((nn / 2) + 31) / 32 * 32, n2 = nn - n1;
    double* x = X + xoff;
    const long long child = xoff + static_cast<long long>(n1) * n2;  // deeper levels' scratch
    auto at = [&](double* base, int r, int c) { return base + r + static_cast<size_t>(c) * ld; };
    inv(off, n1, child);                                                     // B11
    gemm(CUBLAS_OP_N, CUBLAS_OP_N, n1, n2, n1, 1.0, at(B, off, off), ld, at(A, off, off + n1), ld, 0.0, x, n1, stride,
         stride, xstride);                                                   // X = B11 A12
    gemm(CUBLAS_OP_N, CUBLAS_OP_N, n2, n2, n1, -1.0, at(A, off + n1, off), ld, x, n1, 1.0, at(A, off + n1, off + n1), ld,
         stride, xstride, stride);                                           // S = A22 - A21 X
    inv(off + n1, n2, child);                                                // B22 = inv(S)
    gemm(CUBLAS_OP_N, CUBLAS_OP_N, n1, n2, n2, -1.0, x, n1, at(B, off + n1, off + n1), ld, 0.0, at(B, off, off + n1), ld,
         xstride, stride, stride);                                           // B12 = -X B22
    gemm(CUBLAS_OP_N, CUBLAS_OP_T, n1, n1, n2, -1.0, at(B, off, off + n1), ld, x, n1, 1.0, at(B, off, off), ld, stride,
         xstride, stride);                                                   // B11 -= B12 X^T
    block_transpose_launch(at(B, off, off + n1), at(B, off + n1, off), n2, n1, ld, stride, batch, st);  // B21
    count_launch();
  }
};

// scratch doubles per matrix for the recursion (sum of every level's n1 x n2)
long long spd_inverse_scratch(int nn) {
  if (nn <= 64) return 0;
  const int n1 = ((nn / 2) + 31) / 32 * 32, n2 = nn - n1;
  return static_cast<long long>(n1) * n2 + std::max(spd_inverse_scratch(n1), spd_inverse_scratch(n2));
}

void spd_inverse_recursive(gpk_ctx* ctx, cudaStream_t st, double* mats, int dim, int batch, double* inv,
                           double* scratch) {
  if (cublasSetStream(ctx->blas, st) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  if (batch > 4096) throw InvalidArgument("gpk: at most 4096 AP blocks");
  if (!ctx->info_host) GPK_CUDA(cudaMallocHost(&ctx->info_host, sizeof(int) * 4096));
  int* info = ctx->info.ensure(batch);
  GPK_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * batch, st));
  SpdRec r{ctx, st, mats, inv, scratch, info, dim, batch, static_cast<long long>(dim) * dim,
           std::max<long long>(1, spd_inverse_scratch(dim))};
  r.inv(0, dim, 0);
  GPK_CUDA(cudaMemcpyAsync(ctx->info_host, info, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
  if (cublasSetStream(ctx->blas, ctx->stream) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
}

void spd_inverse_check(gpk_ctx* ctx, int batch) {  // after a synchronisation that covers the aux stream
  for (int k = 0; k < batch; ++k)
    if (ctx->info_host[k] != 0)
      throw NumericError("solve_ap: block Cholesky failed; block is not positive definite (noise scale too small)");
}

// Enqueues every AP diagonal block H[blk, blk] and its FP64 inverse on the
// auxiliary stream (after the main stream's pending work: the scaled inputs),
// keyed on the operator's hyperparameter version; solve_ap joins on ev_aux.
void ap_prepare(gpk_batch* b, int block) {
  gpk_operator* op = b->op;
  gpk_ctx* ctx = op->ctx;
  const int n = b->n, nblocks = (n + block - 1) / block;
  const size_t bb = static_cast<size_t>(block) * block;
  double* mats = b->w1.ensure(bb * nblocks);
  double* inv = b->blocks.ensure(bb * nblocks);
  GPK_CUDA(cudaEventRecord(ctx->ev_m2a, ctx->stream));
  GPK_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_m2a, 0));
  const size_t xs = static_cast<size_t>(std::max<long long>(1, spd_inverse_scratch(block)));
  double* scratch = ctx->spd_inverse == 1 ? b->w5.ensure(xs * nblocks) : nullptr;
  double* hyp = op->hyp_dev.p;
  auto enqueue = [&](cudaStream_t st) {
    ap_blocks_launch(op->xs64.p, n, op->d, hyp, block, nblocks, mats, st);
    if (ctx->spd_inverse == 1)
      spd_inverse_recursive(ctx, st, mats, block, nblocks, inv, scratch);
    else
      spd_inverse_batched(ctx, st, mats, block, nblocks, inv);
  };
  // the ~45 launches of the recursive inverse are captured once (fixed
  // buffers, hyperparameters read from the device) and replayed every step
  int* info = ctx->info.ensure(nblocks);  // allocated before the key: the graph captures its address
  if (!ctx->info_host) GPK_CUDA(cudaMallocHost(&ctx->info_host, sizeof(int) * 4096));
  const std::array<const void*, 6> key{op->xs64.p, mats, inv, scratch, hyp, info};
  const bool graphable = ctx->graphs && ctx->spd_inverse == 1;
  if (graphable && !(b->ap_graph && b->ap_graph_key == key && b->ap_graph_dims == std::make_pair(block, nblocks))) {
    if (b->ap_graph) {
      cudaGraphExecDestroy(b->ap_graph);
      b->ap_graph = nullptr;
    }
    const long long before = g_launch_counter ? *g_launch_counter : 0;
    cudaGraph_t g = nullptr;
    GPK_CUDA(cudaStreamBeginCapture(ctx->aux, cudaStreamCaptureModeRelaxed));
    try {
      enqueue(ctx->aux);
    } catch (...) {
      cudaStreamEndCapture(ctx->aux, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    GPK_CUDA(cudaStreamEndCapture(ctx->aux, &g));
    const cudaError_t e = cudaGraphInstantiate(&b->ap_graph, g, 0);
    cudaGraphDestroy(g);
    GPK_CUDA(e);
    b->ap_graph_key = key;
    b->ap_graph_dims = {block, nblocks};
    b->ap_graph_launches = (g_launch_counter ? *g_launch_counter : 0) - before;
    if (g_launch_counter) *g_launch_counter = before;  // counted on replay
  }
  if (graphable) {
    GPK_CUDA(cudaGraphLaunch(b->ap_graph, ctx->aux));
    count_launch(static_cast<int>(b->ap_graph_launches));
  } else {
    enqueue(ctx->aux);
  }
  GPK_CUDA(cudaEventRecord(ctx->ev_aux, ctx->aux));
  b->ap_ready = true;
  b->ap_block = block;
  b->ap_version = op->hyper_version;
}

void solve_ap(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* rep) {
  validate(c);
  const auto start = Clock::now();
  gpk_operator* op = b->op;
  gpk_ctx* ctx = op->ctx;
  cudaStream_t s = ctx->stream;
  const int n = b->n, m = b->m;
  if (m > kMaxRhs) throw InvalidArgument("gpk: batches wider than 65 columns are not supported by the solvers");
  std::memset(rep, 0, sizeof(*rep));
  const int block = std::min(c->block_size, n);
  const int nblocks = (n + block - 1) / block;
  const double max_iterations = static_cast<double>(c->max_epochs) * n / block;  // solvers.cpp:118
  const int budget = static_cast<int>(std::ceil(max_iterations));
  const bool tc = ctx->kernel == 1;
  // inverse of every diagonal block H[blk, blk] (FP64), on the auxiliary
  // stream (possibly enqueued earlier by the optimiser: ap_prepare)
  const size_t bb = static_cast<size_t>(block) * block;
  if (!(b->ap_ready && b->ap_block == block && b->ap_version == op->hyper_version)) ap_prepare(b, block);
  b->ap_ready = false;  // consumed by this solve
  double* inv = b->blocks.p;
  double* inv_scales_dev = b->vec1.ensure(m);
  inv_scales_launch(b->scales_dev.p, m, inv_scales_dev, s);
  // reduction groups per AP block: one resident wave (3 x 148 blocks of 8 row-warps) keeps enough
  // row loads in flight for the latency-bound fused reduce
  const int gpb = std::max(1, std::min(block / 8, 3 * ctx->sms / nblocks));
  const int groups = nblocks * gpb;
  double* spart = b->vec2.ensure(groups);
  // fused slab iterations (run_kv): one partial per 128-row tile, block scores
  // from block/128 tiles; the tail tiles of a partial last block stay zero
  const bool fused = tc && ctx->fused_ap && block % 128 == 0 && m <= 96 && nblocks <= 1024;
  const int tiles = (n + 127) / 128, gpb_t = block / 128;
  double* spart_t = nullptr;
  if (fused) {
    spart_t = b->spart_t.ensure(static_cast<size_t>(nblocks) * gpb_t);
    GPK_CUDA(cudaMemsetAsync(spart_t, 0, sizeof(double) * nblocks * gpb_t, s));
  }
  double* part = b->red.ensure(static_cast<size_t>(std::max(groups, tiles)) * m + 8);
  int* sel = b->ibuf.ensure(1);
  double* Rs = b->w3.ensure(static_cast<size_t>(block) * m);
  double* upd64 = b->w2.ensure(static_cast<size_t>(block) * m);
  float* upd32 = tc ? nullptr : b->f32.ensure(static_cast<size_t>(std::max(block, n)) * kv_ld_for(m));
  double** ptrs = ctx->ptr_b.ensure(4);
  {
    double* hp[3] = {Rs, inv, upd64};
    GPK_CUDA(cudaMemcpyAsync(ptrs, hp, sizeof(hp), cudaMemcpyHostToDevice, s));
  }
  init_ctl(b, budget, -1);
  CgCtl* ctl = b->ctl.p;
  const int* stop = &ctl->stop;
  if (!b->ticket.p) {
    b->ticket.ensure(1);
    GPK_CUDA(cudaMemsetAsync(b->ticket.p, 0, sizeof(unsigned), s));
  }
  unsigned* ticket = b->ticket.p;
  float* vpk_blk = tc ? b->apk.ensure(kv_tc_pack_floats(m, block)) : nullptr;
  // the GEMM reads R_blk in place when the zero padding covers the last block
  const bool in_place = tc && (static_cast<long long>(nblocks) * block - n) <= kResidPad;

  // refresh_residuals (solvers.cpp:98) with the fused norms and block scores
  float* v32 = b->f32.ensure(static_cast<size_t>(std::max(block, n)) * kv_ld_for(m));
  to_f32_launch(b->solutions.p, n, m, m, v32, kv_ld_for(m), nullptr, s);
  {
    KvCall kc;
    kc.v = v32;
    kc.m = m;
    kc.R = n;
    kc.C = n;
    kc.vdiag = b->solutions.p;
    kc.out = b->residuals.p;
    kc.ldo = m;
    kc.base = b->targets.p;
    kc.ldb = m;
    kc.alpha = -1.0;
    kc.dotw = b->residuals.p;
    kc.dpart = part;
    kc.groups = groups;
    kc.inv_scales = inv_scales_dev;
    kc.spart = spart;
    kc.score_block = block;
    kc.gpb = gpb;
    kc.ctl = ctl;  // fused initial test (iters -1 -> 0) and first block choice
    kc.scales = b->scales_dev.p;
    kc.tol = c->tolerance;
    kc.sel_out = sel;
    kc.nblocks = nblocks;
    kc.ticket = ticket;
    if (in_place) {
      kc.ap_ptrs = ptrs;
      kc.ap_inv = inv;
      kc.ap_bb = static_cast<long long>(bb);
      kc.ap_upd = upd64;
    }
    run_kv(op, kc);
  }

  g_phase.mark("ap_refresh");
  GPK_CUDA(cudaStreamWaitEvent(s, ctx->ev_aux, 0));  // block inverses ready before the first update
  ap_info_gate_launch(ctx->info.p, nblocks, ctl, s);  // a failed block inverse: no update runs
  g_phase.mark("ap_inverse_wait");
  if (cublasSetStream(ctx->blas, s) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  auto iteration = [&]() {  // solvers.cpp:120-140
    if (tc) {
      // upd = R_blk^T Hinv (batched GEMM, pointers written by the previous reduce
      // or by the gather) -> V += upd and TF32 images -> slab -> fused reduce
      // (norms, termination test, next block, next GEMM pointers)
      if (!in_place) ap_gather_launch(b->residuals.p, n, m, block, sel, Rs, inv, upd64, ptrs, stop, s);
      const double one = 1.0, zero = 0.0;
      if (cublasDgemmBatched(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, m, block, block, &one,
                             const_cast<const double* const*>(ptrs), m, const_cast<const double* const*>(ptrs + 1),
                             block, &zero, ptrs + 2, m, 1) != CUBLAS_STATUS_SUCCESS)
        throw CudaError("cublasDgemmBatched");
      count_launch();
      ap_apply_pack_launch(upd64, n, m, block, sel, b->solutions.p, vpk_blk, kv_tc_npad(m), stop, s);
      KvCall kc;
      kc.vpk = vpk_blk;
      kc.m = m;
      kc.R = n;
      kc.sel = sel;
      kc.sel_block = block;
      kc.vdiag = upd64;
      kc.out = b->residuals.p;
      kc.ldo = m;
      kc.base = b->residuals.p;
      kc.ldb = m;
      kc.alpha = -1.0;
      kc.skip = stop;
      kc.dotw = b->residuals.p;
      kc.dpart = part;
      kc.groups = fused ? tiles : groups;
      kc.inv_scales = inv_scales_dev;
      kc.spart = fused ? spart_t : spart;
      kc.score_block = block;
      kc.gpb = fused ? gpb_t : gpb;
      kc.ctl = ctl;
      kc.scales = b->scales_dev.p;
      kc.tol = c->tolerance;
      kc.sel_out = sel;
      kc.nblocks = nblocks;
      kc.ticket = ticket;
      kc.fused = fused;
      if (in_place) {
        kc.ap_ptrs = ptrs;
        kc.ap_inv = inv;
        kc.ap_bb = static_cast<long long>(bb);
        kc.ap_upd = upd64;
      }
      run_kv(op, kc);
      return;
    }
    ap_select_groups_launch(spart, nblocks, gpb, sel, stop, s);
    ap_gather_launch(b->residuals.p, n, m, block, sel, Rs, inv, upd64, ptrs, stop, s);
    // upd (m x block, column-major == row-major [block][m]) = R_blk^T Hinv  (Hinv symmetric)
    const double one = 1.0, zero = 0.0;
    if (cublasDgemmBatched(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, m, block, block, &one,
                           const_cast<const double* const*>(ptrs), m, const_cast<const double* const*>(ptrs + 1),
                           block, &zero, ptrs + 2, m, 1) != CUBLAS_STATUS_SUCCESS)
      throw CudaError("cublasDgemmBatched");
    count_launch();
    ap_apply_update_launch(upd64, n, m, block, sel, b->solutions.p, upd32, kv_ld_for(m), stop, s);
    KvCall kc;
    kc.v = upd32;
    kc.m = m;
    kc.R = n;
    kc.sel = sel;
    kc.sel_block = block;
    kc.vdiag = upd64;
    kc.out = b->residuals.p;
    kc.ldo = m;
    kc.base = b->residuals.p;
    kc.ldb = m;
    kc.alpha = -1.0;
    kc.skip = stop;
    kc.dotw = b->residuals.p;  // fused ||R_j||^2 and block scores of the updated residual
    kc.dpart = part;
    kc.groups = groups;
    kc.inv_scales = inv_scales_dev;
    kc.spart = spart;
    kc.score_block = block;
    kc.gpb = gpb;
    run_kv(op, kc);
    ap_check_launch(part, groups, m, b->scales_dev.p, c->tolerance, ctl, s);
  };
  const bool persistent = fused && in_place && ctx->ap_persistent && ap_persistent_supported(n, m, block, ctx->sms);
  if (persistent) {
    // every iteration in one cooperative launch (ap_persistent.cu)
    ApPersistArgs pa{};
    // tensor-core Gram distances when the operator has their images, else the
    // FP32 Gram image for d >= 21 (as run_kv)
    pa.xtg = op->tg ? op->xtg.p : nullptr;
    pa.xs = (op->dpg && !op->tg) ? op->xg32.p : op->xs32.p;
    pa.n = n;
    pa.d = op->d;
    pa.dp = (op->dpg && !op->tg) ? op->dpg : op->dp;
    pa.m = m;
    pa.npad = kv_tc_npad(m);
    pa.log2_s2 = static_cast<float>(std::log2(op->s2));
    pa.sigma2 = op->sigma2;
    pa.block = block;
    pa.nblocks = nblocks;
    pa.gpb = gpb_t;
    pa.budget = budget;
    pa.R = b->residuals.p;
    pa.V = b->solutions.p;
    pa.inv = inv;
    pa.bb = static_cast<long long>(bb);
    pa.upd = upd64;
    pa.cpart = b->ap_cpart.ensure(static_cast<size_t>(8) * block * m);
    pa.vpk = vpk_blk;
    pa.dpart = part;
    pa.spart = spart_t;
    pa.inv_scales = inv_scales_dev;
    pa.scales = b->scales_dev.p;
    pa.tol = c->tolerance;
    pa.ctl = ctl;
    pa.sel = sel;
    pa.gbar = b->gbar.ensure(32);  // [0..5) barrier, ticket, flag, sel, stop; [8..28) optional phase clock
    pa.stats = ctx->stats;
    GPK_CUDA(cudaMemsetAsync(pa.gbar, 0, 8 * sizeof(unsigned), s));  // barrier, ticket, flag, sel, stop
    cudaEvent_t* prof_end = nullptr;
    if (ctx->profiling) {  // timed as one operator launch (it also runs the block updates)
      if (ctx->prof_used == ctx->prof.size()) {
        cudaEvent_t e0, e1;
        GPK_CUDA(cudaEventCreate(&e0));
        GPK_CUDA(cudaEventCreate(&e1));
        ctx->prof.push_back({e0, e1});
      }
      auto& pr = ctx->prof[ctx->prof_used++];
      GPK_CUDA(cudaEventRecord(pr.first, s));
      prof_end = &pr.second;
    }
    static const bool phase_clock = std::getenv("GPK_AP_PROF") != nullptr;  // development: phase split
    if (phase_clock) {
      pa.prof = b->ap_prof.ensure(16 + 64 * 160);
      GPK_CUDA(cudaMemsetAsync(pa.prof, 0, (16 + 64 * 160) * sizeof(unsigned long long), s));
    }
    ap_persistent_launch(pa, s);
    if (prof_end) GPK_CUDA(cudaEventRecord(*prof_end, s));
    GPK_CUDA(cudaStreamSynchronize(s));
    if (phase_clock) {
      std::vector<unsigned long long> hv(16 + 64 * 160);
      GPK_CUDA(cudaMemcpy(hv.data(), pa.prof, hv.size() * 8, cudaMemcpyDeviceToHost));
      const unsigned long long* h = hv.data();
      {  // ticket spread (first ticket -> last ticket) and last ticket -> decision release, ns
        double spread = 0, rel = 0;
        int cnt = 0;
        for (int it = 0; it < 64 && it < static_cast<int>(h[9]); ++it) {
          const unsigned long long* row = h + 16 + it * 160;
          unsigned long long lo = ~0ull, hi = 0;
          for (int c = 0; c < (n + 127) / 128; ++c) {
            lo = std::min(lo, row[c]);
            hi = std::max(hi, row[c]);
          }
          if (row[159] == 0 || lo == 0) continue;
          spread += static_cast<double>(hi - lo);
          rel += static_cast<double>(row[159] - hi);
          ++cnt;
        }
        (void)rel;
        if (cnt) std::fprintf(stderr, "ap_persistent tickets: spread %.2f us\n", spread / cnt / 1e3);
        double seg[3] = {0, 0, 0};
        int c2 = 0;
        for (int it = 0; it < 64 && it < static_cast<int>(h[9]); ++it) {
          const unsigned long long* row = h + 16 + it * 160;
          unsigned long long hi = 0;
          for (int c = 0; c < (n + 127) / 128; ++c) hi = std::max(hi, row[c]);
          if (!row[155] || !row[156] || !row[157] || !row[159]) continue;  // SM clock64 stamps of the last CTA
          seg[0] += static_cast<double>(row[156] - row[155]);
          seg[1] += static_cast<double>(row[157] - row[156]);
          seg[2] += static_cast<double>(row[159] - row[157]);
          ++c2;
        }
        if (c2) std::fprintf(stderr, "ap_persistent last CTA (us at 1.9 GHz): ticket->partials %.2f, sums %.2f, select %.2f\n",
                             seg[0] / c2 / 1.9e3, seg[1] / c2 / 1.9e3, seg[2] / c2 / 1.9e3);
      }
      const double it = static_cast<double>(h[9]) * 1.9e3;  // cycles -> us at ~1.9 GHz
      std::fprintf(stderr,
                   "ap_persistent phases (us/iteration at 1.9 GHz, %llu iterations): C1load %.2f C1 %.2f Csync %.2f C2 %.2f sync1 %.2f "
                   "S %.2f ticket %.2f B %.2f\n",
                   h[9], h[6] / it, h[7] / it, h[8] / it, h[0] / it, h[1] / it, h[2] / it, h[3] / it, h[4] / it);
    }
  } else {
    drive(b, ctl, 8, budget, iteration, true);
  }
  g_phase.mark("ap_iterations");
  spd_inverse_check(ctx, nblocks);
  const CgCtl h = read_ctl(b);
  rep->iterations = h.iters;
  rep->epochs_consumed = static_cast<double>(h.iters) * block / n;
  finalise(b, c->tolerance, rep, start);
}

// SGD on the tcgen05 operator, single rank or row-sharded: the
// minibatch rows idx are contracted against this rank's own rows only; the
// b x m partial gradients (+ the owning rank's target and diagonal terms) are
// all-gathered and summed in rank order, so every rank holds the same g and
// takes the same termination decision, and updates only its own rows of
// momentum, solution and residual estimate -- writing the solution's TF32
// operator images in the same pass, so the next contraction reads them as is.
void solve_sgd_tc(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* rep, int bs, int budget,
                  double step, Clock::time_point start) {
  gpk_operator* op = b->op;
  cudaStream_t s = op->ctx->stream;
  const int n = op->n, nloc = b->n, m = b->m, G = kReduceGroups, nr = op->nr;
  const int row0 = op->sharded ? op->row0 : 0;
  const size_t nm = static_cast<size_t>(nloc) * m;
  GPK_CUDA(cudaMemcpyAsync(b->residuals.p, b->targets.p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, s));
  double* M = b->w1.ensure(nm);
  GPK_CUDA(cudaMemsetAsync(M, 0, sizeof(double) * nm, s));
  const int npad = kv_tc_npad(m);
  float* vpk = b->apk.ensure(kv_tc_pack_floats(m, nloc));
  kv_tc_pack_launch(b->solutions.p, nullptr, m, nloc, m, nullptr, 0, n, vpk, nullptr, s);
  double* hv = b->w2.ensure(static_cast<size_t>(bs) * m);
  double* grad = b->w3.ensure(static_cast<size_t>(bs) * m);
  const long long stride = (static_cast<long long>(bs) * m + m + 1 + 31) / 32 * 32;  // doubles per rank slice
  double* gbuf = b->w4.ensure(static_cast<size_t>(nr) * stride);
  double* part = b->red.ensure(static_cast<size_t>(nr) * G * 2 * m + 8);
  double* sumsq = b->vec1.ensure(m);
  int* pos = b->ibuf2.ensure(nloc);
  GPK_CUDA(cudaMemsetAsync(pos, 0xff, sizeof(int) * nloc, s));  // -1
  int* nonfinite = b->flag.ensure(1);
  GPK_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s));
  col_reduce_launch(b->residuals.p, nullptr, nloc, m, m, 2, part + static_cast<size_t>(op->rk) * G * m, G, nullptr,
                    s);
  gather_inplace(op, part, sizeof(double) * G * m);
  sum_partials_launch(part, G * nr, m, sumsq, nullptr, s);
  init_ctl(b, budget, -1);
  CgCtl* ctl = b->ctl.p;
  const int* stop = &ctl->stop;
  sgd_check_launch(sumsq, m, b->scales_dev.p, c->tolerance, nonfinite, ctl, s);  // initial test

  const int chunk = 256;
  int* idxbuf = b->ibuf.ensure(static_cast<size_t>(chunk) * bs);
  int t = 0;
  auto iteration = [&]() {  // solvers.cpp:164-178
    if (t % chunk == 0) sgd_batches_launch(c->seed, c->substream, n, bs, t, std::min(chunk, budget - t), idxbuf, s);
    const int* idx = idxbuf + static_cast<size_t>(t % chunk) * bs;
    KvCall kc;
    kc.vpk = vpk;
    kc.m = m;
    kc.row_idx = idx;
    kc.R = bs;
    kc.c0 = row0;
    kc.C = nloc;
    kc.vdiag = b->solutions.p;
    kc.out = hv;
    kc.ldo = m;
    kc.skip = stop;
    run_kv(op, kc);
    double* slice = gbuf + static_cast<size_t>(op->sharded ? op->rk : 0) * stride;
    sgd_prep_launch(hv, idx, bs, b->targets.p, b->residuals.p, row0, nloc, m, pos, nonfinite, slice, stop, s);
    gather_inplace(op, gbuf, sizeof(double) * stride);
    sgd_gsum_launch(gbuf, nr, stride, bs, m, grad, stop, s);
    sgd_check_sharded_launch(gbuf, nr, stride, grad, bs, m, sumsq, b->scales_dev.p, c->tolerance, ctl, s);
    // the update runs for the iteration the check just counted (skip reads
    // stop before it is set for the next one: test the pre-check flag)
    sgd_update_pack_launch(M, b->solutions.p, b->residuals.p, vpk, npad, pos, grad, c->momentum, step, nloc, m,
                           nonfinite, &ctl->pad, s);
    // one rank: abort in the iteration that formed the non-finite iterate;
    // sharded: a rank's own non-finite rows reach every rank through its next
    // slice, so all ranks stop at the same iteration (one later)
    if (!op->sharded) sgd_diverge_now_launch(nonfinite, ctl, s);
    sgd_unscatter_launch(idx, bs, row0, nloc, pos, &ctl->pad, s);
    ++t;
  };
  drive(b, ctl, std::max(1, iteration_group(n) * 4), budget, iteration);
  const CgCtl h = read_ctl(b);
  rep->iterations = h.iters;
  rep->epochs_consumed = static_cast<double>(h.iters) * bs / n;
  rep->aborted = h.aborted;
  if (h.aborted) std::strncpy(rep->abort_reason, "sgd divergence: non-finite iterate", 127);
  finalise(b, c->tolerance, rep, start);
}

// Per-launch CUDA-event bracket of an operator launch while profiling is on
// (gpk_ctx_stats' launch count and milliseconds).
cudaEvent_t* prof_begin(gpk_ctx* ctx, cudaStream_t s) {
  if (!ctx->profiling) return nullptr;
  if (ctx->prof_used == ctx->prof.size()) {
    cudaEvent_t e0, e1;
    GPK_CUDA(cudaEventCreate(&e0));
    GPK_CUDA(cudaEventCreate(&e1));
    ctx->prof.push_back({e0, e1});
  }
  auto& pr = ctx->prof[ctx->prof_used++];
  GPK_CUDA(cudaEventRecord(pr.first, s));
  return &pr.second;
}

// SGD with lazily evaluated momentum (sgd_lazy.cu): per iteration the
// minibatch product on the tensor cores builds V(t) from the rows' FP32
// records, and only the b minibatch rows of the state are written. One rank
// or row-sharded: the slab contracts against this rank's rows,
// the b x m partials (+ own diagonal / target terms, old residual squares)
// are all-gathered and summed in rank order, so every rank holds the same g
// and takes the same decisions. Iterations run as CUDA graphs of 256
// (minibatches for the group generated at its start from the device counter).
bool sgd_lazy_supported(gpk_operator* op, int m, int bs) {
  return op->ctx->kernel == 1 && op->ctx->sgd_lazy && m <= 80 && op->dp <= 16 && bs <= 1024;
}

void solve_sgd_lazy(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* rep, int bs, int budget,
                    double step, Clock::time_point start) {
  gpk_operator* op = b->op;
  gpk_ctx* ctx = op->ctx;
  cudaStream_t s = ctx->stream;
  const int n = op->n, nloc = b->n, m = b->m, G = kReduceGroups, nr = op->nr;
  const int row0 = op->sharded ? op->row0 : 0;
  const size_t nm = static_cast<size_t>(nloc) * m;
  GPK_CUDA(cudaMemcpyAsync(b->residuals.p, b->targets.p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, s));
  double* Mb = b->w1.ensure(nm);
  GPK_CUDA(cudaMemsetAsync(Mb, 0, sizeof(double) * nm, s));
  int moff = 0;
  int s32_sat = 0;  // first Delta from which the FP32 S table is constant
  const int rw = sgd_record_width(m, &moff);
  const int rows_pad = (nloc + 31) / 32 * 32;
  // one record per 32-row chunk, plus a zero record past the end (64-column slab chunks)
  float* rec = b->sgd_rec.ensure(static_cast<size_t>(rows_pad / 32 + 1) * rw);
  int* tau = b->sgd_tau.ensure(rows_pad + 32);
  sgd_records_init_launch(b->solutions.p, nloc, rows_pad, m, rw, moff, rec, tau, s);
  // P(Delta) = rho^Delta, S(Delta) = rho + ... + rho^Delta by the recurrence an
  // untouched row follows in the reference (momentum *= rho; solutions += momentum)
  {
    std::vector<double> tab(2 * static_cast<size_t>(budget + 1));
    std::vector<float> t32(budget + 1);
    double* S = tab.data();
    double* P = tab.data() + budget + 1;
    P[0] = 1.0;
    S[0] = 0.0;
    for (int k = 1; k <= budget; ++k) {
      P[k] = P[k - 1] * c->momentum;
      S[k] = S[k - 1] + P[k];
    }
    for (int k = 0; k <= budget; ++k) t32[k] = static_cast<float>(S[k]);
    // S(Delta) is non-decreasing and converges to rho / (1 - rho): in FP32 it is
    // constant from some Delta on (rho = 0.9: ~170), so the slab clamps Delta
    // there -- the same values, a table of a few hundred entries in shared
    // memory instead of 4096, and no global look-ups for long-untouched rows
    s32_sat = budget;
    while (s32_sat > 0 && t32[s32_sat - 1] == t32[budget]) --s32_sat;
    GPK_CUDA(cudaMemcpyAsync(b->sgd_tab.ensure(tab.size()), tab.data(), sizeof(double) * tab.size(),
                             cudaMemcpyHostToDevice, s));
    GPK_CUDA(cudaMemcpyAsync(b->sgd_s32.ensure(t32.size()), t32.data(), sizeof(float) * t32.size(),
                             cudaMemcpyHostToDevice, s));
    GPK_CUDA(cudaStreamSynchronize(s));
  }
  const double* s64 = b->sgd_tab.p;
  const double* p64 = b->sgd_tab.p + budget + 1;
  const int tiles = (bs + 127) / 128;
  // d <= 4: the 64-column slab pipeline (GPK_SGD_CH64=0: 32-column chunks)
  static const bool ch64_env = [] {
    const char* e = std::getenv("GPK_SGD_CH64");
    return !(e && std::atoi(e) == 0);
  }();
  const bool ch64 = ch64_env && op->dp == 4;
  // the 64-column slab as CTA pairs (cta_group::2, each CTA builds half of the
  // B operand; GPK_SGD_PAIR=0: one CTA per row tile)
  static const bool pair_env = [] {
    const char* e = std::getenv("GPK_SGD_PAIR");
    return !(e && std::atoi(e) == 0);
  }();
  const bool pair = ch64 && pair_env && kv_tc_npad(m) % 16 == 0;
  const int cq = ch64 ? 64 : 32;
  int splits = std::max(1, ctx->sms / (pair ? (tiles + 1) / 2 * 2 : tiles));
  int cps = (nloc + splits - 1) / splits;
  cps = (cps + cq - 1) / cq * cq;
  splits = std::max(1, (nloc + cps - 1) / cps);
  double* part = b->sgd_part.ensure(static_cast<size_t>(splits) * bs * m);
  const long long stride = (static_cast<long long>(bs) * m + m + 1 + 31) / 32 * 32;  // doubles per rank slice
  double* gbuf = b->w4.ensure(static_cast<size_t>(stride));
  double* red = b->red.ensure(static_cast<size_t>(nr) * G * 2 * m + 8);
  double* sumsq = b->vec1.ensure(m);
  int* flags = b->sgd_flags.ensure(2);
  GPK_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
  unsigned* ticket = b->ticket.ensure(1);
  GPK_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  double* gpart = b->sgd_gpart.ensure(static_cast<size_t>(sgd_finish_blocks(bs)) * m);  // APPLY_ROWS == FIN_ROWS
  col_reduce_launch(b->residuals.p, nullptr, nloc, m, m, 2, red + static_cast<size_t>(op->rk) * G * m, G, nullptr, s);
  gather_inplace(op, red, sizeof(double) * G * m);
  sum_partials_launch(red, G * nr, m, sumsq, nullptr, s);
  init_ctl(b, budget, -1);
  CgCtl* ctl = b->ctl.p;
  sgd_check_launch(sumsq, m, b->scales_dev.p, c->tolerance, flags, ctl, s);  // initial test (loop head)
  const int chunk = 256;
  int* idxbuf = b->ibuf.ensure(static_cast<size_t>(chunk) * bs);

  SgdSlabArgs sa{};
  sa.xs = op->xs32.p;
  sa.n = n;
  sa.dp = op->dp;
  sa.d = op->d;
  sa.idxbuf = idxbuf;
  sa.idx_chunk = chunk;
  sa.R = bs;
  sa.c0 = row0;
  sa.C = nloc;
  sa.rec = rec;
  sa.rw = rw;
  sa.moff = moff;
  sa.tau = tau;
  sa.s32 = b->sgd_s32.p;
  sa.budget = s32_sat < 4096 ? s32_sat : budget;  // Delta clamp: S32(Delta) == S32(s32_sat) beyond it
  sa.ntab = std::min(sa.budget + 1, 4096);         // staged in shared memory (<= 16 KB)
  // Gram-form distances when the padded row has a free slot for |x|^2
  // (GPK_SGD_GRAM=1; measured: no faster at C4 and 8x the distance rounding
  // at d = 11, so direct differences by default)
  static const bool sgd_gram = [] {
    const char* e = std::getenv("GPK_SGD_GRAM");
    return e && std::atoi(e) != 0;
  }();
  if (op->dp == 4) {  // d <= 4: the slab evaluates two columns per FP32x2 instruction from SoA coordinates
    float* xq = b->sgd_xsoa.ensure(static_cast<size_t>(n + 128) * op->dp);
    sgd_soa_image_launch(op->xs32.p, n + 128, op->dp, xq, s);
    sa.xsoa = xq;
  }
  if (sgd_gram && op->d < op->dp) {
    float* xg = b->sgd_xg.ensure(static_cast<size_t>(n + 128) * op->dp);
    sgd_gram_image_launch(op->xs32.p, n + 128, n, op->d, op->dp, xg, s);
    sa.xg = xg;
  }
  sa.ctl = ctl;
  sa.log2_s2 = static_cast<float>(std::log2(op->s2));
  sa.part = part;
  sa.m = m;
  sa.splits = splits;
  sa.cols_per_split = cps;
  static const int flush = [] {
    const char* e = std::getenv("GPK_SGD_FLUSH");  // FP32 TMEM accumulation span in 32-column chunks
    return e ? std::max(5, std::atoi(e)) : 8;
  }();
  sa.flush = ch64 ? std::max(3, flush / 2) : flush;  // same FP32 accumulation span in 64-column chunks
  sa.ch64 = ch64 ? 1 : 0;
  sa.pair = pair ? 1 : 0;
  sa.stats = ctx->stats;
  SgdStepArgs ta{};
  ta.ctl = ctl;
  ta.idxbuf = idxbuf;
  ta.idx_chunk = chunk;
  ta.b = bs;
  ta.m = m;
  ta.row0 = row0;
  ta.nloc = nloc;
  ta.part = part;
  ta.splits = splits;
  ta.resid = b->residuals.p;
  ta.Vb = b->solutions.p;
  ta.Mb = Mb;
  ta.B = b->targets.p;
  ta.tau = tau;
  ta.s64 = s64;
  ta.p64 = p64;
  ta.budget = budget;
  ta.sigma2 = op->sigma2;
  ta.rho = c->momentum;
  ta.step = step;
  ta.tol = c->tolerance;
  // one FP64 all-reduce of the b x m partials (+ old residual squares, flag)
  // per iteration: every rank reads the same sums
  ta.slice = gbuf;
  ta.gbuf = gbuf;
  ta.stride = stride;
  ta.nr = 1;
  ta.sharded = op->sharded ? 1 : 0;
  ta.nonfinite = flags;
  ta.nonfinite_now = flags + 1;
  ta.rec = rec;
  ta.rw = rw;
  ta.moff = moff;
  ta.gpart = gpart;
  ta.ticket = ticket;
  ta.sumsq = sumsq;
  ta.scales = b->scales_dev.p;
  // one rank: reduce + apply fused into one kernel (GPK_SGD_FUSED_FINISH=0: separate)
  static const bool finish_env = [] {
    const char* e = std::getenv("GPK_SGD_FUSED_FINISH");
    return !(e && std::atoi(e) == 0);
  }();
  const bool fused_finish = finish_env && !op->sharded;
  // slab -> finish -> slab chained by programmatic dependent launch: each
  // kernel's launch and prologue (barriers, TMEM, S table, zero B groups)
  // overlap its predecessor's tail (GPK_SGD_PDL=0: plain stream order)
  static const bool pdl_env = [] {
    const char* e = std::getenv("GPK_SGD_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  const bool pdl = pdl_env && fused_finish && ch64 && !ctx->profiling;
  sa.pdl = pdl ? 1 : 0;
  ta.pdl = 0;
  SgdStepArgs tf = ta;
  tf.pdl = pdl ? 1 : 0;
  if (fused_finish) tf.gpart = b->sgd_gpart2.ensure(static_cast<size_t>(sgd_finish_blocks(bs)) * 2 * m);
  int t = 0;
  auto iteration = [&]() {  // solvers.cpp:164-178
    if (t % chunk == 0) sgd_batches_dev_launch(c->seed, c->substream, n, bs, &ctl->iters, chunk, idxbuf, &ctl->stop, s);
    // profiling brackets the slab; GPK_PROF_SGD_FINISH=1 (development) brackets the finish kernel instead
    static const bool prof_finish = [] {
      const char* e = std::getenv("GPK_PROF_SGD_FINISH");
      return e && std::atoi(e) != 0;
    }();
    cudaEvent_t* pe = prof_finish ? nullptr : prof_begin(ctx, s);
    sgd_slab_launch(sa, s);
    if (pe) GPK_CUDA(cudaEventRecord(*pe, s));
    if (fused_finish) {
      pe = prof_finish ? prof_begin(ctx, s) : nullptr;
      sgd_finish_launch(tf, s);
      if (pe) GPK_CUDA(cudaEventRecord(*pe, s));
    } else {
      sgd_reduce_launch(ta, s);
      allreduce_inplace(op, gbuf, static_cast<size_t>(bs) * m + m + 1);
      sgd_apply_launch(ta, s);
    }
    ++t;
  };
  drive(b, ctl, chunk, budget, iteration, true);
  sgd_materialise_launch(b->solutions.p, Mb, tau, s64, budget, ctl, nloc, m, s);
  const CgCtl h = read_ctl(b);
  rep->iterations = h.iters;
  rep->epochs_consumed = static_cast<double>(h.iters) * bs / n;
  rep->aborted = h.aborted;
  if (h.aborted) std::strncpy(rep->abort_reason, "sgd divergence: non-finite iterate", 127);
  finalise(b, c->tolerance, rep, start);
}

void solve_sgd(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* rep) {
  validate(c);
  const auto start = Clock::now();
  gpk_operator* op = b->op;
  cudaStream_t s = op->ctx->stream;
  const int n = op->n, m = b->m, G = kReduceGroups;  // global rows (b->n is the shard on a sharded operator)
  if (m > kMaxRhs) throw InvalidArgument("gpk: batches wider than 65 columns are not supported by the solvers");
  std::memset(rep, 0, sizeof(*rep));
  rep->residuals_estimated = 1;
  const int bs = std::min(c->batch_size, n);
  const double max_iterations = static_cast<double>(c->max_epochs) * n / bs;
  const int budget = static_cast<int>(std::ceil(max_iterations));
  const double step = c->learning_rate / bs;
  if (sgd_lazy_supported(op, m, bs)) return solve_sgd_lazy(b, c, rep, bs, budget, step, start);
  if (op->ctx->kernel == 1) return solve_sgd_tc(b, c, rep, bs, budget, step, start);
  if (op->nr > 1) throw InvalidArgument("gpk: the sharded operator needs the tcgen05 kernel");
  const size_t nm = static_cast<size_t>(n) * m;
  const int ld = kv_ld_for(m);
  GPK_CUDA(cudaMemcpyAsync(b->residuals.p, b->targets.p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, s));
  double* M = b->w1.ensure(nm);
  GPK_CUDA(cudaMemsetAsync(M, 0, sizeof(double) * nm, s));
  float* V32 = b->f32.ensure(static_cast<size_t>(n) * ld);
  to_f32_launch(b->solutions.p, n, m, m, V32, ld, nullptr, s);
  double* hv = b->w2.ensure(static_cast<size_t>(bs) * m);
  double* grad = b->w3.ensure(static_cast<size_t>(bs) * m);
  double* part = b->red.ensure(static_cast<size_t>(G) * 2 * m + 8);
  double* sumsq = b->vec1.ensure(m);
  int* pos = b->ibuf2.ensure(n);
  GPK_CUDA(cudaMemsetAsync(pos, 0xff, sizeof(int) * n, s));  // -1
  int* nonfinite = b->flag.ensure(1);
  GPK_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s));
  col_reduce_launch(b->residuals.p, nullptr, n, m, m, 2, part, G, nullptr, s);
  sum_partials_launch(part, G, m, sumsq, nullptr, s);
  init_ctl(b, budget, -1);
  CgCtl* ctl = b->ctl.p;
  const int* stop = &ctl->stop;
  sgd_check_launch(sumsq, m, b->scales_dev.p, c->tolerance, nonfinite, ctl, s);  // initial test

  const int chunk = 256;
  int* idxbuf = b->ibuf.ensure(static_cast<size_t>(chunk) * bs);
  int t = 0;
  auto iteration = [&]() {  // solvers.cpp:164-178
    if (t % chunk == 0) sgd_batches_launch(c->seed, c->substream, n, bs, t, std::min(chunk, budget - t), idxbuf, s);
    const int* idx = idxbuf + static_cast<size_t>(t % chunk) * bs;
    KvCall kc;
    kc.v = V32;
    kc.m = m;
    kc.row_idx = idx;
    kc.R = bs;
    kc.C = n;
    kc.vdiag = b->solutions.p;
    kc.out = hv;
    kc.ldo = m;
    kc.skip = stop;
    run_kv(op, kc);
    sgd_step_launch(hv, idx, bs, b->targets.p, grad, m, stop, s);
    sgd_scatter_launch(idx, bs, pos, 1, stop, s);
    sgd_update_launch(M, b->solutions.p, V32, ld, pos, grad, c->momentum, step, n, m, nonfinite, stop, s);
    sgd_residual_launch(b->residuals.p, idx, bs, grad, m, sumsq, stop, s);
    sgd_scatter_launch(idx, bs, pos, 0, stop, s);
    sgd_check_launch(sumsq, m, b->scales_dev.p, c->tolerance, nonfinite, ctl, s);
    ++t;
  };
  // Batches of a chunk are generated before its first iteration; the driver
  // must not run ahead past a chunk boundary with a stale buffer, which the
  // in-order stream guarantees.
  drive(b, ctl, std::max(1, iteration_group(n) * 4), budget, iteration);
  const CgCtl h = read_ctl(b);
  rep->iterations = h.iters;
  rep->epochs_consumed = static_cast<double>(h.iters) * bs / n;
  rep->aborted = h.aborted;
  if (h.aborted) std::strncpy(rep->abort_reason, "sgd divergence: non-finite iterate", 127);
  finalise(b, c->tolerance, rep, start);
}

void solve_dispatch(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* rep) {  // solvers.cpp:186-202
  switch (c->kind) {
    case GPK_CG:
      if (c->preconditioner_rank > 0) {
        if (!b->pc) b->pc = std::make_unique<gpk_precond>();
        gpk_precond* pc = b->pc.get();
        pc->op = b->op;
        pc->n = b->n;
        pc->rank = std::min(c->preconditioner_rank, b->op->n);
        build_precond(pc);
        return solve_cg(b, c, pc, rep);
      }
      return solve_cg(b, c, nullptr, rep);
    case GPK_AP:
      return solve_ap(b, c, rep);
    case GPK_SGD:
      return solve_sgd(b, c, rep);
  }
  throw std::logic_error("solve: unknown solver kind");
}

// ------------------------------------------------------------- gradients
// Quadratic forms for pairs given as device FP64 row-major matrices with a
// column offset (so batch solutions can be used in place). out: npairs x (d+2).
struct PairDev {
  const double* u;
  const double* w;
  int ldu, ldw, col0, cols;
};

__global__ void extract_f32_kernel(const double* src, int n, int lds, int col0, int cols, float* dst, int ldd) {
  const long long total = static_cast<long long>(n) * ldd;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / ldd), j = static_cast<int>(e % ldd);
    dst[e] = j < cols ? static_cast<float>(src[static_cast<size_t>(i) * lds + col0 + j]) : 0.f;
  }
}

__global__ void pair_dot_kernel(const double* u, const double* w, int n, int ldu, int ldw, int col0, int cols,
                                double* part) {
  __shared__ double red[256];
  const int g = blockIdx.x, G = gridDim.x;
  const long long rb = static_cast<long long>(n) * g / G, re = static_cast<long long>(n) * (g + 1) / G;
  double acc = 0.0;
  for (long long e = rb * cols + threadIdx.x; e < re * cols; e += blockDim.x) {
    const long long i = e / cols;
    const int j = static_cast<int>(e % cols);
    acc += u[i * ldu + col0 + j] * w[i * ldw + col0 + j];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[g] = red[0];
}

// Pairs are given by this rank's rows (nloc of them). On a sharded operator the
// FP32 copies of U and W are all-gathered to full height (every tile needs all
// columns), the global tile list is split evenly across ranks, and the per-block
// partial sums are all-gathered and summed in (rank, block) order.
// combine (nullable, one coefficient per pair): return the single form
// sum_p combine[p] forms_p -- on the tensor-core pass accumulated per entry.
std::vector<std::vector<double>> quad_forms_dev(gpk_operator* op, const std::vector<PairDev>& pairs,
                                                const double* combine = nullptr) {
  cudaStream_t s = op->ctx->stream;
  const int n = op->n, d = op->d, P = static_cast<int>(pairs.size());
  const int nloc = op->nloc, nr = op->nr, rk = op->rk;
  const int rows_alloc = op->S * nr;  // >= n; slot r holds rows [r*S, r*S + S)
  if (P < 1 || P > 2) throw InvalidArgument("derivative_quadratic_forms: 1 or 2 pairs supported");
  DBuf<float>* bufs = op->gbuf;
  GradArgs a{};
  a.xs = op->xs32.p;
  a.n = n;
  a.d = d;
  a.dp = op->dp;
  a.npairs = P;
  a.symmetric = 1;
  for (int p = 0; p < P; ++p) {
    const PairDev& pd = pairs[p];
    const int ld = (pd.cols + 3) / 4 * 4;
    float* u32 = bufs[2 * p].ensure(static_cast<size_t>(rows_alloc) * ld);
    const long long tot = static_cast<long long>(nloc) * ld;
    const int nb = static_cast<int>(std::min<long long>((tot + 255) / 256, 148 * 16));
    extract_f32_kernel<<<nb, 256, 0, s>>>(pd.u, nloc, pd.ldu, pd.col0, pd.cols, u32 + static_cast<size_t>(op->row0) * ld,
                                          ld);
    check_launch("extract_f32");
    gather_inplace(op, u32, sizeof(float) * op->S * ld);
    const float* w32 = u32;
    if (pd.w != pd.u || pd.ldw != pd.ldu) {
      float* wb = bufs[2 * p + 1].ensure(static_cast<size_t>(rows_alloc) * ld);
      extract_f32_kernel<<<nb, 256, 0, s>>>(pd.w, nloc, pd.ldw, pd.col0, pd.cols,
                                            wb + static_cast<size_t>(op->row0) * ld, ld);
      check_launch("extract_f32");
      gather_inplace(op, wb, sizeof(float) * op->S * ld);
      w32 = wb;
      a.symmetric = 0;
    }
    a.u[p] = u32;
    a.w[p] = w32;
    a.mcols[p] = pd.cols;
    a.ldu[p] = ld;
  }
  a.s2 = static_cast<float>(op->s2);
  a.log2_s2 = static_cast<float>(std::log2(op->s2));
  const int per = P * (d + 1);
  DBuf<double>& part = op->gpart;
  DBuf<double>& tot = op->gtot;
  DBuf<double>& dots = op->gdots;
  // tensor-core pass: one wide pair (1 < s <= 64) and at most one narrow pair
  int pw = -1, pn = -1;
  for (int p = 0; p < P; ++p) {
    if (a.mcols[p] > 1 && pw < 0)
      pw = p;
    else if (a.mcols[p] == 1 && pn < 0)
      pn = p;
  }
  const bool tc = op->ctx->kernel == 1 && pw >= 0 && a.mcols[pw] <= 64 && (P == 1 || pn >= 0);
  const bool comb = tc && combine && P == 2;  // one accumulated form
  const int pk = comb ? d + 1 : per;          // per-block partial entries
  if (tc) {
    GradTcArgs t{};
    t.xs = op->xs32.p;
    t.n = n;
    t.d = d;
    t.dp = op->dp;
    t.ua = a.u[pw];
    t.lda = a.ldu[pw];
    t.cols = a.mcols[pw];
    t.kp = grad_tc_kp(t.cols);
    const int rows_pad = grad_tc_rows_pad(n);
    float* bpk = op->gpk_b.ensure(grad_tc_pack_floats(n, t.kp));
    float* nar = pn >= 0 ? op->gpk_n.ensure(static_cast<size_t>(2) * rows_pad) : nullptr;
    grad_tc_pack_launch(a.w[pw], a.ldu[pw], n, t.cols, t.kp, bpk, pn >= 0 ? a.u[pn] : nullptr,
                        pn >= 0 ? a.w[pn] : nullptr, pn >= 0 ? a.ldu[pn] : 0, nar, nar ? nar + rows_pad : nullptr, s);
    t.bpk = bpk;
    t.u1 = nar;
    t.w1 = nar ? nar + rows_pad : nullptr;
    t.symmetric = a.symmetric;
    t.pw = pw;
    t.pn = pn >= 0 ? pn : 0;
    t.npairs = comb ? 1 : P;
    t.combined = comb ? 1 : 0;
    t.cw = comb ? static_cast<float>(combine[pw]) : 0.f;
    t.cn = comb ? static_cast<float>(combine[pn]) : 0.f;
    t.blocks = op->ctx->sms;
    static const bool grad_dx = [] {  // GPK_GRAD_DX=0: padded-dimension evaluation at d <= 4
      const char* e = std::getenv("GPK_GRAD_DX");
      return !(e && std::atoi(e) == 0);
    }();
    if (grad_dx && op->dp == 4) {  // SoA column coordinates for the exact-dimension path
      const size_t rows = static_cast<size_t>(rows_pad);
      float* xq = op->gpk_xsoa.ensure(rows * 4);
      sgd_soa_image_launch(op->xs32.p, rows_pad, 4, xq, s);
      t.xsoa = xq;
    }
    const long long ntiles = grad_tc_tiles(n, a.symmetric);
    t.tile_begin = ntiles * rk / nr;
    t.tile_end = ntiles * (rk + 1) / nr;
    a.blocks = t.blocks;
    part.ensure(static_cast<size_t>(nr) * a.blocks * pk);
    t.part = part.p + static_cast<size_t>(rk) * a.blocks * pk;
    grad_tc_launch(t, s);
  } else {
    a.blocks = 2 * op->ctx->sms;
    const long long T = (n + 63) / 64;
    const long long ntiles = a.symmetric ? T * (T + 1) / 2 : T * T;
    a.tile_begin = ntiles * rk / nr;
    a.tile_end = ntiles * (rk + 1) / nr;
    part.ensure(static_cast<size_t>(nr) * a.blocks * per);
    a.part = part.p + static_cast<size_t>(rk) * a.blocks * per;
    grad_launch(a, s);
  }
  tot.ensure(pk);
  gather_inplace(op, part.p, sizeof(double) * a.blocks * pk);
  sum_partials_launch(part.p, a.blocks * nr, pk, tot.p, nullptr, s);
  // noise terms: sum u.w (FP64) over this rank's rows, gathered
  const int G = kReduceGroups;
  dots.ensure(static_cast<size_t>(nr) * G * P);
  for (int p = 0; p < P; ++p) {
    pair_dot_kernel<<<G, 256, 0, s>>>(pairs[p].u, pairs[p].w, nloc, pairs[p].ldu, pairs[p].ldw, pairs[p].col0,
                                      pairs[p].cols, dots.p + static_cast<size_t>(rk) * G * P + static_cast<size_t>(p) * G);
    check_launch("pair_dot");
  }
  gather_inplace(op, dots.p, sizeof(double) * G * P);
  std::vector<double> th(pk), dh(static_cast<size_t>(nr) * G * P);
  GPK_CUDA(cudaMemcpyAsync(th.data(), tot.p, sizeof(double) * pk, cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaMemcpyAsync(dh.data(), dots.p, sizeof(double) * nr * G * P, cudaMemcpyDeviceToHost, s));
  GPK_CUDA(cudaStreamSynchronize(s));
  std::vector<double> uw(P, 0.0);
  for (int p = 0; p < P; ++p)
    for (int r = 0; r < nr; ++r)
      for (int g = 0; g < G; ++g) uw[p] += dh[static_cast<size_t>(r) * G * P + static_cast<size_t>(p) * G + g];
  const int nf = comb ? 1 : P;  // forms computed on the device
  std::vector<std::vector<double>> out(nf, std::vector<double>(d + 2, 0.0));
  for (int p = 0; p < nf; ++p) {
    const double u = comb ? combine[0] * uw[0] + combine[1] * uw[1] : uw[p];
    out[p][d + 1] = 2.0 * op->sigma * u;                                      // kernel.cpp:249-252
    out[p][d] = (2.0 / op->s) * (op->s2 * th[static_cast<size_t>(p) * (d + 1) + d]);  // kernel.cpp:264
    for (int k = 0; k < d; ++k)                                                // kernel.cpp:265-268
      out[p][k] = op->inv_ls[k] * (3.0 * op->s2 * th[static_cast<size_t>(p) * (d + 1) + k]);
  }
  if (combine && !comb) {  // combined on the host from the per-pair forms
    std::vector<double> c(d + 2, 0.0);
    for (int p = 0; p < P; ++p)
      for (int k = 0; k < d + 2; ++k) c[k] += combine[p] * out[p][k];
    return {c};
  }
  return out;
}



void assemble(const std::vector<std::vector<double>>& f, int s_count, int P, double* values, double* quad,
              double* trace) {  // gradients.cpp:39-50
  for (int k = 0; k < P; ++k) {
    const double q = f[0][k], t = f[1][k] / s_count;
    if (quad) quad[k] = q;
    if (trace) trace[k] = t;
    if (values) values[k] = 0.5 * q - 0.5 * t;
  }
}

// ------------------------------------------------------------------ RFF
// Normal draw i of RandomStream(seed, stream, substream) (rng.cpp:64-77):
// draw pair q = i/2 takes u64 words 2q and 2q+1 of the Philox stream (block
// q/2), Box-Muller returns the cosine first and the cached sine second. Same
// arithmetic as the sequential stream, so any slice of a stream can be drawn
// on its own (bit-identical to the sequential order).
double gauss_at(uint64_t seed, uint64_t stream, uint64_t sub, uint64_t i) {
  const uint64_t q = i >> 1;
  const U64x4 blk = philox4x64(q >> 1, sub, 0, 0, seed, stream);
  const int w = static_cast<int>(q & 1) * 2;
  const double u1 = static_cast<double>((blk.v[w] >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(blk.v[w + 1] >> 11) * 0x1.0p-53;
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  return (i & 1) ? radius * std::sin(angle) : radius * std::cos(angle);
}

// runs body(lo, hi) over [0, count) on up to 16 host threads
template <class F>
void host_parallel(size_t count, size_t min_per_thread, F body) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const size_t T = std::max<size_t>(1, std::min<size_t>(hw, count / std::max<size_t>(min_per_thread, 1)));
  if (T == 1) {
    body(size_t{0}, count);
    return;
  }
  std::vector<std::thread> pool;
  for (size_t t = 1; t < T; ++t) pool.emplace_back([&, t] { body(count * t / T, count * (t + 1) / T); });
  body(size_t{0}, count / T);
  for (auto& th : pool) th.join();
}

void build_basis_host(gpk_rff_basis* b) {  // rff.cpp:10-34
  const int P = b->pairs, d = b->d, S = b->samples;
  b->freq.assign(static_cast<size_t>(P) * d, 0.0);
  // frequency row p consumes normals [p(3+d), (p+1)(3+d)) of stream kFrequencies:
  // three for the chi-square scale, then d directions
  host_parallel(static_cast<size_t>(P), 64, [&](size_t lo, size_t hi) {
    for (size_t p = lo; p < hi; ++p) {
      const uint64_t base = static_cast<uint64_t>(p) * (3 + d);
      double chi2 = 0.0;
      for (int i = 0; i < 3; ++i) {
        const double g = gauss_at(b->seed, 3, b->substream, base + i);
        chi2 += g * g;
      }
      const double scale = std::sqrt(3.0 / chi2);
      for (int k = 0; k < d; ++k)
        b->freq[static_cast<size_t>(k) * P + p] = scale * gauss_at(b->seed, 3, b->substream, base + 3 + k);
    }
  });
  b->weights.assign(static_cast<size_t>(2 * P) * S, 0.0);
  host_parallel(b->weights.size(), 4096, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) b->weights[i] = gauss_at(b->seed, 4, b->substream, i);
  });
}

// prior (row-major [rows][s]) = F W: FP64 feature rows (rff_features_kernel)
// in chunks of <= 512 MB, contracted with the weights by cuBLAS DGEMM
// (prior^T = W^T F^T in column-major terms; W is stored [samples][2P]).
// prior (row-major [rows][s_count]) = Phi(x) W: the streaming kernel (Phi never
// materialised); GPK_RFF_STREAM=0 selects the earlier features + cuBLAS DGEMM
// path (row chunks of <= 512 MB of Phi) for A/B runs.
void rff_prior_gemm(gpk_ctx* ctx, const double* x64, int rows, int d, const double* fd, int P, const double* W,
                    int s_count, double amplitude, double* prior) {
  cudaStream_t s = ctx->stream;
  static const bool stream_k5 = [] {
    const char* e = std::getenv("GPK_RFF_STREAM");
    return !(e && std::atoi(e) == 0);
  }();
  if (stream_k5) {
    rff_prior_launch(x64, rows, d, fd, P, amplitude, W, 2 * P, s_count, prior, s);
    return;
  }
  const int F = 2 * P;
  const long long chunk = std::max<long long>(1, std::min<long long>(rows, (512LL << 20) / (8LL * F)));
  double* feat = ctx->rff_feat.ensure(static_cast<size_t>(chunk) * F);
  if (cublasSetStream(ctx->blas, s) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  for (long long r0 = 0; r0 < rows; r0 += chunk) {
    const int len = static_cast<int>(std::min<long long>(chunk, rows - r0));
    rff_features_launch(x64 + r0 * d, len, d, fd, P, amplitude, feat, s);
    count_launch();
    const double one = 1.0, zero = 0.0;
    if (cublasDgemm(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, s_count, len, F, &one, W, F, feat, F, &zero,
                    prior + r0 * s_count, s_count) != CUBLAS_STATUS_SUCCESS)
      throw CudaError("cublasDgemm (RFF prior)");
    count_launch();
  }
}

// prior (row-major [n][s]) at the operator's inputs; freq divided by current l.
void rff_prior_dev(gpk_operator* op, gpk_rff_basis* b, int s_count, double* prior) {
  cudaStream_t s = op->ctx->stream;
  const int P = b->pairs, d = op->d;
  std::vector<double> f(static_cast<size_t>(P) * d);  // [d][P], scaled by 1/l
  for (int k = 0; k < d; ++k)
    for (int p = 0; p < P; ++p) f[static_cast<size_t>(k) * P + p] = b->freq[static_cast<size_t>(k) * P + p] * op->inv_ls[k];
  double* fd = b->freq_dev.ensure(f.size());
  GPK_CUDA(cudaMemcpyAsync(fd, f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice, s));
  if (!b->w_dev.p) {
    b->w_dev.ensure(b->weights.size());
    GPK_CUDA(cudaMemcpyAsync(b->w_dev.p, b->weights.data(), sizeof(double) * b->weights.size(),
                             cudaMemcpyHostToDevice, s));
  }
  const double amplitude = op->s / std::sqrt(static_cast<double>(P));  // rff.cpp:47
  // this rank's rows only (all rows on one GPU)
  rff_prior_gemm(op->ctx, op->x64.p + static_cast<size_t>(op->row0) * d, op->nloc, d, fd, P, b->w_dev.p, s_count,
                 amplitude, prior);
  // no synchronisation: the pageable uploads above are staged before return
}

// ------------------------------------------------------------- posterior
// Query points (host column-major p x d) -> pts64 [p][d] raw, pts32 [p+32][dp]
// scaled by the operator's current lengthscales (kernel.cpp:59-61).
void upload_points(gpk_operator* op, const double* points, int p) {
  cudaStream_t s = op->ctx->stream;
  const int d = op->d, dp = op->dp;
  double* p64 = op->pts64.ensure(static_cast<size_t>(p) * d);
  upload_colmajor(op, points, p, d, p64);
  float* p32 = op->pts32.ensure(static_cast<size_t>(p + 32) * dp);
  GPK_CUDA(cudaMemsetAsync(p32, 0, sizeof(float) * (p + 32) * dp, s));
  prescale_launch(p64, p, d, dp, op->inv_ls_dev.p, p32, op->pts64s.ensure(static_cast<size_t>(p) * d), s);
  if (op->dpg) {
    float* pg = op->ptsg32.ensure(static_cast<size_t>(p + 32) * op->dpg);
    GPK_CUDA(cudaMemsetAsync(pg, 0, sizeof(float) * (p + 32) * op->dpg, s));
    gram_image_launch(p32, p, d, dp, op->dpg, pg, s);
  }
}

// out [p][m] = k(P, X) v, v device FP64 [n][m] (cross_kernel_apply, kernel.cpp:72-81; no noise term)
void cross_apply_dev(gpk_operator* op, int p, const double* v64, int m, double* out) {
  KvCall c;
  c.xs_rows = op->pts32.p;
  c.m = m;
  c.R = p;
  c.C = op->n;
  c.vdiag = v64;  // packing source for the tensor-core kernel
  if (op->ctx->kernel != 1) {
    float* v32 = op->v32.ensure(static_cast<size_t>(op->n) * kv_ld_for(m));
    to_f32_launch(v64, op->n, m, m, v32, kv_ld_for(m), nullptr, op->ctx->stream);
    c.v = v32;
  }
  c.out = out;
  c.ldo = m;
  run_kv(op, c);
}

// Prior samples f_j(P), j < s, from the RFF basis at the query points (rff.cpp:56-62).
void prior_at_points(gpk_operator* op, gpk_rff_basis* b, int p, int s_count, double* prior) {
  cudaStream_t s = op->ctx->stream;
  const int P = b->pairs, d = op->d;
  std::vector<double> f(static_cast<size_t>(P) * d);  // [d][P], scaled by 1/l
  for (int k = 0; k < d; ++k)
    for (int q = 0; q < P; ++q) f[static_cast<size_t>(k) * P + q] = b->freq[static_cast<size_t>(k) * P + q] * op->inv_ls[k];
  double* fd = b->freq_dev.ensure(f.size());
  GPK_CUDA(cudaMemcpyAsync(fd, f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice, s));
  if (!b->w_dev.p) {
    b->w_dev.ensure(b->weights.size());
    GPK_CUDA(cudaMemcpyAsync(b->w_dev.p, b->weights.data(), sizeof(double) * b->weights.size(),
                             cudaMemcpyHostToDevice, s));
  }
  const double amplitude = op->s / std::sqrt(static_cast<double>(P));
  rff_prior_gemm(op->ctx, op->pts64.p, p, d, fd, P, b->w_dev.p, s_count, amplitude, prior);
  GPK_CUDA(cudaStreamSynchronize(s));
}

__global__ void posterior_corr_kernel(const double* vy, const double* zhat, int n, int s, double* corr) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * s;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    corr[e] = vy[e / s] - zhat[e];  // v_y - zhat_j (posterior.cpp:24)
}

// samples [p][s] = f_j(P) + k(P, X)(v_y - zhat_j) for all j (posterior.cpp:19-27); basis null: zero prior.
void sample_posterior_dev(gpk_operator* op, gpk_rff_basis* basis, int p, const double* vy_host, const double* zhat_host,
                          int s, double* samples_dev) {
  cudaStream_t st = op->ctx->stream;
  const int n = op->n;
  DBuf<double> vy, z, corr, prior;
  vy.ensure(n);
  z.ensure(static_cast<size_t>(n) * s);
  corr.ensure(static_cast<size_t>(n) * s);
  GPK_CUDA(cudaMemcpyAsync(vy.p, vy_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  upload_colmajor(op, zhat_host, n, s, z.p);
  posterior_corr_kernel<<<std::max(1, std::min(148 * 16, static_cast<int>((static_cast<long long>(n) * s + 255) / 256))),
                          256, 0, st>>>(vy.p, z.p, n, s, corr.p);
  check_launch("posterior_corr");
  cross_apply_dev(op, p, corr.p, s, samples_dev);
  if (basis) {
    prior.ensure(static_cast<size_t>(p) * s);
    prior_at_points(op, basis, p, s, prior.p);
    xi_assemble_launch(samples_dev, prior.p, p, s, 1.0, samples_dev, s, 0, nullptr, st);  // samples += prior
  }
  GPK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* gpk_last_error(void) { return g_err.c_str(); }
const char* gpk_version(void) { return "gpk 0.1 (sm_100a)"; }
int gpk_rhs_ld(int m) { return kv_ld_for(m); }

gpk_status gpk_ctx_create(int device, gpk_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<gpk_ctx>();
    c->device = device;
    GPK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    GPK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError("gpk: libgpk is built for sm_100a (B200); device is sm_" +
                                          std::to_string(prop.major) + std::to_string(prop.minor));
    c->sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("GPK_FUSED_AP")) c->fused_ap = std::atoi(e) != 0;  // A/B switches
    if (const char* e = std::getenv("GPK_SPD_INVERSE")) c->spd_inverse = std::atoi(e);
    if (const char* e = std::getenv("GPK_KV_DEEP")) c->kv_deep = std::atoi(e);
    if (const char* e = std::getenv("GPK_KV_STREAMK")) c->kv_streamk = std::atoi(e) != 0;
    if (const char* e = std::getenv("GPK_AP_PERSISTENT")) c->ap_persistent = std::atoi(e) != 0;
    if (const char* e = std::getenv("GPK_GRAPHS")) c->graphs = std::atoi(e) != 0;
    if (const char* e = std::getenv("GPK_SGD_LAZY")) c->sgd_lazy = std::atoi(e) != 0;
    GPK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    {  // the auxiliary stream (AP block inverses: chains of small latency-bound
       // launches) runs at the highest priority, so its blocks are scheduled
       // between the waves of the main stream's large operator launches
      int lo = 0, hi = 0;
      GPK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const char* e = std::getenv("GPK_AUX_PRIORITY");
      GPK_CUDA(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, (e && std::atoi(e) == 0) ? lo : hi));
    }
    GPK_CUDA(cudaEventCreateWithFlags(&c->ev_m2a, cudaEventDisableTiming));
    GPK_CUDA(cudaEventCreateWithFlags(&c->ev_aux, cudaEventDisableTiming));
    if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate");
    // explicit workspace: cuBLAS calls inside captured CUDA graphs must not allocate
    GPK_CUDA(cudaMalloc(&c->blas_ws, kBlasWorkspace));
    if (cublasSetWorkspace(c->blas, c->blas_ws, kBlasWorkspace) != CUBLAS_STATUS_SUCCESS)
      throw CudaError("cublasSetWorkspace");
    if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate");
    GPK_CUDA(cudaMallocHost(&c->ctl_host, 2 * sizeof(CgCtl)));
    GPK_CUDA(cudaEventCreateWithFlags(&c->ev[0], cudaEventDisableTiming));
    GPK_CUDA(cudaEventCreateWithFlags(&c->ev[1], cudaEventDisableTiming));
    GPK_CUDA(cudaMalloc(&c->stats, 3 * sizeof(double)));
    GPK_CUDA(cudaMemset(c->stats, 0, 3 * sizeof(double)));
    *out = c.release();
  });
}

gpk_status gpk_ctx_destroy(gpk_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->aux);
    cublasDestroy(c->blas);
    cudaFree(c->blas_ws);
    cusolverDnDestroy(c->solver);
    cudaFreeHost(c->ctl_host);
    cudaEventDestroy(c->ev[0]);
    cudaEventDestroy(c->ev[1]);
    for (auto& pr : c->prof) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    cudaFree(c->stats);
    if (c->comm) nccl().comm_destroy(c->comm);
    cudaEventDestroy(c->ev_m2a);
    cudaEventDestroy(c->ev_aux);
    cudaStreamDestroy(c->aux);
    cudaStreamDestroy(c->stream);
    if (c->info_host) cudaFreeHost(c->info_host);
    delete c;
  });
}

gpk_status gpk_ctx_synchronize(gpk_ctx* c) {
  return guarded([&] { GPK_CUDA(cudaStreamSynchronize(c->stream)); });
}
gpk_status gpk_ctx_join(gpk_ctx* c) {
  return guarded([&] {
    GPK_CUDA(cudaSetDevice(c->device));
    GPK_CUDA(cudaEventRecord(c->ev_aux, c->aux));
    GPK_CUDA(cudaStreamWaitEvent(c->stream, c->ev_aux, 0));
  });
}
gpk_status gpk_ctx_launch_count(gpk_ctx* c, long long* out) {
  return guarded([&] { *out = c->launches; });
}
gpk_status gpk_ctx_stream(gpk_ctx* c, void** out) {
  return guarded([&] { *out = static_cast<void*>(c->stream); });
}
gpk_status gpk_ctx_set_operator_kernel(gpk_ctx* c, int kernel) {
  return guarded([&] {
    if (kernel < 0 || kernel > 1) throw InvalidArgument("gpk_ctx_set_operator_kernel: 0 (SIMT) or 1 (tcgen05)");
    c->kernel = kernel;
  });
}
gpk_status gpk_ctx_set_profiling(gpk_ctx* c, int enable) {
  return guarded([&] { c->profiling = enable != 0; });
}
gpk_status gpk_ctx_reset_stats(gpk_ctx* c) {
  return guarded([&] {
    GPK_CUDA(cudaSetDevice(c->device));
    GPK_CUDA(cudaStreamSynchronize(c->stream));
    GPK_CUDA(cudaMemset(c->stats, 0, 3 * sizeof(double)));
    c->prof_used = 0;
  });
}
gpk_status gpk_ctx_stats(gpk_ctx* c, double* out) {
  return guarded([&] {
    GPK_CUDA(cudaSetDevice(c->device));
    GPK_CUDA(cudaStreamSynchronize(c->stream));
    double dev[3];
    GPK_CUDA(cudaMemcpy(dev, c->stats, 3 * sizeof(double), cudaMemcpyDeviceToHost));
    out[0] = dev[0];
    out[1] = dev[1];
    out[4] = dev[2];
    double ms = 0.0;
    for (size_t i = 0; i < c->prof_used; ++i) {
      float t = 0.f;
      GPK_CUDA(cudaEventElapsedTime(&t, c->prof[i].first, c->prof[i].second));
      ms += t;
    }
    out[2] = static_cast<double>(c->prof_used);
    out[3] = ms;
  });
}

gpk_status gpk_comm_unique_id(unsigned char* id128) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    const ncclResult_t r = nccl().get_unique_id(&id);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclGetUniqueId: ") + nccl().error_string(r));
    std::memcpy(id128, &id, sizeof(id));
  });
}

gpk_status gpk_ctx_init_comm(gpk_ctx* ctx, const unsigned char* id128, int nranks, int rank) {
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "gpk_ctx_init_comm: 0 <= rank < nranks");
    GPK_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (ctx->comm) nccl().comm_destroy(ctx->comm);
    const ncclResult_t r = nccl().comm_init_rank(&ctx->comm, nranks, id, rank);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclCommInitRank: ") + nccl().error_string(r));
    ctx->nranks = nranks;
    ctx->rank = rank;
    if (const char* e = std::getenv("GPK_RING_GATHER")) ctx->ring_gather = std::atoi(e) != 0;
    if (!ctx->comm_stream) {
      GPK_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
      GPK_CUDA(cudaEventCreateWithFlags(&ctx->ring_start, cudaEventDisableTiming));
    }
    for (cudaEvent_t e : ctx->ring_ev) cudaEventDestroy(e);
    ctx->ring_ev.assign(nranks, nullptr);
    for (auto& e : ctx->ring_ev) GPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  });
}

gpk_status gpk_shard_rows(int n, int nranks, int rank, int* row0, int* row1) {
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "gpk_shard_rows: 0 <= rank < nranks");
    const int S = (((n + nranks - 1) / nranks) + 31) / 32 * 32;  // whole 32-row operator chunks
    *row0 = std::min(n, rank * S);
    *row1 = std::min(n, (rank + 1) * S);
  });
}

gpk_status gpk_operator_create(gpk_ctx* ctx, const double* inputs, int n, int d, const double* raw,
                               gpk_operator** out) {
  return guarded([&] {
    LaunchScope ls(ctx);
    require(n >= 1 && d >= 1, "KernelOperator: n >= 1 and d >= 1");
    if (d > 32) throw InvalidArgument("gpk: input dimension > 32 is not supported");
    require(all_finite(inputs, static_cast<size_t>(n) * d), "KernelOperator: non-finite input");
    auto op = std::make_unique<gpk_operator>();
    op->ctx = ctx;
    op->n = n;
    op->d = d;
    op->dp = (d + 3) / 4 * 4;
    op->nloc = n;
    op->S = n;
    op->x64.ensure(static_cast<size_t>(n) * d);
    // 128 zero rows of padding: the tensor-core kernels bulk-copy whole 32-row
    // (operator) and 64-row (gradient pass) chunks up to the 128-row tile edge
    op->xs32.ensure(static_cast<size_t>(n + 128) * op->dp);
    GPK_CUDA(cudaMemsetAsync(op->xs32.p, 0, sizeof(float) * (n + 128) * op->dp, ctx->stream));
    op->xs64.ensure(static_cast<size_t>(n) * d);
    op->tg = tg_enabled(d);
    if (op->tg) op->xtg.ensure(tg_image_floats(n, d));
    op->dpg = gram_dp(d);
    if (op->dpg) {
      op->xg32.ensure(static_cast<size_t>(n + 128) * op->dpg);
      GPK_CUDA(cudaMemsetAsync(op->xg32.p, 0, sizeof(float) * (n + 128) * op->dpg, ctx->stream));
    }
    upload_colmajor(op.get(), inputs, n, d, op->x64.p);
    set_hyper(op.get(), raw);
    *out = op.release();
  });
}

gpk_status gpk_operator_set_hyperparameters(gpk_operator* op, const double* raw) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    set_hyper(op, raw);
  });
}

gpk_status gpk_operator_destroy(gpk_operator* op) {
  return guarded([&] { delete op; });
}

gpk_status gpk_operator_set_dense_cache(gpk_operator* op, int enable) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(!op->sharded, "KernelOperator: dense_cache on a row-sharded operator");
    op->dense = enable != 0;
    if (op->dense && dense_dgemm()) {
      dense_block64_launch(op->xs64.p, op->n, op->d, op->s2, op->sigma2, 0, op->n, 0, op->n,
                           op->kdense.ensure(static_cast<size_t>(op->n) * op->n), op->n, 0, op->ctx->stream);
      GPK_CUDA(cudaStreamSynchronize(op->ctx->stream));
    }
  });
}

gpk_status gpk_operator_size(const gpk_operator* op, int* n, int* d) {
  return guarded([&] {
    *n = op->n;
    *d = op->d;
  });
}

gpk_status gpk_apply(gpk_operator* op, const double* v, int m, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(m >= 1, "KernelOperator::apply: m >= 1");
    require(all_finite(v, static_cast<size_t>(op->n) * m), "KernelOperator::apply: non-finite input");  // kernel.cpp:135
    const int n = op->n;
    double* v64 = op->v64.ensure(static_cast<size_t>(n) * m);
    double* o64 = op->out64.ensure(static_cast<size_t>(n) * m);
    upload_colmajor(op, v, n, m, v64);
    std::vector<double> tmp(static_cast<size_t>(n) * std::min(m, kMaxRhs));
    for (int j0 = 0; j0 < m; j0 += kMaxRhs) {
      const int mm = std::min(kMaxRhs, m - j0);
      DBuf<double> sub, so;
      const double* src = v64;
      double* dst = o64;
      if (mm != m) {
        sub.ensure(static_cast<size_t>(n) * mm);
        so.ensure(static_cast<size_t>(n) * mm);
        // gather columns j0..j0+mm of row-major v64
        GPK_CUDA(cudaMemcpy2DAsync(sub.p, sizeof(double) * mm, v64 + j0, sizeof(double) * m, sizeof(double) * mm, n,
                                   cudaMemcpyDeviceToDevice, op->ctx->stream));
        src = sub.p;
        dst = so.p;
      }
      float* v32 = op->v32.ensure(static_cast<size_t>(n) * kv_ld_for(mm));
      apply_dev64(op, src, mm, dst, nullptr, 1.0, v32, nullptr);
      if (mm != m)
        GPK_CUDA(cudaMemcpy2DAsync(o64 + j0, sizeof(double) * m, so.p, sizeof(double) * mm, sizeof(double) * mm, n,
                                   cudaMemcpyDeviceToDevice, op->ctx->stream));
      if (mm != m) GPK_CUDA(cudaStreamSynchronize(op->ctx->stream));
    }
    download_colmajor(op, o64, n, m, out);
  });
}

gpk_status gpk_apply_device(gpk_operator* op, const float* v, int m, double* out, int ldo) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(m >= 1 && m <= kMaxRhs, "gpk_apply_device: 1 <= m <= 65");
    KvCall c;
    c.v = v;
    c.m = m;
    c.R = op->n;
    c.C = op->n;
    c.out = out;
    c.ldo = ldo;
    run_kv(op, c);
  });
}

gpk_status gpk_apply_rows(gpk_operator* op, const int* rows, int count, const double* v, int m, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(m >= 1 && m <= kMaxRhs, "apply_rows: 1 <= m <= 65");
    require(count >= 1, "apply_rows: count >= 1");
    for (int r = 0; r < count; ++r)
      if (rows[r] < 0 || rows[r] >= op->n) throw OutOfRange("apply_rows: row index");
    const int n = op->n;
    cudaStream_t s = op->ctx->stream;
    double* v64 = op->v64.ensure(static_cast<size_t>(n) * m);
    upload_colmajor(op, v, n, m, v64);
    float* v32 = op->v32.ensure(static_cast<size_t>(n) * kv_ld_for(m));
    to_f32_launch(v64, n, m, m, v32, kv_ld_for(m), nullptr, s);
    int* idx = op->idx.ensure(count);
    GPK_CUDA(cudaMemcpyAsync(idx, rows, sizeof(int) * count, cudaMemcpyHostToDevice, s));
    double* o64 = op->out64.ensure(static_cast<size_t>(count) * m);
    KvCall c;
    c.v = v32;
    c.m = m;
    c.row_idx = idx;
    c.R = count;
    c.C = n;
    c.vdiag = v64;
    c.out = o64;
    c.ldo = m;
    run_kv(op, c);
    download_colmajor(op, o64, count, m, out);
  });
}

gpk_status gpk_apply_columns(gpk_operator* op, int c0, int len, const double* u, int m, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(m >= 1 && m <= kMaxRhs, "apply_columns: 1 <= m <= 65");
    if (c0 < 0 || len < 1 || c0 + len > op->n) throw OutOfRange("apply_columns: column range");
    const int n = op->n;
    cudaStream_t s = op->ctx->stream;
    double* u64 = op->v64.ensure(static_cast<size_t>(len) * m);
    upload_colmajor(op, u, len, m, u64);
    float* u32 = op->v32.ensure(static_cast<size_t>(len) * kv_ld_for(m));
    to_f32_launch(u64, len, m, m, u32, kv_ld_for(m), nullptr, s);
    double* o64 = op->out64.ensure(static_cast<size_t>(n) * m);
    KvCall c;
    c.v = u32;
    c.m = m;
    c.R = n;
    c.c0 = c0;
    c.C = len;
    c.vdiag = u64;
    c.out = o64;
    c.ldo = m;
    run_kv(op, c);
    download_colmajor(op, o64, n, m, out);
  });
}

gpk_status gpk_dense_block(gpk_operator* op, int r0, int rows, int c0, int cols, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    if (r0 < 0 || c0 < 0 || rows < 0 || cols < 0 || r0 + rows > op->n || c0 + cols > op->n)
      throw OutOfRange("dense_block: range");
    if (rows == 0 || cols == 0) return;
    double* o = op->out64.ensure(static_cast<size_t>(rows) * cols);
    dense_block64_launch(op->xs64.p, op->n, op->d, op->s2, op->sigma2, r0, rows, c0, cols, o, cols, 1,
                         op->ctx->stream);
    download_colmajor(op, o, rows, cols, out);
  });
}

gpk_status gpk_derivative_apply(gpk_operator* op, int k, const double* v, int m, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    const int n = op->n, d = op->d;
    if (k < 0 || k >= d + 2) throw OutOfRange("KernelOperator::derivative_apply: parameter index");
    require(m >= 1 && m <= 80, "KernelOperator::derivative_apply: 1 <= columns <= 80");
    if (k == d + 1) {  // dH/dsigma = 2 sigma I (kernel.cpp:205-208)
      const double two_sigma = 2.0 * op->sigma;
      for (size_t e = 0; e < static_cast<size_t>(n) * m; ++e) out[e] = two_sigma * v[e];
      return;
    }
    double* v64 = op->v64.ensure(static_cast<size_t>(n) * m);
    upload_colmajor(op, v, n, m, v64);
    double* o = op->out64.ensure(static_cast<size_t>(n) * m);
    const double coef = k == d ? 2.0 / op->s : 3.0 * op->s2 * op->inv_ls[k];
    deriv_apply_launch(op->xs64.p, n, d, k, op->s2, coef, v64, m, o, op->ctx->stream);
    download_colmajor(op, o, n, m, out);
  });
}

gpk_status gpk_kernel_column(gpk_operator* op, int i, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    if (i < 0 || i >= op->n) throw OutOfRange("kernel_column: index");
    double* o = op->out64.ensure(op->n);
    dense_block64_launch(op->xs64.p, op->n, op->d, op->s2, op->sigma2, i, 1, 0, op->n, o, op->n, 0, op->ctx->stream);
    GPK_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * op->n, cudaMemcpyDeviceToHost, op->ctx->stream));
    GPK_CUDA(cudaStreamSynchronize(op->ctx->stream));
  });
}

gpk_status gpk_kernel_diagonal(gpk_operator* op, double* out) {
  return guarded([&] {
    for (int i = 0; i < op->n; ++i) out[i] = op->s2;
  });
}

gpk_status gpk_derivative_quadratic_forms_many(gpk_operator* op, int npairs, const double* const* u,
                                               const double* const* w, const int* cols, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(npairs >= 1 && npairs <= 2, "derivative_quadratic_forms: 1 or 2 pairs supported");
    const int n = op->n;
    std::vector<std::unique_ptr<DBuf<double>>> bufs;
    std::vector<PairDev> pairs;
    for (int p = 0; p < npairs; ++p) {
      require(cols[p] >= 1, "derivative_quadratic_forms: shape mismatch");
      auto ub = std::make_unique<DBuf<double>>();
      ub->ensure(static_cast<size_t>(n) * cols[p]);
      upload_colmajor(op, u[p], n, cols[p], ub->p);
      const double* wp = ub->p;
      if (w[p] != u[p]) {
        auto wb = std::make_unique<DBuf<double>>();
        wb->ensure(static_cast<size_t>(n) * cols[p]);
        upload_colmajor(op, w[p], n, cols[p], wb->p);
        wp = wb->p;
        bufs.push_back(std::move(wb));
      }
      pairs.push_back({ub->p, wp, cols[p], cols[p], 0, cols[p]});
      bufs.push_back(std::move(ub));
    }
    const auto f = quad_forms_dev(op, pairs);
    for (int p = 0; p < npairs; ++p)
      for (int k = 0; k < op->d + 2; ++k) out[static_cast<size_t>(p) * (op->d + 2) + k] = f[p][k];
  });
}

// ---- precond ----
gpk_status gpk_precond_create(gpk_operator* op, int rank, gpk_precond** out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    if (rank < 0 || rank > op->n) throw InvalidArgument("PivotedCholeskyPreconditioner: rank must be in [0, n]");
    auto p = std::make_unique<gpk_precond>();
    p->op = op;
    p->n = op->n;
    p->rank = rank;
    build_precond(p.get());
    *out = p.release();
  });
}
gpk_status gpk_precond_destroy(gpk_precond* p) {
  return guarded([&] { delete p; });
}
gpk_status gpk_precond_info(const gpk_precond* p, int* achieved, int* stopped) {
  return guarded([&] {
    *achieved = p->achieved;
    *stopped = p->stopped;
  });
}
gpk_status gpk_precond_factor(gpk_precond* p, double* factor, int* pivots) {
  return guarded([&] {
    LaunchScope ls(p->op->ctx);
    const int r = p->achieved, n = p->n;
    if (r == 0) return;
    cudaStream_t s = p->op->ctx->stream;
    std::vector<double> h(static_cast<size_t>(n) * p->rank);
    GPK_CUDA(cudaMemcpyAsync(h.data(), p->L.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    std::vector<int> pv(p->rank);
    GPK_CUDA(cudaMemcpyAsync(pv.data(), p->pivots.p, sizeof(int) * p->rank, cudaMemcpyDeviceToHost, s));
    GPK_CUDA(cudaStreamSynchronize(s));
    if (factor)
      for (int k = 0; k < r; ++k)
        for (int i = 0; i < n; ++i) factor[static_cast<size_t>(k) * n + i] = h[static_cast<size_t>(i) * p->rank + k];
    if (pivots) std::memcpy(pivots, pv.data(), sizeof(int) * r);
  });
}
gpk_status gpk_precond_apply(gpk_precond* p, const double* v, int m, double* out) {
  return guarded([&] {
    gpk_operator* op = p->op;
    LaunchScope ls(op->ctx);
    const int n = op->n;
    DBuf<double> v64, o64;
    v64.ensure(static_cast<size_t>(n) * m);
    o64.ensure(static_cast<size_t>(n) * m);
    upload_colmajor(op, v, n, m, v64.p);
    precond_apply_dev(p, op, v64.p, m, o64.p, nullptr);
    download_colmajor(op, o64.p, n, m, out);
  });
}

// ---- batch ----
gpk_status gpk_batch_create(gpk_operator* op, const double* targets, int m, gpk_batch** out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(m >= 1, "LinearSystemBatch: at least one column");
    auto b = std::make_unique<gpk_batch>();
    b->op = op;
    b->n = op->n;
    b->m = m;
    const size_t nm = static_cast<size_t>(op->n) * m;
    b->targets.ensure(nm);
    b->solutions.ensure(nm);
    b->residuals.ensure(nm + static_cast<size_t>(kResidPad) * m);
    upload_colmajor(op, targets, op->n, m, b->targets.p);
    GPK_CUDA(cudaMemsetAsync(b->solutions.p, 0, sizeof(double) * nm, op->ctx->stream));
    GPK_CUDA(cudaMemsetAsync(b->residuals.p, 0, sizeof(double) * (nm + static_cast<size_t>(kResidPad) * m),
                             op->ctx->stream));
    b->scales.resize(m);
    for (int j = 0; j < m; ++j) {  // linear_system.cpp:21
      double acc = 0.0;
      const double* col = targets + static_cast<size_t>(j) * op->n;
      for (int i = 0; i < op->n; ++i) acc += col[i] * col[i];
      b->scales[j] = std::sqrt(acc) + 1e-12;
    }
    b->scales_dev.ensure(m);
    GPK_CUDA(cudaMemcpyAsync(b->scales_dev.p, b->scales.data(), sizeof(double) * m, cudaMemcpyHostToDevice,
                             op->ctx->stream));
    GPK_CUDA(cudaStreamSynchronize(op->ctx->stream));
    *out = b.release();
  });
}
gpk_status gpk_batch_destroy(gpk_batch* b) {
  return guarded([&] { delete b; });
}
gpk_status gpk_batch_warm_start(gpk_batch* b, const double* prev) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    upload_colmajor(b->op, prev, b->n, b->m, b->solutions.p);
    GPK_CUDA(cudaStreamSynchronize(b->op->ctx->stream));
  });
}
gpk_status gpk_batch_warm_start_from(gpk_batch* b, const gpk_batch* prev) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    if (prev->n != b->n || prev->m != b->m) throw InvalidArgument("LinearSystemBatch::warm_start: shape mismatch");
    GPK_CUDA(cudaMemcpyAsync(b->solutions.p, prev->solutions.p, sizeof(double) * b->n * b->m,
                             cudaMemcpyDeviceToDevice, b->op->ctx->stream));
  });
}
gpk_status gpk_batch_refresh_residuals(gpk_batch* b) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    refresh_residuals(b);
    GPK_CUDA(cudaStreamSynchronize(b->op->ctx->stream));
  });
}
gpk_status gpk_batch_get(gpk_batch* b, int which, double* out) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    if (which == 3) {
      if (b->scales_stale) {
        GPK_CUDA(cudaMemcpy(b->scales.data(), b->scales_dev.p, sizeof(double) * b->m, cudaMemcpyDeviceToHost));
        b->scales_stale = false;
      }
      std::memcpy(out, b->scales.data(), sizeof(double) * b->m);
      return;
    }
    const double* src = which == 0 ? b->targets.p : which == 1 ? b->solutions.p : which == 2 ? b->residuals.p : nullptr;
    if (!src) throw OutOfRange("gpk_batch_get: which");
    download_colmajor(b->op, src, b->n, b->m, out);
  });
}
gpk_status gpk_batch_set(gpk_batch* b, int which, const double* in) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    double* dst = which == 0 ? b->targets.p : which == 1 ? b->solutions.p : which == 2 ? b->residuals.p : nullptr;
    if (!dst) throw OutOfRange("gpk_batch_set: which");
    upload_colmajor(b->op, in, b->n, b->m, dst);
    GPK_CUDA(cudaStreamSynchronize(b->op->ctx->stream));
  });
}
gpk_status gpk_termination_check(gpk_batch* b, double tol, double* mean, double* probe, int* done) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    batch_norms(b, b->residuals.p, tol, mean, probe, done);
  });
}

// ---- solvers ----
gpk_status gpk_solve_cg(gpk_batch* b, const gpk_solver_config* c, gpk_precond* p, gpk_solver_report* r) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    solve_cg(b, c, p, r);
  });
}
gpk_status gpk_solve_ap(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* r) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    solve_ap(b, c, r);
  });
}
gpk_status gpk_solve_sgd(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* r) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    solve_sgd(b, c, r);
  });
}
gpk_status gpk_solve(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* r) {
  return guarded([&] {
    LaunchScope ls(b->op->ctx);
    solve_dispatch(b, c, r);
  });
}
gpk_status gpk_sgd_batches(gpk_ctx* ctx, int n, const gpk_solver_config* c, int first, int count, int* out) {
  return guarded([&] {
    LaunchScope ls(ctx);
    const int bs = std::min(c->batch_size, n);
    DBuf<int> buf;
    buf.ensure(static_cast<size_t>(count) * bs);
    sgd_batches_launch(c->seed, c->substream, n, bs, first, count, buf.p, ctx->stream);
    GPK_CUDA(cudaMemcpyAsync(out, buf.p, sizeof(int) * count * bs, cudaMemcpyDeviceToHost, ctx->stream));
    GPK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- gradients ----
gpk_status gpk_estimate_gradient_pathwise(gpk_operator* op, const double* v_y, const double* zhat, int s,
                                          double* values, double* quad, double* trace) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(s >= 1, "estimate_gradient_pathwise: shape mismatch");
    const int n = op->n;
    DBuf<double> vy, z;
    vy.ensure(n);
    z.ensure(static_cast<size_t>(n) * s);
    GPK_CUDA(cudaMemcpyAsync(vy.p, v_y, sizeof(double) * n, cudaMemcpyHostToDevice, op->ctx->stream));
    upload_colmajor(op, zhat, n, s, z.p);
    const auto f = quad_forms_dev(op, {{vy.p, vy.p, 1, 1, 0, 1}, {z.p, z.p, s, s, 0, s}});
    assemble(f, s, op->d + 2, values, quad, trace);
  });
}
gpk_status gpk_estimate_gradient_standard(gpk_operator* op, const double* v_y, const double* sol,
                                          const double* probes, int s, double* values, double* quad, double* trace) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(s >= 1, "estimate_gradient_standard: shape mismatch");
    const int n = op->n;
    DBuf<double> vy, z, pr;
    vy.ensure(n);
    z.ensure(static_cast<size_t>(n) * s);
    pr.ensure(static_cast<size_t>(n) * s);
    GPK_CUDA(cudaMemcpyAsync(vy.p, v_y, sizeof(double) * n, cudaMemcpyHostToDevice, op->ctx->stream));
    upload_colmajor(op, sol, n, s, z.p);
    upload_colmajor(op, probes, n, s, pr.p);
    const auto f = quad_forms_dev(op, {{vy.p, vy.p, 1, 1, 0, 1}, {z.p, pr.p, s, s, 0, s}});
    assemble(f, s, op->d + 2, values, quad, trace);
  });
}
gpk_status gpk_batch_gradient_pathwise(gpk_batch* b, double* values, double* quad, double* trace) {
  return guarded([&] {
    gpk_operator* op = b->op;
    LaunchScope ls(op->ctx);
    require(b->m >= 2, "estimate_gradient_pathwise: shape mismatch");
    const int m = b->m;
    const auto f = quad_forms_dev(op, {{b->solutions.p, b->solutions.p, m, m, 0, 1},
                                       {b->solutions.p, b->solutions.p, m, m, 1, m - 1}});
    assemble(f, m - 1, op->d + 2, values, quad, trace);
  });
}

// ---- RFF ----
gpk_status gpk_rff_basis_build(gpk_ctx* ctx, int d, int m_pairs, int sample_count, uint64_t seed, uint64_t substream,
                               gpk_rff_basis** out) {
  return guarded([&] {
    if (m_pairs < 1) throw InvalidArgument("build_rff_basis: m_pairs >= 1");
    if (sample_count < 1) throw InvalidArgument("build_rff_basis: sample_count >= 1");
    auto b = std::make_unique<gpk_rff_basis>();
    b->ctx = ctx;
    b->d = d;
    b->pairs = m_pairs;
    b->samples = sample_count;
    b->seed = seed;
    b->substream = substream;
    build_basis_host(b.get());
    *out = b.release();
  });
}
gpk_status gpk_rff_basis_destroy(gpk_rff_basis* b) {
  return guarded([&] { delete b; });
}
gpk_status gpk_rff_basis_get(const gpk_rff_basis* b, double* freq, double* weights) {
  return guarded([&] {
    if (freq) std::memcpy(freq, b->freq.data(), sizeof(double) * b->freq.size());
    if (weights) std::memcpy(weights, b->weights.data(), sizeof(double) * b->weights.size());
  });
}
gpk_status gpk_pathwise_targets(gpk_operator* op, gpk_rff_basis* basis, int s, uint64_t seed, uint64_t substream,
                                double* prior, double* noise, double* xi) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    if (s < 1) throw InvalidArgument("pathwise_targets: s >= 1");
    if (s > basis->samples) throw InvalidArgument("pathwise_targets: basis holds fewer samples than requested");
    if (basis->d != op->d) throw InvalidArgument("rff_features: point dimension does not match basis");
    const int n = op->n;
    cudaStream_t st = op->ctx->stream;
    DBuf<double> pr, no, x;
    pr.ensure(static_cast<size_t>(n) * s);
    no.ensure(static_cast<size_t>(n) * s);
    x.ensure(static_cast<size_t>(n) * s);
    rff_prior_dev(op, basis, s, pr.p);
    gaussian_fill_launch(seed, 5, substream, static_cast<int64_t>(n) * s, n, s, no.p, st);
    xi_assemble_launch(pr.p, no.p, n, s, op->sigma, nullptr, 0, 0, x.p, st);
    if (prior) download_colmajor(op, pr.p, n, s, prior);
    if (noise) download_colmajor(op, no.p, n, s, noise);
    if (xi) download_colmajor(op, x.p, n, s, xi);
  });
}

// ---- outer loop (outer_loop.cpp:57-246) ----
}  // extern "C"

struct gpk_optimiser {
  gpk_ctx* ctx = nullptr;
  gpk_outer_config cfg{};
  int n = 0, d = 0, s = 0, P = 0, m = 0;
  std::vector<double> raw, am, av;
  int astep = 0, t = 0;
  bool sgd_halved = false, have_previous = false, have_noise = false, aborted = false;
  uint64_t noise_sub = ~0ull;
  gpk_solver_config sc{};
  std::unique_ptr<gpk_operator> op;
  std::unique_ptr<gpk_batch> batch;
  std::unique_ptr<gpk_rff_basis> basis;
  DBuf<double> prev, prior, noise, probes, ycol;
  // ExactDense prior: fixed weights W [n][s], dense kernel matrix and its factor
  DBuf<double> exact_w, dense, chol, work;
  bool have_exact_w = false;
};

namespace {

void optimiser_init(gpk_optimiser* o, gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                    const gpk_outer_config* cfg, const double* init_constrained) {
  validate(&cfg->solver);
  if (cfg->steps < 0) throw InvalidArgument("optimise: steps >= 0");
  o->ctx = ctx;
  o->cfg = *cfg;
  o->n = n;
  o->d = d;
  o->s = cfg->probe_count;
  o->P = d + 2;
  o->m = o->s + 1;
  if (o->s < 1) throw InvalidArgument("optimise: probe_count >= 1");
  if (cfg->estimator != 1 && (cfg->probe_distribution < 0 || cfg->probe_distribution > 1))
    throw InvalidArgument("gpk_optimise: probe_distribution 0 (Gaussian) or 1 (Rademacher)");
  if (cfg->prior_mode < 0 || cfg->prior_mode > 1)
    throw InvalidArgument("gpk_optimise: prior_mode 0 (random features) or 1 (exact dense)");
  o->raw.resize(o->P);
  for (int k = 0; k < o->P; ++k) o->raw[k] = softplus_inverse(init_constrained ? init_constrained[k] : cfg->init_value);
  o->am.assign(o->P, 0.0);
  o->av.assign(o->P, 0.0);
  o->sc = cfg->solver;
  o->sc.warm_start = cfg->warm_start;
  gpk_operator* opp = nullptr;
  if (gpk_operator_create(ctx, inputs, n, d, o->raw.data(), &opp) != GPK_OK) throw InvalidArgument(g_err);
  o->op.reset(opp);
  if (ctx->comm) {  // row shard of this rank (X stays replicated)
    if (cfg->solver.kind == GPK_AP)
      throw InvalidArgument("gpk_optimise: multi-GPU row sharding is implemented for the CG and SGD solvers");
    if (ctx->kernel != 1) throw InvalidArgument("gpk_optimise: multi-GPU needs the tcgen05 operator kernel");
    opp->sharded = true;
    opp->nr = ctx->nranks;
    opp->rk = ctx->rank;
    gpk_shard_rows(n, ctx->nranks, ctx->rank, &opp->row0, &opp->nloc);
    opp->nloc -= opp->row0;
    opp->S = (((n + ctx->nranks - 1) / ctx->nranks) + 31) / 32 * 32;
    if (opp->nloc < 1) throw InvalidArgument("gpk_optimise: fewer rows than ranks * 32");
  }
  if (!opp->sharded && n <= dense_cache_cap()) {  // outer_loop.cpp:72: options.dense_cache = n <= cap
    opp->dense = true;  // FP64 products (cached matrix + DGEMM; GPK_DENSE_KV64=1: kv64_kernel on the fly)
    if (dense_dgemm())
      dense_block64_launch(opp->xs64.p, n, d, opp->s2, opp->sigma2, 0, n, 0, n,
                           opp->kdense.ensure(static_cast<size_t>(n) * n), n, 0, ctx->stream);
  }
  const int nloc = opp->nloc;
  cudaStream_t stream = ctx->stream;
  o->batch = std::make_unique<gpk_batch>();
  gpk_batch* b = o->batch.get();
  b->op = opp;
  b->n = nloc;
  b->m = o->m;
  const size_t nm = static_cast<size_t>(nloc) * o->m;
  b->targets.ensure(nm);
  b->solutions.ensure(nm);
  b->residuals.ensure(nm + static_cast<size_t>(kResidPad) * o->m);
  GPK_CUDA(cudaMemsetAsync(b->residuals.p, 0, sizeof(double) * (nm + static_cast<size_t>(kResidPad) * o->m), stream));
  b->scales.resize(o->m);
  b->scales_dev.ensure(o->m);
  o->prev.ensure(nm);
  o->ycol.ensure(nloc);
  GPK_CUDA(cudaMemcpyAsync(o->ycol.p, targets + opp->row0, sizeof(double) * nloc, cudaMemcpyHostToDevice, stream));
  GPK_CUDA(cudaMemcpy2DAsync(b->targets.p, sizeof(double) * o->m, o->ycol.p, sizeof(double), sizeof(double), nloc,
                             cudaMemcpyDeviceToDevice, stream));
  o->prior.ensure(static_cast<size_t>(nloc) * o->s);
  o->noise.ensure(static_cast<size_t>(nloc) * o->s);
  GPK_CUDA(cudaStreamSynchronize(stream));
}

// One outer step (outer_loop.cpp:125-238). Returns false once the run aborted.
__global__ void add_diag_kernel(double* a, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[static_cast<size_t>(i) * n + i] += v;
}

// ExactDense prior (outer_loop.cpp:140-153, exact.cpp:52-61): K = dense(H) -
// sigma^2 I in FP64, L = chol(K + jitter mean(diag K) I) for the first jitter
// in 1e-10 .. 1e-6 that factors (cuSOLVER potrf), prior = L W with fixed
// Gaussian weights W from (feature_seed, kPriorSample = 8, substream).
void exact_prior_dev(gpk_optimiser* o, uint64_t substream, double* prior) {
  gpk_ctx* ctx = o->ctx;
  gpk_operator* op = o->op.get();
  cudaStream_t st = ctx->stream;
  const int n = o->n, s = o->s;
  if (op->sharded) throw InvalidArgument("gpk_optimise: the exact dense prior runs on one GPU");
  if (n > 4096) throw InvalidArgument("optimise: exact prior draws need n within the dense cap");
  if (!o->have_exact_w || !o->cfg.warm_start) {
    gaussian_fill_rows_launch(o->cfg.feature_seed, 8, substream, n, s, 0, n, o->exact_w.ensure(static_cast<size_t>(n) * s),
                              st);
    o->have_exact_w = true;
  }
  const size_t nn = static_cast<size_t>(n) * n;
  double* K = o->dense.ensure(nn);
  dense_block64_launch(op->xs64.p, n, op->d, op->s2, op->sigma2, 0, n, 0, n, K, n, 1, st);  // symmetric
  add_diag_kernel<<<(n + 255) / 256, 256, 0, st>>>(K, n, -op->sigma2);
  check_launch("add_diag");
  // every diagonal entry is (s2 + sigma2) - sigma2 (r = 0): their mean is that value
  const double mean_diag = (op->s2 + op->sigma2) - op->sigma2;
  if (cusolverDnSetStream(ctx->solver, st) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnSetStream");
  int lwork = 0;
  double* L = o->chol.ensure(nn);
  if (cusolverDnDpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, L, n, &lwork) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDpotrf_bufferSize");
  double* work = o->work.ensure(static_cast<size_t>(std::max(lwork, 1)));
  int* info = ctx->info.ensure(1);
  bool ok = false;
  for (double jitter = 1e-10; jitter <= 1.0000001e-6; jitter *= 10.0) {
    GPK_CUDA(cudaMemcpyAsync(L, K, sizeof(double) * nn, cudaMemcpyDeviceToDevice, st));
    add_diag_kernel<<<(n + 255) / 256, 256, 0, st>>>(L, n, jitter * mean_diag);
    check_launch("add_diag");
    if (cusolverDnDpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, L, n, work, lwork, info) != CUSOLVER_STATUS_SUCCESS)
      throw CudaError("cusolverDnDpotrf");
    count_launch(2);
    int h = 0;
    GPK_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    GPK_CUDA(cudaStreamSynchronize(st));
    if (h == 0) {
      ok = true;
      break;
    }
  }
  if (!ok) throw NumericError("jittered_kernel_cholesky: factorisation failed beyond 1e-6 jitter");
  // prior (row-major [n][s] = column-major s x n) = (L W)^T^T: prior^T = W^T L^T
  if (cublasSetStream(ctx->blas, st) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream");
  const double one = 1.0;
  if (cublasDtrmm(ctx->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, s, n, &one, L,
                  n, o->exact_w.p, s, prior, s) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrmm (exact prior)");
  count_launch();
}

bool optimiser_one_step(gpk_optimiser* o, double* row) {
  const auto t0 = Clock::now();
  gpk_ctx* ctx = o->ctx;
  cudaStream_t stream = ctx->stream;
  gpk_operator* op = o->op.get();
  gpk_batch* b = o->batch.get();
  const int n = o->n, s = o->s, m = o->m, P = o->P, t = o->t;
  const int nloc = op->nloc;
  const gpk_outer_config& cfg = o->cfg;
  const bool pathwise = cfg.estimator == 1;
  const size_t nm = static_cast<size_t>(nloc) * m;
  g_phase.start(stream);
  set_hyper(op, o->raw.data());
  // AP: factor the diagonal blocks on the auxiliary stream while the targets
  // and the residual refresh run on the main stream
  if (o->sc.kind == GPK_AP && !op->sharded) {
    const int blk = std::min(o->sc.block_size, nloc);
    if (!(b->ap_ready && b->ap_block == blk && b->ap_version == op->hyper_version)) ap_prepare(b, blk);
  }
  g_phase.mark("set_hyper");
  const uint64_t substream = cfg.warm_start ? 0 : static_cast<uint64_t>(t);
  if (pathwise) {
    if (cfg.prior_mode == 1) {  // outer_loop.cpp:140-153 (no RFF basis in this mode)
      exact_prior_dev(o, substream, o->prior.p);
    } else {  // outer_loop.cpp:134-139
      if (!o->basis || !cfg.warm_start) {
        gpk_rff_basis* bp = nullptr;
        if (gpk_rff_basis_build(ctx, o->d, cfg.rff_pairs, s, cfg.feature_seed, substream, &bp) != GPK_OK)
          throw InvalidArgument(g_err);
        o->basis.reset(bp);
      }
      rff_prior_dev(op, o->basis.get(), s, o->prior.p);
    }
    if (!o->have_noise || o->noise_sub != substream) {  // rows of this rank of the n x s draw
      gaussian_fill_rows_launch(cfg.feature_seed, 5, substream, n, s, op->row0, nloc, o->noise.p, stream);
      o->have_noise = true;
      o->noise_sub = substream;
    }
    xi_assemble_launch(o->prior.p, o->noise.p, nloc, s, op->sigma, b->targets.p, m, 1, nullptr, stream);
    g_phase.mark("targets");
  } else {
    if (!o->have_noise || !cfg.warm_start) {
      o->probes.ensure(static_cast<size_t>(nloc) * s);
      if (cfg.probe_distribution == 1)  // gradients.cpp:21-22, rng.cpp:92-96
        rademacher_fill_rows_launch(cfg.probe_seed, 2, substream, n, s, op->row0, nloc, o->probes.p, stream);
      else
        gaussian_fill_rows_launch(cfg.probe_seed, 2, substream, n, s, op->row0, nloc, o->probes.p, stream);
      o->have_noise = true;
    }
    GPK_CUDA(cudaMemcpy2DAsync(b->targets.p + 1, sizeof(double) * m, o->probes.p, sizeof(double) * s,
                               sizeof(double) * s, nloc, cudaMemcpyDeviceToDevice, stream));
  }
  {  // scales = ||b_j|| + eps (linear_system.cpp:21); column sums over all ranks' rows
    const int G = kReduceGroups, nr = op->nr;
    double* part = b->red.ensure(static_cast<size_t>(nr) * G * 2 * m + 8);
    double* ss = b->vec1.ensure(m);
    col_reduce_launch(b->targets.p, nullptr, nloc, m, m, 2, part + static_cast<size_t>(op->rk) * G * m, G, nullptr,
                      stream);
    gather_inplace(op, part, sizeof(double) * G * m);
    sum_partials_launch(part, G * nr, m, ss, nullptr, stream);
    scales_launch(ss, m, b->scales_dev.p, nullptr, stream);  // no host round trip
    b->scales_stale = true;                                   // host copy refreshed on demand
  }
  if (cfg.warm_start && o->have_previous)
    GPK_CUDA(cudaMemcpyAsync(b->solutions.p, o->prev.p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, stream));
  else
    GPK_CUDA(cudaMemsetAsync(b->solutions.p, 0, sizeof(double) * nm, stream));
  GPK_CUDA(cudaMemsetAsync(b->residuals.p, 0, sizeof(double) * nm, stream));
  o->sc.substream = static_cast<uint64_t>(t);
  o->sc.seed = cfg.solver_seed;
  gpk_solver_report rep{};
  g_phase.mark("scales_warm");
  solve_dispatch(b, &o->sc, &rep);
  g_phase.mark("solve");
  const double solver_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  const int stride = 2 * P + 8;
  std::memset(row, 0, sizeof(double) * stride);
  for (int k = 0; k < P; ++k) row[k] = softplus(o->raw[k]);
  row[2 * P + 0] = rep.mean_residual_norm;
  row[2 * P + 1] = rep.probe_residual_norm;
  row[2 * P + 2] = rep.epochs_consumed;
  row[2 * P + 4] = rep.iterations;
  row[2 * P + 5] = rep.aborted;
  bool keep_going = true;
  if (rep.aborted) {
    if (cfg.divergence_policy == 1) {
      o->aborted = true;
      keep_going = false;
    } else if (o->sc.kind == GPK_SGD && !o->sgd_halved) {
      o->sc.learning_rate *= 0.5;
      o->sgd_halved = true;
    }
  } else {
    std::vector<double> g(P);
    std::vector<std::vector<double>> f;
    // values = q/2 - t/(2s) (gradients.cpp:39-50), accumulated as one form
    const double coef[2] = {0.5, -0.5 / s};
    if (pathwise)
      f = quad_forms_dev(op, {{b->solutions.p, b->solutions.p, m, m, 0, 1}, {b->solutions.p, b->solutions.p, m, m, 1, s}},
                         coef);
    else
      f = quad_forms_dev(op, {{b->solutions.p, b->solutions.p, m, m, 0, 1}, {b->solutions.p, b->targets.p, m, m, 1, s}},
                         coef);
    for (int k = 0; k < P; ++k) g[k] = f[0][k];
    g_phase.mark("gradient");
    double inf = 0.0;
    for (int k = 0; k < P; ++k) {
      row[P + k] = g[k];
      inf = std::max(inf, std::abs(g[k]));
    }
    row[2 * P + 3] = inf;
    // raw += adam.update(-raw_gradient(g, raw)) (outer_loop.cpp:42-55, 229-230)
    const double lr = cfg.learning_rate, b1 = 0.9, b2 = 0.999, eps = 1e-8;
    ++o->astep;
    const double ms = 1.0 / (1.0 - std::pow(b1, o->astep));
    const double vs = 1.0 / (1.0 - std::pow(b2, o->astep));
    std::vector<double> upd(P);
    for (int k = 0; k < P; ++k) {
      const double gr = -(g[k] * sigmoid(o->raw[k]));
      o->am[k] = b1 * o->am[k] + (1.0 - b1) * gr;
      o->av[k] = b2 * o->av[k] + (1.0 - b2) * (gr * gr);
      upd[k] = (-lr) * (ms * o->am[k] / (std::sqrt(vs * o->av[k]) + eps));
    }
    for (int k = 0; k < P; ++k) o->raw[k] += upd[k];
    GPK_CUDA(cudaMemcpyAsync(o->prev.p, b->solutions.p, sizeof(double) * nm, cudaMemcpyDeviceToDevice, stream));
    o->have_previous = true;
    // AP: the next step's hyperparameters are known now -- scale the inputs and
    // start factoring its diagonal blocks on the auxiliary stream, so the work
    // overlaps the caller's gap between steps and the next targets/refresh
    if (o->sc.kind == GPK_AP && !op->sharded && t + 1 < cfg.steps) {
      set_hyper(op, o->raw.data());
      ap_prepare(b, std::min(o->sc.block_size, nloc));
    }
    g_phase.mark("adam");
    g_phase.finish();
  }
  GPK_CUDA(cudaStreamSynchronize(stream));
  row[2 * P + 6] = std::chrono::duration<double>(Clock::now() - t0).count();
  row[2 * P + 7] = solver_seconds;
  ++o->t;
  return keep_going;
}

}  // namespace

extern "C" {

gpk_status gpk_optimiser_create(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                                const gpk_outer_config* cfg, const double* init_constrained, gpk_optimiser** out) {
  return guarded([&] {
    LaunchScope ls(ctx);
    auto o = std::make_unique<gpk_optimiser>();
    optimiser_init(o.get(), ctx, inputs, targets, n, d, cfg, init_constrained);
    *out = o.release();
  });
}

gpk_status gpk_optimiser_step(gpk_optimiser* o, int steps, double* trace, int* rows_written) {
  return guarded([&] {
    LaunchScope ls(o->ctx);
    *rows_written = 0;
    const int stride = 2 * o->P + 8;
    for (int k = 0; k < steps && !o->aborted; ++k) {
      const bool go = optimiser_one_step(o, trace + static_cast<size_t>(k) * stride);
      *rows_written = k + 1;
      if (!go) break;
    }
  });
}

gpk_status gpk_optimiser_state(gpk_optimiser* o, double* raw, int* step, int* aborted) {
  return guarded([&] {
    if (raw) std::memcpy(raw, o->raw.data(), sizeof(double) * o->P);
    if (step) *step = o->t;
    if (aborted) *aborted = o->aborted;
  });
}

gpk_status gpk_optimiser_destroy(gpk_optimiser* o) {
  return guarded([&] { delete o; });
}

gpk_status gpk_optimise(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                        const gpk_outer_config* cfg, const double* init_constrained, double* trace, int* rows_written,
                        double* final_raw, int* aborted) {
  return guarded([&] {
    LaunchScope ls(ctx);
    gpk_optimiser o;
    optimiser_init(&o, ctx, inputs, targets, n, d, cfg, init_constrained);
    *rows_written = 0;
    const int stride = 2 * o.P + 8;
    for (int k = 0; k < cfg->steps; ++k) {
      const bool go = optimiser_one_step(&o, trace + static_cast<size_t>(k) * stride);
      *rows_written = k + 1;
      if (!go) break;
    }
    std::memcpy(final_raw, o.raw.data(), sizeof(double) * o.P);
    *aborted = o.aborted;
  });
}

gpk_status gpk_cross_apply(gpk_operator* op, const double* points, int p, const double* v, int m, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(p >= 1 && m >= 1 && m <= kMaxRhs, "cross_kernel_apply: 1 <= m <= 65 and p >= 1");
    const int n = op->n;
    upload_points(op, points, p);
    DBuf<double> v64, o64;
    v64.ensure(static_cast<size_t>(n) * m);
    o64.ensure(static_cast<size_t>(p) * m);
    upload_colmajor(op, v, n, m, v64.p);
    cross_apply_dev(op, p, v64.p, m, o64.p);
    download_colmajor(op, o64.p, p, m, out);
  });
}

gpk_status gpk_predict_mean(gpk_operator* op, const double* points, int p, const double* v_y, double* out) {
  return gpk_cross_apply(op, points, p, v_y, 1, out);
}

gpk_status gpk_sample_posterior(gpk_operator* op, gpk_rff_basis* basis, const double* points, int p,
                                const double* v_y, const double* zhat, int s, double* out) {
  return guarded([&] {
    LaunchScope ls(op->ctx);
    require(p >= 1 && s >= 1 && s <= kMaxRhs, "sample_posterior: 1 <= s <= 65 and p >= 1");
    if (basis && (basis->d != op->d || s > basis->samples))
      throw InvalidArgument("sample_posterior: basis does not match the samples");
    upload_points(op, points, p);
    DBuf<double> smp;
    smp.ensure(static_cast<size_t>(p) * s);
    sample_posterior_dev(op, basis, p, v_y, zhat, s, smp.p);
    download_colmajor(op, smp.p, p, s, out);
  });
}

gpk_status gpk_test_metrics(gpk_operator* op, gpk_rff_basis* basis, const double* points, int p,
                            const double* targets, const double* v_y, const double* zhat, int s, double target_scale,
                            double* out4) {
  return guarded([&] {  // posterior.cpp:29-59
    LaunchScope ls(op->ctx);
    require(p >= 1, "test_metrics: p >= 1");
    std::vector<double> mean(p);
    {
      gpk_status st = gpk_predict_mean(op, points, p, v_y, mean.data());
      if (st != GPK_OK) throw InvalidArgument(g_err);
    }
    std::vector<double> err(p);
    double se = 0.0;
    for (int i = 0; i < p; ++i) {
      err[i] = targets[i] - mean[i];
      se += err[i] * err[i];
    }
    out4[0] = std::sqrt(se / p);
    out4[2] = out4[0] * target_scale;
    out4[1] = out4[3] = std::nan("");
    if (s >= 2 && basis) {
      std::vector<double> smp(static_cast<size_t>(p) * s);
      gpk_status st = gpk_sample_posterior(op, basis, points, p, v_y, zhat, s, smp.data());
      if (st != GPK_OK) throw InvalidArgument(g_err);
      const double noise_var = op->sigma2;
      double llh = 0.0;
      for (int i = 0; i < p; ++i) {
        double mu = 0.0;
        for (int j = 0; j < s; ++j) mu += smp[static_cast<size_t>(j) * p + i];
        mu /= s;
        double var = 0.0;
        for (int j = 0; j < s; ++j) {
          const double t = smp[static_cast<size_t>(j) * p + i] - mu;
          var += t * t;
        }
        var = var / (s - 1) + noise_var;
        llh += -0.5 * std::log(2.0 * 3.141592653589793 * var) - 0.5 * err[i] * err[i] / var;
      }
      out4[1] = llh / p;
      out4[3] = out4[1] - std::log(target_scale);
    }
  });
}

// ---------------------------------------------- exact MLL (row f4, exact.cpp)
namespace {

struct ExactWork {
  DBuf<double> H, alpha, y, work, part;
  DBuf<int> info;
};

// exact_gradient (exact.cpp:33-50) for the operator's current hyperparameters:
// H = dense (FP64), Cholesky, alpha = H^-1 y, H^-1 (potri), then one fused
// pass sum_ij W_ij dH_ij/dtheta with W = (alpha alpha^T - H^-1) / 2.
std::vector<double> exact_gradient_dev(gpk_operator* op, ExactWork& w) {
  gpk_ctx* ctx = op->ctx;
  cudaStream_t st = ctx->stream;
  const int n = op->n, d = op->d;
  const size_t nn = static_cast<size_t>(n) * n;
  double* H = w.H.ensure(nn);
  dense_block64_launch(op->xs64.p, n, d, op->s2, op->sigma2, 0, n, 0, n, H, n, 1, st);  // symmetric
  if (cusolverDnSetStream(ctx->solver, st) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnSetStream");
  int lw1 = 0, lw2 = 0;
  if (cusolverDnDpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, H, n, &lw1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, H, n, &lw2) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDn buffer size");
  const int lwork = std::max(1, std::max(lw1, lw2));
  double* work = w.work.ensure(static_cast<size_t>(lwork));
  int* info = w.info.ensure(1);
  if (cusolverDnDpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, H, n, work, lwork, info) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDpotrf");
  int h = 0;
  GPK_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  GPK_CUDA(cudaStreamSynchronize(st));
  if (h != 0) throw NumericError("build_dense_problem: H is not positive definite");
  double* alpha = w.alpha.ensure(n);
  GPK_CUDA(cudaMemcpyAsync(alpha, w.y.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (cusolverDnDpotrs(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, 1, H, n, alpha, n, info) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDpotrs");
  if (cusolverDnDpotri(ctx->solver, CUBLAS_FILL_MODE_LOWER, n, H, n, work, lwork, info) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDpotri");
  count_launch(3);
  const long long blocks = exact_forms_blocks(n);
  double* part = w.part.ensure(static_cast<size_t>(blocks) * (d + 2));
  exact_forms_launch(op->xs64.p, n, d, H, alpha, part, st);
  std::vector<double> hp(static_cast<size_t>(blocks) * (d + 2));
  GPK_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, st));
  GPK_CUDA(cudaStreamSynchronize(st));
  std::vector<double> sum(d + 2, 0.0);
  for (long long b = 0; b < blocks; ++b)  // fixed block order
    for (int k = 0; k < d + 2; ++k) sum[k] += hp[static_cast<size_t>(b) * (d + 2) + k];
  std::vector<double> g(d + 2);
  for (int k = 0; k < d; ++k) g[k] = 3.0 * op->s2 * op->inv_ls[k] * sum[k];  // kernel.cpp:222-228
  g[d] = (2.0 / op->s) * op->s2 * sum[d];                                     // kernel.cpp:215-217
  g[d + 1] = 2.0 * op->sigma * sum[d + 1];                                    // kernel.cpp:207-209
  return g;
}

// optimise_exact (outer_loop.cpp:248-262) on a device-resident dataset.
std::vector<double> optimise_exact_dev(gpk_ctx* ctx, const double* inputs_colmajor, const double* targets, int n, int d,
                                       std::vector<double> raw, int steps, double lr, double* trajectory) {
  gpk_operator* opp = nullptr;
  if (gpk_operator_create(ctx, inputs_colmajor, n, d, raw.data(), &opp) != GPK_OK) throw InvalidArgument(g_err);
  std::unique_ptr<gpk_operator> op(opp);
  ExactWork w;
  w.y.ensure(n);
  GPK_CUDA(cudaMemcpyAsync(w.y.p, targets, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  const int P = d + 2;
  std::vector<double> m(P, 0.0), v(P, 0.0);
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  for (int t = 0; t < steps; ++t) {
    set_hyper(op.get(), raw.data());
    if (trajectory)
      for (int k = 0; k < P; ++k) trajectory[static_cast<size_t>(t) * P + k] = softplus(raw[k]);
    const std::vector<double> g = exact_gradient_dev(op.get(), w);
    const double ms = 1.0 / (1.0 - std::pow(b1, t + 1)), vs = 1.0 / (1.0 - std::pow(b2, t + 1));
    std::vector<double> upd(P);
    for (int k = 0; k < P; ++k) {  // outer_loop.cpp:42-55 on -raw_gradient
      const double gr = -(g[k] * sigmoid(raw[k]));
      m[k] = b1 * m[k] + (1.0 - b1) * gr;
      v[k] = b2 * v[k] + (1.0 - b2) * (gr * gr);
      upd[k] = (-lr) * (ms * m[k] / (std::sqrt(vs * v[k]) + eps));
    }
    for (int k = 0; k < P; ++k) raw[k] += upd[k];
  }
  return raw;
}

}  // namespace

gpk_status gpk_optimise_exact(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                              const double* init_constrained, int steps, double learning_rate, double* trajectory,
                              double* final_raw) {
  return guarded([&] {
    LaunchScope ls(ctx);
    require(ctx && inputs && targets && final_raw && n >= 1 && d >= 1 && steps >= 0, "optimise_exact: arguments");
    std::vector<double> raw(d + 2);
    for (int k = 0; k < d + 2; ++k) raw[k] = softplus_inverse(init_constrained ? init_constrained[k] : 1.0);
    raw = optimise_exact_dev(ctx, inputs, targets, n, d, raw, steps, learning_rate, trajectory);
    std::memcpy(final_raw, raw.data(), sizeof(double) * (d + 2));
  });
}

gpk_status gpk_init_heuristic(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d, int n_centroids,
                              int subset, uint64_t seed, int adam_steps, double learning_rate, double* constrained) {
  return guarded([&] {
    LaunchScope ls(ctx);
    require(ctx && inputs && targets && constrained && n >= 1 && d >= 1 && n_centroids >= 1 && subset >= 1,
            "init_heuristic: arguments");
    const int P = d + 2;
    const std::vector<double> init(P, softplus_inverse(1.0));
    if (subset >= n) {  // outer_loop.cpp:268-270
      const std::vector<double> raw = optimise_exact_dev(ctx, inputs, targets, n, d, init, adam_steps, learning_rate,
                                                         nullptr);
      for (int k = 0; k < P; ++k) constrained[k] = softplus(raw[k]);
      return;
    }
    HostStream stream(seed, 9, 0);  // kCentroids
    std::vector<double> acc(P, 0.0), local_x(static_cast<size_t>(subset) * d), local_y(subset);
    std::vector<int> order(n);
    std::vector<double> dist2(n);
    for (int c = 0; c < n_centroids; ++c) {
      const int centroid = static_cast<int>(stream.next_u64() % static_cast<uint64_t>(n));
      for (int i = 0; i < n; ++i) {  // squared distance in column order (inputs column-major)
        double s2 = 0.0;
        for (int k = 0; k < d; ++k) {
          const double t = inputs[static_cast<size_t>(k) * n + i] - inputs[static_cast<size_t>(k) * n + centroid];
          s2 += t * t;
        }
        dist2[i] = s2;
      }
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dist2[a] < dist2[b]; });
      for (int i = 0; i < subset; ++i) {
        for (int k = 0; k < d; ++k) local_x[static_cast<size_t>(k) * subset + i] = inputs[static_cast<size_t>(k) * n + order[i]];
        local_y[i] = targets[order[i]];
      }
      const std::vector<double> raw = optimise_exact_dev(ctx, local_x.data(), local_y.data(), subset, d, init,
                                                         adam_steps, learning_rate, nullptr);
      for (int k = 0; k < P; ++k) acc[k] += softplus(raw[k]);
    }
    for (int k = 0; k < P; ++k) {
      const double mean = acc[k] / n_centroids;
      constrained[k] = softplus(softplus_inverse(mean));  // Hyperparameters::from_constrained round trip
    }
  });
}

gpk_status gpk_spd_inverse(gpk_ctx* ctx, const double* mats, int dim, int batch, int mode, double* inv) {
  return guarded([&] {
    require(ctx && mats && inv && dim >= 1 && batch >= 1, "gpk_spd_inverse: invalid arguments");
    GPK_CUDA(cudaSetDevice(ctx->device));
    const size_t bb = static_cast<size_t>(dim) * dim * batch;
    DBuf<double> a, o, x;
    a.ensure(bb);
    o.ensure(bb);
    GPK_CUDA(cudaMemcpy(a.p, mats, sizeof(double) * bb, cudaMemcpyHostToDevice));
    if (mode == 1)
      spd_inverse_recursive(ctx, ctx->stream, a.p, dim, batch, o.p,
                            x.ensure(static_cast<size_t>(std::max<long long>(1, spd_inverse_scratch(dim))) * batch));
    else
      spd_inverse_batched(ctx, ctx->stream, a.p, dim, batch, o.p);
    GPK_CUDA(cudaStreamSynchronize(ctx->stream));
    spd_inverse_check(ctx, batch);
    GPK_CUDA(cudaMemcpy(inv, o.p, sizeof(double) * bb, cudaMemcpyDeviceToHost));
  });
}

// trace.cpp:7-44: shortest round-trip doubles, same header and columns.
gpk_status gpk_write_trace_csv(const char* path, const double* trace, int rows, int d) {
  return guarded([&] {
    auto fmt = [](double value) {
      char buffer[40];
      for (int precision = 15; precision <= 17; ++precision) {
        std::snprintf(buffer, sizeof(buffer), "%.*g", precision, value);
        double parsed = 0.0;
        std::sscanf(buffer, "%lf", &parsed);
        if (parsed == value) return std::string(buffer);
      }
      std::snprintf(buffer, sizeof(buffer), "%.17g", value);
      return std::string(buffer);
    };
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error(std::string("gpk_write_trace_csv: cannot open ") + path);
    std::string h = "step";
    for (int i = 0; i < d; ++i) h += ",lengthscale_" + std::to_string(i);
    h += ",signal_scale,noise_scale,mean_residual_norm,probe_residual_norm,epochs";
    h += ",solver_seconds_cum,total_seconds_cum,test_rmse,test_llh,grad_inf_norm,diverged";
    std::fprintf(f, "%s\n", h.c_str());
    const int P = d + 2, stride = 2 * P + 8;
    double solver_cum = 0.0, total_cum = 0.0;
    for (int t = 0; t < rows; ++t) {
      const double* r = trace + static_cast<size_t>(t) * stride;
      solver_cum += r[2 * P + 7];
      total_cum += r[2 * P + 6];
      std::string line = std::to_string(t);
      for (int k = 0; k < P; ++k) line += "," + fmt(r[k]);
      line += "," + fmt(r[2 * P + 0]) + "," + fmt(r[2 * P + 1]) + "," + fmt(r[2 * P + 2]);
      line += "," + fmt(solver_cum) + "," + fmt(total_cum) + ",,";
      line += "," + fmt(r[2 * P + 3]) + "," + (r[2 * P + 5] != 0.0 ? "1" : "0");
      std::fprintf(f, "%s\n", line.c_str());
    }
    std::fclose(f);
  });
}

gpk_status gpk_sinsum_dataset(int n, int d, int uniform, double noise, uint64_t seed, float* x_rowmajor, float* yout) {
  return guarded([&] {
    require(n >= 1 && d >= 1, "gpk_sinsum_dataset: n >= 1 and d >= 1");
    auto gauss = [](HostStream& st) -> double {  // rng.cpp:64-77
      if (st.has_cached) {
        st.has_cached = false;
        return st.cached;
      }
      const double u1 = static_cast<double>((st.next_u64() >> 11) + 1) * 0x1.0p-53;
      const double u2 = static_cast<double>(st.next_u64() >> 11) * 0x1.0p-53;
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * 3.141592653589793 * u2;
      st.cached = radius * std::sin(angle);
      st.has_cached = true;
      return radius * std::cos(angle);
    };
    std::vector<double> x(static_cast<size_t>(n) * d);  // column-major fill order
    HostStream xs(seed, 7, 0);
    if (uniform) {
      for (auto& v : x) v = 2.0 * (static_cast<double>(xs.next_u64() >> 11) * 0x1.0p-53) - 1.0;
    } else {
      for (auto& v : x) v = gauss(xs);
    }
    std::vector<double> w(static_cast<size_t>(d) * 4);
    HostStream ws(seed, 7, 1);
    for (auto& v : w) v = gauss(ws);
    const double wscale = 1.0 / std::sqrt(static_cast<double>(d));
    std::vector<double> eps(n);
    HostStream es(seed, 7, 2);
    for (auto& v : eps) v = gauss(es);
    std::vector<double> yy(n);
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k < 4; ++k) {
        double dot = 0.0;
        for (int q = 0; q < d; ++q)
          dot += x[static_cast<size_t>(q) * n + i] * (w[static_cast<size_t>(k) * d + q] * wscale);
        acc += std::sin(dot);
      }
      yy[i] = acc + noise * eps[i];
    }
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
    for (int i = 0; i < n; ++i) yout[i] = static_cast<float>((yy[i] - mean) / scale);
  });
}

}  // extern "C"

