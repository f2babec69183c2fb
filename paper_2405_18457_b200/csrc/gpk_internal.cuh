// Internal declarations shared by the CUDA kernels and the host C++ of libgpk.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace gpk {

struct CgCtl;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define GPK_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::gpk::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

// Launch-count bookkeeping (bench.py reports gpu_launches).
extern thread_local long long* g_launch_counter;
inline void count_launch(int k = 1) {
  if (g_launch_counter) *g_launch_counter += k;
}
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
}

constexpr double kSqrt3 = 1.7320508075688772;

// ---- operator slab (K1/K2/K3) -------------------------------------------
// out_part[split][r][j] = sum over the split's columns c of k(x_row(r), x_c) v[c - c0][j]
// (kernel only; the sigma^2 diagonal is added by kv_reduce).
struct KvArgs {
  const float* xs;     // scaled inputs FP32 [n][dp]
  int n, dp;
  const int* row_idx;  // device row indices (SGD) or null
  int r0, R;           // rows r0..r0+R (when row_idx null)
  int c0, C;           // column range
  const int* sel;      // device block index (AP) or null: c0 = *sel*sel_block
  int sel_block;
  const float* v;      // FP32 RHS [C][ldv]; row (c - c0) <-> column c
  int ldv, m;
  float log2_s2;       // log2(signal variance)
  double* part;        // [splits][R][m]
  int splits, cols_per_split, flush_chunks;
  int sk_ctas;         // stream-K launch (MODE 3): persistent CTAs
  const int* skip;     // device flag: nonzero => no-op (solver predication)
  double* stats;       // device counters [evals x RHS, algorithmic flops] or null
  int d;               // true input dimension (flop accounting)
  const float* xs_rows;  // scaled FP32 inputs of the rows (cross kernel k(P, X)); null: xs
  const float* xtg;      // tensor-core Gram column images (tg_image_kernel) or null; needs c0 % 32 == 0
};
int kv_tc_for(int m);        // columns-per-lane template parameter for m
int kv_ld_for(int m);        // FP32 RHS leading dimension for m
void kv_slab_launch(const KvArgs& a, int dmax, cudaStream_t s);
int kv_choose_splits(int R, int C, int sms, int rows_per_cta = 256);
int kv_tc_choose_splits(int R, int C, int sms, int ctas_per_sm = 2);

// tcgen05 (3xTF32) variant of the operator slab (kv_tc_kernel.cu)
int kv_tc_npad(int m);
size_t kv_tc_pack_floats(int m, int rows);
void kv_tc_pack_launch(const double* v64, const float* v32, int ldv, int rows_max, int m, const int* sel,
                       int sel_block, int n, float* vpk, const int* skip, cudaStream_t s, int rows_valid = -1);
void kv_tc_launch(const KvArgs& a, const float* vpk, cudaStream_t s, int mode = 0);  // 0 normal, 2 deep, 3 stream-K (grid = a.sk_G)
struct KvReduceArgs;
// stream-K decomposition of a full operator product (kv_tc_kernel MODE 3):
// U = tiles x Q chunk units over G persistent CTAs, CTA b owns units
// [b U / G, (b + 1) U / G); tile t is split among CTAs sk_first(t)..sk_last(t)
__host__ __device__ inline long long sk_first(long long t, int Q, int G, long long U) {
  return ((t * Q + 1) * G - 1) / U;
}
__host__ __device__ inline long long sk_last(long long t, int Q, int G, long long U) {
  return (((t + 1) * Q) * G - 1) / U;
}
// AP slab with the reduce fused into the tensor-core kernel (splits == 1,
// one accumulation group, score_block a multiple of 128): writes out, the
// per-tile dpart/spart partials and runs the AP epilogue in the last CTA.
void kv_tc_fused_launch(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s);

struct KvReduceArgs {
  const double* part;
  int splits, R, m;
  // stream-K operator launch (kv_tc_kernel MODE 3): tile t's partials are the
  // split slots 0..nseg(t)-1 written by CTAs sk_first(t).. (sk_G == 0: splits)
  int sk_G, sk_Q;
  long long sk_U;
  const double* vdiag;  // FP64 RHS for the diagonal term, [C][ldvd] (row c - c0), or null
  int ldvd;
  const float* vdiag32; // fallback FP32 RHS for the diagonal
  int ldv32;
  const int* row_idx;
  int r0, c0, C;
  const int* sel;
  int sel_block, n;
  double sigma2;
  double* out;
  int ldo;
  const double* base;   // out = base + alpha * (H v)
  int ldb;
  double alpha;
  const int* skip;
  int vshift;           // diagonal RHS row = gi - c0 - vshift (row shard offset)
  int nodiag;           // cross kernel k(P, X): no sigma^2 diagonal
  // optional fused column reduction of the result: dpart[g][j] = sum over the
  // group's rows of out[r][j] * w[r][j] (w = dotw, or out itself when
  // dotw == out). Deterministic grouping as col_reduce.
  const double* dotw;
  double* dpart;
  int groups;
  // optional AP block scores (solvers.cpp:123-132): spart[g] = sum over the
  // group's rows of (sum_j out[r][j] * inv_scales[j])^2. Groups are then laid
  // out inside AP blocks: gpb groups per block of `score_block` rows.
  const double* inv_scales;
  double* spart;
  int score_block, gpb;
  // optional fused AP epilogue, run by the last block to finish (ticket):
  // iteration count + termination test (ap_check) and next block choice
  // (ap_select) from the complete partials, in a fixed order.
  CgCtl* ctl;
  const double* scales;
  double tol;
  int* sel_out;
  int nblocks;
  unsigned* ticket;
  // and the next block update's batched-GEMM pointers: {R + sel*b*m, Hinv[sel], upd}
  double** ap_ptrs;
  double* ap_inv;
  long long ap_bb;
  double* ap_upd;
};
void kv_reduce_launch(const KvReduceArgs& a, cudaStream_t s);
// tensor-core Gram-distance operator kernels (kv_tc_tg.cu); mode as kv_tc_launch, 1 = fused AP slab
void kv_tc_tg_launch(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s, int mode);

// ---- gradient pass (K4) ---------------------------------------------------
struct GradArgs {
  const float* xs;      // [n][dp] scaled FP32
  int n, d, dp;
  const float* u[2];    // per pair: [n][ldu] FP32
  const float* w[2];
  int mcols[2], ldu[2];
  int npairs;
  int symmetric;        // all pairs have U == W
  float log2_s2, s2;
  double* part;         // [blocks][npairs*(d+1)]
  int blocks;
  long long tile_begin, tile_end;  // global tile range of this rank (tile_end < 0: all tiles)
};
void grad_launch(const GradArgs& a, cudaStream_t s);

// Persistent AP solver (ap_persistent.cu): one cooperative launch per solve.
struct ApPersistArgs {
  const float* xs;        // scaled inputs FP32 [n + 128][dp]
  int n, d, dp, m, npad;
  float log2_s2;
  double sigma2;
  int block, nblocks, gpb, budget;
  double* R;              // residuals [n + pad][m] (read and updated)
  double* V;              // solutions [n][m]
  const double* inv;      // block inverses [nblocks][block][block]
  long long bb;
  double* upd;            // [block][m]
  double* cpart;          // [8][block][m] phase-C1 partials
  float* vpk;             // TF32 images of upd
  double* dpart;          // [tiles][m]
  double* spart;          // [nblocks * gpb]
  const double* inv_scales;
  const double* scales;
  double tol;
  CgCtl* ctl;
  int* sel;
  unsigned* gbar;         // [0] grid-barrier arrivals, [1] slab ticket, [2] decision flag, [3] sel, [4] stop (zeroed)
  double* stats;          // evals x RHS, FP32-equivalent flops, FP32-pipe flops
  unsigned long long* prof;  // optional phase clock (ns, CTA 0): C, sync1, S, sync2, B, iterations
  const float* xtg;       // tensor-core Gram column images (tg_image_launch) or null; xs plain when set
};
bool ap_persistent_supported(int n, int m, int block, int sms);
void ap_persistent_launch(const ApPersistArgs& a, cudaStream_t s);

// Tensor-core gradient pass (grad_tc_kernel.cu): one wide pair (G on tcgen05)
// plus optionally one narrow (single-column) pair.
struct GradTcArgs {
  const float* xs;      // [rows_pad][dp] scaled FP32 (zero rows beyond n)
  int n, d, dp;
  const float* ua;      // wide pair U rows, FP32 [n][lda]
  int lda, cols;
  const float* bpk;     // wide pair W, packed TF32 hi|lo images per 64-row chunk
  int kp;               // cols rounded up to 16
  const float* u1;      // narrow pair U, W as contiguous [rows_pad] (nullptr: none)
  const float* w1;
  int symmetric;
  int pw, pn;           // output slots of the wide / narrow pair
  int npairs;
  int combined;         // accumulate cw G + cn u w^T as one form (npairs = 1)
  float cw, cn;
  double* part;         // [blocks][npairs*(d+1)]
  int blocks;
  long long tile_begin, tile_end;  // 128 x 128 tiles of this rank
  int wave;                         // row-wave tile schedule (set by the launcher: rows >= 8 CTAs)
  const float* xsoa;    // d <= 4: column coordinates per 32-row chunk in SoA order (nullptr: AoS xs)
};
int grad_tc_kp(int cols);
int grad_tc_rows_pad(int n);
size_t grad_tc_pack_floats(int n, int kp);
long long grad_tc_tiles(int n, int symmetric);
void grad_tc_pack_launch(const float* w32, int ld, int n, int cols, int kp, float* bpk, const float* n_u,
                         const float* n_w, int n_ld, float* u1, float* w1, cudaStream_t s);
void grad_tc_launch(const GradTcArgs& a, cudaStream_t s);

// ---- SGD with lazily evaluated momentum (sgd_lazy.cu) ----------------------
// Per 32-row chunk of local rows: an FP32 record [V32 image | M32 image] of
// rw floats (sgd_record_width; M32 at moff), each image in the B operand's
// canonical K-major layout; per row the FP64 base state (Vb = the batch's
// solutions, Mb) and tau = the iteration of its last update (-1: none).
struct SgdSlabArgs {
  const float* xs;      // scaled inputs FP32 [n + 128][dp] (global rows)
  int n, dp, d;
  const int* idxbuf;    // minibatches: iteration t uses idxbuf + (t % idx_chunk) * R
  int idx_chunk;
  int R;                // minibatch size (output rows)
  int c0, C;            // this rank's columns (global row0, local count)
  const float* rec;     // [rows_pad / 32][rw]
  int rw, moff;
  const int* tau;       // [rows_pad]
  const float* s32;     // S(Delta), Delta = 0..budget
  int budget;
  int ntab;             // leading entries of s32 staged in shared memory
  const float* xg;      // Gram column image (-2 x, |x|^2, 0...) [n + 128][dp] or null (direct differences)
  const float* xsoa;    // d <= 4: column coordinates per 32-row chunk in SoA order [chunk][dp][32]
  const CgCtl* ctl;     // iteration t = ctl->iters; no-op once ctl->stop
  float log2_s2;
  double* part;         // [splits][R][m] FP64 partials
  int m, splits, cols_per_split, flush;
  double* stats;
  int ch64;             // 64-column pipeline (d <= 4 with xsoa; cols_per_split a multiple of 64)
  int pair;             // ch64 as CTA pairs (cta_group::2, M = 256; needs NPAD % 16 == 0)
  int pdl;              // launch with programmatic stream serialization (prologue overlaps the previous kernel)
};
struct SgdStepArgs {
  CgCtl* ctl;
  const int* idxbuf;
  int idx_chunk, b, m, row0, nloc;
  const double* part;   // slab partials
  int splits;
  double* resid;        // R [nloc][m] (tracked residual estimate)
  double* Vb;           // [nloc][m]
  double* Mb;           // [nloc][m]
  const double* B;      // targets [nloc][m]
  int* tau;
  const double* s64;    // S(Delta)
  const double* p64;    // rho^Delta
  int budget;
  double sigma2, rho, step, tol;
  double* slice;        // this rank's slice of gbuf: [b*m] partial g, [m] old R^2, [1] flag
  const double* gbuf;   // all ranks' slices (stride doubles apart)
  long long stride;
  int nr;               // slices to sum (1 after an all-reduce)
  int sharded;          // several ranks: own-row divergence is carried to the next iteration
  int* nonfinite;       // carried divergence flag (own rows)
  int* nonfinite_now;   // this iteration's (bit 0 any, bit 1 g itself)
  float* rec;
  int rw, moff;
  double* gpart;        // [blocks][m]
  unsigned* ticket;     // kept at 0 between launches
  double* sumsq;        // [m] tracked sum of R^2 per column
  const double* scales;
  int pdl;              // sgd_finish: launch with programmatic stream serialization
};
int sgd_record_width(int m, int* moff);
void sgd_slab_launch(const SgdSlabArgs& a, cudaStream_t s);
void sgd_reduce_launch(const SgdStepArgs& a, cudaStream_t s);
void sgd_gram_image_launch(const float* xs, int rows, int n, int d, int dp, float* xg, cudaStream_t s);
void sgd_soa_image_launch(const float* xs, int rows, int dp, float* out, cudaStream_t s);  // [rows/32][dp][32]
void sgd_apply_launch(const SgdStepArgs& a, cudaStream_t s);
void sgd_finish_launch(const SgdStepArgs& a, cudaStream_t s);  // single rank: reduce + apply fused
int sgd_finish_blocks(int b);
void sgd_records_init_launch(const double* V, int nloc, int rows_pad, int m, int rw, int moff, float* rec, int* tau,
                             cudaStream_t s);
void sgd_materialise_launch(double* Vb, const double* Mb, const int* tau, const double* s64, int budget,
                            const CgCtl* ctl, int nloc, int m, cudaStream_t s);
// minibatches for iterations [*first, *first + count) (device-read start)
void sgd_batches_dev_launch(uint64_t seed, uint64_t substream, int n, int b, const int* first, int count, int* out,
                            const int* skip, cudaStream_t s);

// ---- misc device kernels (la_kernels.cu) ---------------------------------
void prescale_launch(const double* x64, int n, int d, int dp, const double* inv_ls, float* xs32,
                     double* xs64, cudaStream_t s);
// Gram-form operator image (x, |x|^2, 0...) [n][dpg] for d >= 21 (la_kernels.cu)
void gram_image_launch(const float* xs32, int n, int d, int dp, int dpg, float* xg, cudaStream_t s);
// tensor-core Gram column images (kv_tc_kernel TG): per 32-column chunk
// [B hi | B lo] (-2 x', canonical K-major TF32 images, K = kg) and |x'|^2
int tg_kg(int d);
size_t tg_image_floats(int n, int d);
void tg_image_launch(const float* xs32, int n, int d, int dp, float* xtg, cudaStream_t s);
// tensor-core operator kernels take the Gram image for d in [8, 31]
#ifndef GPK_GRAM
#define GPK_GRAM 1  // build-time A/B switch (make NVEXTRA=-DGPK_GRAM=0): direct differences everywhere
#endif
// Gram form for d >= 21 (measured: C2 d = 26 refresh -5%, d = 8 / 11 / 20 +2..12%);
// image width 4 ceil((d + 1) / 4), i.e. DP4 >= 6 <=> Gram in the kernels (d = 32: DP4 9)
inline int gram_dp(int d) { return (GPK_GRAM && d >= 21) ? (d + 4) / 4 * 4 : 0; }
void to_f32_launch(const double* src, int n, int m, int lds, float* dst, int ldd, const int* skip,
                   cudaStream_t s);
void transpose_launch(const double* src, int rows, int cols, int lds, double* dst, int ldd,
                      cudaStream_t s);  // dst[c][r] = src[r][c]

// Deterministic column reductions: part[g][k*m + j] for nout outputs.
// mode 0: sum a*b ; mode 1: (sum a*b, sum a*a) ; mode 2: sum a*a
void col_reduce_launch(const double* a, const double* b, int n, int m, int lda, int mode,
                       double* part, int groups, const int* skip, cudaStream_t s);
constexpr int kReduceGroups = 296;

// CG scalar kernels (single block), all predicated on ctl.
struct CgCtl {
  int done;        // termination reached
  int aborted;     // breakdown
  int stop;        // done || aborted (skip flag for predicated kernels)
  int iters;       // iterations taken
  int budget;      // max iterations
  int pad;
  double mean_norm, probe_norm;
};
void cg_init_scalars_launch(const double* part, int groups, int m, const double* scales, double tol,
                            double* gamma, CgCtl* ctl, cudaStream_t s);
void cg_alpha_launch(const double* part, int groups, int m, const double* gamma, double* alpha,
                     CgCtl* ctl, cudaStream_t s);
void cg_update_launch(double* v, double* r, const double* d, const double* hd, const double* alpha,
                      int n, int m, const int* skip, cudaStream_t s);
void cg_beta_launch(const double* part, int groups, int m, const double* scales, double tol,
                    double* gamma, double* beta, CgCtl* ctl, cudaStream_t s);
void cg_direction_launch(double* d, const double* p, const double* beta, int n, int m, float* d32,
                         int ldv, const int* skip, cudaStream_t s);
void norms_launch(const double* part, int groups, int m, const double* scales, double tol,
                  double* out3, cudaStream_t s);  // mean, probe, done

// preconditioner (K7)
void argmax_partials_launch(const double* diag, int n, double* pval, int* pidx, int groups,
                            cudaStream_t s);
void pchol_step_launch(const double* xs64, int n, int d, double s2, const double* pval,
                       const int* pidx, int groups, double* L, int ldl, int mcol, double* diag,
                       int* pivots, int* stop_flag, cudaStream_t s);
void gram_partials_launch(const double* L, int n, int r, int ldl, double* part, int groups,
                          cudaStream_t s);
void lt_times_launch(const double* L, int n, int r, int ldl, const double* R, int m, double* part,
                     int groups, const int* skip, cudaStream_t s);
void sum_partials_launch(const double* part, int groups, int count, double* out, const int* skip,
                         cudaStream_t s);
void small_gemm_launch(const double* A, int ra, int ca, const double* B, int cb, double* C,
                       const int* skip, cudaStream_t s);  // C = A(ra x ca, row-major) B(ca x cb)
void woodbury_launch(const double* R, const double* L, int n, int r, int ldl, const double* inner,
                     int m, double sigma2, double* out, const int* skip, cudaStream_t s);
void scale_launch(const double* src, int count, double factor, double* dst, const int* skip,
                  cudaStream_t s);
void dense_block64_launch(const double* xs64, int n, int d, double s2, double sigma2, int r0,
                          int rows, int c0, int cols, double* out, int ldo, int add_noise,
                          cudaStream_t s);  // out row-major [rows][ldo]

void ap_blocks_launch(const double* xs64, int n, int d, const double* hyp, int block, int nblocks, double* mats,
                      cudaStream_t s);  // hyp: device {s2, sigma2}
void spd_leaf_inverse_launch(const double* a, double* out, int off, int nn, int ld, long long stride, int batch,
                             int* info, cudaStream_t s);
void block_transpose_launch(const double* src, double* dst, int rows, int cols, int ld, long long stride, int batch,
                            cudaStream_t s);
void exact_forms_launch(const double* xs64, int n, int d, const double* hinv, const double* alpha, double* part,
                        cudaStream_t s);
long long exact_forms_blocks(int n);
void scales_launch(const double* ss, int m, double* scales, double* inv, cudaStream_t s);
void inv_scales_launch(const double* scales, int m, double* inv, cudaStream_t s);
void set_identity_launch(double* mats, int dim, int batch, cudaStream_t s);

// AP (K8)
void ap_scores_launch(const double* R, int n, int m, const double* inv_scales, int block,
                      int nblocks, double* scores, const int* skip, cudaStream_t s);
void ap_select_launch(const double* scores, int nblocks, int* sel, const int* skip, cudaStream_t s);
// scores from per-group partials (gpb groups per block), then argmax
void ap_select_groups_launch(const double* spart, int nblocks, int gpb, int* sel, const int* skip, cudaStream_t s);
// R block -> zero-padded staging [block][m]; pointer arrays for the batched GEMM upd = Hinv[sel] R_blk
void ap_gather_launch(const double* R, int n, int m, int block, const int* sel, double* Rs, const double* inv_blocks,
                      double* upd, double** ptrs, const int* skip, cudaStream_t s);
// V[blk] += upd; optional FP32 copy of upd for the SIMT operator kernel
void ap_apply_update_launch(const double* upd, int n, int m, int block, const int* sel, double* V, float* upd32,
                            int ldv32, const int* skip, cudaStream_t s);
// Fused block step: upd = Hinv[sel] R_blk (FP64), V[blk] += upd, upd64 for the
// diagonal term, and upd's TF32 hi/lo operator images (tcgen05 layout) in vpk.
void ap_update_pack_launch(const double* R, int n, int m, int block, const int* sel, const double* inv_blocks,
                           double* V, double* upd64, float* vpk, int npad, const int* skip, cudaStream_t s);
// V[blk] += upd (upd from the batched GEMM) and upd's TF32 images.
void ap_apply_pack_launch(const double* upd64, int n, int m, int block, const int* sel, double* V, float* vpk,
                          int npad, const int* skip, cudaStream_t s);
void ap_block_update_launch(const double* inv_blocks, int block, int n, const int* sel,
                            const double* R, int m, double* V, double* upd64, float* upd32,
                            int ldv32, const int* skip, cudaStream_t s);
void ap_check_launch(const double* part, int groups, int m, const double* scales, double tol,
                     CgCtl* ctl, cudaStream_t s);

// SGD (K2 + K9)
void sgd_batches_launch(uint64_t seed, uint64_t substream, int n, int b, int first, int count,
                        int* out, cudaStream_t s);
void sgd_step_launch(const double* hv_part_reduced, const int* idx, int b, const double* targets,
                     double* grad, int m, const int* skip, cudaStream_t s);  // grad = hv - t[idx]
void sgd_update_launch(double* M, double* V, float* V32, int ldv, const int* pos, const double* grad,
                       double rho, double step, int n, int m, int* nonfinite, const int* skip,
                       cudaStream_t s);
void sgd_scatter_launch(const int* idx, int b, int* pos, int value_is_q, const int* skip,
                        cudaStream_t s);
void sgd_residual_launch(double* R, const int* idx, int b, const double* grad, int m,
                         double* sumsq, const int* skip, cudaStream_t s);
void sgd_check_launch(const double* sumsq, int m, const double* scales, double tol,
                      const int* nonfinite, CgCtl* ctl, cudaStream_t s);

// Row-sharded SGD on the tcgen05 operator (one rank = one row shard; with
// one rank the same kernels run without the all-gather). Exchange slice per
// rank: [b*m gradient partials | m own old-residual squares | 1 non-finite flag].
void sgd_prep_launch(const double* hv_part, const int* idx, int b, const double* targets, const double* R,
                     int row0, int nloc, int m, int* pos, const int* nonfinite, double* slice, const int* skip,
                     cudaStream_t s);
void sgd_gsum_launch(const double* gbuf, int nr, long long stride, int b, int m, double* grad, const int* skip,
                     cudaStream_t s);
void sgd_check_sharded_launch(const double* gbuf, int nr, long long stride, const double* grad, int b, int m,
                              double* sumsq, const double* scales, double tol, CgCtl* ctl, cudaStream_t s);
void sgd_update_pack_launch(double* M, double* V, double* R, float* vpk, int npad, const int* pos,
                            const double* grad, double rho, double step, int nloc, int m, int* nonfinite,
                            const int* skip, cudaStream_t s);
void sgd_unscatter_launch(const int* idx, int b, int row0, int nloc, int* pos, const int* skip, cudaStream_t s);
void ap_info_gate_launch(const int* info, int nblocks, CgCtl* ctl, cudaStream_t s);
void sgd_diverge_now_launch(const int* nonfinite, CgCtl* ctl, cudaStream_t s);

// RFF (K5) + noise (K9)
// FP64 on-the-fly operator (n <= dense_cache_cap): split partials for kv_reduce
int kv64_splits(int R, int n, int sms);
int kv64_splits_for(int R, int n, int m, int d, int sms);
void kv64_launch(const double* xs64, int n, int d, double sv, int r0, int R, const double* v, int m, int splits,
                 double* part, const int* skip, cudaStream_t s);
// derivative_apply for k <= d (kernel.cpp:200-236), FP64: out [n][m] row-major;
// coef = 3 s2 / l_k (k < d) or 2 / s (k == d)
void deriv_apply_launch(const double* xs64, int n, int d, int k, double sv, double coef, const double* v, int m,
                        double* out, cudaStream_t s);
// streaming K5: prior [n][s_count] = Phi(x) W without materialising Phi (W column-major, ld ldw)
void rff_prior_launch(const double* x64, int n, int d, const double* freq, int pairs, double amplitude,
                      const double* W, int ldw, int s_count, double* prior, cudaStream_t s);
void rff_features_launch(const double* x64, int n, int d, const double* freq, int pairs, double amplitude, double* F,
                         cudaStream_t s);
  // prior row-major [n][s]
void gaussian_fill_launch(uint64_t seed, uint64_t stream, uint64_t substream, int64_t count,
                          int n, int s, double* out_rowmajor, cudaStream_t st);  // col-major order
// rows [row0, row0 + nloc) of the same n x s column-major fill, row-major [nloc][s]
void gaussian_fill_rows_launch(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s, int row0, int nloc,
                               double* out_rowmajor, cudaStream_t st);
// Rademacher +-1 from the low bit of u64 draw j*n + i (rng.cpp:92-96)
void rademacher_fill_rows_launch(uint64_t seed, uint64_t stream, uint64_t substream, int n, int s, int row0, int nloc,
                                 double* out_rowmajor, cudaStream_t st);
void xi_assemble_launch(const double* prior, const double* noise, int n, int s, double sigma,
                        double* out, int ldo, int col0, double* xi_copy, cudaStream_t st);

}  // namespace gpk
