// K4 on the 5th-generation tensor cores: the fused hyperparameter-gradient
// quadratic forms of KernelOperator::derivative_quadratic_forms_many
// (/root/reference/proj/core/src/kernel.cpp:238-272), for the estimator's
// usual pair set: one wide pair (U, W with s probe columns) and optionally one
// narrow pair (the mean solve, one column). For every entry (i, c):
//   g_ic    = sum_j U[i,j] W[c,j]          -> tcgen05 (3xTF32), D in TMEM
//   signal += k_ic g_ic ; l_k += e_ic g_ic (x_ck - x_ik)^2     -> FP32 SIMT
// (same sums and FP32 evaluation as grad_kernel.cu, whose SIMT phase-1 GEMM
// this replaces; the host scales them exactly as kernel.cpp:264-268).
//
// CTA (one per SM, persistent over a contiguous range of 128 x 128 tiles of
// the symmetric (ti <= tc) or full tile list; each tile = two 64-column chunks):
//   warps 0-7  A operand: on every row-block change each thread writes its
//              row of U (TF32 hi | lo) into TMEM with tcgen05.st; per chunk it
//              reads 32 G values of its row (tcgen05.ld), evaluates the kernel
//              against the chunk's x_c (smem broadcast) and accumulates the
//              d + 1 sums per pair in FP32; per tile the sums are reduce-
//              scattered across the warp (butterfly) into FP64 per-warp slots.
//   warp 8     producer: cp.async.bulk of the chunk's pre-packed W images,
//              x_c rows and narrow-pair w values into a 3-stage ring.
//   warp 9     one thread issues 6 x KP/8 tcgen05.mma.kind::tf32 (M=128,
//              N=64, A from TMEM, B from smem) per chunk into one of two TMEM
//              D buffers; tcgen05.commit releases the stage and the buffer.
// Operands are split exactly into three TF32 pieces, x = hi + mid + lo
// (hi, mid: 11 significant bits by truncation; lo: the <= 3 remaining bits),
// and G takes the six products down to 2^-22 relative (hi.hi, hi.mid, mid.hi,
// mid.mid, hi.lo, lo.hi): FP32-grade G, as the SIMT pass. G = Z Z^T sums
// terms of both signs and the trace forms are sensitive to it; the two-piece
// 3xTF32 split used by the K.V operator (whose kernel values are positive)
// measured ~10x worse here.
// Deterministic: fixed tile ranges, fixed butterfly, fixed warp order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gpk_internal.cuh"
#include "tc_util.cuh"

namespace gpk {

namespace {

using namespace tc;

constexpr int TBM = 128;  // tile edge (rows per CTA pass, columns per tile)
constexpr int CN = 64;    // columns per chunk == MMA N
constexpr int STAGES = 3;
// Evaluation warps: 16 (a quarter of each 64-column chunk each, four per SM
// sub-partition: with 8 the C4 pass ran at 15 % warp occupancy and 48 % issue)
// while the wider distance loops fit the 96-register budget of 18 warps: d <= 12
// for every pair set, d <= 20 for the estimator's combined / single-pair passes
// (LEAN; the two-pair pass spills from d = 13); 8 above (half a chunk each).
// Measured at d = 11, n = 524288: 0.797 -> 0.730 s per gradient call. The
// first 8 warps also write the row tile's U pieces into TMEM; then the
// producer warp and the MMA warp.
constexpr int A_WRITERS = 8;
template <int DP4, bool LEAN>
struct GradRoles {
  static constexpr int EW = (DP4 <= 3 || (LEAN && DP4 <= 5)) ? 16 : 8;
  static constexpr int NT = 32 * (EW + 2);
  static constexpr int CW = CN / (EW / 4);  // chunk columns per evaluation warp
};
constexpr int TMEM_COLS = 512;  // one CTA per SM
constexpr int A_BASE = 2 * CN;  // D buffers at TMEM columns [0, 64) and [64, 128); A pieces from 128
constexpr int NPIECE = 3;

__host__ __device__ __forceinline__ void tile_coords_tc(long long L, int T, int symmetric, int& ti, int& tc) {
  if (!symmetric) {
    ti = static_cast<int>(L / T);
    tc = static_cast<int>(L % T);
    return;
  }
  const double b = 2.0 * T + 1.0;
  int r = static_cast<int>((b - sqrt(b * b - 8.0 * static_cast<double>(L))) / 2.0);
  r = max(0, min(r, T - 1));
  auto off = [&](long long rr) { return rr * T - rr * (rr - 1) / 2; };
  while (r > 0 && off(r) > L) --r;
  while (r + 1 < T && off(r + 1) <= L) ++r;
  ti = r;
  tc = r + static_cast<int>(L - off(r));
}

// The tile pairs of one CTA, in the order it visits them. The rank's share of
// the tile list is the linear range [tb, te) (rows ti, columns tc >= ti of the
// symmetric list, or all T x T); two schedules:
//  * contiguous (small problems): CTA b takes the b-th 1/G of the range in
//    list order -- even shares for any T, but every CTA streams its own
//    columns, so the column images are re-read from DRAM once they exceed L2;
//  * waves (rows >= 8 G): CTA b takes whole rows, one per wave of G rows (the
//    position within the wave alternates direction, so the shares stay within
//    one row of each other), and walks each row from its LAST column down:
//    all CTAs of a wave start at column tile T - 1 and move in step, so a
//    column tile is fetched from DRAM once per wave and read by the other
//    CTAs from L2 (C4: 359 GB -> ~8 GB of DRAM reads per pass).
// Every role builds the same walk; next() is one step per tile pair (the
// closed-form FP64 sqrt ran per chunk in every warp: 5 % of the pass's stalls).
struct TileWalk {
  int ti, tc, T, sym;
  // waves
  int wave, G, b, w, R, r0, c0, r1, c1, lo;
  __device__ __forceinline__ int row_lo(int r) const { return r == r0 ? c0 : (sym ? r : 0); }
  __device__ __forceinline__ int row_hi(int r) const { return r == r1 ? c1 : T - 1; }
  __device__ __forceinline__ bool next_row() {
    ++w;
    const int idx = w * G + ((w & 1) ? G - 1 - b : b);
    if (idx >= R) return false;
    ti = r0 + idx;
    lo = row_lo(ti);
    tc = row_hi(ti);
    return true;
  }
  // returns the number of tile pairs of this CTA
  __device__ __forceinline__ long long init(long long tb, long long te, int T_, int sym_, int wave_, int G_, int b_) {
    T = T_;
    sym = sym_;
    wave = wave_;
    G = G_;
    b = b_;
    if (te <= tb) return 0;
    if (!wave) {
      const long long per = (te - tb + G - 1) / G;
      const long long L0 = tb + b * per;
      const long long L1 = min(te, L0 + per);
      if (L1 <= L0) return 0;
      tile_coords_tc(L0, T, sym, ti, tc);
      return L1 - L0;
    }
    tile_coords_tc(tb, T, sym, r0, c0);
    tile_coords_tc(te - 1, T, sym, r1, c1);
    R = r1 - r0 + 1;
    long long cnt = 0;
    for (int ww = 0; ww * G < R; ++ww) {
      const int idx = ww * G + ((ww & 1) ? G - 1 - b : b);
      if (idx < R) cnt += row_hi(r0 + idx) - row_lo(r0 + idx) + 1;
    }
    w = -1;
    if (cnt > 0) next_row();
    return cnt;
  }
  __device__ __forceinline__ void next() {
    if (wave) {
      if (tc > lo)
        --tc;
      else
        next_row();
      return;
    }
    if (++tc == T) {
      ++ti;
      tc = sym ? ti : 0;
    }
  }
};

// exact three-piece TF32 split: x == hi + mid + lo in FP32 arithmetic
__device__ __forceinline__ void split3_tf32(float x, uint32_t& hi, uint32_t& mid, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xFFFFE000u;
  const float r1 = x - __uint_as_float(hi);
  mid = __float_as_uint(r1) & 0xFFFFE000u;
  lo = __float_as_uint(r1 - __uint_as_float(mid));
}

// Adds the warp's per-lane FP32 sums v[0..NV) into FP64 slots: each 32-value
// slab is widened to FP64 and reduce-scattered across the lanes (5 halvings,
// fixed order), after which every lane owns one slab entry.
template <int NV>
__device__ __forceinline__ void butterfly_flush(const float (&v)[NV], int lane, double* slot, int nused,
                                                double weight) {
#pragma unroll
  for (int sl = 0; sl < NV / 32; ++sl) {
    double w[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) w[k] = static_cast<double>(v[sl * 32 + k]);
    int base = 0;
#pragma unroll
    for (int o = 16, cnt = 32; o > 0; o >>= 1, cnt >>= 1) {
      const int half = cnt / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const double send = up ? w[k] : w[k + half];
        const double keep = up ? w[k + half] : w[k];
        w[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      if (up) base += half;
    }
    const int idx = sl * 32 + base;
    if (idx < nused) slot[idx] += w[0] * weight;
  }
}

// COMB (with NARROW): the estimator's combination cw G + cn u w^T is formed
// per entry and accumulated once (one set of d + 1 sums instead of two).
// DX > 0 (d = DX <= 4): the column coordinates come as SoA pairs (the
// operator's xsoa image) and every FP32x2 instruction evaluates two columns
// (distances, kernel profile, lengthscale sums) instead of two padded
// dimensions of one column -- about half the FMA-pipe work per entry, which
// bounds this pass at small d.
template <int DP4, bool NARROW, bool COMB, int DX = 0>
__global__ void __launch_bounds__((GradRoles<DP4, (COMB || !NARROW)>::NT), 1) grad_tc_kernel(const GradTcArgs a) {
  using Roles = GradRoles<DP4, (COMB || !NARROW)>;
  constexpr int EVAL_WARPS = Roles::EW, NTHREADS = Roles::NT, CW = Roles::CW;
  constexpr int DP = 4 * DP4;
  constexpr int NPR = (NARROW && !COMB) ? 2 : 1;
  constexpr int NUSED = NPR * (DP + 1);
  constexpr int NV = NUSED <= 32 ? 32 : (NUSED <= 64 ? 64 : 128);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int KP = a.kp;
  const int img = CN * KP;  // floats per TF32 image of a chunk
  float* smB = reinterpret_cast<float*>(smem_raw);  // [STAGES][NPIECE * img]
  float* smX = smB + STAGES * NPIECE * img;          // [STAGES][CN][DP]
  float* smW = smX + STAGES * CN * DP;               // [STAGES][CN]
  double* wacc = reinterpret_cast<double*>(smW + STAGES * CN);  // [EVAL_WARPS][NV]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wacc + EVAL_WARPS * NV);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* d_full = bars + 2 * STAGES;
  uint64_t* d_empty = d_full + 2;
  uint64_t* a_full = d_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = (a.n + TBM - 1) / TBM;
  const long long ntiles = a.symmetric ? static_cast<long long>(T) * (T + 1) / 2 : static_cast<long long>(T) * T;
  const long long tb = a.tile_end >= 0 ? a.tile_begin : 0;
  const long long te = a.tile_end >= 0 ? min(a.tile_end, ntiles) : ntiles;
  int nq;
  {
    TileWalk tw0;
    nq = static_cast<int>(2 * tw0.init(tb, te, T, a.symmetric, a.wave, gridDim.x, blockIdx.x));
  }

  for (int e = tid; e < EVAL_WARPS * NV; e += NTHREADS) wacc[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + EVAL_WARPS);  // MMA commit + every eval warp (x_c, w reads)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&d_empty[b], EVAL_WARPS);
    }
    mbar_init(a_full, A_WRITERS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // one CTA per SM allocating all 512 columns: the allocation starts at 0
  // (a compile-time base keeps the MMA issue warp-uniform, tc_util.cuh)
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0) __trap();

  if (warp == EVAL_WARPS) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint32_t bbytes = NPIECE * img * 4u, xbytes = CN * DP * 4u, wbytes = NARROW ? CN * 4u : 0u;
      TileWalk tw;
      tw.init(tb, te, T, a.symmetric, a.wave, gridDim.x, blockIdx.x);
      for (int k = 0; k < nq; ++k) {
        const int s = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[s], ((k - STAGES) / STAGES) & 1);
        if (k > 0 && (k & 1) == 0) tw.next();
        const int ti = tw.ti, tcol = tw.tc;
        const int col0 = tcol * TBM + (k & 1) * CN;
        mbar_expect_tx(&full[s], bbytes + xbytes + wbytes);
        bulk_g2s(smB + s * NPIECE * img, a.bpk + static_cast<size_t>(col0 / CN) * NPIECE * img, bbytes, &full[s]);
        bulk_g2s(smX + s * CN * DP, (DX > 0 ? a.xsoa : a.xs) + static_cast<size_t>(col0) * DP, xbytes, &full[s]);
        if (NARROW) bulk_g2s(smW + s * CN, a.w1 + col0, wbytes, &full[s]);
      }
    }
  } else if (warp == EVAL_WARPS + 1) {
    // ---------------- MMA issuer ----------------
    {  // whole warp: waits and operands; one elected lane issues (tc_util.cuh)
      constexpr uint32_t idesc = tf32_idesc(CN, TBM);
      const uint32_t HI = tc_desc_hi(static_cast<uint32_t>(KP / 4) * 128u);
      int prev_ti = -1, rows_loaded = 0;
      TileWalk tw;
      tw.init(tb, te, T, a.symmetric, a.wave, gridDim.x, blockIdx.x);
      for (int k = 0; k < nq; ++k) {
        const int s = k % STAGES, b = k & 1;
        if (k > 0 && (k & 1) == 0) tw.next();
        const int ti = tw.ti, tcol = tw.tc;
        if (ti != prev_ti) {  // new A rows in TMEM
          mbar_wait(a_full, rows_loaded & 1);
          ++rows_loaded;
          prev_ti = ti;
        }
        mbar_wait(&full[s], (k / STAGES) & 1);
        if (k >= 2) mbar_wait(&d_empty[b], ((k - 2) / 2) & 1);
        tc_fence_after();
        const uint32_t bh = tc_desc_lo(smem_u32(smB + s * NPIECE * img), 128);
        const uint32_t bm = bh + ((img * 4) >> 4), bl = bm + ((img * 4) >> 4);
        const uint32_t dt = tmem + b * CN;
        const uint32_t ah = tmem + A_BASE, am = ah + KP, al = am + KP;
        if (tc_elect_one()) {
          for (int kk = 0; kk < KP / 8; ++kk) {
            tc_mma_ur<idesc>(dt, ah + kk * 8, bh + kk * 16, HI, kk == 0 ? 0u : 1u);
            tc_mma_ur<idesc>(dt, ah + kk * 8, bm + kk * 16, HI, 1u);
            tc_mma_ur<idesc>(dt, am + kk * 8, bh + kk * 16, HI, 1u);
            tc_mma_ur<idesc>(dt, am + kk * 8, bm + kk * 16, HI, 1u);
            tc_mma_ur<idesc>(dt, ah + kk * 8, bl + kk * 16, HI, 1u);
            tc_mma_ur<idesc>(dt, al + kk * 8, bh + kk * 16, HI, 1u);
          }
          tc_commit_u(&empty[s]);
          tc_commit_u(&d_full[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- A writers + evaluation ----------------
    const int lg = warp & 3, half = warp >> 2;  // half: A-writer column half (warps < 8); quarter of the chunk
    const uint32_t lane_addr = static_cast<uint32_t>(lg * 32) << 16;
    uint64_t xi2[2 * DP4];
    float u1i = 0.f;
    uint64_t lw[DP / 2], ln[(NARROW && !COMB) ? DP / 2 : 1];
    float sw = 0.f, sn = 0.f;
    // DX path: per-dimension sums as (even, odd column) pairs, and the row's
    // coordinates duplicated into pairs
    constexpr int NX = DX > 0 ? DX : 1;
    uint64_t lwp[NX], lnp[NX], swp = 0ull, snp = 0ull, xik2[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) lwp[k] = lnp[k] = xik2[k] = 0ull;
#pragma unroll
    for (int k = 0; k < DP / 2; ++k) lw[k] = 0ull;
#pragma unroll
    for (int k = 0; k < ((NARROW && !COMB) ? DP / 2 : 1); ++k) ln[k] = 0ull;
    int prev_ti = -1;
    TileWalk tw;
    tw.init(tb, te, T, a.symmetric, a.wave, gridDim.x, blockIdx.x);
    for (int k = 0; k < nq; ++k) {
      const int s = k % STAGES, b = k & 1;
      if (k > 0 && (k & 1) == 0) tw.next();
      const int ti = tw.ti, tcol = tw.tc;
      if (ti != prev_ti) {
        // the previous chunk's D was consumed, so every MMA reading the old A is done
        prev_ti = ti;
        const int i = ti * TBM + lg * 32 + lane;  // < T * 128: xs / u1 are padded to that
        const bool row_ok = i < a.n;
        const float* urow = a.ua + static_cast<size_t>(row_ok ? i : 0) * a.lda;
        if (warp < A_WRITERS) {
        for (int q = 0; q < KP / 16; ++q) {
          uint32_t hi[8], md[8], lo[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = half * (KP / 2) + q * 8 + e;
            const float x = (row_ok && col < a.cols) ? __ldg(urow + col) : 0.f;
            split3_tf32(x, hi[e], md[e], lo[e]);
          }
          const uint32_t at = tmem + lane_addr + A_BASE + half * (KP / 2) + q * 8;
          tc_st8(at, hi);
          tc_st8(at + KP, md);
          tc_st8(at + 2 * KP, lo);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full);
        }
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(a.xs + static_cast<size_t>(i) * DP) + u);
          asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(v.x), "f"(v.y));
          asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(v.z), "f"(v.w));
        }
        if (NARROW) u1i = __ldg(a.u1 + i);
        if constexpr (DX > 0) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(a.xs + static_cast<size_t>(i) * DP));
          const float xe[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < DX; ++k) asm("mov.b64 %0, {%1, %1};" : "=l"(xik2[k]) : "f"(xe[k]));
        }
      }
      mbar_wait(&full[s], (k / STAGES) & 1);
      mbar_wait(&d_full[b], (k / 2) & 1);
      tc_fence_after();
      const uint32_t xbase = smem_u32(smX + s * CN * DP + half * CW * DP);  // half: the warp's column group here
      const float* wc = smW + s * CN + half * CW;
#pragma unroll 1
      for (int q = 0; q < CW / 8; ++q) {
        uint32_t g[8];
        tc_ld8(tmem + lane_addr + b * CN + half * CW + q * 8, g);
        tc_wait_ld();
        if (q == CW / 8 - 1) {  // D buffer fully read: let the next-but-one chunk's MMAs in
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[b]);
        }
        if constexpr (DX > 0) {
          const int cc0 = half * CW + q * 8;  // first chunk column of this group of 8
          const uint32_t xg = smem_u32(smX + s * CN * DP + (cc0 >> 5) * DP * 32 + (cc0 & 31));
          uint64_t k_s3, k_one, k_c;
          asm("mov.b64 %0, {%1, %1};" : "=l"(k_s3) : "f"(kSqrt3f));
          asm("mov.b64 %0, {%1, %1};" : "=l"(k_one) : "f"(1.f));
          asm("mov.b64 %0, {%1, %1};" : "=l"(k_c) : "f"(kNegSqrt3Log2e));
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            uint64_t sqv[DX], r2 = 0ull;
#pragma unroll
            for (int qd = 0; qd < DX; ++qd) {
              uint64_t cc, dd;
              asm volatile("ld.shared.b64 %0, [%1];" : "=l"(cc) : "r"(xg + (qd * 32 + e) * 4));
              asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(cc), "l"(xik2[qd]));
              asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sqv[qd]) : "l"(dd));
              if (qd == 0)
                r2 = sqv[0];
              else
                asm("add.rn.f32x2 %0, %0, %1;" : "+l"(r2) : "l"(sqv[qd]));
            }
            float ra, rb;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r2));
            ra = sqrt_approx(ra);
            rb = sqrt_approx(rb);
            uint64_t rr, uu, ee, kv2, gw2, cw2;
            asm("mov.b64 %0, {%1, %2};" : "=l"(rr) : "f"(ra), "f"(rb));
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(uu) : "l"(rr), "l"(k_c));
            float ua, ub;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(ua), "=f"(ub) : "l"(uu));
            ua = ex2_approx(ua);  // exp(-sqrt3 r)
            ub = ex2_approx(ub);
            asm("mov.b64 %0, {%1, %2};" : "=l"(ee) : "f"(ua), "f"(ub));
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(kv2) : "l"(rr), "l"(k_s3), "l"(k_one));
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(kv2) : "l"(kv2), "l"(ee));  // k / s^2
            const float ga = __uint_as_float(g[e]), gb = __uint_as_float(g[e + 1]);
            const float gwa = COMB ? fmaf(a.cn, u1i * wc[q * 8 + e], a.cw * ga) : ga;
            const float gwb = COMB ? fmaf(a.cn, u1i * wc[q * 8 + e + 1], a.cw * gb) : gb;
            asm("mov.b64 %0, {%1, %2};" : "=l"(gw2) : "f"(gwa), "f"(gwb));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(swp) : "l"(kv2), "l"(gw2));
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(cw2) : "l"(ee), "l"(gw2));
#pragma unroll
            for (int qd = 0; qd < DX; ++qd) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(lwp[qd]) : "l"(sqv[qd]), "l"(cw2));
            if constexpr (NARROW && !COMB) {
              uint64_t gn2, cn2;
              asm("mov.b64 %0, {%1, %2};" : "=l"(gn2) : "f"(u1i * wc[q * 8 + e]), "f"(u1i * wc[q * 8 + e + 1]));
              asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(snp) : "l"(kv2), "l"(gn2));
              asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(cn2) : "l"(ee), "l"(gn2));
#pragma unroll
              for (int qd = 0; qd < DX; ++qd)
                asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(lnp[qd]) : "l"(sqv[qd]), "l"(cn2));
            }
          }
          continue;
        }
#pragma unroll(DP4 <= 2 ? 8 : 2)
        for (int e = 0; e < 8; ++e) {
          const int c = q * 8 + e;
          uint64_t sq[DP / 2];
          uint64_t r2a = 0ull, r2b = 0ull;
#pragma unroll
          for (int u = 0; u < DP4; ++u) {
            uint64_t c01, c23, d01, d23;
            asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xbase + (c * DP + 4 * u) * 4));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(c01), "l"(xi2[2 * u]));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(c23), "l"(xi2[2 * u + 1]));
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq[2 * u]) : "l"(d01));
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(sq[2 * u + 1]) : "l"(d23));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(r2a) : "l"(sq[2 * u]));
            asm("add.rn.f32x2 %0, %0, %1;" : "+l"(r2b) : "l"(sq[2 * u + 1]));
          }
          uint64_t r2s;
          asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r2s) : "l"(r2a), "l"(r2b));
          float q0, q1;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(q0), "=f"(q1) : "l"(r2s));
          const float r = sqrt_approx(q0 + q1);
          const float e0 = ex2_approx(r * kNegSqrt3Log2e);  // exp(-sqrt3 r)
          const float kv = fmaf(r, kSqrt3f, 1.f) * e0;      // k / s^2
          const float gw = COMB ? fmaf(a.cn, u1i * wc[c], a.cw * __uint_as_float(g[e])) : __uint_as_float(g[e]);
          sw = fmaf(kv, gw, sw);
          uint64_t cw2;
          const float cw = e0 * gw;
          asm("mov.b64 %0, {%1, %1};" : "=l"(cw2) : "f"(cw));
#pragma unroll
          for (int t = 0; t < DP / 2; ++t) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(lw[t]) : "l"(sq[t]), "l"(cw2));
          if constexpr (NARROW && !COMB) {
            const float gn = u1i * wc[c];
            sn = fmaf(kv, gn, sn);
            uint64_t cn2;
            const float cnv = e0 * gn;
            asm("mov.b64 %0, {%1, %1};" : "=l"(cn2) : "f"(cnv));
#pragma unroll
            for (int t = 0; t < DP / 2; ++t)
              asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(ln[t]) : "l"(sq[t]), "l"(cn2));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // x_c / w reads of this stage done
      if (k & 1) {  // tile pair complete (two chunks): flush its FP32 sums into the warp's FP64 slots
        float v[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) v[t] = 0.f;
        if constexpr (DX > 0) {  // (even, odd) column pairs -> one sum each
          auto fold = [](uint64_t& p) {
            float x, y;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p));
            p = 0ull;
            return x + y;
          };
#pragma unroll
          for (int qd = 0; qd < DX; ++qd) v[qd] = fold(lwp[qd]);
          v[DP] = fold(swp);
          if constexpr (NARROW && !COMB) {
#pragma unroll
            for (int qd = 0; qd < DX; ++qd) v[DP + 1 + qd] = fold(lnp[qd]);
            v[2 * DP + 1] = fold(snp);
          }
        } else {
#pragma unroll
        for (int t = 0; t < DP / 2; ++t) {
          asm("mov.b64 {%0, %1}, %2;" : "=f"(v[2 * t]), "=f"(v[2 * t + 1]) : "l"(lw[t]));
          lw[t] = 0ull;
        }
        v[DP] = sw;
        sw = 0.f;
        if constexpr (NARROW && !COMB) {
#pragma unroll
          for (int t = 0; t < DP / 2; ++t) {
            asm("mov.b64 {%0, %1}, %2;" : "=f"(v[DP + 1 + 2 * t]), "=f"(v[DP + 2 + 2 * t]) : "l"(ln[t]));
            ln[t] = 0ull;
          }
          v[2 * DP + 1] = sn;
          sn = 0.f;
        }
        }
        const double weight = (a.symmetric && tcol != ti) ? 2.0 : 1.0;
        butterfly_flush<NV>(v, lane, wacc + warp * NV, NUSED, weight);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
  // block result in the caller's pair order: fixed-order sum over warps
  const int d = a.d, per_pair = d + 1;
  for (int e = tid; e < NPR * per_pair; e += NTHREADS) {
    const int p = e / per_pair, k = e % per_pair;
    const int slot = p * (DP + 1) + (k == d ? DP : k);
    double acc = 0.0;
    for (int w = 0; w < EVAL_WARPS; ++w) acc += wacc[w * NV + slot];
    const int po = COMB ? 0 : (p == 0 ? a.pw : a.pn);
    a.part[static_cast<size_t>(blockIdx.x) * a.npairs * per_pair + po * per_pair + k] = acc;
  }
}

// W (rows x cols, FP32, ld) -> per-64-row-chunk TF32 hi | mid | lo images in the
// canonical K-major no-swizzle layout: element (r, k) of chunk r / 64 at
// ((r%64/8) * (KP/4) + k/4) * 32 + (r%8) * 4 + k%4 of each image. Rows >= n
// and columns >= cols are zero. Narrow-pair vectors go to contiguous arrays.
__global__ void grad_tc_pack_kernel(const float* w32, int ld, int n, int cols, int kp, int rows_pad, float* bpk,
                                    const float* n_u, const float* n_w, int n_ld, float* u1, float* w1) {
  const long long total = static_cast<long long>(rows_pad) * kp;
  const int img = CN * kp;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / kp), k = static_cast<int>(e % kp);
    const float x = (r < n && k < cols) ? w32[static_cast<size_t>(r) * ld + k] : 0.f;
    uint32_t hi, md, lo;
    split3_tf32(x, hi, md, lo);
    const int q = r / CN, rr = r % CN;
    float* base = bpk + static_cast<size_t>(q) * NPIECE * img;
    const int off = ((rr / 8) * (kp / 4) + k / 4) * 32 + (rr % 8) * 4 + (k % 4);
    base[off] = __uint_as_float(hi);
    base[img + off] = __uint_as_float(md);
    base[2 * img + off] = __uint_as_float(lo);
    if (k == 0 && u1) {
      u1[r] = r < n ? n_u[static_cast<size_t>(r) * n_ld] : 0.f;
      w1[r] = r < n ? n_w[static_cast<size_t>(r) * n_ld] : 0.f;
    }
  }
}

template <int DP4, bool NARROW, bool COMB, int DX = 0>
void launch_one(const GradTcArgs& a, cudaStream_t s) {
  constexpr int DP = 4 * DP4;
  constexpr int NPR = (NARROW && !COMB) ? 2 : 1;
  constexpr int NUSED = NPR * (DP + 1);
  constexpr int NV = NUSED <= 32 ? 32 : (NUSED <= 64 ? 64 : 128);
  // >= 120 KB keeps one CTA per SM: each allocates all 512 TMEM columns
  const size_t smem = std::max<size_t>(
      sizeof(float) * (STAGES * NPIECE * CN * a.kp + STAGES * CN * DP + STAGES * CN) +
          sizeof(double) * GradRoles<DP4, (COMB || !NARROW)>::EW * NV + 16 * sizeof(uint64_t),
      120 * 1024);
  static size_t configured = 0;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(grad_tc_kernel<DP4, NARROW, COMB, DX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  grad_tc_kernel<DP4, NARROW, COMB, DX><<<a.blocks, GradRoles<DP4, (COMB || !NARROW)>::NT, smem, s>>>(a);
  check_launch("grad_tc_kernel");
}

template <int DP4, int DX = 0>
void launch_dx(const GradTcArgs& a, cudaStream_t s) {
  if (a.u1 && a.combined)
    launch_one<DP4, true, true, DX>(a, s);
  else if (a.u1)
    launch_one<DP4, true, false, DX>(a, s);
  else
    launch_one<DP4, false, false, DX>(a, s);
}
template <int DP4>
void launch_dp(const GradTcArgs& a, cudaStream_t s) {
  if constexpr (DP4 == 1) {
    if (a.xsoa) switch (a.d) {  // exact-dimension column-pair evaluation
        case 1: return launch_dx<1, 1>(a, s);
        case 2: return launch_dx<1, 2>(a, s);
        case 3: return launch_dx<1, 3>(a, s);
        case 4: return launch_dx<1, 4>(a, s);
        default: break;
      }
  }
  launch_dx<DP4>(a, s);
}

}  // namespace

int grad_tc_kp(int cols) { return (cols + 15) / 16 * 16; }
int grad_tc_rows_pad(int n) { return (n + TBM - 1) / TBM * TBM; }
size_t grad_tc_pack_floats(int n, int kp) { return static_cast<size_t>(grad_tc_rows_pad(n)) * NPIECE * kp; }
long long grad_tc_tiles(int n, int symmetric) {
  const long long T = (n + TBM - 1) / TBM;
  return symmetric ? T * (T + 1) / 2 : T * T;
}

void grad_tc_pack_launch(const float* w32, int ld, int n, int cols, int kp, float* bpk, const float* n_u,
                         const float* n_w, int n_ld, float* u1, float* w1, cudaStream_t s) {
  const int rows_pad = grad_tc_rows_pad(n);
  const long long total = static_cast<long long>(rows_pad) * kp;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  grad_tc_pack_kernel<<<blocks, 256, 0, s>>>(w32, ld, n, cols, kp, rows_pad, bpk, n_u, n_w, n_ld, u1, w1);
  check_launch("grad_tc_pack");
}

void grad_tc_launch(const GradTcArgs& a0, cudaStream_t s) {
  GradTcArgs a = a0;
  if (a.kp < 16 || a.kp > 64 || a.kp % 16) throw std::invalid_argument("gpk: tensor-core grad pass needs 1 < s <= 64");
  {  // row-wave schedule once the rank's share spans >= 8 rows per CTA (GPK_GRAD_WAVE=0 / 1: never / always)
    static const int wave_env = [] {
      const char* e = std::getenv("GPK_GRAD_WAVE");
      return e ? std::atoi(e) : -1;
    }();
    const int T = (a.n + TBM - 1) / TBM;
    const long long ntiles = grad_tc_tiles(a.n, a.symmetric);
    const long long tb = a.tile_end >= 0 ? a.tile_begin : 0;
    const long long te = a.tile_end >= 0 ? std::min(a.tile_end, ntiles) : ntiles;
    int rows = 0;
    if (te > tb) {
      int r0, c0, r1, c1;
      tile_coords_tc(tb, T, a.symmetric, r0, c0);
      tile_coords_tc(te - 1, T, a.symmetric, r1, c1);
      rows = r1 - r0 + 1;
    }
    a.wave = wave_env >= 0 ? (wave_env != 0) : (rows >= 8 * a.blocks);
  }
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
