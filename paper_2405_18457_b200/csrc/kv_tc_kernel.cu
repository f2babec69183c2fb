// K1/K2/K3 on the 5th-generation tensor cores: fused ARD distance ->
// Matérn-3/2 -> K.V with the contraction on tcgen05 (3xTF32, FP32 accumulate
// in TMEM), replacing KernelOperator::apply / apply_rows / apply_columns
// (/root/reference/proj/core/src/kernel.cpp:133-177).
//
// CTA = 128 output rows (one per TMEM lane) x NPAD RHS columns (m rounded up
// to a multiple of 16). Warp roles (10 warps):
//   warps 0-7  evaluate K: warp w owns TMEM lanes 32(w%4).. and half (w/4)
//              of every 32-column chunk; each thread computes 16 kernel
//              entries k(x_row, x_c) (FP32, MUFU sqrt/ex2), splits them into
//              TF32 hi + lo and writes both into TMEM with tcgen05.st — the
//              A operand never touches shared memory.
//   warp 8     producer: cp.async.bulk of the pre-packed V chunk (hi and lo
//              images in the canonical no-swizzle K-major UMMA layout) and of
//              the chunk's x_c rows into a 3-stage smem ring (mbarrier
//              complete_tx).
//   warp 9     one elected thread issues, per 32-column chunk, 12
//              tcgen05.mma.kind::tf32 (M=128, N=NPAD, K=8):
//              D += A_hi B_hi + A_hi B_lo + A_lo B_hi, and tcgen05.commit
//              frees the smem stage and the TMEM A buffer.
// Every `flush_chunks` chunks the eval warps drain D (tcgen05.ld) into the
// FP64 per-split partial (deterministic, each thread owns its outputs) and the
// next group restarts accumulation. kv_reduce (kv_kernel.cu) sums splits and
// adds sigma^2 V on the diagonal.
#include <cuda_runtime.h>

#include <algorithm>

#include "gpk_internal.cuh"
#include "tc_util.cuh"
#include "ap_epilogue.cuh"

namespace gpk {

namespace {

constexpr int TBM = 128;
constexpr int TBK = 32;
constexpr int STAGES = 3;
constexpr int NTHREADS = 320;
constexpr int EVAL_WARPS = 8;
constexpr int TMEM_COLS = 256;
constexpr int A_BASE = 128;  // TMEM column of the first A buffer (D uses [0, NPAD))

#ifndef GPK_EVAL_F32X2
#define GPK_EVAL_F32X2 1  // packed FP32x2 distance loop (FADD2/FFMA2)
#endif

using namespace tc;

template <int NPAD>
struct TcLayout {
  static constexpr int IMG_FLOATS = NPAD * TBK;                 // one TF32 image of a chunk
  static constexpr int CHUNK_FLOATS = 2 * IMG_FLOATS;           // hi + lo
  static constexpr uint32_t CHUNK_BYTES = CHUNK_FLOATS * 4;
};

template <int EW>
__device__ __forceinline__ void eval_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory"); }
constexpr int FUSED_SCRATCH_DOUBLES = 4 * 80 + 512 + 8 + 96 + 1024 + 8;  // fused_drain scratch (NPAD <= 80)

// Fused reduce for an AP slab (splits == 1): each eval thread owns one row and
// half of the D columns. out = base + alpha (D + sigma^2 upd on the diagonal);
// the CTA's column sums of out^2 and its AP block-score partial
// sum_r (sum_j out[r][j] inv_scales[j])^2 go to dpart[tile] / spart[tile] in a
// fixed order (warp reduce-scatter, then lane groups in order), and the last
// CTA (ticket) runs the AP epilogue. Replaces kv_reduce_dot_kernel for slabs.
template <int NPAD, int EW>
__device__ __forceinline__ void fused_drain(const KvArgs& a, const KvReduceArgs& f, uint32_t trow, int er, int gi,
                                            int c0, int C, int qtr, int lg, int lane, int warp, double* scratch,
                                            const double* sbase) {
  constexpr int NQ = EW / 4;          // warps per TMEM lane group
  constexpr int DC = NPAD / NQ;       // D columns drained by this thread (multiple of 4)
  double* red = scratch;              // [4][NPAD] column sums per lane group
  double* rd = red + 4 * NPAD;        // [NQ][128] row-dot parts
  double* ssc = rd + 4 * 128;         // [4]
  double* ss = ssc + 8;               // [96]
  double* bscore = ss + 96;           // [1024]
  unsigned* last = reinterpret_cast<unsigned*>(bscore + 1024);
  const int tid = warp * 32 + lane;
  const bool row_ok = er < a.R;
  const bool diag = row_ok && gi >= c0 && gi < c0 + C;
  const int vr = gi - c0 - f.vshift;
  const int lrow = er - blockIdx.x * 128;
  double rowdot = 0.0;
#pragma unroll 1
  for (int q = 0; q < DC / 4; ++q) {
    const int col0 = qtr * DC + q * 4;
    uint32_t v[4];
    tc_ld4(trow + col0, v);
    tc_wait_ld();
    double cs[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = col0 + e;
      cs[e] = 0.0;
      if (row_ok && j < a.m) {
        double acc = static_cast<double>(__uint_as_float(v[e]));
        if (diag) acc += f.sigma2 * f.vdiag[static_cast<size_t>(vr) * f.ldvd + j];
        const double b = sbase ? sbase[static_cast<size_t>(lrow) * a.m + j]
                               : f.base ? f.base[static_cast<size_t>(er) * f.ldb + j] : 0.0;
        const double val = b + f.alpha * acc;
        f.out[static_cast<size_t>(er) * f.ldo + j] = val;
        cs[e] = val * val;
        rowdot += val * f.inv_scales[j];
      }
    }
    // reduce-scatter the 4 column sums over the 32 rows of this warp
    int base = 0;
#pragma unroll
    for (int o = 16, cnt = 4; o >= 8; o >>= 1, cnt >>= 1) {
      const int hf = cnt / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < hf; ++k) {
        const double send = up ? cs[k] : cs[k + hf];
        const double keep = up ? cs[k + hf] : cs[k];
        cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      if (up) base += hf;
    }
    cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 4);
    cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 2);
    cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 1);
    if ((lane & 7) == 0) red[lg * NPAD + col0 + base] = cs[0];
  }
  rd[qtr * 128 + lg * 32 + lane] = rowdot;
  eval_bar<EW>();
  for (int j = tid; j < a.m; j += 32 * EW)
    f.dpart[static_cast<size_t>(blockIdx.x) * a.m + j] = ((red[j] + red[NPAD + j]) + red[2 * NPAD + j]) + red[3 * NPAD + j];
  if (qtr == 0) {
    double w = rd[lg * 32 + lane];
#pragma unroll
    for (int p = 1; p < NQ; ++p) w += rd[p * 128 + lg * 32 + lane];
    double sc = row_ok ? w * w : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
    if (lane == 0) ssc[lg] = sc;
  }
  eval_bar<EW>();
  if (tid == 0) {
    f.spart[blockIdx.x] = ((ssc[0] + ssc[1]) + ssc[2]) + ssc[3];
    __threadfence();
    *last = (atomicAdd(f.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  eval_bar<EW>();
  if (!*last) return;
  __threadfence();
  ap_epilogue(f, static_cast<int>(gridDim.x), tid, EW, ss, bscore, [] { eval_bar<EW>(); });
}

// MODE 0: two CTAs per SM, 8 evaluation warps, 2 TMEM A buffers (default);
// MODE 1: fused AP slab; MODE 2: "deep" -- one CTA per SM with 16 evaluation
// warps and 4 A buffers (512 TMEM columns), for launches whose per-chunk
// barrier/MMA latency dominates (small d, few rows); MODE 3: the deep CTA as
// a persistent stream-K worker -- one CTA per SM walks a contiguous range of
// the (row tile, 32-column chunk) units, so every SM gets the same number of
// chunks (no partial last wave, one TMEM allocation and pipeline fill per SM)
// and writes one partial per row tile it touches (sk_first .. sk_last).
template <int MODE>
struct TcRoles {
  static constexpr int EW = MODE ? 16 : EVAL_WARPS;  // evaluation warps
  static constexpr int THREADS = 32 * (EW + 2);
  static constexpr int CPT = TBK * 4 / EW;            // chunk columns per eval thread
};

// TG: tensor-core Gram distances. Per 32-column chunk one more set of
// tcgen05 MMAs computes G = -2 X_rows X_c^T (3xTF32: hi.lo + lo.hi + hi.hi,
// M = 128, N = 32, K = KG = 8 ceil(d / 8)) into TMEM columns [TG_COL, +32);
// the evaluation warps read their row's G (one tcgen05.ld per chunk) and form
// r^2 = (|x_i|^2 + |x_c|^2) + G with the norms of the same 22-bit split
// coordinates in FP32, so the per-entry FP32 work is the Matern profile only.
// A operand: the tile's rows as TF32 hi / lo images in TMEM (written by the
// eval warps when a tile starts; A in shared memory would cost the MMA a
// 4 KB operand read per K step); B operand + column norms: per-chunk
// images built once per hyperparameter set (tg_image_kernel), bulk-copied
// with the V chunk.
constexpr int TG_COL = 96;   // TMEM column of the Gram tile (D uses [0, NPAD <= 80))
constexpr int TGA_COL = 384; // TMEM columns of the row images hi | lo (KG each), behind 4 A buffers
template <int DP4>
struct TgShape {
  static constexpr int KG = ((DP4 + 1) / 2) * 8;  // K of the Gram MMAs (multiple of 8, >= 4 DP4)
  static constexpr int CHUNK = 2 * TBK * KG + TBK;  // floats per column chunk: B hi | B lo | |x_c|^2
};

template <int NPAD, int DP4, int MODE, bool TG>
__global__ void __launch_bounds__(TcRoles<MODE>::THREADS, MODE ? 1 : 2)
    kv_tc_kernel(const KvArgs a, const float* __restrict__ vpk, const KvReduceArgs f) {
  constexpr bool FUSED = MODE == 1, DEEP = MODE != 0, SK = MODE == 3;
  static_assert(!(TG && (SK || MODE == 0)), "tensor-core Gram distances: one row tile per CTA, 512 TMEM columns");
  constexpr int EW = TcRoles<MODE>::EW, CPT = TcRoles<MODE>::CPT;
  constexpr int DP = 4 * DP4;
  constexpr bool GRAM = !TG && GPK_GRAM && DP4 >= 6;  // image (x, |x|^2, 0...): host passes it for d >= 21
  constexpr int KG = TgShape<DP4>::KG;
  constexpr int XST = TG ? TgShape<DP4>::CHUNK : TBK * DP;  // floats of column data per stage
  using L = TcLayout<NPAD>;
  // One-CTA-per-SM product launches double-buffer the FP32 accumulator D when
  // the 512 TMEM columns have room for a second one (A ring [128, 384); with
  // tensor-core Gram distances the row images end at 384 + 2 KG): the MMA warp
  // starts the next accumulation group in the other buffer while the
  // evaluation warps drain this one two chunks later, so neither waits.
  constexpr bool DBUF = DEEP && !FUSED && NPAD / (EW / 4) <= 20 && NPAD <= 80 && (!TG || KG <= 24);
  constexpr uint32_t D1_COL = TG ? 432 : 384;
  constexpr int DRAIN_DEFER = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the fused AP slab runs one CTA per SM: 4 TMEM A buffers (512 columns)
  constexpr int NAB = DEEP ? 4 : 2;
  constexpr int TCOLS = DEEP ? 512 : TMEM_COLS;
  float* smB = reinterpret_cast<float*>(smem_raw);                    // [STAGES][CHUNK_FLOATS]
  float* smX = smB + STAGES * L::CHUNK_FLOATS;                        // [STAGES][XST]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smX + STAGES * XST);
  uint64_t* full = bars;              // [STAGES]
  uint64_t* empty = bars + STAGES;    // [STAGES]
  uint64_t* a_full = bars + 2 * STAGES;         // [NAB]
  uint64_t* a_empty = bars + 2 * STAGES + 4;    // [NAB]
  uint64_t* d_full = bars + 2 * STAGES + 8;
  uint64_t* d_empty = bars + 2 * STAGES + 9;
  uint64_t* base_full = bars + 2 * STAGES + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 11);
  uint64_t* g_full = bars + 2 * STAGES + 12;     // TG: Gram tile of the chunk in TMEM
  uint64_t* g_empty = bars + 2 * STAGES + 13;    // TG: eval warps have read it
  uint64_t* arow_full = bars + 2 * STAGES + 14;  // TG: row images written
  uint64_t* d_full1 = bars + 2 * STAGES + 15;    // DBUF: the second accumulator
  uint64_t* d_empty1 = bars + 2 * STAGES + 16;

  if (a.skip && *a.skip) return;
  int c0 = a.c0, C = a.C;
  if (a.sel) {
    c0 = *a.sel * a.sel_block;
    C = min(a.sel_block, a.n - c0);
  }
  const int tile = blockIdx.x, split = blockIdx.y;
  const int cb = split * a.cols_per_split;
  const int ce = min(C, cb + a.cols_per_split);
  const int nq = ce > cb ? (ce - cb + TBK - 1) / TBK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // chunk schedule: stream-K units [u0, u0 + nk) of U = tiles x Q, or this
  // CTA's nq chunks of one tile
  int Q = 1, nk = nq;
  long long U = 1, u0 = 0;
  if constexpr (SK) {
    Q = (C + TBK - 1) / TBK;
    U = static_cast<long long>((a.R + TBM - 1) / TBM) * Q;
    u0 = blockIdx.x * U / gridDim.x;
    nk = static_cast<int>((blockIdx.x + 1) * U / gridDim.x - u0);
  }
  const int flush = a.flush_chunks;
  // walks this CTA's units in order: row tile t, chunk q, accumulation-group
  // boundaries (incremental: no per-chunk 64-bit division)
  struct Walk {
    int t, q, gp, k;
    bool first, last;
  };
  auto walk_begin = [&]() {
    Walk w;
    if constexpr (SK) {
      w.t = static_cast<int>(u0 / Q);
      w.q = static_cast<int>(u0 - static_cast<long long>(w.t) * Q);
    } else {
      w.t = tile;
      w.q = cb / TBK;  // cb is a multiple of TBK
    }
    w.gp = 0;
    w.k = 0;
    w.first = true;
    w.last = nk == 1 || (SK && w.q + 1 == Q) || flush == 1;
    return w;
  };
  auto walk_next = [&](Walk& w) {
    const bool tile_end = SK && w.q + 1 == Q;
    w.gp = w.last ? 0 : w.gp + 1;
    ++w.k;
    if (tile_end) {
      w.q = 0;
      ++w.t;
    } else {
      ++w.q;
    }
    w.first = w.gp == 0;
    w.last = w.k + 1 == nk || (SK && w.q + 1 == Q) || w.gp + 1 == flush;
  };

  if (a.stats && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    const double entries = static_cast<double>(a.R) * C;
    atomicAdd(a.stats, entries * a.m);
    atomicAdd(a.stats + 1, entries * (2.0 * a.m + 3.0 * a.d + 6.0));
    atomicAdd(a.stats + 2, entries * (3.0 * a.d + 6.0));  // FP32 pipe share; the 2m contraction is on tcgen05
  }

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NAB; ++b) {
      mbar_init(&a_full[b], EW);
      mbar_init(&a_empty[b], 1);
    }
    mbar_init(d_full, 1);
    mbar_init(d_empty, EW);
    if (DBUF) {
      mbar_init(d_full1, 1);
      mbar_init(d_empty1, EW);
    }
    if (FUSED) mbar_init(base_full, 1);  // base tile landed
    if (TG) {
      mbar_init(g_full, 1);
      mbar_init(g_empty, EW);
      mbar_init(arow_full, 4);  // the four eval warps of chunk-column group 0 own the 128 rows
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // one CTA per SM allocating all 512 columns (deep variants): the allocation
  // starts at 0, and the compile-time base keeps the MMA issue warp-uniform
  // (tc_util.cuh); two CTAs per SM read their base from the allocation
  constexpr bool UNI = TCOLS == 512;
  const uint32_t tmem = UNI ? 0u : *tmem_slot;
  if (UNI && tid == 0 && *tmem_slot != 0) __trap();

  // fused AP slab: the tile's rows of `base` (the residual) are staged in smem
  // by one bulk copy issued before the chunk loop, so the drain never waits on
  // global loads; sbase sits behind the drain scratch.
  double* sbase = reinterpret_cast<double*>(bars + 64) + FUSED_SCRATCH_DOUBLES;
  bool base_staged = false;
  if constexpr (FUSED) {
    const int rows = min(TBM, a.R - tile * TBM);
    const uint32_t bytes = static_cast<uint32_t>(rows) * f.ldb * 8u;
    base_staged = f.base && f.ldb == a.m && a.m <= 96 && (bytes % 16u) == 0u;
    if (base_staged && warp == EW && lane == 0) {
      mbar_expect_tx(base_full, bytes);
      bulk_g2s(sbase, f.base + static_cast<size_t>(tile) * TBM * f.ldb, bytes, base_full);
    }
  }
  if (warp == EW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      Walk w = walk_begin();
      for (int k = 0; k < nk; ++k, walk_next(w)) {
        const int s = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[s], ((k - STAGES) / STAGES) & 1);
        const int chunk = w.q;
        const uint32_t xbytes = XST * 4;
        mbar_expect_tx(&full[s], L::CHUNK_BYTES + xbytes);
        bulk_g2s(smB + s * L::CHUNK_FLOATS, vpk + static_cast<size_t>(chunk) * L::CHUNK_FLOATS, L::CHUNK_BYTES,
                 &full[s]);
        if constexpr (TG)  // host guarantees c0 % TBK == 0
          bulk_g2s(smX + s * XST, a.xtg + static_cast<size_t>(c0 / TBK + chunk) * XST, xbytes, &full[s]);
        else
          bulk_g2s(smX + s * XST, a.xs + static_cast<size_t>(c0 + chunk * TBK) * DP, xbytes, &full[s]);
      }
    }
  } else if (warp == EW + 1) {
    // ---------------- MMA issuer ----------------
    if (UNI || GPK_MMA_WARP || lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(NPAD, TBM);
      constexpr uint32_t gdesc = tf32_idesc(TBK, TBM);
      constexpr uint32_t GSBO = (KG / 4) * 128, VSBO = (TBK / 4) * 128;
      // TG: G(k) = -2 X_rows X_c(k)^T, the cross terms first and hi.hi last
      // (truncating accumulation: the small terms go in while D is small)
      auto gram_mma = [&](int k) {
        const int s = k % STAGES;
        const uint32_t ah = tmem + TGA_COL, al = ah + KG;
        const uint32_t bh = smem_u32(smX + s * XST), bl = bh + TBK * KG * 4;
        if constexpr (UNI) {
          const uint32_t dh = tc_desc_lo(bh, 128), dl = tc_desc_lo(bl, 128);
          if (tc_elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KG / 8; ++ks) {
              tc_mma_u<tc_desc_hi(GSBO), gdesc>(tmem + TG_COL, ah + ks * 8, dl + ks * 16, ks ? 1u : 0u);
              tc_mma_u<tc_desc_hi(GSBO), gdesc>(tmem + TG_COL, al + ks * 8, dh + ks * 16, 1u);
            }
#pragma unroll
            for (int ks = 0; ks < KG / 8; ++ks)
              tc_mma_u<tc_desc_hi(GSBO), gdesc>(tmem + TG_COL, ah + ks * 8, dh + ks * 16, 1u);
            tc_commit_u(g_full);
          }
          __syncwarp();
        } else {
#pragma unroll
          for (int ks = 0; ks < KG / 8; ++ks) {
            MMA_TF32(tmem + TG_COL, ah + ks * 8, umma_desc(bl + ks * 256, 128, GSBO), gdesc, ks ? 1u : 0u);
            MMA_TF32(tmem + TG_COL, al + ks * 8, umma_desc(bh + ks * 256, 128, GSBO), gdesc, 1u);
          }
#pragma unroll
          for (int ks = 0; ks < KG / 8; ++ks)
            MMA_TF32(tmem + TG_COL, ah + ks * 8, umma_desc(bh + ks * 256, 128, GSBO), gdesc, 1u);
          MMA_COMMIT(g_full);
        }
      };
      if (TG && nk > 0) {
        mbar_wait(arow_full, 0);
        mbar_wait(&full[0], 0);
        tc_fence_after();
        gram_mma(0);
      }
      int g = 0;  // accumulation groups issued
      Walk w = walk_begin();
      for (int k = 0; k < nk; ++k, walk_next(w)) {
        const int s = k % STAGES, b = k % NAB;
        const bool first_in_group = w.first, last_in_group = w.last;
        mbar_wait(&full[s], (k / STAGES) & 1);
        if (TG && k + 1 < nk) {  // next chunk's Gram tile once the eval warps hold this one's
          mbar_wait(&full[(k + 1) % STAGES], ((k + 1) / STAGES) & 1);
          mbar_wait(g_empty, k & 1);
          tc_fence_after();
          gram_mma(k + 1);
        }
        mbar_wait(&a_full[b], (k / NAB) & 1);
        if constexpr (DBUF) {
          if (first_in_group && g >= 2) mbar_wait((g & 1) ? d_empty1 : d_empty, ((g >> 1) - 1) & 1);
        } else {
          if (first_in_group && g > 0) mbar_wait(d_empty, (g - 1) & 1);
        }
        const uint32_t dacc = tmem + ((DBUF && (g & 1)) ? D1_COL : 0u);
        uint64_t* const dfull_g = (DBUF && (g & 1)) ? d_full1 : d_full;
        tc_fence_after();
        const uint32_t bh = smem_u32(smB + s * L::CHUNK_FLOATS);
        const uint32_t bl = bh + L::IMG_FLOATS * 4;
        const uint32_t ah = tmem + A_BASE + b * 64;
        const uint32_t al = ah + 32;
        if constexpr (UNI) {
          const uint32_t dh = tc_desc_lo(bh, 128), dl = tc_desc_lo(bl, 128);
          if (tc_elect_one()) {
#pragma unroll
            for (int kk = 0; kk < TBK / 8; ++kk) {
              tc_mma_u<tc_desc_hi(VSBO), idesc>(dacc, ah + kk * 8, dh + kk * 16, (first_in_group && kk == 0) ? 0u : 1u);
              tc_mma_u<tc_desc_hi(VSBO), idesc>(dacc, ah + kk * 8, dl + kk * 16, 1u);
              tc_mma_u<tc_desc_hi(VSBO), idesc>(dacc, al + kk * 8, dh + kk * 16, 1u);
            }
            tc_commit_u(&empty[s]);
            tc_commit_u(&a_empty[b]);
            if (last_in_group) tc_commit_u(dfull_g);
          }
          __syncwarp();
          if (last_in_group) ++g;
        } else {
#pragma unroll
          for (int kk = 0; kk < TBK / 8; ++kk) {
            const uint64_t dh = umma_desc(bh + kk * 256, 128, VSBO);
            const uint64_t dl = umma_desc(bl + kk * 256, 128, VSBO);
            MMA_TF32(dacc, ah + kk * 8, dh, idesc, (first_in_group && kk == 0) ? 0u : 1u);
            MMA_TF32(dacc, ah + kk * 8, dl, idesc, 1u);
            MMA_TF32(dacc, al + kk * 8, dh, idesc, 1u);
          }
          MMA_COMMIT(&empty[s]);
          MMA_COMMIT(&a_empty[b]);
          if (last_in_group) {
            MMA_COMMIT(dfull_g);
            ++g;
          }
        }
      }
    }
  } else {
    // ---------------- evaluation + epilogue warps ----------------
    const int lg = warp & 3;           // TMEM lane group
    const int half = warp >> 2;        // chunk columns [CPT*half, CPT*half + CPT)
    const int row = lg * 32 + lane;    // row within the tile == TMEM lane
    // per-row-tile state (reloaded when a stream-K CTA moves to the next tile)
    int er = 0, er_c = 0, gi = 0;
#if !GPK_EVAL_F32X2
    static_assert(!GRAM, "the Gram-form operator needs the FP32x2 evaluation loop");
    float4 xi[DP4];
#else
    // Gram form (image width >= 24, i.e. d >= 21): the row keeps (-2 x_i, 1) and
    // |x_i|^2 seeds the accumulator, so r^2 = |x_i|^2 + |x_c|^2 - 2 x_i.x_c is
    // one FFMA2 per two padded dimensions (x_c's image carries |x_c|^2 in slot d)
    uint64_t xi2[2 * DP4];
    uint64_t acc_seed = 0ull;
#endif
    double* part = nullptr;
    // One-CTA-per-SM launches (16 evaluation warps: 20 D columns per thread at
    // NPAD = 80) keep the tile's FP64 partial in registers and write it once
    // per (CTA, tile); the drain used to read-modify-write the partial in
    // global memory every flush_chunks chunks (five serialised L2 round trips
    // with the MMA warp waiting on the single D buffer: 7.3 us per drain, a
    // third of the C5 product's time). Same FP64 adds in the same order.
    constexpr int DCOLS = NPAD / (EW / 4);  // D columns this thread drains
    constexpr bool REGACC = DEEP && !FUSED && DCOLS <= 20;
    double acc64[REGACC ? DCOLS : 1];
    bool wrote = false;
    float tg_ni = 0.f;  // TG: |x_i|^2 of the split coordinates
    auto setup_rows = [&](int t) {
      er = t * TBM + row;
      er_c = er < a.R ? er : 0;
      gi = a.row_idx ? a.row_idx[er_c] : a.r0 + er_c;
      const float* xrow = (a.xs_rows ? a.xs_rows : a.xs) + static_cast<size_t>(gi) * DP;
#if GPK_EVAL_F32X2
      float4 xi[DP4];
#endif
#pragma unroll
      for (int u = 0; u < DP4; ++u) xi[u] = __ldg(reinterpret_cast<const float4*>(xrow) + u);
      if constexpr (TG) {
        // row images for the Gram MMAs (canonical K-major no-swizzle layout:
        // element (row, k) at ((row/8) (KG/4) + k/4) 32 + (row%8) 4 + k%4)
        float hv[4 * DP4], lv[4 * DP4];
        float ni = 0.f;
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          const float* c = reinterpret_cast<const float*>(&xi[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            tg_split(c[e], hv[4 * u + e], lv[4 * u + e]);
            ni = tg_norm_step(ni, hv[4 * u + e], lv[4 * u + e]);
          }
        }
        tg_ni = ni;
        if (half == 0) {  // this warp's 32 rows (TMEM lanes) of the hi | lo row images
          const uint32_t ta = tmem + (static_cast<uint32_t>(lg * 32) << 16) + TGA_COL;
#pragma unroll
          for (int k8 = 0; k8 < KG / 8; ++k8) {
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int k = 8 * k8 + e;
              hw[e] = k < 4 * DP4 ? __float_as_uint(hv[k]) : 0u;
              lw[e] = k < 4 * DP4 ? __float_as_uint(lv[k]) : 0u;
            }
            tc_st8(ta + 8 * k8, hw);
            tc_st8(ta + KG + 8 * k8, lw);
          }
          tc_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(arow_full);
        }
      }
#if GPK_EVAL_F32X2
      float ni = 0.f;
      if constexpr (GRAM) {
#pragma unroll
        for (int u = 0; u < DP4; ++u) gram_row(xi[u], 4 * u, a.d, ni);
      }
      if constexpr (!TG) {
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(xi[u].x), "f"(xi[u].y));
          asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(xi[u].z), "f"(xi[u].w));
        }
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc_seed) : "f"(ni), "f"(0.f));
      }
#endif
      // partial slot: the split, or this CTA's position among the tile's stream-K workers
      const long long slot = SK ? blockIdx.x - sk_first(t, Q, gridDim.x, U) : split;
      part = a.part + static_cast<size_t>(slot) * a.R * a.m;
      wrote = false;
      if constexpr (REGACC) {
#pragma unroll
        for (int e = 0; e < DCOLS; ++e) acc64[e] = 0.0;
      }
    };
    if (!SK) setup_rows(tile);
    const uint32_t lane_addr = static_cast<uint32_t>(lg * 32) << 16;
    int g = 0;  // accumulation groups drained
    [[maybe_unused]] int pending = 0;  // DBUF: a completed group whose drain is deferred

    Walk w = walk_begin();
    for (int k = 0; k < nk; ++k, walk_next(w)) {
      const int s = k % STAGES, b = k % NAB;
      const int q = w.q;
      const bool last_in_group = w.last;
      if (SK && (k == 0 || q == 0)) setup_rows(w.t);
      mbar_wait(&full[s], (k / STAGES) & 1);
      if (k >= NAB) mbar_wait(&a_empty[b], ((k - NAB) / NAB) & 1);
      tc_fence_after();
      const float* xc = smX + s * XST + half * CPT * DP;
      uint32_t hi[CPT], lo[CPT];
      float tg_r2[TG ? CPT : 1];
      if constexpr (TG) {
        mbar_wait(g_full, k & 1);
        tc_fence_after();
        uint32_t gv[CPT];
        if constexpr (CPT == 16)
          tc_ld16(tmem + lane_addr + TG_COL + half * CPT, gv);
        else
          tc_ld8(tmem + lane_addr + TG_COL + half * CPT, gv);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(g_empty);
        const float4* ncs = reinterpret_cast<const float4*>(smX + s * XST + 2 * TBK * KG + half * CPT);
#pragma unroll
        for (int t4 = 0; t4 < CPT / 4; ++t4) {
          const float4 nc = ncs[t4];
          tg_r2[4 * t4] = (tg_ni + nc.x) + __uint_as_float(gv[4 * t4]);
          tg_r2[4 * t4 + 1] = (tg_ni + nc.y) + __uint_as_float(gv[4 * t4 + 1]);
          tg_r2[4 * t4 + 2] = (tg_ni + nc.z) + __uint_as_float(gv[4 * t4 + 2]);
          tg_r2[4 * t4 + 3] = (tg_ni + nc.w) + __uint_as_float(gv[4 * t4 + 3]);
        }
      }
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        if constexpr (TG) {
        const float r = sqrt_approx(fmaxf(tg_r2[t], 0.f));
        const float kv = fmaf(r, kSqrt3f, 1.f) * ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));
        hi[t] = __float_as_uint(kv) & 0xFFFFE000u;
        lo[t] = __float_as_uint(kv - __uint_as_float(hi[t]));
        continue;
        }
#if GPK_EVAL_F32X2
        // packed FP32x2 (FADD2/FFMA2): two dimensions per instruction
        const uint32_t xaddr = smem_u32(xc + t * DP);
        float r;
        if constexpr (GRAM) {
          r = sqrt_approx(gram_r2<DP4>(xaddr, xi2, acc_seed));
        } else {
        uint64_t acc0 = 0ull, acc1 = 0ull;
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          uint64_t c01, c23, d01, d23;
          asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xaddr + 16 * u));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(c01), "l"(xi2[2 * u]));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(c23), "l"(xi2[2 * u + 1]));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc0) : "l"(d01));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc1) : "l"(d23));
        }
        uint64_t accs;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(accs) : "l"(acc0), "l"(acc1));
        float s0, s1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(accs));
        r = sqrt_approx(s0 + s1);
        }
#else
        const float4* xv = reinterpret_cast<const float4*>(xc + t * DP);
        float r2a = 0.f, r2b = 0.f;
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          const float4 c = xv[u];
          const float d0 = c.x - xi[u].x, d1 = c.y - xi[u].y, d2 = c.z - xi[u].z, d3 = c.w - xi[u].w;
          r2a = fmaf(d0, d0, r2a);
          r2b = fmaf(d1, d1, r2b);
          r2a = fmaf(d2, d2, r2a);
          r2b = fmaf(d3, d3, r2b);
        }
        const float r = sqrt_approx(r2a + r2b);
#endif
        const float kv = fmaf(r, kSqrt3f, 1.f) * ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));
        // TF32 split: hi = kv with the 13 low mantissa bits cleared (exact), lo =
        // kv - hi (exact in FP32); the tensor core reads lo's top 19 bits, so
        // hi + lo carries ~21-22 bits of kv.
        hi[t] = __float_as_uint(kv) & 0xFFFFE000u;
        lo[t] = __float_as_uint(kv - __uint_as_float(hi[t]));
      }
      if constexpr (GRAM || TG) {
        // the Gram form leaves O(ulp |x|^2) on the kernel diagonal: pin k(x_i, x_i)
        // to the direct form's value (rare chunks, warp-uniform branch)
        const int cbase = c0 + q * TBK + half * CPT;
        const bool hit = !a.xs_rows && er < a.R && static_cast<unsigned>(gi - cbase) < static_cast<unsigned>(CPT);
        if (__any_sync(0xffffffffu, hit)) gram_pin_diagonal<CPT>(hit, gi - cbase, a.log2_s2, hi, lo);
      }
      const uint32_t abase = tmem + lane_addr + A_BASE + b * 64 + half * CPT;
      if constexpr (CPT == 16) {
        tc_st16(abase, hi);
        tc_st16(abase + 32, lo);
      } else {
        tc_st8(abase, hi);
        tc_st8(abase + 32, lo);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[b]);

      if constexpr (DBUF) {
        // drain of group gd: D buffer gd & 1 -> the FP64 registers
        auto drain_regs = [&](int gd) {
          mbar_wait((gd & 1) ? d_full1 : d_full, (gd >> 1) & 1);
          tc_fence_after();
          const uint32_t dcol = tmem + lane_addr + ((gd & 1) ? D1_COL : 0u) + half * DCOLS;
          uint32_t v[DCOLS];
#pragma unroll
          for (int q4 = 0; q4 < DCOLS / 4; ++q4) tc_ld4(dcol + q4 * 4, *reinterpret_cast<uint32_t(*)[4]>(v + 4 * q4));
          tc_wait_ld();
#pragma unroll
          for (int e = 0; e < DCOLS; ++e) acc64[e] += static_cast<double>(__uint_as_float(v[e]));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive((gd & 1) ? d_empty1 : d_empty);
        };
        // the previous group, DRAIN_DEFER chunks into this one (its MMAs are long done)
        if (pending && (w.gp + 1 == DRAIN_DEFER || last_in_group)) {
          drain_regs(g++);
          pending = 0;
        }
        if (last_in_group) {
          const bool seg_end = k + 1 == nk || (SK && q + 1 == Q);  // the (CTA, tile) segment ends here
          if (seg_end) {
            drain_regs(g++);
            if (er < a.R) {
              double* prow = part + static_cast<size_t>(er_c) * a.m;
#pragma unroll
              for (int e = 0; e < DCOLS; ++e) {
                const int col = half * DCOLS + e;
                if (col < a.m) prow[col] = acc64[e];
              }
            }
            wrote = true;
          } else {
            pending = 1;
          }
        }
      } else
      if (last_in_group) {
        mbar_wait(d_full, g & 1);
        ++g;
        tc_fence_after();
        if constexpr (FUSED) {
          // single accumulation group (host guarantees): D holds the whole slab
          if (base_staged) mbar_wait(base_full, 0);
          fused_drain<NPAD, EW>(a, f, tmem + lane_addr, er, gi, c0, C, half, lg, lane, warp,
                            reinterpret_cast<double*>(bars + 64), base_staged ? sbase : nullptr);
        } else {
        const bool row_ok = er < a.R;
        double* prow = part + static_cast<size_t>(er_c) * a.m;
        if constexpr (REGACC) {
          uint32_t v[DCOLS];
#pragma unroll
          for (int q = 0; q < DCOLS / 4; ++q) tc_ld4(tmem + lane_addr + half * DCOLS + q * 4, *reinterpret_cast<uint32_t(*)[4]>(v + 4 * q));
          tc_wait_ld();
#pragma unroll
          for (int e = 0; e < DCOLS; ++e) acc64[e] += static_cast<double>(__uint_as_float(v[e]));
          // the (CTA, tile) segment ends with this group: write its partial
          const bool seg_end = k + 1 == nk || (SK && q + 1 == Q);
          if (seg_end && row_ok) {
#pragma unroll
            for (int e = 0; e < DCOLS; ++e) {
              const int col = half * DCOLS + e;
              if (col < a.m) prow[col] = acc64[e];
            }
          }
        } else {
#pragma unroll 1
        for (int q = 0; q < DCOLS / 4; ++q) {
          const int col0 = half * DCOLS + q * 4;
          uint32_t v[4];
          tc_ld4(tmem + lane_addr + col0, v);
          tc_wait_ld();
          if (row_ok) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int col = col0 + e;
              if (col < a.m) prow[col] = (wrote ? prow[col] : 0.0) + static_cast<double>(__uint_as_float(v[e]));
            }
          }
        }
        }
        }
        wrote = true;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_empty);
      }
    }
    if (!SK && nq == 0 && er < a.R) {  // empty split: zero partial
      double* prow = part + static_cast<size_t>(er) * a.m;
      for (int col = half * DCOLS; col < min(a.m, (half + 1) * DCOLS); ++col) prow[col] = 0.0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// Packs the FP32 (or FP64) RHS into per-chunk TF32 hi/lo images in the
// canonical K-major no-swizzle layout: element (c, j) of chunk q sits at
// ((j/8) * (TBK/4) + (c%TBK)/4) * 32 + (j%8) * 4 + c%4 within each image.
__global__ void kv_pack_kernel(const double* v64, const float* v32, int ldv, int rows_max, int m, int npad,
                               int nchunks, const int* sel, int sel_block, int n, float* vpk, const int* skip) {
  if (skip && *skip) return;
  int rows = rows_max;  // valid rows (rows beyond are zero-filled up to nchunks * TBK)
  if (sel) rows = min(sel_block, n - *sel * sel_block);
  const long long total = static_cast<long long>(nchunks) * TBK * npad;
  const int img = npad * TBK;
  // e walks the images linearly (coalesced stores): e % img = core * 32 + lane,
  // core = (j/8) * (TBK/4) + kk/4, lane = (j%8) * 4 + kk%4
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(e / img), w = static_cast<int>(e % img);
    const int core = w >> 5, ln = w & 31;
    const int j = (core / (TBK / 4)) * 8 + (ln >> 2);
    const int kk = (core % (TBK / 4)) * 4 + (ln & 3);
    const long long c = static_cast<long long>(q) * TBK + kk;
    float hi = 0.f, lo = 0.f;
    if (c < rows && j < m) {
      if (v64) {
        const double x = v64[c * ldv + j];
        const float h = __uint_as_float(tf32_rna(static_cast<float>(x)));
        hi = h;
        lo = __uint_as_float(tf32_rna(static_cast<float>(x - static_cast<double>(h))));
      } else {
        const float x = v32[c * ldv + j];
        const float h = __uint_as_float(tf32_rna(x));
        hi = h;
        lo = __uint_as_float(tf32_rna(x - h));
      }
    }
    const size_t base = static_cast<size_t>(q) * 2 * img;
    vpk[base + w] = hi;
    vpk[base + img + w] = lo;
  }
}

template <int NPAD, int DP4, int MODE, bool TG>
void launch_tc_one(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s) {
  constexpr bool FUSED = MODE == 1;
  using L = TcLayout<NPAD>;
  constexpr int XST = TG ? TgShape<DP4>::CHUNK : TBK * 4 * DP4;
  // + the fused drain's scratch behind the barriers (bars + 64 words: ~14 KB)
  const size_t need = sizeof(float) * (STAGES * L::CHUNK_FLOATS + STAGES * XST) +
                      32 * sizeof(uint64_t) +
                      (FUSED ? 64 * sizeof(uint64_t) + sizeof(double) * (FUSED_SCRATCH_DOUBLES + TBM * ((a.m + 1) / 2 * 2)) : 0);
  // at most 2 CTAs per SM: each allocates 256 of the 512 TMEM columns
  // one CTA per SM in MODE 1/2 (512 TMEM columns each): >= 120 KB keeps a
  // second CTA off the SM; two per SM otherwise (256 columns each)
  const size_t smem = std::max<size_t>(need, MODE ? 120 * 1024 : 100 * 1024);
  if (smem > 227 * 1024) throw std::invalid_argument("gpk: operator kernel shared memory exceeds 227 KB");
  static size_t configured = 0;
  if (smem > configured) {
    configured = smem;
    GPK_CUDA(cudaFuncSetAttribute(kv_tc_kernel<NPAD, DP4, MODE, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  }
  const dim3 grid = MODE == 3 ? dim3(a.sk_ctas) : dim3((a.R + TBM - 1) / TBM, a.splits);
  kv_tc_kernel<NPAD, DP4, MODE, TG><<<grid, TcRoles<MODE>::THREADS, smem, s>>>(a, vpk, f);
  check_launch("kv_tc_kernel");
}

template <int NPAD, int MODE, bool TG>
void launch_tc_n(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s) {
  switch (a.dp / 4) {
    case 1: return launch_tc_one<NPAD, 1, MODE, TG>(a, vpk, f, s);
    case 2: return launch_tc_one<NPAD, 2, MODE, TG>(a, vpk, f, s);
    case 3: return launch_tc_one<NPAD, 3, MODE, TG>(a, vpk, f, s);
    case 4: return launch_tc_one<NPAD, 4, MODE, TG>(a, vpk, f, s);
    case 5: return launch_tc_one<NPAD, 5, MODE, TG>(a, vpk, f, s);
    case 6: return launch_tc_one<NPAD, 6, MODE, TG>(a, vpk, f, s);
    case 7: return launch_tc_one<NPAD, 7, MODE, TG>(a, vpk, f, s);
    case 8: return launch_tc_one<NPAD, 8, MODE, TG>(a, vpk, f, s);
    case 9:
      if constexpr (!TG) return launch_tc_one<NPAD, 9, MODE, TG>(a, vpk, f, s);  // d = 32 Gram image
      [[fallthrough]];
    default: throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  }
}

template <int MODE, bool TG>
void launch_tc(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s) {
  switch (kv_tc_npad(a.m)) {
    case 16: return launch_tc_n<16, MODE, TG>(a, vpk, f, s);
    case 32: return launch_tc_n<32, MODE, TG>(a, vpk, f, s);
    case 48: return launch_tc_n<48, MODE, TG>(a, vpk, f, s);
    case 64: return launch_tc_n<64, MODE, TG>(a, vpk, f, s);
    case 80: return launch_tc_n<80, MODE, TG>(a, vpk, f, s);
    default: throw std::invalid_argument("gpk: tensor-core operator supports m <= 80");
  }
}

}  // namespace

#if GPK_KV_TC_TG
// tensor-core Gram variants (built in kv_tc_tg.cu: a second translation unit
// keeps the two instantiation sets compiling in parallel)
void kv_tc_tg_launch(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s, int mode) {
  if (mode == 1)
    launch_tc<1, true>(a, vpk, f, s);
  else if (mode == 2)
    launch_tc<2, true>(a, vpk, f, s);
  else
    throw std::logic_error("gpk: tensor-core Gram distances need the one-CTA-per-SM launches (deep, fused)");
}
#else
int kv_tc_npad(int m) { return std::max(16, (m + 15) / 16 * 16); }

size_t kv_tc_pack_floats(int m, int rows) {
  const int nchunks = (rows + TBK - 1) / TBK;
  return static_cast<size_t>(nchunks) * 2 * kv_tc_npad(m) * TBK;
}

void kv_tc_pack_launch(const double* v64, const float* v32, int ldv, int rows_max, int m, const int* sel,
                       int sel_block, int n, float* vpk, const int* skip, cudaStream_t s, int rows_valid) {
  const int npad = kv_tc_npad(m);
  const int nchunks = (rows_max + TBK - 1) / TBK;
  const long long total = static_cast<long long>(nchunks) * TBK * npad;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  kv_pack_kernel<<<std::max(blocks, 1), 256, 0, s>>>(v64, v32, ldv, rows_valid >= 0 ? rows_valid : rows_max, m, npad,
                                                     nchunks, sel, sel_block, n, vpk, skip);
  check_launch("kv_pack_kernel");
}

void kv_tc_launch(const KvArgs& a, const float* vpk, cudaStream_t s, int mode) {
  const KvReduceArgs none{};
  if (a.xtg) return kv_tc_tg_launch(a, vpk, none, s, mode);
  if (mode == 3)
    launch_tc<3, false>(a, vpk, none, s);
  else if (mode == 2)
    launch_tc<2, false>(a, vpk, none, s);
  else
    launch_tc<0, false>(a, vpk, none, s);
}

void kv_tc_fused_launch(const KvArgs& a, const float* vpk, const KvReduceArgs& f, cudaStream_t s) {
  if (a.splits != 1) throw std::invalid_argument("gpk: fused slab reduce needs one column split");
  if (a.xtg) return kv_tc_tg_launch(a, vpk, f, s, 1);
  launch_tc<1, false>(a, vpk, f, s);
}
#endif  // GPK_KV_TC_TG

}  // namespace gpk
