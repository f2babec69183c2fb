// Persistent alternating-projections solver (solvers.cpp:90-145) on the
// tcgen05 operator: one cooperative launch runs every AP iteration of a solve.
//
// One CTA per SM owns one 128-row tile of the residual for the whole solve:
// the tile's inputs stay in registers, its residual rows stay in shared
// memory, TMEM stays allocated and the mbarrier pipeline keeps running across
// iterations. Per iteration, separated by two grid barriers:
//   C  block update for the selected block k: every CTA forms its share of
//      upd = Hinv_k R[blk_k] (FP64), adds it to V[blk_k] and writes the TF32
//      hi/lo operator images of upd (solvers.cpp:133-136);
//   S  slab R[tile] -= H[tile, blk_k] upd: kernel entries evaluated by 16
//      warps into TMEM, 3xTF32 tcgen05 MMAs, fused drain into the smem tile
//      (+ sigma^2 upd on the diagonal rows), the tile's column sums of R^2
//      and block-score partial (the same arithmetic as the fused slab);
//   B  every CTA sums the tile partials in the same fixed order, counts the
//      iteration, tests termination and picks the next block (ap_check /
//      ap_select, strict '>' from -1); CTA 0 publishes the control block.
// Replaces, per iteration, a cuBLAS GEMM, a packing kernel and the fused slab
// launch (their launch gaps, TMEM allocation and pipeline fill).
#include <cuda_runtime.h>

#include <algorithm>

#include "gpk_internal.cuh"
#include "tc_util.cuh"

namespace gpk {

namespace {

using namespace tc;

constexpr int TBM = 128, TBK = 32, STAGES = 3, EW = 16, THREADS = 32 * (EW + 2), CPT = TBK * 4 / EW;
constexpr int NAB = 4, A_BASE = 128, TCOLS = 512;
// tensor-core Gram distances (as kv_tc_kernel TG): Gram tile G = -2 X_tile X_c^T
// at TMEM columns [TG_COL, +32), the tile's row images hi | lo at TGA_COL
constexpr int TG_COL = 96, TGA_COL = 384;
#ifndef AP_DECIDE_ALL
#define AP_DECIDE_ALL 1
#endif
template <int DP4>
struct TgShape {
  static constexpr int KG = ((DP4 + 1) / 2) * 8;
  static constexpr int CHUNK = 2 * TBK * KG + TBK;
};

template <int NPAD>
struct ApLayout {
  static constexpr int IMG_FLOATS = NPAD * TBK;
  static constexpr int CHUNK_FLOATS = 2 * IMG_FLOATS;
  static constexpr uint32_t CHUNK_BYTES = CHUNK_FLOATS * 4;
  // the pipeline ring doubles as phase C1's staging: Hk [32][<=64] + R [<=64][<=NPAD] FP64
  static constexpr int C1_FLOATS = (32 * (64 + 4) + 64 * 88) * 2;
  static constexpr int RING_FLOATS = STAGES * CHUNK_FLOATS > C1_FLOATS ? STAGES * CHUNK_FLOATS : C1_FLOATS;
};

__device__ __forceinline__ void eval_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory"); }

// Grid barrier for a cooperative launch: a monotonic arrival counter (zeroed
// by the host before the launch); barrier g completes at nctas * g arrivals.
// The CTA barrier orders the CTA's writes before thread 0's release fence
// (cumulative), and thread 0's acquire load before everyone's later reads.
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned nctas, unsigned& gen) {
  __syncthreads();
  ++gen;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    const unsigned target = nctas * gen;
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

template <int NPAD, int DP4, bool TG>
__global__ void __launch_bounds__(THREADS, 1) ap_persistent_kernel(const ApPersistArgs a) {
  constexpr int DP = 4 * DP4;
  constexpr bool GRAM = !TG && GPK_GRAM && DP4 >= 6;  // (x, |x|^2, 0...) image for d >= 21, as kv_tc_kernel
  constexpr int KG = TgShape<DP4>::KG;
  constexpr int XST = TG ? TgShape<DP4>::CHUNK : TBK * DP;  // column data floats per stage
  constexpr int NQ = EW / 4;       // warps per TMEM lane group
  constexpr int DC = NPAD / NQ;    // drained D columns per thread
  using L = ApLayout<NPAD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* smB = reinterpret_cast<float*>(smem_raw);
  float* smX = smB + L::RING_FLOATS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smX + STAGES * XST);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* a_full = bars + 2 * STAGES;
  uint64_t* a_empty = a_full + NAB;
  uint64_t* d_full = a_empty + NAB;
  uint64_t* d_empty = d_full + 1;
  uint64_t* r_full = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + 3);
  uint64_t* p_full = d_full + 4;  // tile partials staged for the last CTA's reduction
  uint64_t* g_full = d_full + 5;     // TG: Gram tile of the chunk in TMEM
  uint64_t* g_empty = d_full + 6;    // TG: eval warps have read it
  uint64_t* arow_full = d_full + 7;  // TG: row images written
  double* red = reinterpret_cast<double*>(bars + 32);  // [4][NPAD]
  double* rd = red + 4 * NPAD;                           // [NQ][128]
  double* ssc = rd + NQ * 128;                           // [8]
  double* ss = ssc + 8;                                  // [96]
  double* bscore = ss + 96;                              // [1024]
  double* gemm = bscore + 1024;                          // [2][4 * 96] phase-C K halves
  int* sh = reinterpret_cast<int*>(gemm + 2 * 4 * 96);   // [0] sel, [1] stop
  double* Rt = reinterpret_cast<double*>(sh + 8);        // [128][m] residual tile
  double* scl = Rt + TBM * a.m;                          // [m] column scales (termination test)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, m = a.m, n = a.n;
  const int rows_t = min(TBM, n - tile * TBM);
  const unsigned nctas = gridDim.x;
  unsigned gen = 0;
  for (int j = threadIdx.x; j < a.m; j += blockDim.x) scl[j] = a.scales[j];

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
    mbar_init(r_full, 1);
    mbar_init(p_full, 1);
    if (TG) {
      mbar_init(g_full, 1);
      mbar_init(g_empty, EW);
      mbar_init(arow_full, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh[0] = *a.sel;
    sh[1] = a.ctl->stop;
    sh[2] = a.ctl->iters;
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
  // one CTA per SM allocating all 512 columns: the allocation starts at 0
  // (a compile-time base keeps the MMA issue warp-uniform, tc_util.cuh)
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0) __trap();
  // the residual tile (after the host-side refresh) lives in smem for the solve
  if (tid == 0) {
    const uint32_t bytes = static_cast<uint32_t>(rows_t) * m * 8u;
    mbar_expect_tx(r_full, bytes);
    bulk_g2s(Rt, a.R + static_cast<size_t>(tile) * TBM * m, bytes, r_full);
  }
  mbar_wait(r_full, 0);

  // evaluation-thread constants: row = TMEM lane, inputs in registers
  const int lg = warp & 3, qtr = warp >> 2;
  const int lrow = lg * 32 + lane, er = tile * TBM + lrow;
  const bool row_ok = er < n;
  const uint32_t lane_addr = static_cast<uint32_t>(lg * 32) << 16;
  uint64_t xi2[2 * DP4];
  float ni = 0.f;  // Gram form (d >= 21): |x_i|^2 seeds the distance accumulator
  if (warp < EW && TG) {
    // row images hi | lo of the 22-bit split coordinates in TMEM (the Gram
    // MMAs' A operand) and |x'_i|^2 (kv_tc_kernel TG, tg_image_kernel)
    const float* xrow = a.xs + static_cast<size_t>(row_ok ? er : 0) * DP;
    float hv[4 * DP4], lv[4 * DP4];
#pragma unroll
    for (int u = 0; u < DP4; ++u) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xrow) + u);
      const float c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        tg_split(c[e], hv[4 * u + e], lv[4 * u + e]);
        ni = tg_norm_step(ni, hv[4 * u + e], lv[4 * u + e]);
      }
    }
    if (qtr == 0) {
      const uint32_t ta = tmem + lane_addr + TGA_COL;
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
  } else if (warp < EW) {
    const float* xrow = a.xs + static_cast<size_t>(row_ok ? er : 0) * DP;
#pragma unroll
    for (int u = 0; u < DP4; ++u) {
      float4 v = __ldg(reinterpret_cast<const float4*>(xrow) + u);
      if constexpr (GRAM) gram_row(v, 4 * u, a.d, ni);
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(v.x), "f"(v.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(v.z), "f"(v.w));
    }
  }
  uint64_t acc_seed;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc_seed) : "f"(ni), "f"(0.f));
  const float sigma2f = static_cast<float>(a.sigma2);
  int kg = 0;  // chunk counter across iterations (pipeline phases)
  int pphase = 0;  // uses of p_full (this CTA was last)
  int it = 0;
  int iters = sh[2];
  const int block = a.block, img = a.npad * 32;
  const int rpc = (block + static_cast<int>(nctas) - 1) / static_cast<int>(nctas);  // update rows per CTA

  const bool prof = a.prof && tile == 0 && tid == 0;
  unsigned long long pt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tprev = 0;
  auto mark = [&](int i) {
    if (prof) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (globaltimer is too coarse)
      if (i >= 0) pt[i] += t - tprev;
      tprev = t;
    }
  };
  mark(-1);
  while (!sh[1]) {
    const int sel = sh[0];
    const int r0 = sel * block, len = min(block, n - r0);
    // ---------------- C: block update (upd = Hinv_sel R_blk, V += upd, images) ----------------
    {
      const double* Hk = a.inv + static_cast<size_t>(sel) * a.bb;  // symmetric: row c == column c
      // C1: 2-D split of upd = Hk R_blk over (32-row group rg, K eighth kg):
      // the CTA stages Hk[rg rows][kg cols] and R_blk[kg rows] in the idle
      // pipeline buffers (one round of coalesced loads) and writes its FP64
      // partial to cpart[kg]
      const int kq = block / 8, rgs = block / 32;
      if (tile < rgs * 8) {
        const int rg = tile >> 3, kgi = tile & 7, kb = kgi * kq;
        // FP64 throughout: upd's error must not scale with the block's
        // condition number (an FP32 Hk or FP32 products give relative errors
        // ~1e-7 kappa: a non-contracting block step for kappa ~ 1e6). The
        // 32 x m x kq product runs on the FP64 tensor cores (mma.sync m8n8k4):
        // sH [32][kq + 4] and sR [kq][88] (zero-padded columns) are strided so
        // the fragment loads are bank-conflict free.
        constexpr int SRS = 88;
        const int sha = kq + 4;
        double* sH = reinterpret_cast<double*>(smB);  // [32][kq + 4]
        double* sR = sH + 32 * sha;                   // [kq][SRS]
        // one round of loads (all issued before the first store); columns of sR
        // beyond m only feed discarded output columns and are left as they are
        constexpr int HN = (32 * 64 + THREADS - 1) / THREADS, RN = (64 * 80 + THREADS - 1) / THREADS;
        const int kv = max(0, min(kq, len - kb));
        const double* rsrc = a.R + static_cast<size_t>(r0 + kb) * m;
        double hv[HN], rv[RN];
#pragma unroll
        for (int i = 0; i < HN; ++i) {
          // Hk symmetric: read row kb + k, columns rg*32 + r (32 consecutive words per warp)
          const int e = tid + i * THREADS, k = e >> 5, r = e & 31, row = rg * 32 + r, kk = kb + k;
          hv[i] = (e < 32 * kq && row < len && kk < len) ? Hk[static_cast<size_t>(kk) * block + row] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < RN; ++i) {
          const int e = tid + i * THREADS;
          rv[i] = e < kv * m ? rsrc[e] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < HN; ++i) {
          const int e = tid + i * THREADS;
          if (e < 32 * kq) sH[(e & 31) * sha + (e >> 5)] = hv[i];
        }
#pragma unroll
        for (int i = 0; i < RN; ++i) {
          const int e = tid + i * THREADS;
          if (e < kq * m) sR[(e / m) * SRS + e % m] = rv[i];
        }
        __syncthreads();
        mark(6);
        // warp w < ceil(m / 8): column tile w, all four 8-row tiles
        const int ntiles = (m + 7) / 8;
        if (warp < ntiles) {
          const int fr = lane >> 2, fc = lane & 3;
          double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
          for (int k0 = 0; k0 < kq; k0 += 4) {
            const double bv = sR[(k0 + fc) * SRS + warp * 8 + fr];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
              const double av = sH[(mt * 8 + fr) * sha + k0 + fc];
              asm volatile(
                  "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                  : "+d"(acc[mt][0]), "+d"(acc[mt][1])
                  : "d"(av), "d"(bv));
            }
          }
          const int col = warp * 8 + 2 * fc;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            double* dst = a.cpart + (static_cast<size_t>(kgi) * block + rg * 32 + mt * 8 + fr) * m;
            if (col < m) dst[col] = acc[mt][0];
            if (col + 1 < m) dst[col + 1] = acc[mt][1];
          }
        }
      }
      mark(7);
      grid_sync(a.gbar, nctas, gen);
      mark(8);
      // C2: this CTA's rows of upd = the eight partials in order; V += upd and
      // the TF32 hi/lo images of upd for the slab's MMAs
      const int c_beg = tile * rpc, c_end = min(block, c_beg + rpc);
      for (int e = tid; e < (c_end - c_beg) * a.npad; e += THREADS) {
        const int q = e / a.npad, j = e % a.npad;
        const int c = c_beg + q;
        double u = 0.0;
        if (j < m) {
          if (c < len) {
            double pv[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) pv[g] = __ldcg(a.cpart + (static_cast<size_t>(g) * block + c) * m + j);
            u = pv[0];
#pragma unroll
            for (int g = 1; g < 8; ++g) u += pv[g];
          }
          a.upd[static_cast<size_t>(c) * m + j] = u;
          if (c < len) a.V[static_cast<size_t>(r0 + c) * m + j] += u;
        }
        uint32_t hb, lb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(static_cast<float>(u)));
        const float hf = __uint_as_float(hb);
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(static_cast<float>(u - static_cast<double>(hf))));
        const int kk = c % 32;
        float* base = a.vpk + static_cast<size_t>(c / 32) * 2 * img;
        const int off = ((j / 8) * 8 + kk / 4) * 32 + (j % 8) * 4 + (kk % 4);
        base[off] = hf;
        base[img + off] = __uint_as_float(lb);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // C1 staging writes -> the slab's TMA
    mark(0);
    grid_sync(a.gbar, nctas, gen);
    mark(1);
    // ---------------- S: slab R[tile] -= H[tile, blk] upd ----------------
    const int nq = (len + TBK - 1) / TBK;
    const int c0 = r0;
    if (warp == EW) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic upd-image stores -> TMA reads
        for (int q = 0; q < nq; ++q) {
          const int k = kg + q, s = k % STAGES;
          if (k >= STAGES) mbar_wait(&empty[s], ((k - STAGES) / STAGES) & 1);
          const uint32_t xbytes = XST * 4;
          mbar_expect_tx(&full[s], L::CHUNK_BYTES + xbytes);
          bulk_g2s(smB + s * L::CHUNK_FLOATS, a.vpk + static_cast<size_t>(q) * L::CHUNK_FLOATS, L::CHUNK_BYTES,
                   &full[s]);
          if constexpr (TG)  // block % 32 == 0 (ap_persistent_supported)
            bulk_g2s(smX + s * XST, a.xtg + static_cast<size_t>(c0 / TBK + q) * XST, xbytes, &full[s]);
          else
            bulk_g2s(smX + s * XST, a.xs + static_cast<size_t>(c0 + q * TBK) * DP, xbytes, &full[s]);
        }
      }
    } else if (warp == EW + 1) {
      {  // whole warp: waits and operands; one elected lane issues (tc_util.cuh)
        constexpr uint32_t idesc = tf32_idesc(NPAD, TBM);
        constexpr uint32_t gdesc = tf32_idesc(TBK, TBM);
        constexpr uint32_t GHI = tc_desc_hi((KG / 4) * 128), VHI = tc_desc_hi((TBK / 4) * 128);
        // TG: G(k) = -2 X_tile X_c(k)^T, cross terms first, hi.hi last
        auto gram_mma = [&](int k) {
          const int s = k % STAGES;
          const uint32_t ah = tmem + TGA_COL, al = ah + KG;
          const uint32_t bh = tc_desc_lo(smem_u32(smX + s * XST), 128), bl = bh + ((TBK * KG * 4) >> 4);
          if (tc_elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KG / 8; ++ks) {
              tc_mma_u<GHI, gdesc>(tmem + TG_COL, ah + ks * 8, bl + ks * 16, ks ? 1u : 0u);
              tc_mma_u<GHI, gdesc>(tmem + TG_COL, al + ks * 8, bh + ks * 16, 1u);
            }
#pragma unroll
            for (int ks = 0; ks < KG / 8; ++ks) tc_mma_u<GHI, gdesc>(tmem + TG_COL, ah + ks * 8, bh + ks * 16, 1u);
            tc_commit_u(g_full);
          }
          __syncwarp();
        };
        if (TG && nq > 0) {
          if (it == 0) mbar_wait(arow_full, 0);
          if (kg > 0) mbar_wait(g_empty, (kg - 1) & 1);  // previous slab's last Gram tile read
          mbar_wait(&full[kg % STAGES], (kg / STAGES) & 1);
          tc_fence_after();
          gram_mma(kg);
        }
        if (it > 0) mbar_wait(d_empty, (it - 1) & 1);  // previous slab's D drained
        for (int q = 0; q < nq; ++q) {
          const int k = kg + q, s = k % STAGES, b = k % NAB;
          mbar_wait(&full[s], (k / STAGES) & 1);
          if (TG && q + 1 < nq) {  // next chunk's Gram tile once the eval warps hold this one's
            mbar_wait(&full[(k + 1) % STAGES], ((k + 1) / STAGES) & 1);
            mbar_wait(g_empty, k & 1);
            tc_fence_after();
            gram_mma(k + 1);
          }
          mbar_wait(&a_full[b], (k / NAB) & 1);
          tc_fence_after();
          const uint32_t bh = tc_desc_lo(smem_u32(smB + s * L::CHUNK_FLOATS), 128);
          const uint32_t bl = bh + ((L::IMG_FLOATS * 4) >> 4);
          const uint32_t ah = tmem + A_BASE + b * 64, al = ah + 32;
          if (tc_elect_one()) {
#pragma unroll
            for (int kk = 0; kk < TBK / 8; ++kk) {
              tc_mma_u<VHI, idesc>(tmem, ah + kk * 8, bh + kk * 16, (q == 0 && kk == 0) ? 0u : 1u);
              tc_mma_u<VHI, idesc>(tmem, ah + kk * 8, bl + kk * 16, 1u);
              tc_mma_u<VHI, idesc>(tmem, al + kk * 8, bh + kk * 16, 1u);
            }
            tc_commit_u(&empty[s]);
            tc_commit_u(&a_empty[b]);
          }
          __syncwarp();
        }
        if (tc_elect_one()) tc_commit_u(d_full);
        __syncwarp();
      }
    } else {
      for (int q = 0; q < nq; ++q) {
        const int k = kg + q, s = k % STAGES, b = k % NAB;
        mbar_wait(&full[s], (k / STAGES) & 1);
        if (k >= NAB) mbar_wait(&a_empty[b], ((k - NAB) / NAB) & 1);
        tc_fence_after();
        const uint32_t xbase = smem_u32(smX + s * XST + qtr * CPT * DP);
        uint32_t hi[CPT], lo[CPT];
        float tg_r2[TG ? CPT : 1];
        if constexpr (TG) {
          mbar_wait(g_full, k & 1);
          tc_fence_after();
          uint32_t gv[CPT];
          tc_ld8(tmem + lane_addr + TG_COL + qtr * CPT, gv);
          tc_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(g_empty);
          const float4* ncs = reinterpret_cast<const float4*>(smX + s * XST + 2 * TBK * KG + qtr * CPT);
#pragma unroll
          for (int t4 = 0; t4 < CPT / 4; ++t4) {
            const float4 nc = ncs[t4];
            tg_r2[4 * t4] = (ni + nc.x) + __uint_as_float(gv[4 * t4]);
            tg_r2[4 * t4 + 1] = (ni + nc.y) + __uint_as_float(gv[4 * t4 + 1]);
            tg_r2[4 * t4 + 2] = (ni + nc.z) + __uint_as_float(gv[4 * t4 + 2]);
            tg_r2[4 * t4 + 3] = (ni + nc.w) + __uint_as_float(gv[4 * t4 + 3]);
          }
        }
#pragma unroll
        for (int t = 0; t < CPT; ++t) {
          float r;
          if constexpr (TG) {
            r = sqrt_approx(fmaxf(tg_r2[t], 0.f));
          } else if constexpr (GRAM) {
            r = sqrt_approx(gram_r2<DP4>(xbase + t * DP * 4, xi2, acc_seed));
          } else {
          uint64_t acc0 = 0ull, acc1 = 0ull;
#pragma unroll
          for (int u = 0; u < DP4; ++u) {
            uint64_t c01, c23, d01, d23;
            asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xbase + (t * DP + 4 * u) * 4));
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
          const float kv = fmaf(r, kSqrt3f, 1.f) * ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));
          hi[t] = __float_as_uint(kv) & 0xFFFFE000u;
          lo[t] = __float_as_uint(kv - __uint_as_float(hi[t]));
        }
        {  // diagonal entries: k(x_i, x_i) + sigma^2 (H = K + sigma^2 I on the slab, so
           // the drain needs no upd rows); also pins the Gram form's r = 0
          const int cbase = c0 + q * TBK + qtr * CPT;
          const bool hit = row_ok && static_cast<unsigned>(er - cbase) < static_cast<unsigned>(CPT);
          if (__any_sync(0xffffffffu, hit)) gram_pin_diagonal<CPT>(hit, er - cbase, a.log2_s2, hi, lo, sigma2f);
        }
        const uint32_t abase = tmem + lane_addr + A_BASE + b * 64 + qtr * CPT;
        tc_st8(abase, hi);
        tc_st8(abase + 32, lo);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[b]);
      }
      // ---- drain: R_tile -= D (+ sigma^2 upd on the block's own rows) ----
      mbar_wait(d_full, it & 1);
      tc_fence_after();
      double rowdot = 0.0;
#pragma unroll 1
      for (int q = 0; q < DC / 4; ++q) {
        const int col0 = qtr * DC + q * 4;
        uint32_t v[4];
        tc_ld4(tmem + lane_addr + col0, v);
        tc_wait_ld();
        double cs[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = col0 + e;
          cs[e] = 0.0;
          if (row_ok && j < m) {
            double acc = static_cast<double>(__uint_as_float(v[e]));
            const double val = Rt[static_cast<size_t>(lrow) * m + j] - acc;
            Rt[static_cast<size_t>(lrow) * m + j] = val;
            a.R[static_cast<size_t>(er) * m + j] = val;
            cs[e] = val * val;
            rowdot += val * a.inv_scales[j];
          }
        }
        int basei = 0;
#pragma unroll
        for (int o = 16, cnt = 4; o >= 8; o >>= 1, cnt >>= 1) {
          const int hf = cnt / 2;
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int kk = 0; kk < hf; ++kk) {
            const double send = up ? cs[kk] : cs[kk + hf];
            const double keep = up ? cs[kk + hf] : cs[kk];
            cs[kk] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
          if (up) basei += hf;
        }
        cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 4);
        cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 2);
        cs[0] += __shfl_xor_sync(0xffffffffu, cs[0], 1);
        if ((lane & 7) == 0) red[lg * NPAD + col0 + basei] = cs[0];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty);
      rd[qtr * 128 + lrow] = rowdot;
      eval_bar();
      for (int j = tid; j < m; j += 32 * EW)
        a.dpart[static_cast<size_t>(tile) * m + j] = ((red[j] + red[NPAD + j]) + red[2 * NPAD + j]) + red[3 * NPAD + j];
      if (qtr == 0) {
        double w = rd[lrow];
#pragma unroll
        for (int p = 1; p < NQ; ++p) w += rd[p * 128 + lrow];
        double sc = row_ok ? w * w : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
        if (lane == 0) ssc[lg] = sc;
      }
      eval_bar();
      if (tid == 0) a.spart[tile] = ((ssc[0] + ssc[1]) + ssc[2]) + ssc[3];
    }
    if (a.stats && tile == 0 && tid == 0) {  // device counters, as the operator kernels keep them
      const double entries = static_cast<double>(n) * len;
      atomicAdd(a.stats, entries * m);
      atomicAdd(a.stats + 1, entries * (2.0 * m + 3.0 * a.d + 6.0));
      atomicAdd(a.stats + 2, entries * (3.0 * a.d + 6.0));
    }
    kg += nq;
    ++it;
    mark(2);
    // ---------------- B: termination test and next block ----------------
    // Every CTA (AP_DECIDE_ALL, default) or the last CTA to finish its slab
    // (arrival ticket) sums the tile partials in a fixed order, tests
    // termination and picks the next block (ap_check / ap_select, strict '>'
    // from -1); CTA 0 (or the last CTA) writes the control block. With one
    // deciding CTA the others wait on a release flag carrying the decision;
    // measured: that CTA's rarely-run code path costs ~4 us of instruction
    // fetch per iteration, while a grid barrier + the same bitwise decision
    // in every CTA keeps the path hot on every SM.
    if (tid == 0) iters += 1;  // every CTA counts iterations (budget test)
#if AP_DECIDE_ALL
    grid_sync(a.gbar, nctas, gen);  // every tile's partials are published
    mark(3);
    if (true) {
#else
    __syncthreads();
    if (tid == 0) {
      if (a.prof && it <= 64) {  // development timeline: ticket time of every CTA (globaltimer)
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        a.prof[16 + (it - 1) * 160 + tile] = gt;
      }
      __threadfence();
      const unsigned t = atomicAdd(a.gbar + 1, 1u);
      sh[3] = (t == nctas * static_cast<unsigned>(it) - 1u) ? 1 : 0;
    }
    __syncthreads();
    mark(3);
    if (sh[3]) {
      __threadfence();
#endif
      if (a.prof && it <= 64 && tid == 0 && tile == 0) {  // development timeline
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(gt));
        a.prof[16 + (it - 1) * 160 + 155] = gt;
      }
      // thread (j, p) = (tid / 8, tid % 8) sums column j of the tile partials
      // over tiles p, p + 8, ... then a fixed xor-4/2/1 tree; thread k < nblocks
      // sums block k's score partials in order. The partials arrive by one bulk
      // copy into the idle pipeline buffers when they fit, else as one round of
      // loads per thread (same order either way).
      const int G = static_cast<int>(nctas);
      const uint32_t pbytes = static_cast<uint32_t>(G) * m * 8u;
      const bool staged = pbytes <= (L::RING_FLOATS + STAGES * TBK * DP) * 4u && (pbytes % 16u) == 0u;
      if (staged) {
        if (tid == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");  // other CTAs' generic writes -> bulk read
          mbar_expect_tx(p_full, pbytes);
          bulk_g2s(smB, a.dpart, pbytes, p_full);
        }
        double sp[4] = {0.0, 0.0, 0.0, 0.0};  // gpb <= 4 (ap_persistent_supported)
        if (tid < a.nblocks) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < a.gpb) sp[q] = __ldcg(a.spart + static_cast<size_t>(tid) * a.gpb + q);
        }
        mbar_wait(p_full, pphase & 1);
        if (a.prof && it <= 64 && tid == 0 && tile == 0) {  // development timeline
          unsigned long long gt;
          asm volatile("mov.u64 %0, %%clock64;" : "=l"(gt));
          a.prof[16 + (it - 1) * 160 + 156] = gt;
        }
        const double* st = reinterpret_cast<const double*>(smB);
        const int j = tid >> 3, p = tid & 7;
        double acc = 0.0;
        if (j < m)
          for (int q = p; q < G; q += 8) acc += st[static_cast<size_t>(q) * m + j];
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (p == 0 && j < m) ss[j] = sqrt(acc) / scl[j];
        if (tid < a.nblocks) bscore[tid] = sqrt(((sp[0] + sp[1]) + sp[2]) + sp[3]);
      } else {
        constexpr int QH = 10;  // 2 x 10 x 8 >= 148 tiles (ap_persistent_supported)
        const int j = tid >> 3, p = tid & 7;
        double v[QH];
  #pragma unroll
        for (int i = 0; i < QH; ++i) {
          const int q = p + 8 * i;
          v[i] = (j < m && q < G) ? __ldcg(a.dpart + static_cast<size_t>(q) * m + j) : 0.0;
        }
        double sp[4] = {0.0, 0.0, 0.0, 0.0};  // gpb <= 4 (ap_persistent_supported)
        if (tid < a.nblocks) {
  #pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < a.gpb) sp[q] = __ldcg(a.spart + static_cast<size_t>(tid) * a.gpb + q);
        }
        double acc = 0.0;
  #pragma unroll
        for (int i = 0; i < QH; ++i) acc += v[i];
        if (G > 8 * QH) {
  #pragma unroll
          for (int i = 0; i < QH; ++i) {
            const int q = p + 8 * (QH + i);
            v[i] = (j < m && q < G) ? __ldcg(a.dpart + static_cast<size_t>(q) * m + j) : 0.0;
          }
  #pragma unroll
          for (int i = 0; i < QH; ++i) acc += v[i];
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (p == 0 && j < m) ss[j] = sqrt(acc) / scl[j];
        if (tid < a.nblocks) bscore[tid] = sqrt(((sp[0] + sp[1]) + sp[2]) + sp[3]);
      }
      if (staged) ++pphase;
      __syncthreads();
      if (a.prof && it <= 64 && tid == 0 && tile == 0) {  // development timeline
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(gt));
        a.prof[16 + (it - 1) * 160 + 157] = gt;
      }
      if (warp == 0) {
        // probe mean over columns 1..m-1 and the first maximal block score
        // (the serial strict '>' scan from -1 of ap_select)
        double sum = 0.0;
        for (int jj = 1 + lane; jj < m; jj += 32) sum += ss[jj];
  #pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        double best = -1.0;
        int best_k = 0x7fffffff;
        for (int k = lane; k < a.nblocks; k += 32)
          if (bscore[k] > best) {
            best = bscore[k];
            best_k = k;
          }
  #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int ok = __shfl_xor_sync(0xffffffffu, best_k, o);
          if (ob > best || (ob == best && ok < best_k)) {
            best = ob;
            best_k = ok;
          }
        }
        if (best_k == 0x7fffffff) best_k = 0;
        if (lane == 0) {
          const double mean = ss[0];
          const double probe = m > 1 ? sum / (m - 1) : 0.0;
          const int done = (mean <= a.tol && probe <= a.tol) ? 1 : 0;
          const int stop = (done || iters >= a.budget) ? 1 : 0;
          sh[0] = best_k;
          sh[1] = stop;
          if (!AP_DECIDE_ALL || tile == 0) {
            a.ctl->iters = iters;
            a.ctl->mean_norm = mean;
            a.ctl->probe_norm = probe;
            a.ctl->done = done;
            a.ctl->stop = stop;
            *a.sel = best_k;
          }
          if (a.prof && it <= 64 && tile == 0) {
            unsigned long long gt;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(gt));
            a.prof[16 + (it - 1) * 160 + 159] = gt;
          }
#if !AP_DECIDE_ALL
          // the decision travels in the release word itself (iteration << 12 |
          // stop << 11 | block; nblocks <= 148 here), so a waiting CTA needs one
          // acquire load; this thread's ctl / sel stores are ordered before it
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.gbar + 2),
                       "r"((static_cast<unsigned>(it) << 12) | (static_cast<unsigned>(stop) << 11) |
                           static_cast<unsigned>(best_k))
                       : "memory");
#endif
        }
      }
    } else if (tid == 0) {
      unsigned v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.gbar + 2) : "memory");
        if ((v >> 12) >= static_cast<unsigned>(it)) break;
        __nanosleep(32);
      }
      sh[0] = static_cast<int>(v & 2047u);
      sh[1] = static_cast<int>((v >> 11) & 1u);
    }
    __syncthreads();
    mark(4);
    if (prof) ++pt[9];
  }
  if (prof)
    for (int i = 0; i < 10; ++i) a.prof[i] += pt[i];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

template <int NPAD, int DP4, bool TG>
void launch_one(const ApPersistArgs& a, cudaStream_t s) {
  using L = ApLayout<NPAD>;
  constexpr int XST = TG ? TgShape<DP4>::CHUNK : TBK * 4 * DP4;
  const size_t smem = sizeof(float) * (L::RING_FLOATS + STAGES * XST) + 32 * sizeof(uint64_t) +
                      sizeof(double) * (4 * NPAD + 4 * 128 + 8 + 96 + 1024 + 2 * 4 * 96) + 8 * sizeof(int) +
                      sizeof(double) * (TBM + 1) * a.m + 64;
  if (smem > 227 * 1024) throw std::invalid_argument("gpk: persistent AP kernel shared memory exceeds 227 KB");
  static size_t configured = 0;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(ap_persistent_kernel<NPAD, DP4, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  ApPersistArgs args = a;
  void* params[] = {&args};
  GPK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ap_persistent_kernel<NPAD, DP4, TG>),
                                       dim3((a.n + TBM - 1) / TBM), dim3(THREADS), params, smem, s));
  count_launch();
}

template <int NPAD, bool TG>
void launch_n(const ApPersistArgs& a, cudaStream_t s) {
  switch (a.dp / 4) {
    case 1: return launch_one<NPAD, 1, TG>(a, s);
    case 2: return launch_one<NPAD, 2, TG>(a, s);
    case 3: return launch_one<NPAD, 3, TG>(a, s);
    case 4: return launch_one<NPAD, 4, TG>(a, s);
    case 5: return launch_one<NPAD, 5, TG>(a, s);
    case 6: return launch_one<NPAD, 6, TG>(a, s);
    case 7: return launch_one<NPAD, 7, TG>(a, s);
    case 8: return launch_one<NPAD, 8, TG>(a, s);
    case 9:
      if constexpr (!TG) return launch_one<NPAD, 9, TG>(a, s);  // d = 32 Gram image
      [[fallthrough]];
    default: throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  }
}

template <bool TG>
void launch_tg(const ApPersistArgs& a, cudaStream_t s) {
  switch (kv_tc_npad(a.m)) {
    case 16: return launch_n<16, TG>(a, s);
    case 32: return launch_n<32, TG>(a, s);
    case 48: return launch_n<48, TG>(a, s);
    case 64: return launch_n<64, TG>(a, s);
    case 80: return launch_n<80, TG>(a, s);
    default: throw std::invalid_argument("gpk: persistent AP supports m <= 80");
  }
}

}  // namespace

bool ap_persistent_supported(int n, int m, int block, int sms) {
  const int tiles = (n + TBM - 1) / TBM;
  return tiles <= sms && m <= 80 && block % TBM == 0 && (block + tiles - 1) / tiles <= 4 && block / TBM <= 1024;
}

void ap_persistent_launch(const ApPersistArgs& a, cudaStream_t s) {
  if (a.xtg)
    launch_tg<true>(a, s);
  else
    launch_tg<false>(a, s);
}

}  // namespace gpk
