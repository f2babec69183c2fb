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

template <int NPAD>
struct ApLayout {
  static constexpr int IMG_FLOATS = NPAD * TBK;
  static constexpr int CHUNK_FLOATS = 2 * IMG_FLOATS;
  static constexpr uint32_t CHUNK_BYTES = CHUNK_FLOATS * 4;
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

template <int NPAD, int DP4>
__global__ void __launch_bounds__(THREADS, 1) ap_persistent_kernel(const ApPersistArgs a) {
  constexpr int DP = 4 * DP4;
  constexpr int NQ = EW / 4;       // warps per TMEM lane group
  constexpr int DC = NPAD / NQ;    // drained D columns per thread
  using L = ApLayout<NPAD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* smB = reinterpret_cast<float*>(smem_raw);
  float* smX = smB + STAGES * L::CHUNK_FLOATS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smX + STAGES * TBK * DP);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* a_full = bars + 2 * STAGES;
  uint64_t* a_empty = a_full + NAB;
  uint64_t* d_full = a_empty + NAB;
  uint64_t* d_empty = d_full + 1;
  uint64_t* r_full = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_full + 3);
  double* red = reinterpret_cast<double*>(bars + 32);  // [4][NPAD]
  double* rd = red + 4 * NPAD;                           // [NQ][128]
  double* ssc = rd + NQ * 128;                           // [8]
  double* ss = ssc + 8;                                  // [96]
  double* bscore = ss + 96;                              // [1024]
  double* gemm = bscore + 1024;                          // [2][4 * 96] phase-C K halves
  int* sh = reinterpret_cast<int*>(gemm + 2 * 4 * 96);   // [0] sel, [1] stop
  double* Rt = reinterpret_cast<double*>(sh + 8);        // [128][m] residual tile

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, m = a.m, n = a.n;
  const int rows_t = min(TBM, n - tile * TBM);
  const unsigned nctas = gridDim.x;
  unsigned gen = 0;

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
  const uint32_t tmem = *tmem_slot;
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
  if (warp < EW) {
    const float* xrow = a.xs + static_cast<size_t>(row_ok ? er : 0) * DP;
#pragma unroll
    for (int u = 0; u < DP4; ++u) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xrow) + u);
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(v.x), "f"(v.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(v.z), "f"(v.w));
    }
  }
  int kg = 0;  // chunk counter across iterations (pipeline phases)
  int it = 0;
  int iters = sh[2];
  const int block = a.block, img = a.npad * 32;
  const int rpc = (block + static_cast<int>(nctas) - 1) / static_cast<int>(nctas);  // update rows per CTA

  while (!sh[1]) {
    const int sel = sh[0];
    const int r0 = sel * block, len = min(block, n - r0);
    // ---------------- C: block update (upd = Hinv_sel R_blk, V += upd, images) ----------------
    {
      const int c_beg = tile * rpc, c_end = min(block, c_beg + rpc);
      const double* Hk = a.inv + static_cast<size_t>(sel) * a.bb;
      const int nrow = c_end > c_beg ? c_end - c_beg : 0;
      // work item = (K split ks, column j): 4 rows share every residual load;
      // partials in the idle pipeline buffers, added in K-split order
      constexpr int KS = 16;
      double* gp = reinterpret_cast<double*>(smB);  // [KS][4][m]
      const int kq = (block + KS - 1) / KS;
      for (int w = tid; w < KS * m; w += THREADS) {
        const int ks = w / m, j = w % m;
        const int kb = ks * kq, ke = min(block, kb + kq);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* rr = a.R + static_cast<size_t>(r0) * m + j;
        const double* h0 = Hk + static_cast<size_t>(min(c_beg + 0, block - 1)) * block;  // row c == column c
        const double* h1 = Hk + static_cast<size_t>(min(c_beg + 1, block - 1)) * block;
        const double* h2 = Hk + static_cast<size_t>(min(c_beg + 2, block - 1)) * block;
        const double* h3 = Hk + static_cast<size_t>(min(c_beg + 3, block - 1)) * block;
#pragma unroll 8
        for (int k = kb; k < ke; ++k) {
          const double rv = rr[static_cast<size_t>(k) * m];
          acc[0] = fma(h0[k], rv, acc[0]);
          acc[1] = fma(h1[k], rv, acc[1]);
          acc[2] = fma(h2[k], rv, acc[2]);
          acc[3] = fma(h3[k], rv, acc[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) gp[(ks * 4 + q) * m + j] = acc[q];
      }
      __syncthreads();
      (void)nrow;
      for (int e = tid; e < (c_end - c_beg) * a.npad; e += THREADS) {
        const int q = e / a.npad, j = e % a.npad;
        const int c = c_beg + q;
        double u = 0.0;
        if (j < m) {
          if (c < len) {
            u = gp[q * m + j];
            for (int ks = 1; ks < KS; ++ks) u += gp[(ks * 4 + q) * m + j];
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
    grid_sync(a.gbar, nctas, gen);
    // ---------------- S: slab R[tile] -= H[tile, blk] upd ----------------
    const int nq = (len + TBK - 1) / TBK;
    const int c0 = r0;
    if (warp == EW) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic upd-image stores -> TMA reads
        for (int q = 0; q < nq; ++q) {
          const int k = kg + q, s = k % STAGES;
          if (k >= STAGES) mbar_wait(&empty[s], ((k - STAGES) / STAGES) & 1);
          const uint32_t xbytes = TBK * DP * 4;
          mbar_expect_tx(&full[s], L::CHUNK_BYTES + xbytes);
          bulk_g2s(smB + s * L::CHUNK_FLOATS, a.vpk + static_cast<size_t>(q) * L::CHUNK_FLOATS, L::CHUNK_BYTES,
                   &full[s]);
          bulk_g2s(smX + s * TBK * DP, a.xs + static_cast<size_t>(c0 + q * TBK) * DP, xbytes, &full[s]);
        }
      }
    } else if (warp == EW + 1) {
      if (lane == 0) {
        constexpr uint32_t idesc = tf32_idesc(NPAD, TBM);
        if (it > 0) mbar_wait(d_empty, (it - 1) & 1);  // previous slab's D drained
        for (int q = 0; q < nq; ++q) {
          const int k = kg + q, s = k % STAGES, b = k % NAB;
          mbar_wait(&full[s], (k / STAGES) & 1);
          mbar_wait(&a_full[b], (k / NAB) & 1);
          tc_fence_after();
          const uint32_t bh = smem_u32(smB + s * L::CHUNK_FLOATS);
          const uint32_t bl = bh + L::IMG_FLOATS * 4;
          const uint32_t ah = tmem + A_BASE + b * 64, al = ah + 32;
#pragma unroll
          for (int kk = 0; kk < TBK / 8; ++kk) {
            const uint64_t dh = umma_desc(bh + kk * 256, 128, (TBK / 4) * 128);
            const uint64_t dl = umma_desc(bl + kk * 256, 128, (TBK / 4) * 128);
            tc_mma_tf32(tmem, ah + kk * 8, dh, idesc, (q == 0 && kk == 0) ? 0u : 1u);
            tc_mma_tf32(tmem, ah + kk * 8, dl, idesc, 1u);
            tc_mma_tf32(tmem, al + kk * 8, dh, idesc, 1u);
          }
          tc_commit(&empty[s]);
          tc_commit(&a_empty[b]);
        }
        tc_commit(d_full);
      }
    } else {
      for (int q = 0; q < nq; ++q) {
        const int k = kg + q, s = k % STAGES, b = k % NAB;
        mbar_wait(&full[s], (k / STAGES) & 1);
        if (k >= NAB) mbar_wait(&a_empty[b], ((k - NAB) / NAB) & 1);
        tc_fence_after();
        const uint32_t xbase = smem_u32(smX + s * TBK * DP + qtr * CPT * DP);
        uint32_t hi[CPT], lo[CPT];
#pragma unroll
        for (int t = 0; t < CPT; ++t) {
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
          const float r = sqrt_approx(s0 + s1);
          const float kv = fmaf(r, kSqrt3f, 1.f) * ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));
          hi[t] = __float_as_uint(kv) & 0xFFFFE000u;
          lo[t] = __float_as_uint(kv - __uint_as_float(hi[t]));
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
      const bool diag = row_ok && er >= c0 && er < c0 + len;
      const int vr = er - c0;
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
            if (diag) acc += a.sigma2 * a.upd[static_cast<size_t>(vr) * m + j];
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
    grid_sync(a.gbar, nctas, gen);
    // ---------------- B: termination test and next block (every CTA alike) ----------------
    if (warp < EW) {
      const int G = static_cast<int>(nctas);
      for (int j = warp; j < m; j += EW) {  // G <= 148: at most 5 loads per lane, issued together
        double v[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const int q = lane + 32 * i;
          v[i] = q < G ? __ldcg(a.dpart + static_cast<size_t>(q) * m + j) : 0.0;
        }
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) acc += v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) ss[j] = acc;
      }
      for (int k = warp; k < a.nblocks; k += EW) {
        double t = 0.0;
        for (int q = lane; q < a.gpb; q += 32) t += __ldcg(a.spart + static_cast<size_t>(k) * a.gpb + q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) bscore[k] = sqrt(t);
      }
      eval_bar();
      for (int j = tid; j < m; j += 32 * EW) ss[j] = sqrt(ss[j]) / a.scales[j];
      eval_bar();
      if (tid == 0) {
        iters += 1;
        const double mean = ss[0];
        double sum = 0.0;
        for (int j = 1; j < m; ++j) sum += ss[j];
        const double probe = m > 1 ? sum / (m - 1) : 0.0;
        const int done = (mean <= a.tol && probe <= a.tol) ? 1 : 0;
        const int stop = (done || iters >= a.budget) ? 1 : 0;
        int best_k = 0;
        double best = -1.0;
        for (int k = 0; k < a.nblocks; ++k)
          if (bscore[k] > best) {
            best = bscore[k];
            best_k = k;
          }
        sh[0] = best_k;
        sh[1] = stop;
        if (blockIdx.x == 0) {
          a.ctl->iters = iters;
          a.ctl->mean_norm = mean;
          a.ctl->probe_norm = probe;
          a.ctl->done = done;
          a.ctl->stop = stop;
          *a.sel = best_k;
        }
      }
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

template <int NPAD, int DP4>
void launch_one(const ApPersistArgs& a, cudaStream_t s) {
  using L = ApLayout<NPAD>;
  const size_t smem = sizeof(float) * (STAGES * L::CHUNK_FLOATS + STAGES * TBK * 4 * DP4) + 32 * sizeof(uint64_t) +
                      sizeof(double) * (4 * NPAD + 4 * 128 + 8 + 96 + 1024 + 2 * 4 * 96) + 8 * sizeof(int) +
                      sizeof(double) * TBM * a.m + 64;
  if (smem > 227 * 1024) throw std::invalid_argument("gpk: persistent AP kernel shared memory exceeds 227 KB");
  static size_t configured = 0;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(ap_persistent_kernel<NPAD, DP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  ApPersistArgs args = a;
  void* params[] = {&args};
  GPK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ap_persistent_kernel<NPAD, DP4>),
                                       dim3((a.n + TBM - 1) / TBM), dim3(THREADS), params, smem, s));
  count_launch();
}

template <int NPAD>
void launch_n(const ApPersistArgs& a, cudaStream_t s) {
  switch (a.dp / 4) {
    case 1: return launch_one<NPAD, 1>(a, s);
    case 2: return launch_one<NPAD, 2>(a, s);
    case 3: return launch_one<NPAD, 3>(a, s);
    case 4: return launch_one<NPAD, 4>(a, s);
    case 5: return launch_one<NPAD, 5>(a, s);
    case 6: return launch_one<NPAD, 6>(a, s);
    case 7: return launch_one<NPAD, 7>(a, s);
    case 8: return launch_one<NPAD, 8>(a, s);
    default: throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  }
}

}  // namespace

bool ap_persistent_supported(int n, int m, int block, int sms) {
  const int tiles = (n + TBM - 1) / TBM;
  return tiles <= sms && m <= 80 && block % TBM == 0 && (block + tiles - 1) / tiles <= 4 && block / TBM <= 1024;
}

void ap_persistent_launch(const ApPersistArgs& a, cudaStream_t s) {
  switch (kv_tc_npad(a.m)) {
    case 16: return launch_n<16>(a, s);
    case 32: return launch_n<32>(a, s);
    case 48: return launch_n<48>(a, s);
    case 64: return launch_n<64>(a, s);
    case 80: return launch_n<80>(a, s);
    default: throw std::invalid_argument("gpk: persistent AP supports m <= 80");
  }
}

}  // namespace gpk
