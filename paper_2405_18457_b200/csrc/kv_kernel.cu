// K1/K2/K3: fused ARD distance -> Matérn-3/2 -> FMA into the n x m RHS block.
//
// Replaces KernelOperator::apply / apply_rows / apply_columns
// (/root/reference/proj/core/src/kernel.cpp:133-177, with fill_rows 111-120,
// matern_profile 35-39 and accumulate_rows_product 15-30). K is never
// materialised: each CTA evaluates a 256-row x 32-column tile of K into shared
// memory (one entry per thread per column, x_row held in registers, x_col
// broadcast from smem, MUFU sqrt + ex2), then contracts it with the matching
// 32 rows of V by a register-tiled SIMT GEMM (8 rows x TC cols per lane plus
// one shared "extra" column so m = 8*TC + 1 = 65 needs no padding).
//
// Pipeline (one __syncthreads per 32-column chunk): iteration k waits for the
// cp.async copies of chunk k+1, issues chunk k+2, evaluates K for chunk k+1
// into Ks[(k+1)%2] and runs the GEMM of chunk k on Ks[k%2] — so MUFU/eval work
// of one chunk and FFMA work of the previous overlap across warps.
//
// Precision: FP32 evaluation, FP32 accumulation over at most
// flush_chunks*32 columns, then FP64 accumulation into the per-split partial
// (each thread owns its outputs; no atomics, deterministic). Split-K over
// columns fills the 148 SMs at small row counts; kv_reduce sums splits in a
// fixed order in FP64 and adds sigma^2 V on the diagonal.
#include <cuda_runtime.h>

#include <algorithm>

#include "gpk_internal.cuh"
#include "ap_epilogue.cuh"

namespace gpk {

namespace {

constexpr int BM = 256;
constexpr int BK = 32;
constexpr int NT = 256;

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
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// -log2(e) * sqrt(3): e^{-sqrt3 r} = 2^{r * kNegSqrt3Log2e}
constexpr float kNegSqrt3Log2e = -2.4988211106473432f;  // -sqrt(3) * log2(e)
constexpr float kSqrt3f = 1.7320508075688772f;

template <int TC>
struct Tile {
  static constexpr int MC = 8 * TC;       // columns handled by the 8x4-lane grid
  static constexpr int MP = MC + 4;       // smem/global row stride of V (floats); col MC = extra
};

template <int TC, int DP4>
__global__ void __launch_bounds__(NT, (TC >= 8 ? 1 : 2)) kv_slab_kernel(const KvArgs a) {
  constexpr int MC = Tile<TC>::MC;
  constexpr int MP = Tile<TC>::MP;
  constexpr int DP = 4 * DP4;
  extern __shared__ __align__(16) float smem[];
  float* Ks = smem;               // [2][BK][BM]
  float* Vs = Ks + 2 * BK * BM;   // [3][BK][MP]
  float* Xc = Vs + 3 * BK * MP;   // [3][BK][DP]

  if (a.skip && *a.skip) return;

  int c0 = a.c0, C = a.C;
  if (a.sel) {
    c0 = *a.sel * a.sel_block;
    C = min(a.sel_block, a.n - c0);
  }
  const int tile = blockIdx.x, split = blockIdx.y;
  const int cb = split * a.cols_per_split;
  const int ce = min(C, cb + a.cols_per_split);
  const int nq = ce > cb ? (ce - cb + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.stats && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    const double entries = static_cast<double>(a.R) * C;
    atomicAdd(a.stats, entries * a.m);
    atomicAdd(a.stats + 1, entries * (2.0 * a.m + 3.0 * a.d + 6.0));
    atomicAdd(a.stats + 2, entries * (2.0 * a.m + 3.0 * a.d + 6.0));  // all on the FP32 pipe
  }

  // ---- evaluation role: this thread's K row ----
  const int er = tile * BM + tid;
  const int er_c = er < a.R ? er : 0;
  const int gi = a.row_idx ? a.row_idx[er_c] : a.r0 + er_c;
  const float4* xi_ptr =
      reinterpret_cast<const float4*>((a.xs_rows ? a.xs_rows : a.xs) + static_cast<size_t>(gi) * a.dp);

  // ---- GEMM role ----
  const int rg = warp >> 1, wcg = warp & 1, lr = lane >> 2, lc = lane & 3;
  const int rbase = rg * 64 + lr * 4;  // rows rbase+i (i<4) and rbase+32+i
  const int cbase = wcg * 4 * TC + lc * TC;
  const int q = wcg * 4 + lc;
  const int rext = rg * 64 + (q < 4 ? lr * 4 + q : 32 + lr * 4 + (q - 4));

  float acc[8][TC];
  float acce = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TC; ++j) acc[i][j] = 0.f;

  auto load_chunk = [&](int k) {
    const int buf = k % 3;
    const int col0 = cb + k * BK;  // relative column of the chunk's first row
    const int valid = min(BK, ce - col0);
    // V rows: contiguous BK*MP floats (ldv == MP).
    float* vdst = Vs + buf * BK * MP;
    const float* vsrc = a.v + static_cast<size_t>(col0) * MP;
    constexpr int V16 = BK * MP / 4;
    for (int e = tid; e < V16; e += NT) {
      const int row = (e * 4) / MP;
      const bool ok = row < valid;
      cp_async16(vdst + e * 4, ok ? vsrc + e * 4 : a.v, ok ? 16 : 0);
    }
    float* xdst = Xc + buf * BK * DP;
    const float* xsrc = a.xs + static_cast<size_t>(c0 + col0) * DP;
    constexpr int X16 = BK * DP / 4;
    for (int e = tid; e < X16; e += NT) {
      const int row = (e * 4) / DP;
      const bool ok = row < valid;
      cp_async16(xdst + e * 4, ok ? xsrc + e * 4 : a.xs, ok ? 16 : 0);
    }
  };

  auto eval_chunk = [&](int k) {
    const float* xc = Xc + (k % 3) * BK * DP;
    float* kd = Ks + (k & 1) * BK * BM;
    float4 xi[DP4];
#pragma unroll
    for (int u = 0; u < DP4; ++u) xi[u] = __ldg(xi_ptr + u);
#pragma unroll 4
    for (int t = 0; t < BK; ++t) {
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
      const float e = ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));  // s2 * exp(-sqrt3 r)
      kd[t * BM + tid] = fmaf(r, kSqrt3f, 1.f) * e;
    }
  };

  auto gemm_chunk = [&](int k) {
    const float* kb = Ks + (k & 1) * BK * BM;
    const float* vb = Vs + (k % 3) * BK * MP;
#pragma unroll 4
    for (int t = 0; t < BK; ++t) {
      const float4 a0 = *reinterpret_cast<const float4*>(kb + t * BM + rbase);
      const float4 a1 = *reinterpret_cast<const float4*>(kb + t * BM + rbase + 32);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[TC];
      if constexpr (TC % 4 == 0) {
#pragma unroll
        for (int j = 0; j < TC; j += 4) {
          const float4 b = *reinterpret_cast<const float4*>(vb + t * MP + cbase + j);
          bv[j] = b.x; bv[j + 1] = b.y; bv[j + 2] = b.z; bv[j + 3] = b.w;
        }
      } else if constexpr (TC == 2) {
        const float2 b = *reinterpret_cast<const float2*>(vb + t * MP + cbase);
        bv[0] = b.x; bv[1] = b.y;
      } else {
        bv[0] = vb[t * MP + cbase];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      acce = fmaf(kb[t * BM + rext], vb[t * MP + MC], acce);
    }
  };

  bool first_flush = true;
  auto flush = [&]() {
    double* base = a.part + static_cast<size_t>(split) * a.R * a.m;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = tile * BM + rbase + (i < 4 ? i : 28 + i);
      if (r < a.R) {
        double* row = base + static_cast<size_t>(r) * a.m;
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          const int c = cbase + j;
          if (c < a.m) row[c] = (first_flush ? 0.0 : row[c]) + static_cast<double>(acc[i][j]);
          acc[i][j] = 0.f;
        }
      } else {
#pragma unroll
        for (int j = 0; j < TC; ++j) acc[i][j] = 0.f;
      }
    }
    const int r = tile * BM + rext;
    if (MC < a.m && r < a.R) {
      double* p = base + static_cast<size_t>(r) * a.m + MC;
      *p = (first_flush ? 0.0 : *p) + static_cast<double>(acce);
    }
    acce = 0.f;
    first_flush = false;
  };

  if (nq > 0) {
    load_chunk(0);
    cp_async_commit();
    if (nq > 1) load_chunk(1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    eval_chunk(0);
  }
  int since_flush = 0;
  for (int k = 0; k < nq; ++k) {
    cp_async_wait<0>();
    __syncthreads();
    if (k + 2 < nq) load_chunk(k + 2);
    cp_async_commit();
    if (k + 1 < nq) eval_chunk(k + 1);
    gemm_chunk(k);
    if (++since_flush == a.flush_chunks && k + 1 < nq) {
      flush();
      since_flush = 0;
    }
  }
  flush();
}

template <int TC, int DP4>
void launch_one(const KvArgs& a, cudaStream_t s) {
  constexpr int MP = Tile<TC>::MP;
  const size_t smem = sizeof(float) * (2 * BK * BM + 3 * BK * MP + 3 * BK * 4 * DP4);
  static bool configured = false;
  if (!configured) {
    GPK_CUDA(cudaFuncSetAttribute(kv_slab_kernel<TC, DP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = true;
  }
  dim3 grid((a.R + BM - 1) / BM, a.splits);
  kv_slab_kernel<TC, DP4><<<grid, NT, smem, s>>>(a);
  check_launch("kv_slab_kernel");
}

template <int TC>
void launch_tc(const KvArgs& a, cudaStream_t s) {
  switch (a.dp / 4) {
    case 1: return launch_one<TC, 1>(a, s);
    case 2: return launch_one<TC, 2>(a, s);
    case 3: return launch_one<TC, 3>(a, s);
    case 4: return launch_one<TC, 4>(a, s);
    case 5: return launch_one<TC, 5>(a, s);
    case 6: return launch_one<TC, 6>(a, s);
    case 7: return launch_one<TC, 7>(a, s);
    case 8: return launch_one<TC, 8>(a, s);
    default: throw std::invalid_argument("gpk: input dimension > 32 is not supported");
  }
}

// ---- split reduction + diagonal term ------------------------------------
__device__ __forceinline__ int splits_of_row(const KvReduceArgs& a, int r) {
  if (!a.sk_G) return a.splits;
  const long long t = r / 128;
  return static_cast<int>(sk_last(t, a.sk_Q, a.sk_G, a.sk_U) - sk_first(t, a.sk_Q, a.sk_G, a.sk_U) + 1);
}

__global__ void kv_reduce_kernel(const KvReduceArgs a) {
  if (a.skip && *a.skip) return;
  int c0 = a.c0, C = a.C;
  if (a.sel) {
    c0 = *a.sel * a.sel_block;
    C = min(a.sel_block, a.n - c0);
  }
  const long long total = static_cast<long long>(a.R) * a.m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / a.m), j = static_cast<int>(e % a.m);
    double acc = 0.0;
    const int ns = splits_of_row(a, r);
    for (int s = 0; s < ns; ++s) acc += a.part[(static_cast<size_t>(s) * a.R + r) * a.m + j];
    const int gi = a.row_idx ? a.row_idx[r] : a.r0 + r;
    if (!a.nodiag && gi >= c0 && gi < c0 + C) {
      const int vr = gi - c0 - a.vshift;
      const double vv = a.vdiag ? a.vdiag[static_cast<size_t>(vr) * a.ldvd + j]
                                : static_cast<double>(a.vdiag32[static_cast<size_t>(vr) * a.ldv32 + j]);
      acc += a.sigma2 * vv;
    }
    double* o = a.out + static_cast<size_t>(r) * a.ldo + j;
    const double b = a.base ? a.base[static_cast<size_t>(r) * a.ldb + j] : 0.0;
    *o = b + a.alpha * acc;
  }
}

// Grouped variant (warp per row, coalesced 520-byte row reads): block g owns a
// contiguous row range, writes out = base + alpha * (sum of split partials +
// sigma^2 V on the diagonal), and emits in a fixed order
//   dpart[g][j] = sum_r out[r][j] * w[r][j]            (w = dotw, or out itself)
//   spart[g]    = sum_r (sum_j out[r][j] inv_scales[j])^2   (AP block scores)
__device__ __forceinline__ void group_rows(const KvReduceArgs& a, int g, int& rb, int& re) {
  if (a.spart) {  // gpb groups inside each AP block of score_block rows
    const int blk = g / a.gpb, sub = g % a.gpb;
    const int b0 = blk * a.score_block, len = min(a.score_block, a.R - b0);
    rb = b0 + static_cast<int>(static_cast<long long>(len) * sub / a.gpb);
    re = b0 + static_cast<int>(static_cast<long long>(len) * (sub + 1) / a.gpb);
  } else {
    rb = static_cast<int>(static_cast<long long>(a.R) * g / gridDim.x);
    re = static_cast<int>(static_cast<long long>(a.R) * (g + 1) / gridDim.x);
  }
}

__global__ void __launch_bounds__(256, 3) kv_reduce_dot_kernel(const KvReduceArgs a) {
  if (a.skip && *a.skip) return;
  constexpr int NW = 8, MQ = 3;  // 8 warps; lane owns columns lane + 32 q, q < 3 (m <= 96)
  __shared__ double red[NW][96];
  __shared__ double sred[NW];
  int c0 = a.c0, C = a.C;
  if (a.sel) {
    c0 = *a.sel * a.sel_block;
    C = min(a.sel_block, a.n - c0);
  }
  const int g = blockIdx.x;
  int rb, re;
  group_rows(a, g, rb, re);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double dot[MQ] = {0.0, 0.0, 0.0};
  double sc = 0.0;
  double isc[MQ];
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    const int j = lane + 32 * q;
    isc[q] = (a.spart && j < a.m) ? a.inv_scales[j] : 0.0;
  }
  // Row loop, latency-bound: all loads of a row (split partials, base,
  // diagonal term, dot weights) are issued before any is consumed; the split
  // partials are summed in split order as before.
  for (int r = rb + warp; r < re; r += NW) {
    const int gi = a.row_idx ? a.row_idx[r] : a.r0 + r;
    const bool diag = !a.nodiag && gi >= c0 && gi < c0 + C;
    const int vr = gi - c0 - a.vshift;
    const int ns = splits_of_row(a, r);
    double pv[MQ][2], bv[MQ], dv[MQ], wv[MQ];
#pragma unroll
    for (int q = 0; q < MQ; ++q) {
      const int j = lane + 32 * q;
      const bool ok = j < a.m;
#pragma unroll
      for (int s = 0; s < 2; ++s)
        pv[q][s] = (ok && s < ns) ? __ldcs(a.part + (static_cast<size_t>(s) * a.R + r) * a.m + j) : 0.0;
      bv[q] = (ok && a.base) ? a.base[static_cast<size_t>(r) * a.ldb + j] : 0.0;
      dv[q] = 0.0;
      if (ok && diag)
        dv[q] = a.vdiag ? a.vdiag[static_cast<size_t>(vr) * a.ldvd + j]
                        : static_cast<double>(a.vdiag32[static_cast<size_t>(vr) * a.ldv32 + j]);
      wv[q] = (ok && a.dotw != a.out) ? a.dotw[static_cast<size_t>(r) * a.ldo + j] : 0.0;
    }
    double wsum = 0.0;
#pragma unroll
    for (int q = 0; q < MQ; ++q) {
      const int j = lane + 32 * q;
      if (j < a.m) {
        double acc = pv[q][0];
        if (ns > 1) acc += pv[q][1];
        for (int s = 2; s < ns; ++s) acc += a.part[(static_cast<size_t>(s) * a.R + r) * a.m + j];
        if (diag) acc += a.sigma2 * dv[q];
        const double val = bv[q] + a.alpha * acc;
        a.out[static_cast<size_t>(r) * a.ldo + j] = val;
        const double w = (a.dotw == a.out) ? val : wv[q];
        dot[q] = fma(val, w, dot[q]);
        wsum += val * isc[q];
      }
    }
    if (a.spart) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
      sc += wsum * wsum;
    }
  }
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    const int j = lane + 32 * q;
    if (j < a.m) red[warp][j] = dot[q];
  }
  if (lane == 0) sred[warp] = sc;
  __syncthreads();
  for (int j = threadIdx.x; j < a.m; j += blockDim.x) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += red[w][j];
    a.dpart[static_cast<size_t>(g) * a.m + j] = t;
  }
  if (a.spart && threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += sred[w];
    a.spart[g] = t;
  }
  if (!a.ctl) return;
  // ---- fused AP epilogue in the last block (ticket) ----
  __shared__ unsigned last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double ss[96];
  __shared__ double bscore[1024];
  ap_epilogue(a, static_cast<int>(gridDim.x), threadIdx.x, NW, ss, bscore, [] { __syncthreads(); });
}

}  // namespace

int kv_tc_for(int m) {
  if (m <= 9) return 1;
  if (m <= 17) return 2;
  if (m <= 33) return 4;
  return 8;
}

int kv_ld_for(int m) { return 8 * kv_tc_for(m) + 4; }

// Split-K factor: fill 2 CTAs/SM x 148 SMs in whole waves while keeping each
// split at least one chunk; prefers the split count whose last wave is fullest.
int kv_choose_splits(int R, int C, int sms, int rows_per_cta) {
  const int tiles = (R + rows_per_cta - 1) / rows_per_cta;
  const int slots = 2 * sms;
  const int max_splits = std::max(1, (C + BK - 1) / BK);
  if (tiles >= 4 * slots) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= std::min(max_splits, 4 * slots); ++s) {
    const long long ctas = static_cast<long long>(tiles) * s;
    const long long waves = (ctas + slots - 1) / slots;
    // efficiency of the wave structure, mildly penalising many splits
    double eff = static_cast<double>(ctas) / (waves * slots);
    if (waves < 2) eff *= static_cast<double>(ctas) / slots;  // underfilled single wave
    eff -= 0.002 * s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// Split count for the tensor-core kernel: minimise the busiest SM's work,
// ceil(ctas / SMs) * (chunks per CTA + per-CTA overhead), where the overhead
// (TMEM alloc, pipeline fill, FP64 epilogue, split-K partial traffic) is
// worth ~4 chunks. Favours few long CTAs for short column ranges (AP slabs)
// and enough CTAs to balance 148 SMs for full products.
int kv_tc_choose_splits(int R, int C, int sms, int ctas_per_sm) {
  const int tiles = (R + 127) / 128;
  const int chunks = (C + BK - 1) / BK;
  int best = 1;
  double best_cost = 1e300;
  for (int s = 1; s <= std::max(1, chunks); ++s) {
    const long long ctas = static_cast<long long>(tiles) * s;
    const double per = static_cast<double>((chunks + s - 1) / s) + 4.0;
    const long long slots = static_cast<long long>(ctas_per_sm) * sms;  // co-resident CTAs (TMEM columns)
    const double cost = static_cast<double>((ctas + slots - 1) / slots) * per * (1.0 + 1e-3 * s);
    if (cost < best_cost) {
      best_cost = cost;
      best = s;
    }
    if (ctas > 64LL * sms) break;
  }
  return best;
}

void kv_slab_launch(const KvArgs& a, int /*dmax*/, cudaStream_t s) {
  switch (kv_tc_for(a.m)) {
    case 1: return launch_tc<1>(a, s);
    case 2: return launch_tc<2>(a, s);
    case 4: return launch_tc<4>(a, s);
    default: return launch_tc<8>(a, s);
  }
}

void kv_reduce_launch(const KvReduceArgs& a, cudaStream_t s) {
  if (a.dpart) {
    if (a.m > 96) throw std::invalid_argument("gpk: fused reductions support m <= 96");
    if (a.ctl && a.nblocks > 1024) throw std::invalid_argument("gpk: fused AP epilogue supports <= 1024 blocks");
    kv_reduce_dot_kernel<<<a.groups, 256, 0, s>>>(a);
    check_launch("kv_reduce_dot_kernel");
    return;
  }
  const long long total = static_cast<long long>(a.R) * a.m;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  kv_reduce_kernel<<<std::max(blocks, 1), 256, 0, s>>>(a);
  check_launch("kv_reduce_kernel");
}

}  // namespace gpk
