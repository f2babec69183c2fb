// SGD (solvers.cpp:147-184) with the momentum recurrence evaluated lazily,
// and its minibatch product H[idx, :] V on the tcgen05 tensor cores.
//
// The reference updates every row of the n x m momentum and solution each
// iteration (M *= rho; M[idx] -= (lr/b) g; V += M), i.e. ~4 n m doubles of
// memory traffic per iteration for b = 512 rows of actual change. A row i
// that is not in the minibatch evolves in closed form: if (Vb, Mb) is its
// state right after iteration tau (its last update), then after
// Delta = t - tau - 1 further iterations
//   M(t) = rho^Delta Mb,   V(t) = Vb + S(Delta) Mb,   S(Delta) = rho + ... + rho^Delta.
// So each iteration writes only its b minibatch rows (FP64 base state, their
// FP32 records, tau), and the operator kernel materialises V(t) on the fly
// from the FP32 records while it builds its tensor-core B operand -- the full
// state is read once per iteration by the kernel that needs it anyway, and
// never written. P(Delta) = rho^Delta and S(Delta) are tables built by
// repeated multiplication / addition (the reference's own recurrence for an
// untouched row), so the closed form differs from the reference only in
// rounding (one multiply-add instead of Delta of them).
//
// sgd_slab_kernel: CTA = one 128-row tile of the minibatch x a column range
// (its split); 22 warps:
//   warps 0-15  evaluation: k(x_i, x_c) in FP32 (MUFU sqrt/ex2), TF32 hi/lo
//               split, tcgen05.st into a TMEM A buffer (5-deep ring); every
//               F chunks they drain the FP32 TMEM accumulator into FP64
//               registers (D double-buffered, drain deferred L chunks so the
//               MMA never waits), FP64 partial per split at the end.
//   warp 16     producer: cp.async.bulk of the chunk's 32 FP32 records
//               (V32 | M32), tau and x_c rows into a 4-stage staging ring.
//   warps 17-20 B builders: V(t) = V32 + S(Delta) M32 in FP32, TF32 hi/lo,
//               stored in the canonical K-major UMMA layout (3-stage ring).
//   warp 21     MMA: per 32-column chunk 12 tcgen05.mma.kind::tf32
//               (M = 128, N = NPAD, K = 8): D += A_hi B_hi + A_hi B_lo + A_lo B_hi.
// sgd_reduce_kernel: split partials -> the rank's slice of g (+ sigma^2 V(t)
// and -B on its own rows, old residual squares); sgd_apply_kernel: rank-order
// sum of the slices = g, the lazy update of the own minibatch rows, R[idx] =
// -g, the incremental residual norms and the termination / divergence test.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "gpk_internal.cuh"
#include "tc_util.cuh"

namespace gpk {

namespace {
using namespace tc;

constexpr int TBM = 128, TBK = 32;
constexpr int EW = 16;                 // evaluation warps
constexpr int BW = 4;                  // B-builder warps
constexpr int PROD_WARP = EW;          // 16
constexpr int BUILD_WARP0 = EW + 1;    // 17..20
constexpr int MMA_WARP = EW + 1 + BW;  // 21
constexpr int NTHREADS = 32 * (MMA_WARP + 1);
constexpr int ST = 4;    // staging stages
constexpr int SB = 3;    // B stages
constexpr int NAB = 5;   // TMEM A buffers (64 columns each, from column 192)
constexpr int A_COL0 = 192;
constexpr int D_COL1 = 96;  // second accumulator (the first at column 0)
constexpr int CPT = 8;      // chunk columns per evaluation thread
constexpr int DEFER = 4;    // drain of group g runs after chunk (g + 1) F + DEFER is evaluated

// shared memory: B ring | staging ring | barriers (64 words) | S of the chunk
// columns [SB][32] | S table [ntab]
template <int NPAD>
__host__ __device__ constexpr size_t sgd_smem_bytes(int rw, int dp, int ntab) {
  return sizeof(float) * (SB * 2 * NPAD * 32 + ST * (static_cast<size_t>(rw) + 32 * dp + 32)) +
         64 * sizeof(uint64_t) + SB * 32 * sizeof(float) + static_cast<size_t>(ntab) * sizeof(float);
}

// position of element (c, j) of a chunk's V (or M) image: the canonical
// K-major UMMA layout of the B operand (see kv_pack_kernel)
__host__ __device__ __forceinline__ int sgd_record_pos(int c, int j) {
  return ((j >> 3) * 8 + (c >> 2)) * 32 + (j & 7) * 4 + (c & 3);
}

// Waiting with back-off for the roles that run ahead of the pipeline (producer,
// B builders) or only issue (MMA): a failed probe sleeps `ns` instead of
// re-probing, so the waiting warps leave issue slots and the MIO queue
// (mbarrier probes share it with LDS / MUFU) to the evaluation warps.
template <int NS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (NS > 0) __nanosleep(NS);
  }
}
// spin without suspend hint or sleep (latency-critical consumers)
#ifndef SGD_SPIN
#define SGD_SPIN 1
#endif
#if SGD_SPIN
#define SGD_WAIT mbar_wait_spin
#else
#define SGD_WAIT mbar_wait
#endif
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) { mbar_wait_backoff<0>(bar, parity); }

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int NPAD, int DP4>
struct SgdLayout {
  static constexpr int DP = 4 * DP4;
  static constexpr int IMG = NPAD * TBK;  // floats of one TF32 image of a chunk
};

template <int NPAD, int DP4, bool GRAM, int DX>
__global__ void __launch_bounds__(NTHREADS, 1) sgd_slab_kernel(const SgdSlabArgs a) {
  using L = SgdLayout<NPAD, DP4>;
  constexpr int DP = L::DP;
  constexpr int DC = NPAD / 4;  // D columns drained per evaluation thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int rw = a.rw;                              // floats of one chunk record (V image | M image)
  const int st_floats = rw + TBK * DP + TBK;        // record | x_c | tau
  float* smB = reinterpret_cast<float*>(smem_raw);         // [SB][2 * IMG]
  float* smS = smB + SB * 2 * L::IMG;                      // [ST][st_floats]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smS + ST * st_floats);
  uint64_t* st_full = bars;                 // [ST]
  uint64_t* st_empty = bars + ST;           // [ST]
  uint64_t* b_full = bars + 2 * ST;         // [SB]
  uint64_t* b_empty = b_full + SB;          // [SB]
  uint64_t* a_full = b_empty + SB;          // [NAB]
  uint64_t* a_empty = a_full + NAB;         // [NAB]
  uint64_t* d_full = a_empty + NAB;         // [2]
  uint64_t* d_empty = d_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);
  float* sS = reinterpret_cast<float*>(d_empty + 4);  // [SB][32] S(Delta) of the chunk's columns
  float* stab = sS + SB * 32;                          // [ntab] S(Delta) table

  if (a.ctl->stop) return;
  const int t_iter = a.ctl->iters;
  const int* idx = a.idxbuf + static_cast<size_t>(t_iter % a.idx_chunk) * a.R;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int cb = split * a.cols_per_split;
  const int ce = min(a.C, cb + a.cols_per_split);
  const int nk = ce > cb ? (ce - cb + TBK - 1) / TBK : 0;
  const int F = a.flush;
  const int ngroups = (nk + F - 1) / F;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (a.stats && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    const double entries = static_cast<double>(a.R) * a.C;
    atomicAdd(a.stats, entries * a.m);
    atomicAdd(a.stats + 1, entries * (2.0 * a.m + 3.0 * a.d + 6.0));
    atomicAdd(a.stats + 2, entries * (3.0 * a.d + 6.0));
  }
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], EW + BW);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&b_full[s], BW);
      mbar_init(&b_empty[s], 1);
    }
    for (int b = 0; b < NAB; ++b) {
      mbar_init(&a_full[b], EW);
      mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&d_empty[b], EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < a.ntab; e += NTHREADS) stab[e] = __ldg(a.s32 + e);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PROD_WARP) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint32_t rec_bytes = rw * 4u, x_bytes = TBK * DP * 4u;
      for (int k = 0; k < nk; ++k) {
        const int s = k % ST;
        if (k >= ST) mbar_wait_backoff<256>(&st_empty[s], ((k / ST) - 1) & 1);
        const size_t c = static_cast<size_t>(cb) + static_cast<size_t>(k) * TBK;  // local column of the chunk
        float* dst = smS + s * st_floats;
        mbar_expect_tx(&st_full[s], rec_bytes + x_bytes + TBK * 4u);
        bulk_g2s(dst, a.rec + (c / TBK) * rw, rec_bytes, &st_full[s]);
        bulk_g2s(dst + rw, (GRAM ? a.xg : DX > 0 ? a.xsoa : a.xs) + (a.c0 + c) * DP, x_bytes, &st_full[s]);
        bulk_g2s(dst + rw + TBK * DP, a.tau + c, TBK * 4u, &st_full[s]);
      }
    }
  } else if (warp >= BUILD_WARP0 && warp < MMA_WARP) {
    // ---------------- B builders: V(t) images ----------------
    // The chunk record holds V32 and M32 already in the B operand's canonical
    // K-major layout (j-groups < JG), so V(t) = V32 + S(Delta_c) M32 is float4
    // in, float4 out; per chunk the first builder warp looks up S(Delta_c) of
    // the 32 columns.
    const int bt = tid - BUILD_WARP0 * 32;  // 0..127
    const int jgroups = a.moff / 256;       // JG: j-groups stored (8 j x 32 c each)
    for (int k = 0; k < nk; ++k) {
      const int s = k % ST, sb = k % SB;
      mbar_wait_backoff<64>(&st_full[s], (k / ST) & 1);
      const float* rec = smS + s * st_floats;
      if (warp == BUILD_WARP0) {
        const int* tau = reinterpret_cast<const int*>(rec + rw + TBK * DP);
        const int dl = min(max(t_iter - tau[lane] - 1, 0), a.budget);
        sS[sb * 32 + lane] = dl < a.ntab ? stab[dl] : __ldg(a.s32 + dl);
      }
      if (k >= SB) mbar_wait_backoff<128>(&b_empty[sb], ((k / SB) - 1) & 1);
      asm volatile("bar.sync 1, %0;" ::"n"(32 * BW) : "memory");
      const float4* v4 = reinterpret_cast<const float4*>(rec);
      const float4* m4 = reinterpret_cast<const float4*>(rec + a.moff);
      const float4* s4 = reinterpret_cast<const float4*>(sS + sb * 32);
      float4* bh = reinterpret_cast<float4*>(smB + sb * 2 * L::IMG);
      float4* bl = bh + L::IMG / 4;
#pragma unroll 5
      for (int f = bt; f < L::IMG / 4; f += 32 * BW) {
        const int core = f >> 3;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((core >> 3) < jgroups) {
          const float4 vv = v4[f], mm = m4[f], sc = s4[core & 7];
          v.x = fmaf(sc.x, mm.x, vv.x);
          v.y = fmaf(sc.y, mm.y, vv.y);
          v.z = fmaf(sc.z, mm.z, vv.z);
          v.w = fmaf(sc.w, mm.w, vv.w);
        }
        // hi = v rounded to TF32 (nearest, ties away: add half of the 13
        // dropped bits, clear them), lo = v - hi exactly; the tensor core reads
        // lo's top 19 bits
        float4 h, l;
        h.x = __uint_as_float((__float_as_uint(v.x) + 0x1000u) & 0xFFFFE000u);
        h.y = __uint_as_float((__float_as_uint(v.y) + 0x1000u) & 0xFFFFE000u);
        h.z = __uint_as_float((__float_as_uint(v.z) + 0x1000u) & 0xFFFFE000u);
        h.w = __uint_as_float((__float_as_uint(v.w) + 0x1000u) & 0xFFFFE000u);
        l.x = v.x - h.x;
        l.y = v.y - h.y;
        l.z = v.z - h.z;
        l.w = v.w - h.w;
        bh[f] = h;
        bl[f] = l;
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&b_full[sb]);
        mbar_arrive(&st_empty[s]);
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = tf32_idesc(NPAD, TBM);
    int sb = 0, bph = 0, ab = 0, aph = 0, g = 0, kf = 0;
    for (int k = 0; k < nk; ++k) {
      const bool first = kf == 0, last = kf == F - 1 || k + 1 == nk;
      SGD_WAIT(&b_full[sb], bph);
      SGD_WAIT(&a_full[ab], aph);
      if (first && g >= 2) SGD_WAIT(&d_empty[g & 1], ((g >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t dt = tmem + ((g & 1) ? D_COL1 : 0);
      const uint32_t bh = smem_u32(smB + sb * 2 * L::IMG);
      const uint32_t bl = bh + L::IMG * 4;
      const uint32_t ah = tmem + A_COL0 + ab * 64, al = ah + 32;
#pragma unroll
      for (int kk = 0; kk < TBK / 8; ++kk) {
        const uint64_t dh = umma_desc(bh + kk * 256, 128, (TBK / 4) * 128);
        const uint64_t dl = umma_desc(bl + kk * 256, 128, (TBK / 4) * 128);
        MMA_TF32(dt, ah + kk * 8, dh, idesc, (first && kk == 0) ? 0u : 1u);
        MMA_TF32(dt, ah + kk * 8, dl, idesc, 1u);
        MMA_TF32(dt, al + kk * 8, dh, idesc, 1u);
      }
      MMA_COMMIT(&b_empty[sb]);
      MMA_COMMIT(&a_empty[ab]);
      if (last) MMA_COMMIT(&d_full[g & 1]);
      if (++sb == SB) { sb = 0; bph ^= 1; }
      if (++ab == NAB) { ab = 0; aph ^= 1; }
      if (++kf == F) { kf = 0; ++g; }
    }
  } else {
    // ---------------- evaluation + drain ----------------
    const int lg = warp & 3, quarter = warp >> 2;
    const int row = lg * 32 + lane;
    const int er = tile * TBM + row;
    const bool row_ok = er < a.R;
    const int gi = row_ok ? idx[er] : 0;
    uint64_t xi2[2 * DP4];
    uint64_t seed = 0ull;  // GRAM: (|x_i|^2, 0)
    const float* xrow = a.xs + static_cast<size_t>(gi) * DP;
    float ni = 0.f;
#pragma unroll
    for (int u = 0; u < DP4; ++u) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(xrow) + u);
      float e[4] = {x.x, x.y, x.z, x.w};
      if constexpr (GRAM) {  // (x, 1 at slot d, 0...) against the column image (-2 x, |x|^2, 0...)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (4 * u + q < a.d) ni = fmaf(e[q], e[q], ni);
          e[q] = (4 * u + q == a.d) ? 1.f : e[q];
        }
      }
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u]) : "f"(e[0]), "f"(e[1]));
      asm("mov.b64 %0, {%1, %2};" : "=l"(xi2[2 * u + 1]) : "f"(e[2]), "f"(e[3]));
    }
    asm("mov.b64 %0, {%1, %2};" : "=l"(seed) : "f"(ni), "f"(0.f));
    const uint32_t lane_addr = static_cast<uint32_t>(lg * 32) << 16;
    // this thread's FP64 accumulators: its row, columns quarter * DC .. + DC
    // (registers; measured 12% faster than shared-memory accumulators)
    double acc[DC];
#pragma unroll
    for (int e = 0; e < DC; ++e) acc[e] = 0.0;
    auto drain = [&](int g) {
      mbar_wait(&d_full[g & 1], (g >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + lane_addr + ((g & 1) ? D_COL1 : 0) + quarter * DC;
#pragma unroll
      for (int q = 0; q < DC / 4; ++q) {
        uint32_t v[4];
        tc_ld4(base + 4 * q, v);
        tc_wait_ld();
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[4 * q + e] += static_cast<double>(__uint_as_float(v[e]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty[g & 1]);
    };
    int drained = 0, next_drain = F + DEFER;
    // ring positions kept incrementally (no divisions in the chunk loop)
    int s = 0, sph = 0, ab = 0, aph = 0;  // a_empty waited from the second pass over the ring on
    // DX > 0: the row's coordinates duplicated into FP32x2 pairs, and the
    // profile constants as pairs
    uint64_t xik2[4] = {0ull, 0ull, 0ull, 0ull}, k_s3 = 0ull, k_one = 0ull, k_c = 0ull, k_l2s2 = 0ull;
    if constexpr (DX > 0) {
      const float4 xr = __ldg(reinterpret_cast<const float4*>(xrow));
      const float xe[4] = {xr.x, xr.y, xr.z, xr.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) asm("mov.b64 %0, {%1, %1};" : "=l"(xik2[k]) : "f"(xe[k]));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_s3) : "f"(kSqrt3f));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_one) : "f"(1.f));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_c) : "f"(kNegSqrt3Log2e));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_l2s2) : "f"(a.log2_s2));
    }
    // Chunk k's entries are computed before its A buffer is waited for, and
    // its TMEM stores complete while chunk k + 1 is computed: the wait::st and
    // the a_full arrive of chunk k run at the top of chunk k + 1's store.
    int pend = -1;  // A buffer whose stores are still in flight
    auto publish = [&]() {
      if (pend < 0) return;
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[pend]);
      pend = -1;
    };
    for (int k = 0; k < nk; ++k) {
      SGD_WAIT(&st_full[s], sph);
      const float* xc = smS + s * st_floats + rw + quarter * CPT * DP;
      uint32_t hi[CPT], lo[CPT];
#pragma unroll
      for (int t = 0; t < CPT; ++t) {
        if constexpr (DX > 0) {  // exactly DX <= 4 dimensions, two columns per FP32x2 instruction
          if (t & 1) continue;   // (t, t + 1) done together
          // column coordinates of this chunk in SoA order: xq[k * 32 + c]
          const float* xq = smS + s * st_floats + rw + quarter * CPT + t;
          uint64_t r2;
#pragma unroll
          for (int k = 0; k < DX; ++k) {
            const uint64_t cc = *reinterpret_cast<const uint64_t*>(xq + k * 32);
            uint64_t dd;
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(cc), "l"(xik2[k]));
            if (k == 0)
              asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r2) : "l"(dd));
            else
              asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r2) : "l"(dd));
          }
          float ra, rb;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r2));
          ra = sqrt_approx(ra);
          rb = sqrt_approx(rb);
          uint64_t rr, tt, uu, ee, kk;
          asm("mov.b64 %0, {%1, %2};" : "=l"(rr) : "f"(ra), "f"(rb));
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(tt) : "l"(rr), "l"(k_s3), "l"(k_one));
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(uu) : "l"(rr), "l"(k_c), "l"(k_l2s2));
          float ua, ub;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(ua), "=f"(ub) : "l"(uu));
          ua = ex2_approx(ua);
          ub = ex2_approx(ub);
          asm("mov.b64 %0, {%1, %2};" : "=l"(ee) : "f"(ua), "f"(ub));
          asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(kk) : "l"(tt), "l"(ee));
          float ka, kb;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(ka), "=f"(kb) : "l"(kk));
          hi[t] = __float_as_uint(ka) & 0xFFFFE000u;
          hi[t + 1] = __float_as_uint(kb) & 0xFFFFE000u;
          uint64_t hh, ll;
          asm("mov.b64 %0, {%1, %2};" : "=l"(hh) : "r"(hi[t]), "r"(hi[t + 1]));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ll) : "l"(kk), "l"(hh));
          asm("mov.b64 {%0, %1}, %2;" : "=r"(lo[t]), "=r"(lo[t + 1]) : "l"(ll));
          continue;
        }
        // packed FP32x2 (FADD2/FFMA2): two dimensions per instruction
        const uint32_t xaddr = smem_u32(xc + t * DP);
        uint64_t acc0 = seed, acc1 = 0ull;
#pragma unroll
        for (int u = 0; u < DP4; ++u) {
          uint64_t c01, c23;
          asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xaddr + 16 * u));
          if constexpr (GRAM) {  // r^2 = |x_i|^2 + x_i.(-2 x_c) + |x_c|^2
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc0) : "l"(c01), "l"(xi2[2 * u]));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc1) : "l"(c23), "l"(xi2[2 * u + 1]));
          } else {
            uint64_t d01, d23;
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d01) : "l"(c01), "l"(xi2[2 * u]));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d23) : "l"(c23), "l"(xi2[2 * u + 1]));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc0) : "l"(d01));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc1) : "l"(d23));
          }
        }
        uint64_t accs;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(accs) : "l"(acc0), "l"(acc1));
        float s0, s1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(accs));
        const float r = sqrt_approx(GRAM ? fmaxf(s0 + s1, 0.f) : s0 + s1);
        const float kv = fmaf(r, kSqrt3f, 1.f) * ex2_approx(fmaf(r, kNegSqrt3Log2e, a.log2_s2));
        hi[t] = __float_as_uint(kv) & 0xFFFFE000u;
        lo[t] = __float_as_uint(kv - __uint_as_float(hi[t]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_empty[s]);  // x_c consumed
      if (k >= NAB) SGD_WAIT(&a_empty[ab], aph);
      publish();  // chunk k - 1
      tc_fence_after();
      const uint32_t abase = tmem + lane_addr + A_COL0 + ab * 64 + quarter * CPT;
      tc_st8(abase, hi);
      tc_st8(abase + 32, lo);
      pend = ab;
      if (++s == ST) { s = 0; sph ^= 1; }
      if (++ab == NAB) { ab = 0; if (k >= NAB) aph ^= 1; }
      // deferred drain: group g once chunk (g + 1) F + DEFER is in flight
      if (k == next_drain) {
        drain(drained++);
        next_drain += F;
      }
    }
    publish();
    while (drained < ngroups) drain(drained++);
    if (row_ok) {
      double* prow = a.part + (static_cast<size_t>(split) * a.R + er) * a.m;
#pragma unroll
      for (int e = 0; e < DC; ++e) {
        const int j = quarter * DC + e;
        if (j < a.m) prow[j] = acc[e];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Development instrumentation (build with -DSGD_PROF=1, tools/sgd_prof.sh):
// per-role barrier-wait cycles of the 64-column slab, summed over CTAs and
// warps (lane 0), read back with gpk_debug_sgd_prof.
#ifndef SGD_PROF
#define SGD_PROF 0
#endif
#ifndef SGD_FAKE_DIST
#define SGD_FAKE_DIST 0
#endif
#ifndef SGD_FAKE_MUFU
#define SGD_FAKE_MUFU 0
#endif
#ifndef SGD_FAKE_HALFREC
#define SGD_FAKE_HALFREC 0
#endif
#if SGD_PROF
__device__ unsigned long long g_sgd_prof[16];
#define PROF_T0 prof_t0 = clock64()
#define PROF_ADD(i) prof_acc[i] += clock64() - prof_t0
#else
#define PROF_T0
#define PROF_ADD(i)
#endif

// ---- 64-column pipeline (d <= 4, FP32x2 SoA evaluation) -----------------
// The same roles as sgd_slab_kernel, with 64-column chunks (two 32-column
// records per stage): every evaluation thread computes 16 entries per
// barrier round instead of 8, which halves the per-entry share of the
// mbarrier waits / arrivals, TMEM-address and ring bookkeeping that made up
// ~45% of the evaluation warps' instructions at 32 columns
// (profiles/r02_sass_hot_sgd_slab_C4_v2_soa.txt). TMEM: D double buffer at
// columns 0 / 80, then a ring of five A slots of one 32-column half each
// (hi 32 | lo 32). Stages: staging ring 3 x (2 records + SoA x + tau), B ring
// 2 x (hi | lo of two 32-column images); the B images' zero j-groups are
// written once.
// ---- CTA pairs (cta_group::2) ------------------------------------------------
#ifndef SGD_PAIR_ACQ_CLUSTER
#define SGD_PAIR_ACQ_CLUSTER 0
#endif
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory word in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on a barrier of either CTA of the pair. CTA-scope release (the
// default), as for a local arrive: the data it publishes -- TMEM stores
// (completed by tcgen05.wait::st) and B images (fence.proxy.async) -- is read
// by the pair's tensor core, not by a thread of the other CTA; a cluster-scope
// release here made every evaluation warp ~1.8x slower (per-role profile).
__device__ __forceinline__ void arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}

// programmatic dependent launch (no-ops when the kernel was launched without the attribute)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace c64 {
constexpr int CH = 64;
constexpr int SB = 2;
constexpr int DEFER = 2;
// staging stages and TMEM A half-slots: 3 / 5 for one CTA per row tile; a CTA
// pair stages half-records, so it has room for 4 / 4, and the evaluation warps
// walk the rings in passes of 4 chunks with every stage, slot, barrier address
// and phase a compile-time constant of the position in the pass
template <bool PAIR>
constexpr int st_stages() { return PAIR ? 4 : 3; }
template <bool PAIR>
constexpr int a_slots() { return PAIR ? 4 : 5; }

// NB = B-image rows held by one CTA (NPAD, or NPAD / 2 in a CTA pair), rws =
// staged floats of one 32-column record
template <int NB, int ST>
__host__ __device__ constexpr size_t smem_bytes(int rws, int dp, int ntab) {
  return sizeof(float) * (SB * 4 * static_cast<size_t>(NB) * 32 + ST * (2 * static_cast<size_t>(rws) + 2 * 32 * dp + CH)) +
         64 * sizeof(uint64_t) + SB * CH * sizeof(float) + static_cast<size_t>(ntab) * sizeof(float);
}
}  // namespace c64

// PAIR: the two CTAs of a cluster (row tiles 2p, 2p + 1 of one column split)
// run as one cta_group::2 MMA of M = 256: each keeps its own 128 rows of A in
// its TMEM and receives its 128 rows of D, and each holds half of the B
// operand's N = NPAD RHS rows (CTA r: j-groups [r NPAD/16, (r + 1) NPAD/16)),
// so each stages and builds half of every record -- the B builders' shared
// memory traffic, the single-CTA bound, is halved per CTA. The even CTA's MMA
// warp issues for both; the peer's evaluation, builder and drain warps arrive
// on the leader's barriers, the MMA completions are multicast to both.
template <int NPAD, int DX, int NBW, bool PAIR>
__global__ void __launch_bounds__(32 * (EW + 2 + NBW), 1) sgd_slab64_kernel(const SgdSlabArgs a) {
  constexpr int CH = c64::CH, ST = c64::st_stages<PAIR>(), SB = c64::SB, DEFER = c64::DEFER;
  static_assert(!PAIR || NPAD % 16 == 0, "cta_group::2 needs N a multiple of 16");
  // TMEM: D double buffer at columns 0 / 80, then a ring of NS = 5 A slots of
  // one 32-column half each (hi 32 | lo 32) from column 160: half j of the
  // solve (chunk j / 2, half j % 2) uses slot j % 5
  constexpr int NS = c64::a_slots<PAIR>(), A_COL0 = 160, D1 = 80;
  constexpr int BW = NBW, MMA_WARP = EW + 1 + NBW, NTHREADS = 32 * (MMA_WARP + 1);
  constexpr int NB = PAIR ? NPAD / 2 : NPAD;  // B-image rows (RHS) held by this CTA
  constexpr int LG = NB / 8;                  // their j-groups
  constexpr int IMG = NB * 32;                // floats of this CTA's part of one 32-column TF32 image
  constexpr int DC = NPAD / 4;
  constexpr int DP = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int rw = a.rw;
  const int jgroups = a.moff / 256;
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const int g0 = static_cast<int>(crank) * LG;                         // first j-group held here
  const int lgl = PAIR ? max(0, min(jgroups - g0, LG)) : jgroups;      // live j-groups held here
  const int rws = PAIR ? 2 * LG * 256 : rw;                            // staged floats of one record
  const int mo = PAIR ? LG * 256 : a.moff;                             // M image within a staged record
  const int st_floats = 2 * rws + 2 * 32 * DP + CH;  // 2 records | 2 SoA x | tau
  float* smB = reinterpret_cast<float*>(smem_raw);  // [SB][hi0 | hi1 | lo0 | lo1]
  float* smS = smB + SB * 4 * IMG;                  // [ST][st_floats]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smS + ST * st_floats);
  uint64_t* st_full = bars;
  uint64_t* st_empty = bars + ST;
  uint64_t* b_full = bars + 2 * ST;
  uint64_t* b_empty = b_full + SB;
  uint64_t* a_full = b_empty + SB;  // [NS]
  uint64_t* a_empty = a_full + NS;  // [NS]
  uint64_t* d_full = a_empty + NS;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);
  float* sS = reinterpret_cast<float*>(bars + 64);  // [SB][CH]
  float* stab = sS + SB * CH;

  // Everything up to griddep_wait() touches only this CTA's shared memory,
  // TMEM and launch-constant inputs, so under programmatic dependent launch
  // it overlaps the previous iteration's finish kernel (which wrote ctl, the
  // minibatch rows' records and tau).
  const int tile = blockIdx.x, split = blockIdx.y;
  const int cb = split * a.cols_per_split;  // multiple of 64
  const int ce = min(a.C, cb + a.cols_per_split);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t NPEER = PAIR ? 2u : 1u;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], EW + BW);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&b_full[s], NPEER * BW);
      mbar_init(&b_empty[s], 1);
    }
    for (int b = 0; b < NS; ++b) {
      mbar_init(&a_full[b], NPEER * EW);
      mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&d_empty[b], NPEER * EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  for (int e = tid; e < a.ntab; e += NTHREADS) stab[e] = __ldg(a.s32 + e);
#if SGD_FAKE_HALFREC
  for (int e = tid; e < ST * st_floats; e += NTHREADS) smS[e] = 0.f;
#endif
  // zero j-groups (>= the live ones) of every B image: written once, never rebuilt
  for (int sb = 0; sb < SB; ++sb)
    for (int f = tid; f < 4 * IMG; f += NTHREADS)
      if (((f % IMG) >> 8) >= lgl) smB[sb * 4 * IMG + f] = 0.f;
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  griddep_wait();    // the previous kernel's writes (ctl, records, tau, idx) are visible from here
  griddep_launch();  // the finish kernel may be scheduled as this grid's CTAs retire
  // once the solve has stopped the launch is a no-op: zero chunks, no partials
  const bool stopped = a.ctl->stop != 0;
  const int t_iter = a.ctl->iters;
  const int* idx = a.idxbuf + static_cast<size_t>(t_iter % a.idx_chunk) * a.R;
  const int nk = (!stopped && ce > cb) ? (ce - cb + CH - 1) / CH : 0;
  const int F = a.flush;
  const int ngroups = (nk + F - 1) / F;
  if (!stopped && a.stats && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    const double entries = static_cast<double>(a.R) * a.C;
    atomicAdd(a.stats, entries * a.m);
    atomicAdd(a.stats + 1, entries * (2.0 * a.m + 3.0 * a.d + 6.0));
    atomicAdd(a.stats + 2, entries * (3.0 * a.d + 6.0));
  }
  // one CTA per SM allocating all 512 columns: the allocation starts at
  // column 0, lane 0. The MMA issue uses that constant so ptxas keeps every
  // operand in uniform registers (no per-MMA elect/broadcast of the TMEM
  // addresses: ~18 -> ~6 instructions per MMA).
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0) __trap();
#if SGD_PROF
  const long long prof_start = clock64();
  long long prof_t0 = 0;
  long long prof_acc[10] = {};
#endif

  if (warp == PROD_WARP) {
    // ---------------- producer ----------------
    if (lane == 0) {
#if SGD_FAKE_HALFREC  // timing experiment only (wrong results): half of each chunk's record bytes
      const uint32_t rec_bytes = rw * 4u, x_bytes = 2 * 32 * DP * 4u;
#else
      const uint32_t rec_bytes = PAIR ? 4u * lgl * 1024u : 2 * rw * 4u, x_bytes = 2 * 32 * DP * 4u;
#endif
      for (int k = 0; k < nk; ++k) {
        const int s = k % ST;
        PROF_T0;
        if (k >= ST) mbar_wait_backoff<256>(&st_empty[s], ((k / ST) - 1) & 1);
        PROF_ADD(0);
        const size_t c = static_cast<size_t>(cb) + static_cast<size_t>(k) * CH;
        float* dst = smS + s * st_floats;
        mbar_expect_tx(&st_full[s], rec_bytes + x_bytes + CH * 4u);
        if constexpr (PAIR) {  // this CTA's j-groups of the V and M images of both records
          if (lgl > 0)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float* src = a.rec + (c / 32 + h) * rw + g0 * 256;
              bulk_g2s(dst + h * rws, src, lgl * 1024u, &st_full[s]);
              bulk_g2s(dst + h * rws + mo, src + a.moff, lgl * 1024u, &st_full[s]);
            }
        } else {
          bulk_g2s(dst, a.rec + (c / 32) * rw, rec_bytes, &st_full[s]);
        }
        bulk_g2s(dst + 2 * rws, a.xsoa + (a.c0 + c) * DP, x_bytes, &st_full[s]);
        bulk_g2s(dst + 2 * rws + 2 * 32 * DP, a.tau + c, CH * 4u, &st_full[s]);
      }
    }
  } else if (warp >= BUILD_WARP0 && warp < MMA_WARP) {
    // ---------------- B builders: V(t) = V32 + S(Delta) M32 -> TF32 hi / lo ----------------
    // thread bt handles float4 f = bt + 128 i of the live j-groups of both
    // 32-column images; the S(Delta) quadruple of f is (f / 8) % 8 = (bt / 8) % 8
    // for every i (128 / 8 = 16), so it is loaded once per half
    const int bt = tid - BUILD_WARP0 * 32;  // 0..127
    const int live = lgl * 64;              // float4s of one 32-column image in live j-groups
    const int squad = (bt >> 3) & 7;
    for (int k = 0; k < nk; ++k) {
      const int s = k % ST, sb = k % SB;
      PROF_T0;
      mbar_wait_backoff<64>(&st_full[s], (k / ST) & 1);
      PROF_ADD(1);
      const float* rec = smS + s * st_floats;
      if (warp == BUILD_WARP0) {
        const int* tau = reinterpret_cast<const int*>(rec + 2 * rws + 2 * 32 * DP);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int dl = min(max(t_iter - tau[h * 32 + lane] - 1, 0), a.budget);
          sS[sb * CH + h * 32 + lane] = dl < a.ntab ? stab[dl] : __ldg(a.s32 + dl);
        }
      }
      PROF_T0;
      if (k >= SB) mbar_wait_backoff<128>(&b_empty[sb], ((k / SB) - 1) & 1);
      PROF_ADD(2);
      PROF_T0;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * BW) : "memory");
      PROF_ADD(3);
#if SGD_PROF
      const long long prof_b0 = clock64();
#endif
      float4* bbase = reinterpret_cast<float4*>(smB + sb * 4 * IMG);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 sc = reinterpret_cast<const float4*>(sS + sb * CH + h * 32)[squad];
        const float4* v4 = reinterpret_cast<const float4*>(rec + h * rws);
        const float4* m4 = reinterpret_cast<const float4*>(rec + h * rws + mo);
        float4* bh = bbase + h * (IMG / 4);
        float4* bl = bbase + (2 + h) * (IMG / 4);
        const float2 s01 = make_float2(sc.x, sc.y), s23 = make_float2(sc.z, sc.w);
        // all of this half's loads first (independent registers), then the
        // arithmetic and the stores: the loop-carried register reuse of the
        // rolled loop serialised one shared-memory round trip per float4
        constexpr int MAXI = (NB * 8 + 32 * BW - 1) / (32 * BW);  // float4s per thread per half, at most
        float4 vv[MAXI], mm[MAXI];
#pragma unroll
        for (int i = 0; i < MAXI; ++i) {
          const int f = bt + i * 32 * BW;
          if (f < live) {
            vv[i] = v4[f];
            mm[i] = m4[f];
          }
        }
#pragma unroll
        for (int i = 0; i < MAXI; ++i) {
          const int f = bt + i * 32 * BW;
          if (f < live) {
            // V(t) in packed FP32x2; hi = V(t) truncated to TF32 (one LOP per
            // element), lo = V(t) - hi exactly (the tensor core reads its top 11 bits)
            const float2 v01 = __ffma2_rn(s01, make_float2(mm[i].x, mm[i].y), make_float2(vv[i].x, vv[i].y));
            const float2 v23 = __ffma2_rn(s23, make_float2(mm[i].z, mm[i].w), make_float2(vv[i].z, vv[i].w));
            float4 h;
            h.x = __uint_as_float(__float_as_uint(v01.x) & 0xFFFFE000u);
            h.y = __uint_as_float(__float_as_uint(v01.y) & 0xFFFFE000u);
            h.z = __uint_as_float(__float_as_uint(v23.x) & 0xFFFFE000u);
            h.w = __uint_as_float(__float_as_uint(v23.y) & 0xFFFFE000u);
            const float2 l01 = __fadd2_rn(v01, make_float2(-h.x, -h.y));
            const float2 l23 = __fadd2_rn(v23, make_float2(-h.z, -h.w));
            bh[f] = h;
            bl[f] = make_float4(l01.x, l01.y, l23.x, l23.y);
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          arrive_cluster(mapa_u32(smem_u32(&b_full[sb]), 0));
        else
          mbar_arrive(&b_full[sb]);
        mbar_arrive(&st_empty[s]);
      }
#if SGD_PROF
      prof_acc[4] += clock64() - prof_b0;  // build (slot 14 at the end)
#endif
    }
  } else if (warp == MMA_WARP && crank == 0) {
    // ---------------- MMA issuer: 2 x 12 MMAs per 64-column chunk ----------------
    // (in a pair: the even CTA's, M = 256, completions multicast to both CTAs)
    // Each 32-column half of A starts as soon as the evaluation warps publish
    // it. The whole warp waits; one elected lane issues from an if-block whose
    // operands are all warp-uniform (constant TMEM base, descriptors as 32-bit
    // offsets of one per-stage base word), so ptxas keeps them in uniform
    // registers: ~2.5 instructions per MMA instead of ~18 with the per-MMA
    // elect/broadcast of MMA_TF32 (the issue warp had become the bottleneck).
    constexpr uint32_t idesc = tf32_idesc(NPAD, PAIR ? 2 * TBM : TBM);
    constexpr uint32_t DESC_HI = (1024u >> 4) | (1u << 14);  // SBO 1 KiB, version 1 (bit 46)
    const uint32_t smb0 = smem_u32(smB);
    const uint32_t bfull0 = smem_u32(b_full), bempty0 = smem_u32(b_empty), afull0 = smem_u32(a_full),
                   aempty0 = smem_u32(a_empty), dfull0 = smem_u32(d_full), dempty0 = smem_u32(d_empty);
    auto wait_u = [](uint32_t bar, uint32_t parity) {
      if constexpr (PAIR && SGD_PAIR_ACQ_CLUSTER)  // (development A/B)
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra W_%=;\n\t}" ::"r"(bar),
            "r"(parity)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra W_%=;\n\t}" ::"r"(bar),
            "r"(parity)
            : "memory");
    };
    auto elect_one = []() -> uint32_t {
      uint32_t pred = 0;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      return pred;
    };
    auto mma = [](uint32_t d, uint32_t a, uint32_t blo, uint32_t acc) {
      if constexpr (PAIR)
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\t"
            "mov.b64 bd, {%2, %3};\n\t"
            "setp.ne.b32 p, %5, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d),
            "r"(a), "r"(blo), "n"(DESC_HI), "n"(idesc), "r"(acc)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\t"
            "mov.b64 bd, {%2, %3};\n\t"
            "setp.ne.b32 p, %5, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d),
            "r"(a), "r"(blo), "n"(DESC_HI), "n"(idesc), "r"(acc)
            : "memory");
    };
    auto commit = [](uint32_t bar) {
      if constexpr (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                bar),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
    };
    int sb = 0, bph = 0, ab = 0, aph = 0, g = 0, kf = 0;
    for (int k = 0; k < nk; ++k) {
      const bool first = kf == 0, last = kf == F - 1 || k + 1 == nk;
      PROF_T0;
      wait_u(bfull0 + 8 * sb, bph);
      PROF_ADD(4);
      PROF_T0;
      if (first && g >= 2) wait_u(dempty0 + 8 * (g & 1), ((g >> 1) - 1) & 1);
      PROF_ADD(5);
      const uint32_t dt = tmem + ((g & 1) ? D1 : 0);
      const uint32_t blo0 = (((smb0 + sb * 4 * IMG * 4) & 0x3FFFF) >> 4) | (8u << 16);  // LBO 128 B
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t ah = tmem + A_COL0 + ab * 64;
        PROF_T0;
        wait_u(afull0 + 8 * ab, aph);
        PROF_ADD(6);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = 4 * h + k4;
            const uint32_t bh = blo0 + ((h * IMG * 4 + k4 * 256) >> 4);
            const uint32_t bl = bh + ((2 * IMG * 4) >> 4);
            mma(dt, ah + k4 * 8, bh, (first && kk == 0) ? 0u : 1u);
            mma(dt, ah + k4 * 8, bl, 1u);
            mma(dt, ah + 32 + k4 * 8, bh, 1u);
          }
          commit(aempty0 + 8 * ab);  // the slot is free once these MMAs have read it
        }
        __syncwarp();
        if (++ab == NS) { ab = 0; aph ^= 1; }
      }
      if (elect_one()) {
        commit(bempty0 + 8 * sb);
        if (last) commit(dfull0 + 8 * (g & 1));
      }
      __syncwarp();
      if (++sb == SB) { sb = 0; bph ^= 1; }
      if (++kf == F) { kf = 0; ++g; }
    }
  } else if (warp < EW) {
    // ---------------- evaluation + drain ----------------
    const int lg = warp & 3, quarter = warp >> 2;
    const int row = lg * 32 + lane;
    const int er = tile * TBM + row;
    const bool row_ok = !stopped && er < a.R;
    const int gi = row_ok ? idx[er] : 0;
    const float* xrow = a.xs + static_cast<size_t>(gi) * a.dp;
    const uint32_t lane_addr = static_cast<uint32_t>(lg * 32) << 16;
    double acc[DC];
#pragma unroll
    for (int e = 0; e < DC; ++e) acc[e] = 0.0;
    auto drain = [&](int g) {
      PROF_T0;
      mbar_wait(&d_full[g & 1], (g >> 1) & 1);
      PROF_ADD(7);
      tc_fence_after();
      const uint32_t base = tmem + lane_addr + ((g & 1) ? D1 : 0) + quarter * DC;
#pragma unroll
      for (int q = 0; q < DC / 4; ++q) {
        uint32_t v[4];
        tc_ld4(base + 4 * q, v);
        tc_wait_ld();
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[4 * q + e] += static_cast<double>(__uint_as_float(v[e]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          arrive_cluster(mapa_u32(smem_u32(&d_empty[g & 1]), 0));
        else
          mbar_arrive(&d_empty[g & 1]);
      }
    };
    uint64_t xik2[4], k_s3, k_one, k_c, k_l2s2;
    {
      const float4 xr = __ldg(reinterpret_cast<const float4*>(xrow));
      const float xe[4] = {xr.x, xr.y, xr.z, xr.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) asm("mov.b64 %0, {%1, %1};" : "=l"(xik2[q]) : "f"(xe[q]));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_s3) : "f"(kSqrt3f));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_one) : "f"(1.f));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_c) : "f"(kNegSqrt3Log2e));
      asm("mov.b64 %0, {%1, %1};" : "=l"(k_l2s2) : "f"(a.log2_s2));
    }
    // this thread's 16 columns: 8 q .. 8 q + 7 of each 32-column half (half h:
    // chunk columns 32 h + 8 q ..), so each half of the A buffer is complete --
    // and published to the MMA warp -- after one eval8 of every evaluation warp
    const uint32_t st_base = smem_u32(smS);
    const uint32_t xoff = static_cast<uint32_t>((2 * rws + quarter * 8) * 4);
    constexpr uint32_t XHALF = 32 * DP * 4;  // bytes between the halves' SoA x
    const uint32_t st_full0 = smem_u32(st_full), st_empty0 = smem_u32(st_empty);
    const uint32_t a_full0 = smem_u32(a_full), a_empty0 = smem_u32(a_empty);
    const uint32_t acol = tmem + lane_addr + A_COL0 + quarter * 8;
    auto wait_u32 = [](uint32_t bar, uint32_t parity) {
      uint32_t done = 0;
      do {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
      } while (!done);
    };
    auto arrive_u32 = [](uint32_t bar) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    };
    // eight entries (four FP32x2 column pairs) starting at column pair base xq
    auto eval8 = [&](uint32_t xq, uint32_t (&hi)[8], uint32_t (&lo)[8]) {
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        uint64_t r2;
#if SGD_FAKE_DIST  // timing experiment only (wrong results): no distance work
        r2 = xik2[0] ^ static_cast<uint64_t>(t);
#else
#pragma unroll
        for (int q = 0; q < DX; ++q) {
          uint64_t cc, dd;
          asm volatile("ld.shared.b64 %0, [%1];" : "=l"(cc) : "r"(xq + (q * 32 + t) * 4));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dd) : "l"(cc), "l"(xik2[q]));
          if (q == 0)
            asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r2) : "l"(dd));
          else
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r2) : "l"(dd));
        }
#endif
        float ra, rb;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(ra), "=f"(rb) : "l"(r2));
#if !SGD_FAKE_MUFU
        ra = sqrt_approx(ra);
        rb = sqrt_approx(rb);
#endif
        uint64_t rr, tt, uu, ee, kk;
        asm("mov.b64 %0, {%1, %2};" : "=l"(rr) : "f"(ra), "f"(rb));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(tt) : "l"(rr), "l"(k_s3), "l"(k_one));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(uu) : "l"(rr), "l"(k_c), "l"(k_l2s2));
        float ua, ub;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(ua), "=f"(ub) : "l"(uu));
#if !SGD_FAKE_MUFU
        ua = ex2_approx(ua);
        ub = ex2_approx(ub);
#endif
        asm("mov.b64 %0, {%1, %2};" : "=l"(ee) : "f"(ua), "f"(ub));
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(kk) : "l"(tt), "l"(ee));
        float ka, kb;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(ka), "=f"(kb) : "l"(kk));
        hi[t] = __float_as_uint(ka) & 0xFFFFE000u;
        hi[t + 1] = __float_as_uint(kb) & 0xFFFFE000u;
        uint64_t hh, ll;
        asm("mov.b64 %0, {%1, %2};" : "=l"(hh) : "r"(hi[t]), "r"(hi[t + 1]));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ll) : "l"(kk), "l"(hh));
        asm("mov.b64 {%0, %1}, %2;" : "=r"(lo[t]), "=r"(lo[t + 1]) : "l"(ll));
      }
    };
    int drained = 0, next_drain = F + DEFER;
    int pend = -1;  // a_full barrier (2 ab + h) of the half whose stores are in flight
    const uint32_t a_full_lead = PAIR ? mapa_u32(a_full0, 0) : a_full0;  // the MMA issuer's a_full
    auto publish = [&]() {
      if (pend < 0) return;
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          arrive_cluster(a_full_lead + 8 * pend);
        else
          arrive_u32(a_full0 + 8 * pend);
      }
      pend = -1;
    };
    int s = 0, sph = 0;
    int slot = 0, use = 0;  // the A slot of the next half and its use count
    auto store_half = [&](const uint32_t (&hi)[8], const uint32_t (&lo)[8]) {
      publish();  // the previous half
      PROF_T0;
      if (use > 0) wait_u32(a_empty0 + 8 * slot, (use - 1) & 1);  // the slot's previous half consumed
      PROF_ADD(9);
      tc_fence_after();
      const uint32_t abase = acol + slot * 64;
      tc_st8(abase, hi);
      tc_st8(abase + 32, lo);
      pend = slot;

      if (++slot == NS) {
        slot = 0;
        ++use;
      }
    };
    if constexpr (PAIR) {
      // passes of 4 chunks: chunk u of a pass uses stage u and A slots 2u % 4,
      // (2u + 1) % 4 (half j of the solve uses slot j % 4), so after unrolling
      // every barrier / TMEM address is an immediate and every phase a
      // constant: the ring bookkeeping was ~40 % of the warps' instructions
      static_assert(ST == 4 && NS == 4, "pass layout");
      constexpr uint32_t STB = static_cast<uint32_t>((4 * LG * 256 + 2 * 32 * DP + CH) * 4);  // bytes per stage
      auto pub = [&](int slot) {  // the half in `slot` is stored: hand it to the MMA issuer
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cluster(a_full_lead + 8 * slot);
      };
      auto put = [&](int slot, bool reuse, uint32_t parity, const uint32_t (&hi)[8], const uint32_t (&lo)[8]) {
        PROF_T0;
        if (reuse) wait_u32(a_empty0 + 8 * slot, parity);  // the slot's previous half consumed
        PROF_ADD(9);
        tc_fence_after();
        tc_st8(acol + slot * 64, hi);
        tc_st8(acol + slot * 64 + 32, lo);
      };
      int pass = 0;
      for (int k0 = 0; k0 < nk; k0 += 4, ++pass) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          if (k < nk) {
            const int s0 = (2 * u) % 4, s1 = (2 * u + 1) % 4;
            const bool reuse = pass > 0 || u >= 2;
            const uint32_t aph = u >= 2 ? 0u : 1u;
            PROF_T0;
            wait_u32(st_full0 + 8 * u, static_cast<uint32_t>(pass & 1));
            PROF_ADD(8);
            const uint32_t xq = st_base + u * STB + xoff;
            uint32_t hi[8], lo[8];
            eval8(xq, hi, lo);
            if (k > 0) pub((2 * u + 3) % 4);  // the previous half
            put(s0, reuse, aph, hi, lo);
            eval8(xq + XHALF, hi, lo);
            __syncwarp();
            if (lane == 0) arrive_u32(st_empty0 + 8 * u);  // x_c consumed
            pub(s0);
            put(s1, reuse, aph, hi, lo);
            if (k == next_drain) {
              drain(drained++);
              next_drain += F;
            }
          }
        }
      }
      if (nk > 0) pub((2 * nk - 1) % 4);
    } else {
      for (int k = 0; k < nk; ++k) {
        PROF_T0;
        wait_u32(st_full0 + 8 * s, sph);
        PROF_ADD(8);
        const uint32_t xq = st_base + static_cast<uint32_t>(s * st_floats * 4) + xoff;
        uint32_t hi[8], lo[8];
        eval8(xq, hi, lo);
        store_half(hi, lo);
        eval8(xq + XHALF, hi, lo);
        __syncwarp();
        if (lane == 0) arrive_u32(st_empty0 + 8 * s);  // x_c consumed
        store_half(hi, lo);
        if (++s == ST) { s = 0; sph ^= 1; }
        if (k == next_drain) {
          drain(drained++);
          next_drain += F;
        }
      }
      publish();
    }
    while (drained < ngroups) drain(drained++);
    if (row_ok) {
      double* prow = a.part + (static_cast<size_t>(split) * a.R + er) * a.m;
#pragma unroll
      for (int e = 0; e < DC; ++e) {
        const int j = quarter * DC + e;
        if (j < a.m) prow[j] = acc[e];
      }
    }
  }
#if SGD_PROF
  if (lane == 0) {
    const int slot = warp == PROD_WARP ? 10 : (warp >= BUILD_WARP0 && warp < MMA_WARP) ? 11 : warp == MMA_WARP ? 12 : 13;
    atomicAdd(&g_sgd_prof[slot], static_cast<unsigned long long>(clock64() - prof_start));
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const bool bld = warp >= BUILD_WARP0 && warp < MMA_WARP;
      const int slot = (bld && i == 4) ? 14 : i;
      if (prof_acc[i]) atomicAdd(&g_sgd_prof[slot], static_cast<unsigned long long>(prof_acc[i]));
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's MMAs / arrivals are done before either CTA frees TMEM
  if (warp == 0) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int NPAD, int DX, int NBW, bool PAIR>
void launch_64_t(const SgdSlabArgs& a, cudaStream_t s) {
  constexpr int NB = PAIR ? NPAD / 2 : NPAD;
  const int rws = PAIR ? 2 * (NB / 8) * 256 : a.rw;
  const size_t smem = c64::smem_bytes<NB, c64::st_stages<PAIR>()>(rws, 4, a.ntab);
  if (smem > 227 * 1024) throw std::invalid_argument("gpk: SGD slab kernel (64) shared memory exceeds 227 KB");
  static size_t configured = 0;
  auto kern = sgd_slab64_kernel<NPAD, DX, NBW, PAIR>;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  const int tiles = (a.R + TBM - 1) / TBM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(PAIR ? (tiles + 1) / 2 * 2 : tiles, a.splits, 1);  // PAIR: whole pairs of row tiles
  cfg.blockDim = dim3(32 * (EW + 2 + NBW), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if constexpr (PAIR) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (a.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  GPK_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  check_launch("sgd_slab64_kernel");
}
template <int NPAD, int DX>
void launch_64(const SgdSlabArgs& a, cudaStream_t s) {
  // B-builder warps: 4 (measured at C4 with the loads-first builders: 223 us
  // per launch vs 236 with 8, whose 72-register cap spills in the evaluation
  // warps); GPK_SGD_BW=8 selects eight
  static const int bw = [] {
    const char* e = std::getenv("GPK_SGD_BW");
    return e ? std::atoi(e) : 4;
  }();
  if constexpr (NPAD % 16 == 0)
    if (a.pair) return launch_64_t<NPAD, DX, 4, true>(a, s);
  if (bw == 8) return launch_64_t<NPAD, DX, 8, false>(a, s);
  return launch_64_t<NPAD, DX, 4, false>(a, s);
}

template <int NPAD, int DP4, bool GRAM, int DX = 0>
void launch_one(const SgdSlabArgs& a, cudaStream_t s) {
  constexpr int DP = 4 * DP4;
  const size_t smem = sgd_smem_bytes<NPAD>(a.rw, DP, a.ntab);
  if (smem > 227 * 1024) throw std::invalid_argument("gpk: SGD slab kernel shared memory exceeds 227 KB");
  static size_t configured = 0;
  if (smem > configured) {
    GPK_CUDA(cudaFuncSetAttribute(sgd_slab_kernel<NPAD, DP4, GRAM, DX>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  sgd_slab_kernel<NPAD, DP4, GRAM, DX><<<dim3((a.R + TBM - 1) / TBM, a.splits), NTHREADS, smem, s>>>(a);
  check_launch("sgd_slab_kernel");
}

template <int NPAD>
void launch_n(const SgdSlabArgs& a, cudaStream_t s) {
  switch (a.dp / 4) {
    case 1:
      if (a.xg) return launch_one<NPAD, 1, true>(a, s);
      if (a.ch64) switch (a.d) {  // 64-column pipeline
          case 1: return launch_64<NPAD, 1>(a, s);
          case 2: return launch_64<NPAD, 2>(a, s);
          case 3: return launch_64<NPAD, 3>(a, s);
          default: return launch_64<NPAD, 4>(a, s);
        }
      switch (a.d) {  // exact-dimension scalar distance loops for d <= 4
        case 1: return launch_one<NPAD, 1, false, 1>(a, s);
        case 2: return launch_one<NPAD, 1, false, 2>(a, s);
        case 3: return launch_one<NPAD, 1, false, 3>(a, s);
        default: return launch_one<NPAD, 1, false, 4>(a, s);
      }
    case 2: return a.xg ? launch_one<NPAD, 2, true>(a, s) : launch_one<NPAD, 2, false>(a, s);
    case 3: return a.xg ? launch_one<NPAD, 3, true>(a, s) : launch_one<NPAD, 3, false>(a, s);
    case 4: return a.xg ? launch_one<NPAD, 4, true>(a, s) : launch_one<NPAD, 4, false>(a, s);
    default: throw std::invalid_argument("gpk: the SGD slab kernel supports d <= 16");
  }
}

// ---- per-iteration reduction / update kernels ------------------------------
// slice[q][j] = sum_s part[s][q][j] (+ sigma^2 V(t)[i][j] - B[i][j] if row i =
// idx[q] is this rank's); slice[bm + j] = sum over own q of R[i][j]^2 (old
// residual estimate), slice[bm + m] = this rank's pending divergence flag.
__global__ void sgd_reduce_kernel(SgdStepArgs a) {
  if (a.ctl->stop) return;
  const int t = a.ctl->iters;
  const int* idx = a.idxbuf + static_cast<size_t>(t % a.idx_chunk) * a.b;
  const int m = a.m, bm = a.b * m;
  const int gb = gridDim.x - m;
  if (static_cast<int>(blockIdx.x) >= gb) {
    const int j = blockIdx.x - gb;
    __shared__ double wsum[32];
    double acc = 0.0;
    for (int q = threadIdx.x; q < a.b; q += blockDim.x) {
      const int li = idx[q] - a.row0;
      if (li >= 0 && li < a.nloc) {
        const double r = a.resid[static_cast<size_t>(li) * m + j];
        acc += r * r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += wsum[w];
      a.slice[bm + j] = tot;
      if (j == 0) a.slice[bm + m] = *a.nonfinite ? 1.0 : 0.0;
    }
    return;
  }
  // four lanes per element: lane k of the quad sums splits k, k + 4, ...
  // (independent loads in flight), the quad combines (s0 + s1) + (s2 + s3)
  const int quad = threadIdx.x & 3;
  for (int e4 = blockIdx.x * blockDim.x + threadIdx.x; e4 < 4 * bm; e4 += gb * blockDim.x) {
    const int e = e4 >> 2;
    const int q = e / m, j = e - q * m;
    double g = 0.0;
#pragma unroll 4
    for (int s = quad; s < a.splits; s += 4) g += a.part[static_cast<size_t>(s) * bm + e];
    const unsigned act = __activemask();  // whole quads (4 bm is a multiple of 4)
    g += __shfl_xor_sync(act, g, 1);
    g += __shfl_xor_sync(act, g, 2);
    if (quad != 0) continue;
    const int li = idx[q] - a.row0;
    if (li >= 0 && li < a.nloc) {
      const size_t o = static_cast<size_t>(li) * m + j;
      const int dl = min(max(t - a.tau[li] - 1, 0), a.budget);
      const double v = fma(a.s64[dl], a.Mb[o], a.Vb[o]);  // V(t) of the row
      g = fma(a.sigma2, v, g) - a.B[o];
    }
    a.slice[e] = g;
  }
}

// g = sum of the rank slices (rank order); own minibatch rows: M(t+1) = rho
// M(t) - (lr/b) g, V(t+1) = V(t) + M(t+1) as the new base, tau = t, FP32
// records; R[i] = -g. Block partials of sum_q g^2 per column; the last block
// to finish updates the residual norms and takes the termination decision
// (solvers.cpp:164-178: test after the update, abort on a non-finite iterate).
// minibatch rows per block of the apply / finish kernels (the same in both: their block partials are summed
// in one order). Measured at C4: 4 rows (128 blocks) 20.7 us per finish launch, 8 rows 17.0 us; 16 exceeds 1024 threads.
#ifndef SGD_FIN_ROWS
#define SGD_FIN_ROWS 8
#endif
constexpr int APPLY_ROWS = SGD_FIN_ROWS;
__global__ void sgd_apply_kernel(SgdStepArgs a) {
  if (a.ctl->stop) return;
  const int t = a.ctl->iters;
  const int* idx = a.idxbuf + static_cast<size_t>(t % a.idx_chunk) * a.b;
  const int m = a.m, bm = a.b * m;
  __shared__ double gs[APPLY_ROWS][80];
  __shared__ int bad_g, bad_row;
  __shared__ unsigned last;
  if (threadIdx.x == 0) bad_g = bad_row = 0;
  __syncthreads();
  const int rl = threadIdx.x / m, j = threadIdx.x - rl * m;  // blockDim.x = APPLY_ROWS * m
  const int q = blockIdx.x * APPLY_ROWS + rl;
  double g2 = 0.0;
  if (rl < APPLY_ROWS && q < a.b) {
    double g = a.gbuf[static_cast<size_t>(q) * m + j];
    for (int r = 1; r < a.nr; ++r) g += a.gbuf[static_cast<size_t>(r) * a.stride + static_cast<size_t>(q) * m + j];
    if (!isfinite(g)) bad_g = 1;
    g2 = g * g;
    const int li = idx[q] - a.row0;
    if (li >= 0 && li < a.nloc) {
      const size_t o = static_cast<size_t>(li) * m + j;
      const int dl = min(max(t - a.tau[li] - 1, 0), a.budget);
      const double mb = a.Mb[o];
      const double mt = a.p64[dl] * mb;                      // M(t)
      const double vt = fma(a.s64[dl], mb, a.Vb[o]);         // V(t)
      const double mn = __dsub_rn(__dmul_rn(mt, a.rho), __dmul_rn(a.step, g));
      const double vn = __dadd_rn(vt, mn);
      if (!isfinite(vn) || !isfinite(mn)) bad_row = 1;
      a.Mb[o] = mn;
      a.Vb[o] = vn;
      a.resid[o] = -g;
      const size_t ro = static_cast<size_t>(li / 32) * a.rw + sgd_record_pos(li % 32, j);
      a.rec[ro] = static_cast<float>(vn);
      a.rec[ro + a.moff] = static_cast<float>(mn);
    }
  }
  if (rl < APPLY_ROWS) gs[rl][j] = g2;
  __syncthreads();  // every thread of the block has read tau of its row
  if (rl < APPLY_ROWS && j == 0 && q < a.b) {
    const int li = idx[q] - a.row0;
    if (li >= 0 && li < a.nloc) a.tau[li] = t;
  }
  // block partial of sum g^2 per column (rows in order)
  if (threadIdx.x < m) {
    double s = 0.0;
    for (int r = 0; r < APPLY_ROWS; ++r) s += gs[r][threadIdx.x];
    a.gpart[static_cast<size_t>(blockIdx.x) * m + threadIdx.x] = s;
  }
  if (threadIdx.x == 0 && (bad_g || bad_row)) atomicOr(a.nonfinite_now, bad_g ? 3 : 1);  // bit 1: g itself
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double ss[128];
  __shared__ double red8[8][80];
  {  // column sums of the block partials: thread (jj, k) sums blocks k, k + 8, ... then 8 partials in order
    const int jj = threadIdx.x % m, k = threadIdx.x / m;
    if (k < 8) {
      double s = 0.0;
      for (int b = k; b < static_cast<int>(gridDim.x); b += 8) s += a.gpart[static_cast<size_t>(b) * m + jj];
      red8[k][jj] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int jj = threadIdx.x;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red8[k][jj];
    double old = 0.0;
    for (int r = 0; r < a.nr; ++r) old += a.gbuf[static_cast<size_t>(r) * a.stride + bm + jj];
    const double v = a.sumsq[jj] + (s - old);
    a.sumsq[jj] = v;
    ss[jj] = fmax(v, 0.0);
  }
  __syncthreads();
  // divergence (solvers.cpp:173-177): one rank -- a non-finite updated row, now;
  // sharded -- a non-finite g (identical on every rank) now, a rank's own
  // non-finite row through its next slice, so every rank stops at the same
  // iteration (their collectives must match)
  double pend = 0.0;
  for (int r = 0; r < a.nr; ++r) pend += a.gbuf[static_cast<size_t>(r) * a.stride + bm + m];
  const int now = *a.nonfinite_now;
  const bool diverged = (!a.sharded ? now != 0 : (now & 2) != 0) || pend != 0.0;
  if (threadIdx.x == 0) {
    *a.ticket = 0u;
    if (now) *a.nonfinite = 1;
  }
  if (threadIdx.x < 32) {  // termination_check on the tracked residuals (linear_system.cpp:47-53)
    double probe = 0.0;
    for (int jj = 1 + threadIdx.x; jj < m; jj += 32) probe += sqrt(ss[jj]) / a.scales[jj];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) probe += __shfl_xor_sync(0xffffffffu, probe, o);
    if (threadIdx.x == 0) {
      const double mean = sqrt(ss[0]) / a.scales[0];
      probe = m > 1 ? probe / (m - 1) : 0.0;
      CgCtl* c = a.ctl;
      c->iters += 1;
      c->mean_norm = mean;
      c->probe_norm = probe;
      c->done = mean <= a.tol && probe <= a.tol;
      c->aborted = diverged ? 1 : 0;
      c->stop = (c->done || c->aborted || c->iters >= c->budget) ? 1 : 0;
    }
  }
}

// Single rank: the reduce and apply kernels fused (one launch per iteration
// fewer, no g round trip). Block = FIN_ROWS minibatch rows x m columns; the
// thread of an element sums the split partials in four interleaved chains
// s = c, c + 4, ... and combines (s0 + s1) + (s2 + s3) (sgd_reduce_kernel's
// order), then applies the row's lazy update exactly as sgd_apply_kernel,
// keeping the old residual square for the incremental norms. The last of the
// b / FIN_ROWS = 64 blocks sums the block partials of g^2 and of the old
// squares in block order and takes the termination / divergence decision
// (solvers.cpp:164-178).
constexpr int FIN_ROWS = SGD_FIN_ROWS;
__global__ void sgd_finish_kernel(SgdStepArgs a) {
  // programmatic dependent launch: the next slab kernel may start its prologue
  // now (it waits for this grid's completion before it reads anything this
  // grid writes); this grid waits for the slab's partials
  griddep_launch();
  griddep_wait();
  if (a.ctl->stop) return;
  const int t = a.ctl->iters;
  const int ctl_budget = a.ctl->budget;
  const int* idx = a.idxbuf + static_cast<size_t>(t % a.idx_chunk) * a.b;
  const int m = a.m, bm = a.b * m;
  // (only the last block uses it; loaded here so the load is off its serial tail)
  const double sumsq_old = static_cast<int>(threadIdx.x) < m ? a.sumsq[threadIdx.x] : 0.0;
  __shared__ double gs[FIN_ROWS][80], os[FIN_ROWS][80];
  __shared__ int bad_g, bad_row;
  __shared__ unsigned last;
  if (threadIdx.x == 0) bad_g = bad_row = 0;
  __syncthreads();
  const int rl = threadIdx.x / m, j = threadIdx.x - rl * m;  // blockDim.x = FIN_ROWS m (rounded to 32)
  const int q = blockIdx.x * FIN_ROWS + rl;
  const bool act = rl < FIN_ROWS && q < a.b;
  // FIN_DEEP split partials in flight per round; element e of the splits goes
  // to chain e % 4, each chain in increasing e, whatever the depth. The rounds
  // are unpredicated so that ptxas issues all of a round's loads before the
  // first add (a predicated round compiled, depending on unrelated code, to a
  // load-add-load-add chain: 26.7 instead of 16.8 us per launch at C4's 37
  // splits; depth 4: 24.2 us; depth 20 spills).
#ifndef FIN_DEEP
#define FIN_DEEP 16
#endif
  int li = -1;
  double g = 0.0;
  if (act) {
    const int e = q * m + j;
    double c4[4] = {0.0, 0.0, 0.0, 0.0};
    // unpredicated rounds of FIN_DEEP loads (all in flight before the first
    // add), then rounds of four, then the tail; sp stays a multiple of 4
    int sp = 0;
#if FIN_DEEP > 4
    for (; sp + FIN_DEEP <= a.splits; sp += FIN_DEEP) {
      double v[FIN_DEEP];
#pragma unroll
      for (int i = 0; i < FIN_DEEP; ++i) v[i] = __ldcg(a.part + static_cast<size_t>(sp + i) * bm + e);
#pragma unroll
      for (int i = 0; i < FIN_DEEP; ++i) c4[i & 3] += v[i];
    }
#endif
    for (; sp + 4 <= a.splits; sp += 4) {
      double v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __ldcg(a.part + static_cast<size_t>(sp + c) * bm + e);
#pragma unroll
      for (int c = 0; c < 4; ++c) c4[c] += v[c];
    }
    for (int c = 0; sp + c < a.splits; ++c) c4[c] += __ldcg(a.part + static_cast<size_t>(sp + c) * bm + e);
    g = (c4[0] + c4[1]) + (c4[2] + c4[3]);
  }
  double g2 = 0.0, o2 = 0.0;
  if (act) {
    li = idx[q];
    const size_t o = static_cast<size_t>(li) * m + j;
    const int dl = min(max(t - a.tau[li] - 1, 0), a.budget);
    const double mb = a.Mb[o];
    const double vb = a.Vb[o], bt = a.B[o], old = a.resid[o], sd = a.s64[dl], pd = a.p64[dl];
    const double vt = fma(sd, mb, vb);  // V(t)
    g = fma(a.sigma2, vt, g) - bt;
    if (!isfinite(g)) bad_g = 1;
    g2 = g * g;
    o2 = old * old;
    const double mt = pd * mb;  // M(t)
    const double mn = __dsub_rn(__dmul_rn(mt, a.rho), __dmul_rn(a.step, g));
    const double vn = __dadd_rn(vt, mn);
    if (!isfinite(vn) || !isfinite(mn)) bad_row = 1;
    a.Mb[o] = mn;
    a.Vb[o] = vn;
    a.resid[o] = -g;
    const size_t ro = static_cast<size_t>(li / 32) * a.rw + sgd_record_pos(li % 32, j);
    a.rec[ro] = static_cast<float>(vn);
    a.rec[ro + a.moff] = static_cast<float>(mn);
  }
  if (rl < FIN_ROWS) {
    gs[rl][j] = g2;
    os[rl][j] = o2;
  }
  __syncthreads();  // every thread of the block has read tau of its row
  if (act && j == 0) a.tau[li] = t;
  if (threadIdx.x < m) {  // block partials, rows in order
    double sg = 0.0, so = 0.0;
#pragma unroll
    for (int r = 0; r < FIN_ROWS; ++r) {
      sg += gs[r][threadIdx.x];
      so += os[r][threadIdx.x];
    }
    a.gpart[static_cast<size_t>(blockIdx.x) * 2 * m + threadIdx.x] = sg;
    a.gpart[static_cast<size_t>(blockIdx.x) * 2 * m + m + threadIdx.x] = so;
  }
  if (threadIdx.x == 0 && (bad_g || bad_row)) atomicOr(a.nonfinite_now, bad_g ? 3 : 1);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int now = __ldcg(a.nonfinite_now);
  __shared__ double ss[128];
  __shared__ double red8[8][2][80];
  {  // column sums of the block partials: thread (jj, k) sums blocks k, k + 8, ... then 8 partials in order
    for (int w = threadIdx.x; w < 8 * m; w += blockDim.x) {
      const int jj = w % m, k = w / m;
      double sg = 0.0, so = 0.0;
#pragma unroll 8
      for (int b = k; b < static_cast<int>(gridDim.x); b += 8) {  // loads issued ahead, adds in block order
        sg += __ldcg(a.gpart + static_cast<size_t>(b) * 2 * m + jj);
        so += __ldcg(a.gpart + static_cast<size_t>(b) * 2 * m + m + jj);
      }
      red8[k][0][jj] = sg;
      red8[k][1][jj] = so;
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int jj = threadIdx.x;
    double sg = 0.0, so = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sg += red8[k][0][jj];
      so += red8[k][1][jj];
    }
    const double v = sumsq_old + (sg - so);
    a.sumsq[jj] = v;
    ss[jj] = fmax(v, 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.ticket = 0u;
    if (now) *a.nonfinite = 1;
  }
  if (threadIdx.x < 32) {  // termination_check on the tracked residuals (linear_system.cpp:47-53)
    double probe = 0.0;
    for (int jj = 1 + threadIdx.x; jj < m; jj += 32) probe += sqrt(ss[jj]) / a.scales[jj];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) probe += __shfl_xor_sync(0xffffffffu, probe, o);
    if (threadIdx.x == 0) {
      const double mean = sqrt(ss[0]) / a.scales[0];
      probe = m > 1 ? probe / (m - 1) : 0.0;
      CgCtl* c = a.ctl;
      const int done = (mean <= a.tol && probe <= a.tol) ? 1 : 0;
      c->iters = t + 1;
      c->mean_norm = mean;
      c->probe_norm = probe;
      c->done = done;
      c->aborted = now ? 1 : 0;
      c->stop = (done || now || t + 1 >= ctl_budget) ? 1 : 0;
    }
  }
}

// Gram column image for the SGD slab: (-2 x, |x|^2 at slot d, 0...) of the
// scaled FP32 inputs (rows beyond n zero), |x|^2 by the same FP32 chain the
// kernel uses for its rows
__global__ void sgd_gram_image_kernel(const float* xs, int rows, int n, int d, int dp, float* xg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    float ni = 0.f;
    for (int k = 0; k < dp; ++k) {
      const float x = i < n ? xs[static_cast<size_t>(i) * dp + k] : 0.f;
      if (k < d) ni = fmaf(x, x, ni);
      xg[static_cast<size_t>(i) * dp + k] = k < d ? -2.f * x : 0.f;
    }
    if (i < n) xg[static_cast<size_t>(i) * dp + d] = ni;
  }
}

// Column coordinates per 32-row chunk in SoA order (chunk q: [dp][32]) for
// the exact-dimension FP32x2 evaluation (two columns per instruction)
__global__ void sgd_soa_image_kernel(const float* xs, int rows, int dp, float* out) {
  const long long total = static_cast<long long>(rows) * dp;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / dp), k = static_cast<int>(e % dp);
    out[(static_cast<size_t>(i / 32) * dp + k) * 32 + (i % 32)] = xs[e];
  }
}

// initial records from the warm-start solution: V32 = V0, M32 = 0, tau = -1
__global__ void sgd_records_init_kernel(const double* V, int nloc, int nchunks, int m, int rw, int moff, float* rec,
                                        int* tau) {
  const long long total = static_cast<long long>(nchunks) * rw;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int q = static_cast<int>(e / rw), w = static_cast<int>(e % rw);
    float v = 0.f;
    if (w < moff) {  // V image: element (c, j) at ((j / 8) 8 + c / 4) 32 + (j % 8) 4 + c % 4
      const int core = w >> 5, ln = w & 31;
      const int j = (core >> 3) * 8 + (ln >> 2), c = (core & 7) * 4 + (ln & 3);
      const int i = q * 32 + c;
      if (i < nloc && j < m) v = static_cast<float>(V[static_cast<size_t>(i) * m + j]);
    }
    rec[e] = v;
    if (w < 32) tau[q * 32 + w] = -1;
  }
}

// V(T) for every own row at the end of the solve (in place on the base)
__global__ void sgd_materialise_kernel(double* Vb, const double* Mb, const int* tau, const double* s64, int budget,
                                       const CgCtl* ctl, int nloc, int m) {
  const int T = ctl->iters;
  const long long total = static_cast<long long>(nloc) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / m);
    const int dl = min(max(T - tau[i] - 1, 0), budget);
    Vb[e] = fma(s64[dl], Mb[e], Vb[e]);
  }
}

}  // namespace

int sgd_record_width(int m, int* moff) {
  const int img = 256 * ((m + 7) / 8);  // j-groups of 8 x 32 chunk columns
  if (moff) *moff = img;
  return 2 * img;
}

void sgd_slab_launch(const SgdSlabArgs& a, cudaStream_t s) {
  switch (kv_tc_npad(a.m)) {
    case 16: return launch_n<16>(a, s);
    case 32: return launch_n<32>(a, s);
    case 48: return launch_n<48>(a, s);
    case 64: return launch_n<64>(a, s);
    case 80: return launch_n<80>(a, s);
    default: throw std::invalid_argument("gpk: the SGD slab kernel supports m <= 80");
  }
}

void sgd_gram_image_launch(const float* xs, int rows, int n, int d, int dp, float* xg, cudaStream_t s) {
  sgd_gram_image_kernel<<<std::max(1, std::min(148 * 4, (rows + 255) / 256)), 256, 0, s>>>(xs, rows, n, d, dp, xg);
  check_launch("sgd_gram_image");
}

void sgd_soa_image_launch(const float* xs, int rows, int dp, float* out, cudaStream_t s) {
  const long long total = static_cast<long long>(rows) * dp;
  sgd_soa_image_kernel<<<static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8)), 256, 0, s>>>(xs, rows, dp,
                                                                                                          out);
  check_launch("sgd_soa_image");
}

void sgd_reduce_launch(const SgdStepArgs& a, cudaStream_t s) {
  const int gb = std::max(1, (4 * a.b * a.m + 255) / 256);  // one thread per (element, quarter of the splits)
  sgd_reduce_kernel<<<gb + a.m, 256, 0, s>>>(a);
  check_launch("sgd_reduce");
}

void sgd_apply_launch(const SgdStepArgs& a, cudaStream_t s) {
  if (a.m > 80) throw std::invalid_argument("gpk: SGD apply supports m <= 80");
  const int threads = ((APPLY_ROWS * a.m + 31) / 32) * 32;
  sgd_apply_kernel<<<(a.b + APPLY_ROWS - 1) / APPLY_ROWS, threads, 0, s>>>(a);
  check_launch("sgd_apply");
}

void sgd_finish_launch(const SgdStepArgs& a, cudaStream_t s) {
  if (a.m > 80) throw std::invalid_argument("gpk: SGD finish supports m <= 80");
  const int threads = ((FIN_ROWS * a.m + 31) / 32) * 32;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.b + FIN_ROWS - 1) / FIN_ROWS, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  GPK_CUDA(cudaLaunchKernelEx(&cfg, sgd_finish_kernel, a));
  check_launch("sgd_finish");
}
int sgd_finish_blocks(int b) { return (b + FIN_ROWS - 1) / FIN_ROWS; }

void sgd_records_init_launch(const double* V, int nloc, int rows_pad, int m, int rw, int moff, float* rec, int* tau,
                             cudaStream_t s) {
  const int nchunks = rows_pad / 32 + 1;  // + one zero record: a 64-column chunk may end past rows_pad
  const long long total = static_cast<long long>(nchunks) * rw;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  sgd_records_init_kernel<<<blocks, 256, 0, s>>>(V, nloc, nchunks, m, rw, moff, rec, tau);
  check_launch("sgd_records_init");
}

void sgd_materialise_launch(double* Vb, const double* Mb, const int* tau, const double* s64, int budget,
                            const CgCtl* ctl, int nloc, int m, cudaStream_t s) {
  const long long total = static_cast<long long>(nloc) * m;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  sgd_materialise_kernel<<<blocks, 256, 0, s>>>(Vb, Mb, tau, s64, budget, ctl, nloc, m);
  check_launch("sgd_materialise");
}

}  // namespace gpk

#if SGD_PROF
extern "C" int gpk_debug_sgd_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, gpk::g_sgd_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(gpk::g_sgd_prof, z, sizeof(z));
  }
  return 0;
}
#endif
