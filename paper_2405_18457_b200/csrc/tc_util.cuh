// Shared PTX wrappers for the tcgen05 kernels (kv_tc_kernel.cu,
// grad_tc_kernel.cu): mbarriers, bulk async copies, TMEM loads/stores,
// kind::tf32 MMA with A from TMEM or shared memory, UMMA descriptors.
#pragma once
#include <cstdint>

namespace gpk {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits for the phase with the given parity. The suspend-time hint lets the
// waiting thread sleep until the phase completes (or the hint expires) instead
// of re-issuing try_wait: spinning producer / MMA / waiting eval warps
// otherwise take issue slots from the evaluation warps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-converged variants: every lane of the issuing warp executes them and
// elect.sync picks the one lane that issues (the warp stays converged around
// the MMA stream instead of running it in single-thread divergent code).
__device__ __forceinline__ void tc_mma_tf32_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// Issue loops of the tcgen05 kernels: the whole MMA warp runs them and
// elect.sync issues (GPK_MMA_WARP=0: lane 0 alone, in divergent code, where
// ptxas wraps every MMA in an elect/branch waterfall: measured ~17% slower on
// the C2 operator product)
#ifndef GPK_MMA_WARP
#define GPK_MMA_WARP 1
#endif
#if GPK_MMA_WARP
#define MMA_TF32 tc_mma_tf32_w
#define MMA_COMMIT tc_commit_w
#else
#define MMA_TF32 tc_mma_tf32
#define MMA_COMMIT tc_commit
#endif
// ---- warp-uniform single-thread issue -------------------------------------
// The whole issuing warp runs the waits and the operand arithmetic; one lane,
// chosen by tc_elect_one(), issues from an if-block. With a compile-time TMEM
// base (one CTA per SM allocating all 512 columns: the allocation starts at 0)
// and descriptors formed as 32-bit offsets of one base word (the start-address
// field is the low 14 bits), every operand is warp-uniform, so ptxas keeps
// them in uniform registers: ~2.5 instructions per MMA instead of ~18 for
// MMA_TF32's per-MMA elect and register broadcasts.
__device__ __forceinline__ uint32_t tc_elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred;
}
// low word of umma_desc(saddr, lbo, sbo); the high word is tc_desc_hi(sbo)
__device__ __forceinline__ uint32_t tc_desc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr & 0x3FFFF) >> 4) | ((lbo >> 4) << 16);
}
constexpr uint32_t tc_desc_hi(uint32_t sbo) { return ((sbo >> 4) & 0x3FFF) | (1u << 14); }
template <uint32_t HI, uint32_t IDESC>
__device__ __forceinline__ void tc_mma_u(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\t"
      "mov.b64 bd, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "r"(b_lo), "n"(HI), "n"(IDESC), "r"(accumulate)
      : "memory");
}
// the same with the descriptor's high word at run time (SBO from a kernel argument)
template <uint32_t IDESC>
__device__ __forceinline__ void tc_mma_ur(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\t"
      "mov.b64 bd, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bd, %4, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "r"(b_lo), "r"(b_hi), "n"(IDESC), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_u(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tc_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// Tensor-core Gram distances (kv_tc_kernel TG, tg_image_kernel): a scaled
// coordinate enters as x' = hi + lo, two TF32 values (22 significant bits);
// the MMAs form -2 x'_i.x'_c from hi.hi + hi.lo + lo.hi and both sides compute
// |x'|^2 with this same FP32 chain (zero padding adds nothing), so the row
// and column norms of one point are bitwise equal.
__device__ __forceinline__ void tg_split(float x, float& hi, float& lo) {
  hi = __uint_as_float(tf32_rna(x));
  lo = __uint_as_float(tf32_rna(x - hi));
}
__device__ __forceinline__ float tg_norm_step(float acc, float hi, float lo) {
  const float xp = hi + lo;  // exact: at most 22 significant bits
  return fmaf(xp, xp, acc);
}
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
constexpr float kNegSqrt3Log2e = -2.4988211106473432f;  // -sqrt(3) * log2(e)
constexpr float kSqrt3f = 1.7320508075688772f;

// Canonical no-swizzle K-major UMMA smem descriptor (version 1 = tcgen05):
// core matrices of 8 rows x 16 B; LBO = K-adjacent core-matrix stride,
// SBO = 8-row-group stride (both in bytes).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  return d;                             // base offset 0, lbo mode 0, SWIZZLE_NONE (0)
}

// kind::tf32 instruction descriptor: D F32, A/B TF32, both K-major, M=128.
constexpr uint32_t tf32_idesc(int n, int m = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// ---- Gram-form squared distance (d >= 21; see gram_image_kernel) ----
// Row side: slot d of the image holds |x_i|^2 -> captured into ni and
// replaced by 1; the coordinates are scaled by -2 (exact).
__device__ __forceinline__ void gram_row(float4& v, int k0, int d, float& ni) {
  float* c = reinterpret_cast<float*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (k0 + e == d) {
      ni = c[e];
      c[e] = 1.f;
    } else {
      c[e] = -2.f * c[e];
    }
  }
}
// r^2 = |x_i|^2 + sum_k xt_i[k] xt_c[k] over the padded row, four FFMA2 chains
template <int DP4>
__device__ __forceinline__ float gram_r2(uint32_t xaddr, const uint64_t* xi2, uint64_t seed) {
  uint64_t acc[4] = {seed, 0ull, 0ull, 0ull};
#pragma unroll
  for (int u = 0; u < DP4; ++u) {
    uint64_t c01, c23;
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(c01), "=l"(c23) : "r"(xaddr + 16 * u));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[(2 * u) & 3]) : "l"(c01), "l"(xi2[2 * u]));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[(2 * u + 1) & 3]) : "l"(c23), "l"(xi2[2 * u + 1]));
  }
  uint64_t s01, s23, s;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s01) : "l"(acc[0]), "l"(acc[1]));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s23) : "l"(acc[2]), "l"(acc[3]));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(s01), "l"(s23));
  float s0, s1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(s));
  return fmaxf(s0 + s1, 0.f);
}
// k(x_i, x_i) = s2 exactly as the direct form evaluates it at r = 0, plus
// `add` (the persistent AP slab folds the noise term sigma^2 into the entry)
template <int CPT>
__device__ __forceinline__ void gram_pin_diagonal(bool hit, int tpos, float log2_s2, uint32_t* hi, uint32_t* lo,
                                                  float add = 0.f) {
  const float k0 = ex2_approx(log2_s2) + add;
  const uint32_t h0 = __float_as_uint(k0) & 0xFFFFE000u;
  const uint32_t l0 = __float_as_uint(k0 - __uint_as_float(h0));
#pragma unroll
  for (int t = 0; t < CPT; ++t)
    if (hit && tpos == t) {
      hi[t] = h0;
      lo[t] = l0;
    }
}

}  // namespace tc

}  // namespace gpk
