// Fused AP epilogue shared by kv_reduce_dot_kernel (kv_kernel.cu) and the
// fused tensor-core slab (kv_tc_kernel.cu): run by the last CTA to finish an
// AP slab (ticket), it sums the per-group column partials and block-score
// partials in a fixed order, counts the iteration and tests termination
// (ap_check), picks the next block (ap_select, strict '>' from -1) and writes
// the next block update's batched-GEMM pointers (solvers.cpp:119-141).
#pragma once

#include "gpk_internal.cuh"

namespace gpk {

// Every participating thread calls it; `bar()` synchronises them (tid in
// [0, 32 * nwarps)). ss >= 96 doubles, bscore >= nblocks doubles (<= 1024).
template <class Bar>
__device__ void ap_epilogue(const KvReduceArgs& a, int G, int tid, int nwarps, double* ss, double* bscore, Bar bar) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int j = warp; j < a.m; j += nwarps) {  // sum_g dpart[g][j], fixed xor tree per warp
    double acc = 0.0;
    for (int q = lane; q < G; q += 32) acc += __ldcg(a.dpart + static_cast<size_t>(q) * a.m + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ss[j] = acc;
  }
  for (int k = warp; k < a.nblocks; k += nwarps) {  // fixed xor tree per block
    double t = 0.0;
    for (int q = lane; q < a.gpb; q += 32) t += __ldcg(a.spart + static_cast<size_t>(k) * a.gpb + q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0 && k < 1024) bscore[k] = sqrt(t);
  }
  bar();
  // per-column norm terms in parallel; one thread adds them in column order
  for (int j = tid; j < a.m; j += 32 * nwarps) ss[j] = sqrt(ss[j]) / a.scales[j];
  bar();
  if (tid == 0) {
    CgCtl* c = a.ctl;
    c->iters += 1;
    const double mean = ss[0];
    double sum = 0.0;
    for (int j = 1; j < a.m; ++j) sum += ss[j];
    const double probe = a.m > 1 ? sum / (a.m - 1) : 0.0;
    c->mean_norm = mean;
    c->probe_norm = probe;
    c->done = (mean <= a.tol && probe <= a.tol) ? 1 : 0;
    c->stop = (c->done || c->iters >= c->budget) ? 1 : 0;
    int best_k = 0;
    double best = -1.0;
    for (int k = 0; k < a.nblocks; ++k)
      if (bscore[k] > best) {
        best = bscore[k];
        best_k = k;
      }
    *a.sel_out = best_k;
    if (a.ap_ptrs) {
      a.ap_ptrs[0] = a.out + static_cast<size_t>(best_k) * a.score_block * a.m;  // R rows of the block (padded)
      a.ap_ptrs[1] = a.ap_inv + static_cast<size_t>(best_k) * a.ap_bb;
      a.ap_ptrs[2] = a.ap_upd;
    }
    *a.ticket = 0u;
  }
}

}  // namespace gpk
