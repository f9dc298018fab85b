// solver.cuh -- the conv bucket's solver as the tail of the TF32 plan's
// last backward kernel (conv1's weight gradient, a single-GPU whole step):
// a grid-wide barrier (every block's partials written), then every thread of
// the grid reduces, updates and re-packs a share of the conv parameters.
#pragma once
#include "params.h"
#include "reduce.cuh"
#include "sgd.cuh"
#include "tc_ptx.cuh"

namespace pn {
// W2d (conv2 data-gradient A operand, tc.cu dg::): [5 i][14 planes of 4 f][104 (c,j) rows][4 f]
constexpr int kW2dPlanes = 14, kW2dRows = 104;

// grid-wide barrier over a monotonic counter (every CTA resident: one per SM)
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned ncta) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long old;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    const unsigned long long target = (old / ncta + 1) * ncta;
    unsigned long long cur;
    do {
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
    } while (cur < target);
  }
  __syncthreads();
}

// The conv bucket's solver by every thread of the grid (conv1's weight
// gradient, a single-GPU whole step): output i of a segment with few splits
// is summed by one thread (split_sum_serial), of one with many splits by 8
// lanes (split w of lane w, then lane 0 adds the 8 in order) -- both the
// bucket reduction's exact order -- then SGD and the W2c / W2d copies.
__device__ __forceinline__ unsigned tail_span(const ReduceP& s) {
  return ((s.splits > 64 ? 8 : 1) * s.n + 31) & ~31u;  // (multiples of 32: warp-uniform segments)
}
#ifndef TAIL_ONE_PASS
#define TAIL_ONE_PASS 40
#endif
constexpr int kTailOnePass = TAIL_ONE_PASS;  // splits summed with all loads in flight together
__device__ __forceinline__ void tail_update(const SolverP& sp, const ReduceP& s, int i, long long e, float r, float w,
                                            float v, float lr);
// item t of segments [k0, k1) (t warp-uniform in its 32-block)
__device__ __forceinline__ void solver_item(const SolverP& sp, unsigned t, int k0, int k1, float lr) {
  unsigned l = t;
  int k = k0;
  for (; k < k1 - 1; ++k) {
    const unsigned span = tail_span(sp.seg[k]);
    if (l < span) break;
    l -= span;
  }
  const ReduceP& s = sp.seg[k];
  const bool wide = s.splits > 64;
  const int i = wide ? (int)(l >> 3) : (int)l;
  float r;
  if (wide) {
    const int w = (int)(l & 7), lane = threadIdx.x & 31;
    float acc = 0.f;
    if (i < s.n) {
#pragma unroll 1
      for (int base = w; base < s.splits; base += 8 * 16) {
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          v[q] = base + 8 * q < s.splits ? __ldcg(s.part + (long long)(base + 8 * q) * s.stride + i) : 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += v[q];
      }
    }
    r = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) r += __shfl_sync(0xffffffffu, acc, (lane & ~7) + q);
    if (w != 0) return;
  } else if (kTailOnePass > 0 && s.splits <= kTailOnePass) {
    // split_sum_serial's order with every load (partials, w, v) in one round trip
    if (i >= s.n) return;
    const long long e = (s.out - sp.g) + i;
    float w = sp.w[e], v = sp.v[e];
    float x[kTailOnePass > 0 ? kTailOnePass : 1];
#pragma unroll
    for (int q = 0; q < kTailOnePass; ++q) x[q] = q < s.splits ? __ldcg(s.part + (long long)q * s.stride + i) : 0.f;
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
#pragma unroll
    for (int q = 0; q < kTailOnePass; ++q)
      if (q < s.splits) acc[q & 7] += x[q];
    r = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) r += acc[q];
    tail_update(sp, s, i, e, r, w, v, lr);
    return;
  } else {
    r = i < s.n ? split_sum_serial(s, i) : 0.f;
  }
  if (i >= s.n) return;
  const long long e = (s.out - sp.g) + i;
  float w = sp.w[e], v = sp.v[e];
  tail_update(sp, s, i, e, r, w, v, lr);
}
__device__ __forceinline__ void tail_update(const SolverP& sp, const ReduceP& s, int i, long long e, float r, float w,
                                            float v, float lr) {
  if (s.part != s.out) s.out[i] = r;
  sgd_one(w, r, v, lr, sp.mom, sp.decay, sp.gscale);
  sp.w[e] = w;
  sp.v[e] = v;
  const long long q2 = e - sp.w2_off;
  if (q2 >= 0 && q2 < 25000) {
    const int f = (int)q2 / 500, c = ((int)q2 / 25) % 20, ii = ((int)q2 / 5) % 5, jj = (int)q2 % 5;
    const float wf = tc::tf32f(w);
    sp.w2c[(ii * 5 + jj) * 1000 + (c >> 2) * 200 + f * 4 + (c & 3)] = wf;
    sp.w2t[((ii * kW2dPlanes + (f >> 2)) * kW2dRows + c * 5 + jj) * 4 + (f & 3)] = wf;
  }
}
// Segments [k0, k1), strided over the grid's threads
__device__ __forceinline__ void solver_tail(const SolverP& sp, unsigned u, unsigned nthreads, int k0, int k1) {
  const float lr = sp.lr_dev ? __ldg(sp.lr_dev) : sp.lr;
  unsigned total = 0;
  for (int k = k0; k < k1; ++k) total += tail_span(sp.seg[k]);
  for (unsigned t = u; t < total; t += nthreads) solver_item(sp, t, k0, k1, lr);
}
}  // namespace pn
