// reduce.cuh -- the fixed-order sum of split partials shared by the bucket
// reduction (reduce_partials_multi) and the fused solver (tc.cu): warp w of a
// 256-thread block sums splits w, w+8, w+16, ... of its lane's output in
// ascending order (starting from +0), then warp 0 adds the 8 warp sums in
// order.  A thread's loads of one pass (8, 16 or 32, by the split count) are
// all issued before its adds: one L2 round trip per pass.
#pragma once
#include "params.h"

namespace pn {
template <int L>
__device__ __forceinline__ float split_sum_pass(const ReduceP& s, int i, int w) {
  float acc = 0.f;
#pragma unroll 1
  for (int base = w; base < s.splits; base += 8 * L) {
    float v[L];
#pragma unroll
    for (int q = 0; q < L; ++q) {
      const int j = base + 8 * q;
      v[q] = j < s.splits ? __ldcg(s.part + (long long)j * s.stride + i) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < L; ++q) acc += v[q];  // (+0 padding leaves a non-(-0) sum bit-identical)
  }
  return acc;
}
__device__ __forceinline__ float split_sum_warp(const ReduceP& s, int i, int w) {
  if (i >= s.n) return 0.f;
  if (s.splits <= 8 * 8) return split_sum_pass<8>(s, i, w);
  if (s.splits <= 8 * 16) return split_sum_pass<16>(s, i, w);
  return split_sum_pass<32>(s, i, w);
}
// The same value as split_sum_warp's 8-warp scheme for output i, computed by
// one thread (narrow segments): acc_w over splits w, w+8, ... ascending, then
// ((0 + acc_0) + acc_1) ... + acc_7; loads in batches of 16 ascending.
__device__ __forceinline__ float split_sum_serial(const ReduceP& s, int i) {
  float acc[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) acc[w] = 0.f;
#pragma unroll 1
  for (int base = 0; base < s.splits; base += 16) {
    float v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      v[q] = base + q < s.splits ? __ldcg(s.part + (long long)(base + q) * s.stride + i) : 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (base + q < s.splits) acc[q & 7] += v[q];  // base % 8 == 0: split base+q belongs to warp q % 8
  }
  float r = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) r += acc[w];
  return r;
}
}  // namespace pn
