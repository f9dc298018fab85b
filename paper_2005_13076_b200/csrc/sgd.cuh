// sgd.cuh -- the solver's per-element update (S:536-544 / DESIGN.md R11),
// shared by the generic SGD kernel and the fused LeNet solver (tc.cu): one
// IEEE fp32 rounding per op, no contraction.
#pragma once
__device__ __forceinline__ void sgd_one(float& w, float d, float& v, float lr, float mom, float decay, float gs) {
  float g = __fmul_rn(d, gs);
  g = __fadd_rn(g, __fmul_rn(decay, w));
  v = __fadd_rn(__fmul_rn(mom, v), __fmul_rn(lr, g));
  w = __fsub_rn(w, v);
}
