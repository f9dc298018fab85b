// tc.h -- tcgen05 (5th-gen tensor core) TF32 kernels for the GEMM-shaped
// LeNet layers: conv2 (+bias+pool2+mask), ip1 (+bias+relu), ip1 weight and
// data gradients (the latter fused with pool2's backward), conv2 data and
// weight gradients, and the per-step TF32 weight packing they consume.
// Dense operands are fed by TMA from TF32 copies in global memory; the
// tensor maps are encoded at plan-build time (library-owned buffers).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "params.h"
#include "runtime.h"

namespace pn {
namespace tc {
// Packed TF32 weight copies (see tc.cu "weight packing")
struct PackP {
  const float* w1;  // [500][800]
  const float* w2;  // [50][500]
  float* w1f;       // [500][800]
  float* w1t;       // [800][512]
  float* w2c;       // [25 taps][5][50][4] (conv2 fwd B)
  float* w2t;       // W2d: [5 i][14 planes][104 (c,j)][4 f] + pad (conv2 dgrad A)
};
constexpr int kW1fFloats = 500 * 800, kW1tFloats = 800 * 512, kW2cFloats = 25000, kW2tFloats = 5 * 14 * 104 * 4 + 96;

cudaError_t setup();    // driver entry point + opt-in shared memory sizes
bool tensor_maps_ok();  // false if any cuTensorMapEncodeTiled call failed
Launch pack_weights_launch(const PackP& p);
// the fused solver (reduce + SGD + TF32 weight copies; tc.cu "fused solver")
Launch lenet_solver_launch(const SolverP& p);
// conv2 forward operand layout p1c: per image pair [5 cc][12 h][2 n][12 w][4 c] floats
constexpr int kP1cPairFloats = 5 * 12 * 2 * 12 * 4;
Launch conv2_pool2_launch(const float* w2c, const float* b, const float* p1c, float* p2, float* p2T, uint8_t* m2,
                          int N, int npad, int sms);
Launch pack_p1c_launch(const float* p1, float* p1c, int N);
// the three ip1 GEMMs as 128-row tiles (ip_tile<Op>: per-layer tile width and K
// split over a cluster, partials reduced in DSMEM)
Launch ip1_fwd_launch(const float* p2, const float* w1f, const float* b, float* y, int N);
// fp32 class (PN_3XTF32): the ip1 contractions as 3xTF32 over hi / lo operand copies
struct Split3P {  // hi / lo [R][C] and their transposes [C][ldt] (null: skipped)
  const float* src;
  float* hi;
  float* lo;
  float* hiT;
  float* loT;
  int R, C, ldt;
};
Launch split3_launch(const Split3P& p);
Launch ip1_fwd3_launch(const float* p2h, const float* p2l, const float* w1h, const float* w1l, const float* b, float* y,
                       int N);
Launch ip1_grad3_launch(const float* ah, const float* al, int rows, int K, int lda, const float* bh, const float* bl,
                        int cols, int ldb, float* out, int ldo);
Launch ip1_wgrad_launch(const float* da1T, const float* p2T, float* dw, int N, int npad);
Launch ip1_dgrad_unpool_launch(const float* da1r, const float* w1t, const uint8_t* m2, float* g2, float* part_db2,
                               int N);
int db2_partials(int N);  // conv2 bias-gradient partial rows written by ip1_dgrad_unpool
Launch conv2_dgrad_launch(const float* g2, const float* w2t, float* dp1, int N, int sms);
Launch conv2_wgrad_launch(const float* g2, const float* p1, float* part, int splits, int N);
// conv1 + pool1 on the tensor cores (tc_conv1.cu): implicit GEMM over 128-row
// tiles of (pooled position, window slot), quad-shuffle pooling epilogue
cudaError_t conv1_setup();
Launch conv1_pool1_tc_launch(const Conv1Pool1P& p, int sms);
}  // namespace tc
}  // namespace pn
