// tc.h -- tcgen05 (5th-gen tensor core) TF32 kernels for the GEMM-shaped
// LeNet layers: conv2 (+bias+pool2+mask), ip1 (+bias+relu), ip1 weight and
// data gradients (the latter fused with pool2's backward), conv2 data and
// weight gradients.  Accumulators live in TMEM; operands are staged in shared
// memory in the UMMA canonical K-major layout by producer warps (implicit
// im2col gather with round-to-nearest TF32 conversion).
#pragma once
#include <cuda_runtime.h>

#include "runtime.h"

namespace pn {
namespace tc {
cudaError_t setup();  // opt-in shared memory sizes etc.
Launch conv2_pool2_launch(const float* w, const float* b, const float* p1, float* p2, uint8_t* m2, int N, int sms);
Launch ip_fwd_launch(const float* x, const float* w, const float* b, float* y, int M, int K, int Nout, bool relu,
                     int sms);
Launch ip_wgrad_launch(const float* dy, const float* x, float* dw, float* db, int M, int K, int Nout, int sms);
Launch ip_dgrad_unpool_launch(const float* dy, const float* w, const uint8_t* m2, float* g2, int N, int sms);
Launch pack_w2d_launch(const float* w2, float* w2d);  // W2 -> [c][(f,i,j)] TF32
Launch conv2_dgrad_launch(const float* g2, const float* w2d, float* dp1, int N, int sms);
Launch conv2_wgrad_launch(const float* g2, const float* p1, float* part, int splits, int N, int sms);
}  // namespace tc
}  // namespace pn
