// tc_conv.h -- host entry points of the general tcgen05 TF32 convolution
// (tc_conv.cu): forward, data gradient (as a flipped-filter stride-1
// convolution), split-m weight gradient, and the per-step TF32 weight packing.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "params.h"
#include "runtime.h"

namespace pn {
namespace tcc {
cudaError_t setup(int max_nk);  // opt-in shared memory for K up to max_nk*32
int fwd_rows_pad(int F);        // rows of the packed B image for an output of F channels
size_t fwd_smem_bytes(int F, int nk);
Launch conv_fwd_launch(const ConvTcP& p);
int wgrad_splits(int N, int Ho, int Wo, int F, int K, int bias, int sms);
Launch conv_wgrad_launch(const ConvTcWgradP& p);
Launch pack_launch(const ConvPackP& p);

// weight gradient over materialised TF32 operands (colT, Gm), TMA-fed
struct ConvWgTmaP {
  CUtensorMap ta;  // colT [Kpad][pitch]: box {32 m, 128 k}
  CUtensorMap tb;  // Gm   [Fpad][pitch]: box {32 m, BN f}
  float* part;     // [splits][pstride]: w at f*K + k, b at F*K + f
  int M, K, F, bias, splits, pstride;
};
struct WgTmaPlan {
  int bn, kpad, fpad, pitch, splits;
};
WgTmaPlan wgrad_tma_plan(int N, int Ho, int Wo, int F, int K, int bias, int sms);
Launch im2col_t_launch(const Im2colTP& p);
Launch gm_launch(const GmP& p);
// false if the tensor-map encoding failed
bool wgrad_tma_launch(const WgTmaPlan& w, const float* col, const float* gm, float* part, int M, int K, int F,
                      int bias, int pstride, Launch* out);
}  // namespace tcc
}  // namespace pn
