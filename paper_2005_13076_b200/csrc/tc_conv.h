// tc_conv.h -- host entry points of the general tcgen05 TF32 convolution
// (tc_conv.cu): im2col / col2im materialisation kernels, the TF32 weight
// copies, and the TMA-fed GEMM of the forward, weight and data gradients.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "params.h"
#include "runtime.h"

namespace pn {
namespace tcc {
cudaError_t setup(int max_nk);  // opt-in shared memory (gather kernel: K up to max_nk*32)

// ---- data gradient: implicit GEMM with gathered operand (stride-1 convs):
// dx = W' (*) G, W'[c][(f,i',j')] = W[f][c][kh-1-i'][kw-1-j'], pad kh-1-p
int fwd_rows_pad(int F);  // rows of the packed (swizzled) B image for F output channels
Launch conv_fwd_launch(const ConvTcP& p);
Launch pack_launch(const ConvPackP& p);

// ---- the contractions over materialised TF32 operands (TMA-fed GEMM)
struct ConvGemmP {
  CUtensorMap ta;  // A [rows][Kdim] K-major, box {32, 128}
  CUtensorMap tb;  // B [cols][Kdim] K-major, box {32, BN}
  float* out;
  const float* bias;
  int Kdim, rows, cols, splits;
  int K, F, has_bias, pstride;  // weight gradient
  int HoWo, relu;               // forward
  int bn, ctiles;               // column tile width / count per group (set at launch)
  int G;                        // groups: rows / cols above are per group
};
// shapes of one conv layer's materialised operands and GEMM tilings
struct ConvTmaPlan {
  int M, K, F, bias, howo, G;  // K = (C/G)*kh*kw (per group)
  int pitch_m;  // row pitch of colT / Gm (floats, multiple of 4)
  int kp, fp;   // row pitch of col / Wf (K) and of Gt / Wt (F)
  int wg_bn, wg_kpad, wg_fpad, wg_splits;
  int fw_bn;
  size_t col_floats, g_floats;  // workspace this layer needs
};
ConvTmaPlan conv_tma_plan(int N, int C, int kh, int kw, int F, int Ho, int Wo, int bias, int sms, int G = 1);
Launch im2col_t_launch(const Im2colTP& p);     // colT [k][m] (weight gradient)
Launch im2col_rows_launch(const Im2colTP& p);  // col  [m][k] (forward)
Launch gm_launch(const GmP& p);                // Gm   [f][m] (weight gradient)
Launch pack_plain_launch(const PackPlainP& p);
// false if a tensor-map encoding failed
bool gemm_wgrad_launch(const ConvTmaPlan& w, const float* colT, const float* gm, float* part, int pstride,
                       Launch* out);
bool gemm_fwd_launch(const ConvTmaPlan& w, const float* col, const float* wf, const float* bias, float* y, int relu,
                     Launch* out);

// ---- stride-1 convolution as a TMA tap GEMM over NHWC (forward and data gradient)
struct ConvTapP {
  CUtensorMap ta;  // NHWC activation [N][H][W][cp], box {32, bw, bh, bni}
  CUtensorMap tb;  // per-tap weights [T][rows][ip], box {32, BN, 1}
  const float* bias;
  const float* relu_y;
  float* out;      // NCHW [N][F][Ho][Wo]
  int N, Ho, Wo, F, cp, kh, kw, ph, pw, sgn;
  int bw, bh, bni, tiles_w, tiles_h, relu;
  int bn, ctiles;  // output-channel tile width / tiles per group
  int G, fg, cpg;  // groups, output channels per group, input-channel slots per group
};
// in: NHWC activation (N x Hin x Win x cp); out: F channels of Ho x Wo;
// sgn = +1 forward (input at out + tap - pad), -1 data gradient (out - tap + pad)
// G > 1: grouped convolution -- cp = G * cpg input-channel slots, F = G * fg
// output channels, group g's output channels read slots [g*cpg, (g+1)*cpg)
bool tap_launch(const float* nhwc, int N, int Hin, int Win, int cp, const float* wtaps, int rows, int ip, int kh,
                int kw, int ph, int pw, int sgn, int Ho, int Wo, int F, const float* bias, int relu,
                const float* relu_y, float* out, Launch* l, int G = 1, int cpg = 0);
Launch nhwc_launch(const NhwcP& p);

// ---- weight gradient as a tap GEMM over TMA-staged segments (no im2col)
// dW[f, c, i, j] = sum_{n, yo, xo} G[n, f, yo, xo] X[n, c, yo + i - ph, xo + j - pw]
// for stride-1, ungrouped layers with W = Wo in {8, 16, 32}, C in {16, 32,
// 64, 128}, F % 16 == 0 (F <= 256): the accumulator rows are (tap, c), the
// contraction runs over output positions, one TMA box per segment of R output
// rows brings every shifted input row it needs (tc_conv.cu conv_wgrad_taps).
// Split partials per CTA (segments split evenly) in [f][tap][c] order, summed
// and permuted to [f][c][tap] by wgrad_reduce (ReduceP pc/pk/pt).
struct ShiftCopyP {  // out[n][y][j][c][x] = tf32(x[n][c][y][x + j - pw]), 0 outside
  const float* x;
  float* out;
  int N, C, H, W, kw, pw;
};
struct GwP {  // out[n][yo][f][xo] = tf32(g[n][f][yo][xo])
  const float* g;
  float* out;
  int N, F, Ho, Wo;
};
struct ConvWtapP {
  CUtensorMap tx;  // Xs {W, C, kw, H, N}, box {Wo, C, kw, R + kh, 1}
  CUtensorMap tg;  // Gw {Wo, F, Ho, N}, box {Wo, F, R, 1}
  float* part;     // [splits][pstride]: f*K + t*C + c (t = tap; the reduce permutes); bias at F*K + f
  int N, C, Ho, Wo, F, kh, kw, ph, pw, T, K, bias, pstride;
  int MT, TPT, R, x_bytes, stage_bytes, tx_bytes, seg_per_img, segs, tmem_cols;
};
Launch shift_copies_launch(const ShiftCopyP& p);
Launch gw_launch(const GwP& p);
bool wgrad_taps_ok(int C, int W, int Wo, int F, int kh, int kw, int sh, int sw, int G);
int wgrad_taps_splits(int N, int Ho, int Wo, int C, int F, int kh, int kw, int sms);  // CTAs = split partials
bool wgrad_taps_launch(const float* xs, const float* gw, int N, int C, int H, int W, int Ho, int Wo, int F, int kh,
                       int kw, int ph, int pw, int bias, float* part, int pstride, int splits, Launch* l);
Launch pack_taps_launch(const PackTapsP& p);

// ---- stride-1 convolution over halo-staged 4-channel planes (tc_plane.cu):
// forward (+bias, ReLU) and data gradient (+ the in-place ReLU's mask)
struct PlanePlan {
  int TY, TN, HY, HX, Kq, a_bytes, w_bytes, stages, tiles_x, tiles_y, tiles;
  int ns;  // output-channel splits (w_bytes = one split's weights)
  size_t smem;
};
struct PlanePackP {  // A blocks [tile][cq][HY][TN][HX][4] (TF32)
  const float* src;
  float* out;
  int N, C, H, W, ph, pw, Kq, HY, HX, TY, TN, tiles, tiles_x, tiles_y;
};
struct PlaneWpackP {  // B [split][t][cq][o][4] (TF32); mode 0 forward, 1 data gradient
  const float* w;
  float* out;
  int Cin, Nout, kh, kw, Kq, mode, ns;
};
struct PlaneConvP {
  const float* src;     // A blocks
  const float* wts;     // B
  const float* bias;    // forward bias (nullable)
  const float* relu_y;  // data gradient: the in-place ReLU's output (nullable)
  float* out;           // NCHW [N][Nout][Ho][Wo]
  int N, Ho, Wo, Nout, Kq, kh, kw, TY, TN, HY, HX, tiles, tiles_x, tiles_y, a_bytes, w_bytes, relu, stages;
  int tmem_cols;
  int ns;  // output-channel splits: CTA b computes split b % ns
};
bool plane_plan(int N, int Cin, int Ho, int Wo, int Nout, int kh, int kw, PlanePlan* pl);
Launch plane_pack_launch(const PlanePlan& pl, const float* src, float* out, int N, int C, int H, int W, int ph,
                         int pw);
Launch plane_wpack_launch(const PlanePlan& pl, const float* w, float* out, int Cin, int Nout, int kh, int kw,
                          int mode);
Launch plane_conv_launch(const PlanePlan& pl, const float* src, const float* wts, const float* bias,
                         const float* relu_y, float* out, int N, int Ho, int Wo, int Nout, int kh, int kw, int relu,
                         int sms);
cudaError_t plane_setup();
}  // namespace tcc
}  // namespace pn
