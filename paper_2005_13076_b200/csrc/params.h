// params.h -- kernel parameter blocks (one __grid_constant__ struct per kernel)
// shared by the host runtime (net.cpp) and the CUDA kernels.  Product code
// only: nothing here is shared with oracle/.
#pragma once
#include <stdint.h>

namespace pn {

// ---------------------------------------------------------------- generic
struct ConvFwdP {  // y = W (*) x + b
  const float* x;
  const float* w;
  const float* b;
  float* y;
  int N, C, H, W, F, kh, kw, sh, sw, ph, pw, Ho, Wo;
  int G;  // groups (0 or 1: none); w is [F][C/G][kh][kw]
};
struct ConvBwdDataP {  // dx = col2im(W^T dy) in gather form
  const float* dy;
  const float* w;
  float* dx;
  int N, C, H, W, F, kh, kw, sh, sw, ph, pw, Ho, Wo;
  int G;
};
struct ConvBwdWeightP {  // split-N partials of dW = sum dy col^T and db
  const float* dy;
  const float* x;
  float* part_w;  // [splits][F*C*kh*kw]
  float* part_b;  // [splits][F]
  int N, C, H, W, F, kh, kw, sh, sw, ph, pw, Ho, Wo, splits;
  int pstride;    // floats between consecutive splits of part_w / part_b
  int G;          // groups; grid.x = F * C/G
};
struct ReduceP {  // out[i] = sum_s part[s*stride + i], i < n (fixed order s = 0..)
  const float* part;
  float* out;
  int n, splits, stride;
  // pc > 0: the partials of i < pw are a conv weight gradient in [f][t][c]
  // order (tc_conv.cu conv_wgrad_taps); out index f*pk + c*pt + t (pk = C*T)
  int pw, pk, pc, pt;
};
__host__ __device__ inline int reduce_out_index(const ReduceP& s, int i) {
  if (s.pc <= 0 || i >= s.pw) return i;
  const int f = i / s.pk, r = i - f * s.pk, t = r / s.pc, c = r - t * s.pc;
  return f * s.pk + c * s.pt + t;
}
struct ReduceMultiP {  // several ReduceP segments in one launch
  ReduceP seg[6];
  int nseg, total;
  int late;  // inputs come from >= 2 launches back: wait on the predecessor only at the end (pdl.cuh)
};
// The TF32 LeNet plan's fused solver (tc.cu lenet_solver, solver.cuh solver_tail):
// reduce + SGD + the TF32 weight copies
struct SolverP {
  float* w;        // flat parameters
  float* g;        // flat gradients
  float* v;        // flat momentum history
  float lr, mom, decay, gscale;
  const float* lr_dev;
  long long w1_off, w2_off;  // ip1.w / conv2.w offsets in the flat buffers
  float *w1f, *w1t, *w2c, *w2t;
  ReduceP seg[4];  // gradient = fixed-order sum of partials (part == out: already reduced)
  int nseg, seg_blocks;
  int w1_tiles;  // 0, or the 400 W1 tiles (ip1 weights + W1f / W1t)
  long long plain_lo[3], plain_hi[3];  // other parameters (gradients already reduced)
  int nplain;
};

// The layerwise plans' stem: conv (stride 1, the data input) -> MAX pool ->
// in-place ReLU fused (kernels_generic.cu stem_fwd / stem_wgrad)
struct StemP {
  const float* x;      // [N][C][H][W]
  const float* w;      // [F][C][kh][kw]
  const float* b;      // [F] or nullptr
  float* y;            // pooled, ReLU'd output [N][F][Hp][Wp]
  int32_t* mask;       // pool origins (plane-local h*Wo + w of the conv output)
  const float* dy;     // gradient w.r.t. y (ReLU already back-propagated by its consumer)
  float* part_w;       // [splits][pstride] weight-gradient partials (+ bias at F*C*kh*kw)
  int N, C, H, W, F, kh, kw, ph, pw, Ho, Wo;
  int pk, ps, pp, Hp, Wp;  // pool kernel, stride, pad (square), output
  int splits, pstride, relu;
};
struct PoolFwdP {  // P:215-220; S:357-365 (method 0 MAX, 1 AVE)
  const float* x;
  float* y;
  int32_t* mask;
  int N, C, H, W, kh, kw, sh, sw, ph, pw, Hp, Wp, method;
  int relu;  // 1: an in-place ReLU follows (y = max(pooled, 0); the mask is the pooling's)
};
struct PoolBwdP {  // P:220-222; gather form, ascending output order
  const float* dy;
  const int32_t* mask;
  float* dx;
  int N, C, H, W, kh, kw, sh, sw, ph, pw, Hp, Wp, method;
  const float* relu_y;  // non-null: the bottom is an in-place ReLU (slope 0) output -> dx *= (relu_y > 0)
};
struct GemmP {  // C[m,n] = sum_k A(m,k) B(k,n) (+ bias[n]) (relu)
  const float* A;
  const float* B;
  float* C;
  const float* bias;
  int M, N, K;
  long long sam, sak, sbk, sbn;
  int relu;
  int splits;   // gemm_tiled: > 1 = K split over gridDim.z, raw partials to part[z][M][N] (gemm_splitk_reduce adds them)
  float* part;
};
struct ColSumP {  // out[n] = sum_m a[m*N + n]
  const float* a;
  float* out;
  int M, N;
};
struct ReluP {
  const float* x;   // fwd input / bwd dy
  const float* y;   // bwd: forward output
  float* out;
  long long n;
  float slope;
};
struct SoftmaxLossP {  // P:109-110; S:429-446 (fwd + bwd in one pass)
  const float* logits;
  const int32_t* labels;
  float* prob;
  int32_t* pred;
  float* dlogits;
  float* row_loss;
  unsigned* err;
  int M, D;
  float grad_scale;  // loss_weight / M
};
struct SoftmaxP {  // standalone SoftMax: fwd y = softmax(x); bwd dx = y (dy - <dy, y>)
  const float* x;   // fwd input / bwd top diff
  const float* y;   // bwd: forward output
  float* out;       // fwd y / bwd bottom diff
  int M, D;
};
struct AccuracyP {  // top-k accuracy: flag[i] = rank(label_i) < k
  const float* x;
  const int32_t* labels;
  int32_t* flag;
  unsigned* err;
  int M, D, k;
};
struct AccReduceP {  // acc = (sum of flags) / M, IEEE division
  const int32_t* flag;
  float* out;
  int M;
};
struct LossReduceP {
  const float* row_loss;
  float* loss_out;  // caller's (may be null)
  float* loss_blob;
  int M;
  float inv_M;
};
struct SgdP {  // S:536-544 Caffe SGD, fp32, no FMA
  float* w;
  const float* g;
  float* v;
  long long n;
  float lr, mom, decay, gscale;
  const float* lr_dev;  // if set: the learning rate is read from device memory (pipelined host loop)
};
struct Tf32CopyP {  // src [R][C] -> TF32-rounded copies: dst [R][C] and/or dstT [C][ldt]
  const float* src;
  float* dst;
  float* dstT;
  int R, C, ldt;
};
struct MaskExpandP {  // uint8 window offset <-> int32 plane-local (ABI view)
  uint8_t* m8;
  int32_t* m32;
  int N, C, H, W, kh, kw, sh, sw, ph, pw, Hp, Wp;
  int to32;  // 1: m8 -> m32, 0: m32 -> m8
};

// ------------------------------------------------------------ fused LeNet
// Shapes are compile-time in the kernels; the structs carry pointers only.
struct Conv1Pool1P {  // x[N,1,28,28] -> p1[N,20,12,12], m1 (uint8 offsets)
  const float* x;
  const float* w;  // [20,1,5,5]
  const float* b;  // [20]
  float* p1;
  uint8_t* m1;
  int N;
  int round_tf32;  // store p1 rounded to TF32 (RNA) for the tensor-core plan
  float* p1c;      // optional: TF32 copy in the conv2 tap-GEMM layout (tc.h kP1cPairFloats per pair)
  int per_block;   // pooled (image, position) items per block (grid = ceil(N*144 / per_block))
  // optional byte input (NEXT #4): x = fl(fl(x8 * x_scale) - x_mean[pixel]) replaces x
  const uint8_t* x8;
  float x_scale;
  const float* x_mean;  // [784] or null
};
struct Conv2Pool2P {  // p1[N,20,12,12] -> p2[N,50,4,4], m2
  const float* p1;
  const float* w;  // [50,20,5,5]
  const float* b;
  float* p2;
  uint8_t* m2;
  int N;
};
struct Ip2LossP {  // a1[N,500] -> logits, prob, pred, dz, row_loss
  const float* a1;
  const float* w;  // [10,500]
  const float* b;
  const int32_t* labels;
  float* logits;
  float* prob;
  int32_t* pred;
  float* dz;
  float* row_loss;
  unsigned* err;
  int N;
  float grad_scale;
};
struct Ip2BwdP {  // dz[N,10], a1 -> da1 = relu'(a1) * dz W2 ; dW2 / db2 partials
  const float* dz;
  const float* a1;
  const float* w;  // [10,500]
  float* da1;
  float* part_w;  // [splits][10*500]
  float* part_b;  // [splits][10]
  int N, splits, pstride;
  // TF32 plan only (null otherwise): TF32-rounded copies of da1 for the ip1
  // contractions ([N][500] and transposed [500][npad]) and db1 partials
  float* da1r;
  float* da1rT;
  float* part_b1;  // [splits][500]
  int npad;
};
struct Unpool2P {  // dp2 [N,800] + m2 -> G2 [N,50,8,8] dense
  const float* dp2;
  const uint8_t* m2;
  float* g2;
  int N;
};
struct Conv1WgradP {  // dp1 + m1 + x -> partial dW1, db1
  const float* dp1;
  const uint8_t* m1;
  const float* x;
  float* part_w;  // [splits][500]
  float* part_b;  // [splits][20]
  int N, splits, pstride;
  const uint8_t* x8;  // optional byte input, as Conv1Pool1P
  float x_scale;
  const float* x_mean;
  int tail;                 // 1: the conv bucket's solver after a grid barrier (solver.cuh)
  unsigned long long* bar;  // grid-barrier counter (monotonic)
  SolverP sp;               // the conv bucket: reduce segments, SGD, W2c / W2d copies
};
struct LoopSumP {  // test-hook exchange: rank-order sum of one bucket over n ranks' buffers (net.cu)
  float* buf[8];
  int n;
  long long count;
};
struct IngestP {  // bytes -> fp32 input blob: y = fl(fl(x8 * scale) - mean[i % per])
  const uint8_t* x8;
  float* y;
  long long n;
  int per;
  float scale;
  const float* mean;  // [per] or null
};


// --------------------------------------------- general tensor-core conv (tc_conv.cu)
struct ConvTcP {  // y = W (*) x (+ b) (relu), implicit GEMM on tcgen05
  const float* x;    // gathered activation NCHW [N][C][H][W]
  const float* bpk;  // packed TF32 B image [nk][Fpad][32] (pack_conv_weights)
  const float* bias; // [F] or nullptr
  float* y;          // [N][F][Ho][Wo]
  int N, C, H, W, F, kh, kw, sh, sw, ph, pw, Ho, Wo;
  int K, nk, Fpad;   // K = C*kh*kw, nk = ceil(K/32), Fpad = rows of the B image
  int relu;
  const float* relu_y;  // data gradient: y of the in-place ReLU (slope 0) below -> out *= (relu_y > 0)
};
struct ConvPackP {  // TF32 B image of the forward (mode 0) / data-gradient (mode 1) contraction
  const float* w;   // [F][C][kh][kw]
  float* out;       // [nk][rows][32] SW128
  int F, C, kh, kw, rows, nk, mode;
};
struct NhwcP {  // out[n][h][w][c] = tf32(x[n][c][h][w]), channels padded to cp
  const float* x;
  float* out;
  int N, C, H, W, cp;
  int G, cpg;  // grouped: group g's channels at slots [g*cpg, g*cpg + C/G)
};
struct PackTapsP {  // per-tap TF32 weight matrices (tc_conv.cu pack_taps)
  const float* w;   // [F][C][kh][kw]
  float* out;       // [kh*kw][rows][ip]
  int F, C, kh, kw, ip, mode;  // mode 0: rows f, inner c (forward); 1: rows c, inner f (data gradient)
  int G;                       // groups (inner index group-local)
};
struct Im2colTP {  // colT[k][m] = tf32(col[m][k]) (k < K), 1 (k == K: bias row)
  const float* x;
  float* col;  // [rows][pitch]
  int N, C, H, W, kh, kw, sh, sw, ph, pw, Ho, Wo, K, Kb, pitch;
  int G, Kgb;  // grouped (colT only): Kb = G blocks of Kgb = K + bias rows, K per group
};
struct GmP {  // gm[f][n*HoWo + pos] = tf32(g[n][f][pos])
  const float* g;
  float* gm;  // [rows][pitch]
  int N, F, HoWo, pitch;
};

struct PackPlainP {  // TF32 copy of W [F][K] as [F][pitch]
  const float* w;
  float* out;
  int F, K, pitch;
};

struct IpRowsP {  // y[m,o] = sum_k x[m,k] W[o,k] + b[o] (relu): split-K rows kernel for skinny outputs
  const float* x;   // [M][K]
  const float* w;   // [Nout][K]
  const float* b;   // [Nout] or nullptr
  float* y;         // [M][Nout]
  int M, K, Nout, relu;
};

}  // namespace pn
