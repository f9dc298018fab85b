/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the LeNet-style
 * layer chain of arxiv 2005.13076 ("Using PHAST to port Caffe library").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2005_13076_b200/) never links, imports or calls it,
 * and shares no code, header, table or helper with it.
 *
 * Citations: P:<line> = PAPER.md line, S:<line> = SPEC.md line (section in
 * brackets).  Readings of silent/ambiguous passages are listed in DESIGN.md
 * section "Readings" and repeated at each function.
 *
 * Precision: every reduction is accumulated in double (fp64 "truth"); inputs
 * are the fp32 blob values the caller passes as double.  The solver update is
 * the one exception: SGD state is fp32 and each statement rounds to fp32
 * (Caffe float solver), so orc_sgd_update_f32 works in float with no FMA
 * contraction (built with -ffp-contract=off).
 *
 * Alongside a reduction output the oracle can return S_i = sum |term| (plus
 * |bias|), the scale used by the per-element tolerance |gpu - o| <= rtol*S_i.
 *
 * Return value: 0 on success, -1 on invalid geometry (non-positive output
 * size, non-positive dimension), -2 on label out of range.
 */
#ifndef PN_ORACLE_H
#define PN_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Output sizes. Conv: floor.  Pool: Caffe ceil with the
 * "last window must start inside the image" correction (R4). */
int orc_conv_out_size(int in, int k, int s, int p);
int orc_pool_out_size(int in, int k, int s, int p);

/* im2col / col2im.
 * col is (C*kh*kw) x (Ho*Wo), row index (c,i,j) row-major, column (ho,wo). */
int orc_im2col(const double* x, int C, int H, int W, int kh, int kw, int sh,
               int sw, int ph, int pw, double* col);
int orc_col2im(const double* col, int C, int H, int W, int kh, int kw, int sh,
               int sw, int ph, int pw, double* x);

/* naive GEMM C[M,N] = A[M,K] * B[K,N] (row-major), the paper's gemm step. */
void orc_gemm(int M, int N, int K, const double* A, const double* B, double* C);

/* Convolution forward, plain definition (cross-correlation, no flip; bias
 * after the full sum: Listing 1 order P:160-167).
 * x: N*C*H*W, w: F*C*kh*kw, b: F (may be NULL), y: N*F*Ho*Wo,
 * S (may be NULL): per-output sum |w*x| + |b|. */
int orc_conv_fwd(const double* x, int N, int C, int H, int W, const double* w,
                 int F, int kh, int kw, const double* b, int sh, int sw, int ph,
                 int pw, double* y, double* S);

/* Convolution forward the paper's way: per image im2col, then
 * GEMM  W(F x CKK) * col(CKK x HoWo), then bias added to every row. */
int orc_conv_fwd_im2col(const double* x, int N, int C, int H, int W,
                        const double* w, int F, int kh, int kw, const double* b,
                        int sh, int sw, int ph, int pw, double* y);

/* Convolution backward.  Overwrites.
 * dw: F*C*kh*kw, db: F (NULL to skip), dx: N*C*H*W (NULL to skip: the data
 * layer's conv computes no input gradient).  S* may be NULL. */
int orc_conv_bwd(const double* dy, const double* x, const double* w, int N,
                 int C, int H, int W, int F, int kh, int kw, int sh, int sw,
                 int ph, int pw, double* dw, double* db, double* dx,
                 double* Sdw, double* Sdb, double* Sdx);

/* Pooling.  method 0 = MAX, 1 = AVE.
 * mask (MAX only, may be NULL): plane-local index h*W + w of the first
 * maximum in row-major window scan (strict >).  AVE divides by the window
 * size counted before clipping to the image (= in-bounds count when p = 0). */
int orc_pool_fwd(const double* x, int N, int C, int H, int W, int method,
                 int kh, int kw, int sh, int sw, int ph, int pw, double* y,
                 int32_t* mask);
/* dx overwritten: MAX routes dy[o] to mask[o]; AVE spreads dy/size. */
int orc_pool_bwd(const double* dy, const int32_t* mask, int N, int C, int H,
                 int W, int method, int kh, int kw, int sh, int sw, int ph,
                 int pw, double* dx);

/* The same pooling in Caffe's float arithmetic (float accumulators rounded
 * after every addition, one float division for AVE; SURVEY §8(c) c4-c6
 * bit-exact contract).  Inputs/outputs float. */
int orc_pool_fwd_f32(const float* x, int N, int C, int H, int W, int method,
                     int kh, int kw, int sh, int sw, int ph, int pw, float* y,
                     int32_t* mask);
int orc_pool_bwd_f32(const float* dy, const int32_t* mask, int N, int C, int H,
                     int W, int method, int kh, int kw, int sh, int sw, int ph,
                     int pw, float* dx);

/* InnerProduct (Listings 1-2).  w is [Nout, K]
 * (transpose_ = false).  y = x * w^T + b. */
int orc_ip_fwd(const double* x, int M, int K, const double* w, int Nout,
               const double* b, double* y, double* S);
/* dw = dy^T x, db = sum_m dy, dx = dy w  (gradient only; R7). */
int orc_ip_bwd(const double* dy, const double* x, const double* w, int M, int K,
               int Nout, double* dw, double* db, double* dx, double* Sdw,
               double* Sdb, double* Sdx);

/* (leaky) ReLU.  Backward uses the output sign, valid
 * for slope >= 0 with in-place storage (R8). */
void orc_relu_fwd(const double* x, long n, double slope, double* y);
void orc_relu_bwd(const double* dy, const double* y, long n, double slope,
                  double* dx);

/* Softmax with loss.  prob: M*D, loss: scalar
 * -(1/M) sum log(max(p_label, FLT_MIN)), pred: lowest index of the maximum
 * logit (may be NULL).  Returns -2 on a label outside [0, D). */
int orc_softmax_loss_fwd(const double* logits, const int32_t* labels, int M,
                         int D, double* prob, double* loss, int32_t* pred);
/* dx = loss_weight * (p - onehot) / M */
int orc_softmax_loss_bwd(const double* prob, const int32_t* labels, int M,
                         int D, double loss_weight, double* dx);

/* Caffe learning rate policies: 0 fixed, 1 inv. */
double orc_lr(int policy, double base_lr, double gamma, double power,
              long iter);

/* SGD with momentum + L2 decay, Caffe order, fp32 arithmetic,
 * no FMA.  g = diff*grad_scale; g = g + decay*w; v = mom*v + lr*g; w -= v. */
void orc_sgd_update_f32(float* w, const float* diff, float* v, long n,
                        float lr, float mom, float decay, float grad_scale);

/* Standalone SoftMax forward / backward and top-k accuracy
 * (ties by ascending class index: DESIGN.md R10). */
int orc_softmax_fwd(const double* x, int M, int D, double* p);
int orc_softmax_bwd(const double* p, const double* dy, int M, int D, double* dx);
int orc_accuracy(const double* x, const int32_t* labels, int M, int D, int k, int32_t* correct,
                 double* acc);

#ifdef __cplusplus
}
#endif
#endif
