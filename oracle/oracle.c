/*
 * oracle.c -- plain single-threaded CPU oracle (TEST INFRASTRUCTURE ONLY).
 * See oracle.h for the contract, citations and precision rules.
 *
 * Every function here is the textbook definition written out with loops in
 * ascending order; there is no blocking, fusion or reordering.  A reader can
 * check each against the paper / SPEC passage cited above it.
 *
 * Parity status: every function is pinned by tests/test_oracle_*.py
 * (torch fp64 library routines, brute force, finite differences, closed
 * forms, hand vectors in tests/golden/).  Nothing is "parity unpinned".
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* S:301  H_out = floor((H + 2p - k)/s) + 1 */
int orc_conv_out_size(int in, int k, int s, int p) {
  if (in <= 0 || k <= 0 || s <= 0 || p < 0) return -1;
  int num = in + 2 * p - k;
  if (num < 0) return -1;
  return num / s + 1;
}

/* DESIGN.md R4 (Caffe pooling): ceil((H + 2p - k)/s) + 1, then if p > 0 and
 * the last window would start in the bottom/right padding, drop it. */
int orc_pool_out_size(int in, int k, int s, int p) {
  if (in <= 0 || k <= 0 || s <= 0 || p < 0 || p >= k) return -1;
  int num = in + 2 * p - k;
  if (num < 0) return -1;
  int out = (num + s - 1) / s + 1;
  if (p > 0 && (out - 1) * s >= in + p) out--;
  return out;
}

/* P:122 "maps the input matrix into columns".
 * col[(c*kh + i)*kw + j][ho*Wo + wo] = x[c][ho*sh - ph + i][wo*sw - pw + j]
 * (0 outside the image). */
int orc_im2col(const double* x, int C, int H, int W, int kh, int kw, int sh,
               int sw, int ph, int pw, double* col) {
  int Ho = orc_conv_out_size(H, kh, sh, ph);
  int Wo = orc_conv_out_size(W, kw, sw, pw);
  if (Ho < 1 || Wo < 1 || C < 1) return -1;
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < kh; ++i)
      for (int j = 0; j < kw; ++j) {
        long row = ((long)c * kh + i) * kw + j;
        for (int ho = 0; ho < Ho; ++ho)
          for (int wo = 0; wo < Wo; ++wo) {
            int h = ho * sh - ph + i, w = wo * sw - pw + j;
            double v = 0.0;
            if (h >= 0 && h < H && w >= 0 && w < W)
              v = x[((long)c * H + h) * W + w];
            col[row * (Ho * Wo) + (long)ho * Wo + wo] = v;
          }
      }
  return 0;
}

/* P:139 "usage of col2im to map the gradients to the size of the input";
 * the adjoint of im2col -- every column entry is added back to the
 * pixel it was copied from; padding entries are dropped. */
int orc_col2im(const double* col, int C, int H, int W, int kh, int kw, int sh,
               int sw, int ph, int pw, double* x) {
  int Ho = orc_conv_out_size(H, kh, sh, ph);
  int Wo = orc_conv_out_size(W, kw, sw, pw);
  if (Ho < 1 || Wo < 1 || C < 1) return -1;
  memset(x, 0, sizeof(double) * (size_t)C * H * W);
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < kh; ++i)
      for (int j = 0; j < kw; ++j) {
        long row = ((long)c * kh + i) * kw + j;
        for (int ho = 0; ho < Ho; ++ho)
          for (int wo = 0; wo < Wo; ++wo) {
            int h = ho * sh - ph + i, w = wo * sw - pw + j;
            if (h >= 0 && h < H && w >= 0 && w < W)
              x[((long)c * H + h) * W + w] +=
                  col[row * (Ho * Wo) + (long)ho * Wo + wo];
          }
      }
  return 0;
}

/* The GEMM step of P:160 (caffe_cpu_gemm) / P:193 (phast::dot_product). */
void orc_gemm(int M, int N, int K, const double* A, const double* B,
              double* C) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += A[(long)m * K + k] * B[(long)k * N + n];
      C[(long)m * N + n] = acc;
    }
}

/* Plain definition of the 2-D convolution layer:
 * y[n,f,ho,wo] = sum_{c,i,j} w[f,c,i,j] * x[n,c,ho*sh-ph+i,wo*sw-pw+j] + b[f]
 * (cross-correlation, R1; bias after the sum, Listing 1). */
int orc_conv_fwd(const double* x, int N, int C, int H, int W, const double* w,
                 int F, int kh, int kw, const double* b, int sh, int sw, int ph,
                 int pw, double* y, double* S) {
  int Ho = orc_conv_out_size(H, kh, sh, ph);
  int Wo = orc_conv_out_size(W, kw, sw, pw);
  if (Ho < 1 || Wo < 1 || N < 0 || C < 1 || F < 1) return -1;
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f)
      for (int ho = 0; ho < Ho; ++ho)
        for (int wo = 0; wo < Wo; ++wo) {
          double acc = 0.0, s = 0.0;
          for (int c = 0; c < C; ++c)
            for (int i = 0; i < kh; ++i)
              for (int j = 0; j < kw; ++j) {
                int h = ho * sh - ph + i, ww = wo * sw - pw + j;
                if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
                double t = w[(((long)f * C + c) * kh + i) * kw + j] *
                           x[(((long)n * C + c) * H + h) * W + ww];
                acc += t;
                s += fabs(t);
              }
          if (b) {
            acc += b[f];
            s += fabs(b[f]);
          }
          long o = (((long)n * F + f) * Ho + ho) * Wo + wo;
          y[o] = acc;
          if (S) S[o] = s;
        }
  return 0;
}

/* The paper's algorithm (Fig. 3): im2col + gemm + bias rows
 * (matrixPlusVectorRows). */
int orc_conv_fwd_im2col(const double* x, int N, int C, int H, int W,
                        const double* w, int F, int kh, int kw, const double* b,
                        int sh, int sw, int ph, int pw, double* y) {
  int Ho = orc_conv_out_size(H, kh, sh, ph);
  int Wo = orc_conv_out_size(W, kw, sw, pw);
  if (Ho < 1 || Wo < 1 || C < 1 || F < 1) return -1;
  long K = (long)C * kh * kw, P = (long)Ho * Wo;
  double* col = (double*)malloc(sizeof(double) * K * P);
  if (!col) return -1;
  for (int n = 0; n < N; ++n) {
    orc_im2col(x + (long)n * C * H * W, C, H, W, kh, kw, sh, sw, ph, pw, col);
    double* yn = y + (long)n * F * P;
    orc_gemm(F, (int)P, (int)K, w, col, yn);
    if (b)
      for (int f = 0; f < F; ++f)
        for (long p = 0; p < P; ++p) yn[f * P + p] += b[f];
  }
  free(col);
  return 0;
}

/* Convolution backward, plain definitions:
 * dw[f,c,i,j] = sum_n sum_{ho,wo} dy[n,f,ho,wo] * x[n,c,ho*sh-ph+i, wo*sw-pw+j]
 * db[f]       = sum_n sum_{ho,wo} dy[n,f,ho,wo]
 * dx          = col2im(W^T dy), i.e.
 * dx[n,c,h,w] = sum over (f,i,j,ho,wo) with ho*sh-ph+i = h, wo*sw-pw+j = w
 *               of w[f,c,i,j] * dy[n,f,ho,wo]. */
int orc_conv_bwd(const double* dy, const double* x, const double* w, int N,
                 int C, int H, int W, int F, int kh, int kw, int sh, int sw,
                 int ph, int pw, double* dw, double* db, double* dx,
                 double* Sdw, double* Sdb, double* Sdx) {
  int Ho = orc_conv_out_size(H, kh, sh, ph);
  int Wo = orc_conv_out_size(W, kw, sw, pw);
  if (Ho < 1 || Wo < 1 || C < 1 || F < 1) return -1;
  for (int f = 0; f < F; ++f)
    for (int c = 0; c < C; ++c)
      for (int i = 0; i < kh; ++i)
        for (int j = 0; j < kw; ++j) {
          double acc = 0.0, s = 0.0;
          for (int n = 0; n < N; ++n)
            for (int ho = 0; ho < Ho; ++ho)
              for (int wo = 0; wo < Wo; ++wo) {
                int h = ho * sh - ph + i, ww = wo * sw - pw + j;
                if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
                double t = dy[(((long)n * F + f) * Ho + ho) * Wo + wo] *
                           x[(((long)n * C + c) * H + h) * W + ww];
                acc += t;
                s += fabs(t);
              }
          long o = (((long)f * C + c) * kh + i) * kw + j;
          dw[o] = acc;
          if (Sdw) Sdw[o] = s;
        }
  if (db)
    for (int f = 0; f < F; ++f) {
      double acc = 0.0, s = 0.0;
      for (int n = 0; n < N; ++n)
        for (int p = 0; p < Ho * Wo; ++p) {
          double t = dy[((long)n * F + f) * Ho * Wo + p];
          acc += t;
          s += fabs(t);
        }
      db[f] = acc;
      if (Sdb) Sdb[f] = s;
    }
  if (dx) {
    long nx = (long)N * C * H * W;
    memset(dx, 0, sizeof(double) * nx);
    if (Sdx) memset(Sdx, 0, sizeof(double) * nx);
    for (int n = 0; n < N; ++n)
      for (int c = 0; c < C; ++c)
        for (int f = 0; f < F; ++f)
          for (int i = 0; i < kh; ++i)
            for (int j = 0; j < kw; ++j)
              for (int ho = 0; ho < Ho; ++ho)
                for (int wo = 0; wo < Wo; ++wo) {
                  int h = ho * sh - ph + i, ww = wo * sw - pw + j;
                  if (h < 0 || h >= H || ww < 0 || ww >= W) continue;
                  double t = w[(((long)f * C + c) * kh + i) * kw + j] *
                             dy[(((long)n * F + f) * Ho + ho) * Wo + wo];
                  long o = (((long)n * C + c) * H + h) * W + ww;
                  dx[o] += t;
                  if (Sdx) Sdx[o] += fabs(t);
                }
  }
  return 0;
}

/* Pooling forward ("maximum ... or mean"; "we stored the origin
 * of each output value").  Window (Caffe, R4/R5):
 *   hs = ph_*s - p;  he = min(hs + k, H + p);  size = (he-hs)*(we-ws);
 *   hs = max(hs, 0); he = min(he, H).
 * MAX: first maximum in row-major scan, strict >; mask = h*W + w.
 * AVE: sum of in-window values / size. */
int orc_pool_fwd(const double* x, int N, int C, int H, int W, int method,
                 int kh, int kw, int sh, int sw, int ph, int pw, double* y,
                 int32_t* mask) {
  int Hp = orc_pool_out_size(H, kh, sh, ph);
  int Wp = orc_pool_out_size(W, kw, sw, pw);
  if (Hp < 1 || Wp < 1 || (method != 0 && method != 1)) return -1;
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      const double* xp = x + ((long)n * C + c) * H * W;
      for (int a = 0; a < Hp; ++a)
        for (int bq = 0; bq < Wp; ++bq) {
          int hs = a * sh - ph, ws = bq * sw - pw;
          int he = hs + kh < H + ph ? hs + kh : H + ph;
          int we = ws + kw < W + pw ? ws + kw : W + pw;
          int size = (he - hs) * (we - ws);
          if (hs < 0) hs = 0;
          if (ws < 0) ws = 0;
          if (he > H) he = H;
          if (we > W) we = W;
          long o = (((long)n * C + c) * Hp + a) * Wp + bq;
          if (method == 0) {
            double best = xp[(long)hs * W + ws];
            int arg = hs * W + ws;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w)
                if (xp[(long)h * W + w] > best) {
                  best = xp[(long)h * W + w];
                  arg = h * W + w;
                }
            y[o] = best;
            if (mask) mask[o] = arg;
          } else {
            double acc = 0.0;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w) acc += xp[(long)h * W + w];
            y[o] = acc / size;
          }
        }
    }
  return 0;
}

/* Pooling backward, overwrites dx.
 * MAX: dx[n,c,mask[o]] += dy[o] for outputs o in ascending order.
 * AVE: every in-window position of output o gains dy[o]/size. */
int orc_pool_bwd(const double* dy, const int32_t* mask, int N, int C, int H,
                 int W, int method, int kh, int kw, int sh, int sw, int ph,
                 int pw, double* dx) {
  int Hp = orc_pool_out_size(H, kh, sh, ph);
  int Wp = orc_pool_out_size(W, kw, sw, pw);
  if (Hp < 1 || Wp < 1 || (method != 0 && method != 1)) return -1;
  memset(dx, 0, sizeof(double) * (size_t)N * C * H * W);
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      double* dxp = dx + ((long)n * C + c) * H * W;
      for (int a = 0; a < Hp; ++a)
        for (int bq = 0; bq < Wp; ++bq) {
          long o = (((long)n * C + c) * Hp + a) * Wp + bq;
          if (method == 0) {
            int m = mask[o];
            if (m < 0 || m >= H * W) return -1;
            dxp[m] += dy[o];
          } else {
            int hs = a * sh - ph, ws = bq * sw - pw;
            int he = hs + kh < H + ph ? hs + kh : H + ph;
            int we = ws + kw < W + pw ? ws + kw : W + pw;
            int size = (he - hs) * (we - ws);
            if (hs < 0) hs = 0;
            if (ws < 0) ws = 0;
            if (he > H) he = H;
            if (we > W) we = W;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w) dxp[(long)h * W + w] += dy[o] / size;
          }
        }
    }
  return 0;
}

/* Pooling in Caffe's float arithmetic (SURVEY.md §8(c) implementation rule
 * "acc = float (Caffe-faithful)"; rows c4-c6 are a bit-exact contract).
 * Same windows, scan order and output order as orc_pool_fwd / orc_pool_bwd
 * (S:357-374); every sum is a float accumulator rounded after each
 * addition and the AVE quotient is one IEEE float division:
 *   fwd AVE:  acc = 0f; acc += x (h, w ascending); y = acc / (float)size
 *   fwd MAX:  identical to orc_pool_fwd (a max selects an input: no rounding)
 *   bwd MAX:  dx = 0f; for o ascending: dx[mask[o]] += dy[o]
 *   bwd AVE:  q = dy[o] / (float)size; every in-window position += q, o ascending
 * Inputs and outputs are float. */
int orc_pool_fwd_f32(const float* x, int N, int C, int H, int W, int method,
                     int kh, int kw, int sh, int sw, int ph, int pw, float* y,
                     int32_t* mask) {
  int Hp = orc_pool_out_size(H, kh, sh, ph);
  int Wp = orc_pool_out_size(W, kw, sw, pw);
  if (Hp < 1 || Wp < 1 || (method != 0 && method != 1)) return -1;
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      const float* xp = x + ((long)n * C + c) * H * W;
      for (int a = 0; a < Hp; ++a)
        for (int bq = 0; bq < Wp; ++bq) {
          int hs = a * sh - ph, ws = bq * sw - pw;
          int he = hs + kh < H + ph ? hs + kh : H + ph;
          int we = ws + kw < W + pw ? ws + kw : W + pw;
          int size = (he - hs) * (we - ws);
          if (hs < 0) hs = 0;
          if (ws < 0) ws = 0;
          if (he > H) he = H;
          if (we > W) we = W;
          long o = (((long)n * C + c) * Hp + a) * Wp + bq;
          if (method == 0) {
            float best = xp[(long)hs * W + ws];
            int arg = hs * W + ws;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w)
                if (xp[(long)h * W + w] > best) {
                  best = xp[(long)h * W + w];
                  arg = h * W + w;
                }
            y[o] = best;
            if (mask) mask[o] = arg;
          } else {
            float acc = 0.0f;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w) acc = acc + xp[(long)h * W + w];
            y[o] = acc / (float)size;
          }
        }
    }
  return 0;
}

int orc_pool_bwd_f32(const float* dy, const int32_t* mask, int N, int C, int H,
                     int W, int method, int kh, int kw, int sh, int sw, int ph,
                     int pw, float* dx) {
  int Hp = orc_pool_out_size(H, kh, sh, ph);
  int Wp = orc_pool_out_size(W, kw, sw, pw);
  if (Hp < 1 || Wp < 1 || (method != 0 && method != 1)) return -1;
  memset(dx, 0, sizeof(float) * (size_t)N * C * H * W);
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) {
      float* dxp = dx + ((long)n * C + c) * H * W;
      for (int a = 0; a < Hp; ++a)
        for (int bq = 0; bq < Wp; ++bq) {
          long o = (((long)n * C + c) * Hp + a) * Wp + bq;
          if (method == 0) {
            int m = mask[o];
            if (m < 0 || m >= H * W) return -1;
            dxp[m] = dxp[m] + dy[o];
          } else {
            int hs = a * sh - ph, ws = bq * sw - pw;
            int he = hs + kh < H + ph ? hs + kh : H + ph;
            int we = ws + kw < W + pw ? ws + kw : W + pw;
            int size = (he - hs) * (we - ws);
            if (hs < 0) hs = 0;
            if (ws < 0) ws = 0;
            if (he > H) he = H;
            if (we > W) we = W;
            const float q = dy[o] / (float)size;
            for (int h = hs; h < he; ++h)
              for (int w = ws; w < we; ++w) dxp[(long)h * W + w] = dxp[(long)h * W + w] + q;
          }
        }
    }
  return 0;
}

/* InnerProduct forward (Listing 1: gemm NoTrans x Trans, then the
 * bias row add).  y[m,o] = sum_k x[m,k] w[o,k] + b[o]. */
int orc_ip_fwd(const double* x, int M, int K, const double* w, int Nout,
               const double* b, double* y, double* S) {
  if (M < 0 || K < 1 || Nout < 1) return -1;
  for (int m = 0; m < M; ++m)
    for (int o = 0; o < Nout; ++o) {
      double acc = 0.0, s = 0.0;
      for (int k = 0; k < K; ++k) {
        double t = x[(long)m * K + k] * w[(long)o * K + k];
        acc += t;
        s += fabs(t);
      }
      if (b) {
        acc += b[o];
        s += fabs(b[o]);
      }
      y[(long)m * Nout + o] = acc;
      if (S) S[(long)m * Nout + o] = s;
    }
  return 0;
}

/* InnerProduct backward (read as gradient only, R7;
 * S:384-392):  dw[o,k] = sum_m dy[m,o] x[m,k];  db[o] = sum_m dy[m,o];
 * dx[m,k] = sum_o dy[m,o] w[o,k]. */
int orc_ip_bwd(const double* dy, const double* x, const double* w, int M, int K,
               int Nout, double* dw, double* db, double* dx, double* Sdw,
               double* Sdb, double* Sdx) {
  if (M < 0 || K < 1 || Nout < 1) return -1;
  for (int o = 0; o < Nout; ++o)
    for (int k = 0; k < K; ++k) {
      double acc = 0.0, s = 0.0;
      for (int m = 0; m < M; ++m) {
        double t = dy[(long)m * Nout + o] * x[(long)m * K + k];
        acc += t;
        s += fabs(t);
      }
      dw[(long)o * K + k] = acc;
      if (Sdw) Sdw[(long)o * K + k] = s;
    }
  if (db)
    for (int o = 0; o < Nout; ++o) {
      double acc = 0.0, s = 0.0;
      for (int m = 0; m < M; ++m) {
        acc += dy[(long)m * Nout + o];
        s += fabs(dy[(long)m * Nout + o]);
      }
      db[o] = acc;
      if (Sdb) Sdb[o] = s;
    }
  if (dx)
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) {
        double acc = 0.0, s = 0.0;
        for (int o = 0; o < Nout; ++o) {
          double t = dy[(long)m * Nout + o] * w[(long)o * K + k];
          acc += t;
          s += fabs(t);
        }
        dx[(long)m * K + k] = acc;
        if (Sdx) Sdx[(long)m * K + k] = s;
      }
  return 0;
}

/* P:107 leaky ReLU; y = x > 0 ? x : slope*x */
void orc_relu_fwd(const double* x, long n, double slope, double* y) {
  for (long i = 0; i < n; ++i) y[i] = x[i] > 0 ? x[i] : slope * x[i];
}

/* S:402-410 with the in-place reading (R8): the sign of the output
 * equals the sign of the input for slope >= 0. */
void orc_relu_bwd(const double* dy, const double* y, long n, double slope,
                  double* dx) {
  for (long i = 0; i < n; ++i) dx[i] = dy[i] * (y[i] > 0 ? 1.0 : slope);
}

/* P:109-110.  Per row: m = max x, e = exp(x - m), s = sum e
 * (ascending), p = e / s.  loss = -(1/M) sum_i log(max(p[i,y_i], FLT_MIN))
 * (R9).  pred = lowest index of the maximum logit (R10). */
int orc_softmax_loss_fwd(const double* logits, const int32_t* labels, int M,
                         int D, double* prob, double* loss, int32_t* pred) {
  if (M < 0 || D < 1) return -1;
  double total = 0.0;
  for (int i = 0; i < M; ++i) {
    const double* x = logits + (long)i * D;
    double* p = prob + (long)i * D;
    int y = labels[i];
    if (y < 0 || y >= D) return -2;
    double m = x[0];
    int arg = 0;
    for (int j = 1; j < D; ++j)
      if (x[j] > m) {
        m = x[j];
        arg = j;
      }
    double s = 0.0;
    for (int j = 0; j < D; ++j) {
      p[j] = exp(x[j] - m);
      s += p[j];
    }
    for (int j = 0; j < D; ++j) p[j] /= s;
    double py = p[y] > (double)FLT_MIN ? p[y] : (double)FLT_MIN;
    total += -log(py);
    if (pred) pred[i] = arg;
  }
  if (loss) *loss = M > 0 ? total / M : 0.0;
  return 0;
}

/* dx[i,j] = loss_weight * (p[i,j] - [j == y_i]) / M */
int orc_softmax_loss_bwd(const double* prob, const int32_t* labels, int M,
                         int D, double loss_weight, double* dx) {
  if (M < 0 || D < 1) return -1;
  for (int i = 0; i < M; ++i) {
    int y = labels[i];
    if (y < 0 || y >= D) return -2;
    for (int j = 0; j < D; ++j)
      dx[(long)i * D + j] =
          loss_weight * (prob[(long)i * D + j] - (j == y ? 1.0 : 0.0)) / M;
  }
  return 0;
}

/* Standalone SoftMax ("maps any set of numbers to probabilities that
 * will add up to 1").  Per row: m = max x, e = exp(x - m),
 * s = sum e (ascending), p = e / s. */
int orc_softmax_fwd(const double* x, int M, int D, double* p) {
  if (M < 0 || D < 1) return -1;
  for (int i = 0; i < M; ++i) {
    const double* xr = x + (long)i * D;
    double* pr = p + (long)i * D;
    double m = xr[0];
    for (int j = 1; j < D; ++j)
      if (xr[j] > m) m = xr[j];
    double s = 0.0;
    for (int j = 0; j < D; ++j) {
      pr[j] = exp(xr[j] - m);
      s += pr[j];
    }
    for (int j = 0; j < D; ++j) pr[j] /= s;
  }
  return 0;
}

/* SoftMax backward: per row dx[i] = p[i] (dy[i] - sum_j dy[j] p[j]),
 * the inner sum ascending in j. */
int orc_softmax_bwd(const double* p, const double* dy, int M, int D, double* dx) {
  if (M < 0 || D < 1) return -1;
  for (int i = 0; i < M; ++i) {
    const double* pr = p + (long)i * D;
    const double* gr = dy + (long)i * D;
    double dot = 0.0;
    for (int j = 0; j < D; ++j) dot += gr[j] * pr[j];
    for (int j = 0; j < D; ++j) dx[(long)i * D + j] = pr[j] * (gr[j] - dot);
  }
  return 0;
}

/* Accuracy ("calculates the accuracy of the network for a specific set
 * of inputs"): the fraction of rows whose label ranks among the
 * top k scores, ranking by descending score with ties broken by ascending
 * class index (R10): rank(y) = #{j : x_j > x_y or (x_j == x_y and
 * j < y)}; correct iff rank < k.  correct[i] (may be NULL) gets 0/1. */
int orc_accuracy(const double* x, const int32_t* labels, int M, int D, int k, int32_t* correct,
                 double* acc) {
  if (M < 0 || D < 1 || k < 1 || k > D) return -1;
  long hits = 0;
  for (int i = 0; i < M; ++i) {
    const double* xr = x + (long)i * D;
    int y = labels[i];
    if (y < 0 || y >= D) return -2;
    int rank = 0;
    for (int j = 0; j < D; ++j)
      if (xr[j] > xr[y] || (xr[j] == xr[y] && j < y)) ++rank;
    int ok = rank < k;
    if (correct) correct[i] = ok;
    hits += ok;
  }
  if (acc) *acc = M > 0 ? (double)hits / M : 0.0;
  return 0;
}

/* lr = base_lr * (1 + gamma*iter)^(-power) for inv, base_lr for fixed */
double orc_lr(int policy, double base_lr, double gamma, double power,
              long iter) {
  if (policy == 1) return base_lr * pow(1.0 + gamma * (double)iter, -power);
  return base_lr;
}

/* S:536-544 (Caffe SGD, R11/R12), one fp32 rounding per op:
 *   g = diff * grad_scale      (grad_scale = 1/G under data parallelism)
 *   g = g + decay * w
 *   v = mom * v + lr * g
 *   w = w - v                                                            */
void orc_sgd_update_f32(float* w, const float* diff, float* v, long n,
                        float lr, float mom, float decay, float grad_scale) {
  for (long i = 0; i < n; ++i) {
    float g = diff[i] * grad_scale;
    float dwd = decay * w[i];
    g = g + dwd;
    float mv = mom * v[i];
    float lg = lr * g;
    v[i] = mv + lg;
    w[i] = w[i] - v[i];
  }
}
