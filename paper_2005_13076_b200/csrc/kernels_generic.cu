// kernels_generic.cu -- one generic fp32 SIMT kernel per Caffe layer
// (PN_LAYERWISE plan, and the fallback for nets with no fused pattern).
//
// Each kernel implements the layer definition the paper's blocks compute
// for any geometry; reductions are in fixed order so reruns are
// bitwise identical (no atomics on data).  The fused LeNet kernels in
// kernels_lenet.cu / kernels_tc.cu are the performance path.
#include <cfloat>
#include <cstdint>

#include "kernels.h"
#include "reduce.cuh"
#include "sgd.cuh"

namespace pn {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in fixed order (warp trees, then warp 0 over warp partials).
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  float r = 0.f;
  if (w == 0) {
    r = (l < NT / 32) ? sm[l] : 0.f;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// ---------------------------------------------------------------- conv fwd
// each output is the inner product of a filter with one sliding
// window (cross-correlation, R1); bias after the sum (Listing 1).
// (32-bit index math throughout: every blob has fewer than 2^31 elements)
__global__ void conv_fwd_generic(const __grid_constant__ ConvFwdP p) {
  pdl_enter();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int HoWo = p.Ho * p.Wo;
  if (idx >= p.N * p.F * HoWo) return;
  const int nf = idx / HoWo, pos = idx - nf * HoWo, n = nf / p.F, f = nf - n * p.F;
  const int ho = pos / p.Wo, wo = pos - ho * p.Wo;
  const int h0 = ho * p.sh - p.ph, w0 = wo * p.sw - p.pw;
  const int i0 = max(0, -h0), i1 = min(p.kh, p.H - h0), j0 = max(0, -w0), j1 = min(p.kw, p.W - w0);
  const int G = max(1, p.G), Cg = p.C / G, c0 = (f / (p.F / G)) * Cg;  // filter f sees its group's channels
  float acc = 0.f;
  for (int cl = 0; cl < Cg; ++cl) {
    const float* xp = p.x + ((size_t)n * p.C + c0 + cl) * p.H * p.W + h0 * p.W + w0;
    const float* wp = p.w + ((size_t)f * Cg + cl) * p.kh * p.kw;
    for (int i = i0; i < i1; ++i)
      for (int j = j0; j < j1; ++j) acc = fmaf(__ldg(wp + i * p.kw + j), __ldg(xp + i * p.W + j), acc);
  }
  if (p.b) acc += __ldg(p.b + f);
  p.y[idx] = acc;
}

// col2im(W^T dy) evaluated per input element (gather form): the
// output positions whose window covers (h, w) are a rectangle [ho0, ho1] x
// [wo0, wo1] (no per-tap divisibility tests).
__global__ void conv_bwd_data_generic(const __grid_constant__ ConvBwdDataP p) {
  pdl_enter();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int HW = p.H * p.W, HoWo = p.Ho * p.Wo;
  if (idx >= p.N * p.C * HW) return;
  const int nc = idx / HW, r = idx - nc * HW, n = nc / p.C, c = nc - n * p.C;
  const int h = r / p.W, w = r - h * p.W;
  const int th = h + p.ph, tw = w + p.pw;  // ho*sh + i = th, wo*sw + j = tw
  const int ho0 = th >= p.kh ? (th - p.kh) / p.sh + 1 : 0, ho1 = min(th / p.sh, p.Ho - 1);
  const int wo0 = tw >= p.kw ? (tw - p.kw) / p.sw + 1 : 0, wo1 = min(tw / p.sw, p.Wo - 1);
  const int G = max(1, p.G), Cg = p.C / G, Fg = p.F / G, g = c / Cg;  // channel c feeds its group's filters
  float acc = 0.f;
  for (int f = g * Fg; f < (g + 1) * Fg; ++f) {
    const float* dyp = p.dy + ((size_t)n * p.F + f) * HoWo;
    const float* wp = p.w + ((size_t)f * Cg + (c - g * Cg)) * p.kh * p.kw;
    for (int ho = ho0; ho <= ho1; ++ho) {
      const int i = th - ho * p.sh;
      for (int wo = wo0; wo <= wo1; ++wo)
        acc = fmaf(__ldg(wp + i * p.kw + (tw - wo * p.sw)), __ldg(dyp + ho * p.Wo + wo), acc);
    }
  }
  p.dx[idx] = acc;
}

// dW[f,c,i,j] partial over the images of split s; 16 taps per pass.
// grid = (F*C, splits), block = 256.
__global__ void __launch_bounds__(256) conv_bwd_weight_generic(
    const __grid_constant__ ConvBwdWeightP p) {
  pdl_enter();
  __shared__ float sm[32];
  const int G = max(1, p.G), Cg = p.C / G;
  const int f = blockIdx.x / Cg, cl = blockIdx.x % Cg, c = (f / (p.F / G)) * Cg + cl, s = blockIdx.y;
  const int n0 = (int)((long long)p.N * s / p.splits);
  const int n1 = (int)((long long)p.N * (s + 1) / p.splits);
  const int P = p.Ho * p.Wo;
  const int cnt = (n1 - n0) * P;
  const int taps = p.kh * p.kw;
  for (int t0 = 0; t0 < taps; t0 += 16) {
    float acc[16];
    int ti[16], tj[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      acc[q] = 0.f;
      ti[q] = (t0 + q) / p.kw;
      tj[q] = (t0 + q) - ti[q] * p.kw;
    }
    float bacc = 0.f;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int nn = e / P, pos = e - nn * P, n = n0 + nn;
      const int ho = pos / p.Wo, wo = pos - ho * p.Wo;
      const float g = __ldg(p.dy + ((size_t)n * p.F + f) * P + pos);
      if (t0 == 0) bacc += g;
      const int h0 = ho * p.sh - p.ph, w0 = wo * p.sw - p.pw;
      const float* xp = p.x + ((size_t)n * p.C + c) * p.H * p.W;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int h = h0 + ti[q], w = w0 + tj[q];
        if (t0 + q < taps && (unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W)
          acc[q] = fmaf(g, __ldg(xp + h * p.W + w), acc[q]);
      }
    }
#pragma unroll 1
    for (int q = 0; q < 16; ++q) {
      if (t0 + q >= taps) break;
      float r = block_sum<256>(acc[q], sm);
      if (threadIdx.x == 0)
        p.part_w[(long long)s * p.pstride + ((long long)f * Cg + cl) * taps + t0 + q] = r;
    }
    if (t0 == 0 && cl == 0 && p.part_b) {
      float r = block_sum<256>(bacc, sm);
      if (threadIdx.x == 0) p.part_b[(long long)s * p.pstride + f] = r;
    }
  }
}

__global__ void reduce_partials(const __grid_constant__ ReduceP p) {
  pdl_enter();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  // independent loads issued in batches of 8, summed in ascending split order
  float acc = 0.f;
  int s = 0;
  for (; s + 8 <= p.splits; s += 8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcg(p.part + (long long)(s + q) * p.stride + i);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += v[q];
  }
  for (; s < p.splits; ++s) acc += __ldcg(p.part + (long long)s * p.stride + i);
  p.out[i] = acc;
}

// All split-partial reductions of a gradient bucket in one launch.  Block =
// 8 warps x 32 consecutive outputs of one segment: warp w sums splits
// w, w+8, ... (coalesced 128-B rows, ascending), then warp 0 adds the 8 warp
// sums in order -- a fixed order, so reruns are bitwise identical.
// p.total = number of 32-output blocks over all segments.
__global__ void __launch_bounds__(256) reduce_partials_multi(const __grid_constant__ ReduceMultiP p) {
  const int stk = p.late ? ST_RED_IP : ST_RED_CONV;
  ST_BEGIN(stk);
  if (!p.late) pdl_enter_k(stk);
  __shared__ float sm[8][33];
  int b = blockIdx.x, k = 0;
  while (k < p.nseg - 1 && b >= (p.seg[k].n + 31) / 32) b -= (p.seg[k++].n + 31) / 32;
  const ReduceP& s = p.seg[k];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = b * 32 + lane;
  sm[w][lane] = split_sum_warp(s, i, w);  // splits w, w+8, ... ascending (reduce.cuh)
  __syncthreads();
  if (w == 0 && i < s.n) {
    float r = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) r += sm[q][lane];
    s.out[reduce_out_index(s, i)] = r;
  }
  if (p.late) pdl_enter_k(stk);
  ST_END(stk);
}

// ---------------------------------------------------------------- stem
// The cifar10_quick stem (conv1 -> MAX pool1 -> in-place ReLU; Caffe
// pooling R4/R5) fused: the conv output never reaches HBM.
// Forward: block = (image n, 8 filters): the zero-padded image in shared
// memory, the 8 filters' conv plane computed there (thread = 4 adjacent
// outputs x 8 filters, fp32 FMAs in ascending (c, i, j)), + bias (one fp32
// add, as the conv epilogue), then the pooled max over each window in
// row-major scan order (strict >: the first maximum) with its origin, and
// the ReLU: y = max(best, 0).
constexpr int STEM_FG = STEM_FG_HOST;
__global__ void __launch_bounds__(256) stem_fwd(const __grid_constant__ StemP p) {
  pdl_enter();
  extern __shared__ __align__(16) float sm[];
  const int n = blockIdx.y, f0 = blockIdx.x * STEM_FG, tid = threadIdx.x;
  const int Hpad = p.H + 2 * p.ph, Wpad = p.W + 2 * p.pw, K = p.C * p.kh * p.kw;
  const int Wq = (p.Wo + 3) & ~3;                 // conv plane row pitch (4-output strips)
  float* xs = sm;                                 // [C][Hpad][Wpad + 8]
  const int xpitch = Wpad + 8;
  float* ws = xs + p.C * Hpad * xpitch;           // [K][8 filters]
  float* cs = ws + K * STEM_FG;                   // [8][Ho][Wq]
  for (int i = tid; i < p.C * Hpad * xpitch; i += 256) {
    const int c = i / (Hpad * xpitch), r = i - c * Hpad * xpitch, h = r / xpitch - p.ph, w = r % xpitch - p.pw;
    xs[i] = (h >= 0 && h < p.H && w >= 0 && w < p.W) ? __ldg(p.x + (((size_t)n * p.C + c) * p.H + h) * p.W + w) : 0.f;
  }
  for (int i = tid; i < K * STEM_FG; i += 256) {
    const int k = i / STEM_FG, f = f0 + i % STEM_FG;
    ws[i] = f < p.F ? __ldg(p.w + (size_t)f * K + k) : 0.f;
  }
  __syncthreads();
  const int strips = p.Ho * (Wq / 4);
  for (int s = tid; s < strips; s += 256) {
    const int h = s / (Wq / 4), w0 = (s % (Wq / 4)) * 4;
    float acc[4][STEM_FG];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int f = 0; f < STEM_FG; ++f) acc[q][f] = 0.f;
    for (int c = 0; c < p.C; ++c)
#pragma unroll 1
      for (int i = 0; i < 5; ++i) {  // (the stem's kernel is 5 x 5: net.cu checks)
        const float* xr = xs + (c * Hpad + h + i) * xpitch + w0;
        float xv[8];  // the 4 outputs' row segment: w0 .. w0 + 3 + (kw - 1), two 16-B loads
        {  // (w0 and the row pitch are multiples of 4 floats: conflict-free quarter-warp phases)
          const float4 a = *reinterpret_cast<const float4*>(xr), b = *reinterpret_cast<const float4*>(xr + 4);
          xv[0] = a.x, xv[1] = a.y, xv[2] = a.z, xv[3] = a.w, xv[4] = b.x, xv[5] = b.y, xv[6] = b.z, xv[7] = b.w;
        }
        const float* wr = ws + ((c * 5 + i) * 5) * STEM_FG;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const float4 wa = *reinterpret_cast<const float4*>(wr + j * STEM_FG);
          const float4 wb = *reinterpret_cast<const float4*>(wr + j * STEM_FG + 4);
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int f = 0; f < STEM_FG; ++f) acc[q][f] = fmaf(wv[f], xv[q + j], acc[q][f]);
        }
      }
#pragma unroll
    for (int f = 0; f < STEM_FG; ++f) {
      const float bb = (p.b && f0 + f < p.F) ? __ldg(p.b + f0 + f) : 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (w0 + q < p.Wo) cs[(f * p.Ho + h) * Wq + w0 + q] = p.b ? acc[q][f] + bb : acc[q][f];
    }
  }
  __syncthreads();
  const int HWp = p.Hp * p.Wp;
  for (int e = tid; e < STEM_FG * HWp; e += 256) {
    const int f = e / HWp, r = e - f * HWp;
    if (f0 + f >= p.F) continue;
    const int a = r / p.Wp, bq = r - a * p.Wp;
    int hs = a * p.ps - p.pp, wst = bq * p.ps - p.pp;
    int he = min(hs + p.pk, p.Ho + p.pp), we = min(wst + p.pk, p.Wo + p.pp);
    hs = max(hs, 0);
    wst = max(wst, 0);
    he = min(he, p.Ho);
    we = min(we, p.Wo);
    const float* cp = cs + f * p.Ho * Wq;
    float best = cp[hs * Wq + wst];
    int arg = hs * p.Wo + wst;
    for (int h = hs; h < he; ++h)
      for (int w = wst; w < we; ++w) {
        const float v = cp[h * Wq + w];
        if (v > best) {
          best = v;
          arg = h * p.Wo + w;
        }
      }
    const size_t idx = ((size_t)n * p.F + f0 + f) * HWp + r;
    p.y[idx] = p.relu ? fmaxf(best, 0.f) : best;
    p.mask[idx] = arg;
  }
}

// Weight gradient of the stem: dW[f,c,i,j] = sum_n sum_q g[n,f,q] x[n,c,
// h_q+i-ph, w_q+j-pw] with (h_q, w_q) the conv position pool q routed its
// gradient to (P:220-222 composed with the conv weight gradient; no
// conv-output gradient is formed: overlapping windows that pick the same
// position just add), db[f] = sum g.  g = dy: the ReLU's backward was applied
// by its consumer (the next conv's data gradient).  grid = image splits;
// lane = filter (F <= 32), warp w the pooled positions q = w, w+8, ...: at a
// given q the 32 filters' windows start at <= 9 distinct origins (dy, dx in
// the pooling window), whose words fall in distinct banks (dy * Wpad + dx
// mod 32), so every window load of the warp is one conflict-free wavefront
// (lanes on one q but different positions gathered the same rows in many
// banks).  The image's gradients and origins are staged per filter row
// (pitch HWp + 1: conflict-free column reads), the 75 accumulators of a
// thread cover its filter's taps; warps combined in order at the end.
constexpr int STEM_KMAX = kStemKmax;
__global__ void __launch_bounds__(256) stem_wgrad(const __grid_constant__ StemP p) {
  pdl_enter();
  extern __shared__ __align__(16) float sm[];
  const int s = blockIdx.x, f = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n0 = (int)((long long)p.N * s / p.splits), n1 = (int)((long long)p.N * (s + 1) / p.splits);
  const int Hpad = p.H + 2 * p.ph, Wpad = p.W + 2 * p.pw, HWp = p.Hp * p.Wp, GP = HWp + 1;
  const int XN = p.C * Hpad * Wpad;
  float* xs = sm;                              // [C][Hpad][Wpad] zero-padded image
  float* gs = xs + XN;                         // [32 f][GP] gradients
  int* os = reinterpret_cast<int*>(gs + 32 * GP);  // [32 f][GP] origins
  const bool live = f < p.F;
  float acc[STEM_KMAX], bacc = 0.f;
#pragma unroll
  for (int k = 0; k < STEM_KMAX; ++k) acc[k] = 0.f;
  for (int n = n0; n < n1; ++n) {
    __syncthreads();  // the previous image's reads are done
    for (int i = threadIdx.x; i < XN; i += 256) {
      const int c = i / (Hpad * Wpad), r = i - c * Hpad * Wpad, h = r / Wpad - p.ph, ww = r % Wpad - p.pw;
      xs[i] = (h >= 0 && h < p.H && ww >= 0 && ww < p.W) ? __ldg(p.x + (((size_t)n * p.C + c) * p.H + h) * p.W + ww) : 0.f;
    }
    for (int i = threadIdx.x; i < p.F * HWp; i += 256) {  // coalesced along q
      const int ff = i / HWp, q = i - ff * HWp;
      const size_t src = ((size_t)n * p.F + ff) * HWp + q;
      gs[ff * GP + q] = __ldg(p.dy + src);
      os[ff * GP + q] = __ldg(p.mask + src);
    }
    __syncthreads();
    if (!live) continue;
    for (int q = w; q < HWp; q += 8) {
      const float g = gs[f * GP + q];
      const int o = os[f * GP + q], h = o / p.Wo, ww = o - h * p.Wo;
      bacc += g;
      const float* xp = xs + h * Wpad + ww;  // conv output (h, w) reads padded rows h..h+kh-1
#pragma unroll
      for (int k = 0; k < STEM_KMAX; ++k) {
        const int c = k / 25, i = (k / 5) % 5, j = k % 5;  // (C kh kw = 3 x 5 x 5)
        acc[k] = fmaf(g, xp[(c * Hpad + i) * Wpad + j], acc[k]);
      }
    }
  }
  // combine the 8 warps in order: [w][f][76] over the staging area
  __syncthreads();
  float* red = sm;
  if (live) {
#pragma unroll
    for (int k = 0; k < STEM_KMAX; ++k) red[(w * 32 + f) * (STEM_KMAX + 1) + k] = acc[k];
    red[(w * 32 + f) * (STEM_KMAX + 1) + STEM_KMAX] = bacc;
  }
  __syncthreads();
  float* out = p.part_w + (size_t)s * p.pstride;
  for (int e = threadIdx.x; e < p.F * (STEM_KMAX + 1); e += 256) {
    const int ff = e / (STEM_KMAX + 1), k = e - ff * (STEM_KMAX + 1);
    float v = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += red[(ww * 32 + ff) * (STEM_KMAX + 1) + k];
    if (k < STEM_KMAX) out[ff * STEM_KMAX + k] = v;
    else if (p.b) out[p.F * STEM_KMAX + ff] = v;
  }
}

size_t stem_wgrad_smem(int C, int H, int W, int ph, int pw, int HWp) {
  const size_t a = (size_t)C * (H + 2 * ph) * (W + 2 * pw) + 2 * 32 * (size_t)(HWp + 1);
  const size_t r = (size_t)8 * 32 * (kStemKmax + 1);
  return 4 * (a > r ? a : r);
}

// ------------------------------------------------------------------ pooling
// P:215-220; Caffe window (R4-R6).  MAX keeps the first maximum of
// a row-major scan (strict >) and stores its plane-local index h*W+w.
// exact a / d for 0 <= a < 2^22, d >= 1: MUFU reciprocal estimate (relative
// error ~2^-22, so the estimate is within one) + one-step correction
__device__ __forceinline__ int qdiv(int a, int d) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)d));
  int q = __float2int_rz(((float)a + 0.5f) * r);
  q -= (q * d > a);
  q += ((q + 1) * d <= a);
  return q;
}

// grid (positions of a plane / 256, planes): one output per thread, no
// 64-bit or long integer division on the per-element path
__global__ void pool_fwd_generic(const __grid_constant__ PoolFwdP p) {
  // thread per output over all planes (grid-stride): small planes (cifar's
  // 8x8 / 4x4 outputs) keep every lane busy
  pdl_enter();
  const int HWp = p.Hp * p.Wp;
  const long long total = (long long)p.N * p.C * HWp;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long nc = idx / HWp;
    const int r = (int)(idx - nc * HWp);
    const int a = qdiv(r, p.Wp), b = r - a * p.Wp;
    int hs = a * p.sh - p.ph, ws = b * p.sw - p.pw;
    int he = min(hs + p.kh, p.H + p.ph), we = min(ws + p.kw, p.W + p.pw);
    const int size = (he - hs) * (we - ws);
    hs = max(hs, 0);
    ws = max(ws, 0);
    he = min(he, p.H);
    we = min(we, p.W);
    const float* xp = p.x + (size_t)nc * p.H * p.W;
    if (p.method == 0) {
      float best = __ldg(xp + hs * p.W + ws);
      int arg = hs * p.W + ws;
      for (int h = hs; h < he; ++h)
        for (int w = ws; w < we; ++w) {
          float v = __ldg(xp + h * p.W + w);
          if (v > best) {
            best = v;
            arg = h * p.W + w;
          }
        }
      p.y[idx] = p.relu ? fmaxf(best, 0.f) : best;
      p.mask[idx] = arg;
    } else {
      float acc = 0.f;
      for (int h = hs; h < he; ++h)
        for (int w = ws; w < we; ++w) acc += __ldg(xp + h * p.W + w);
      const float v = __fdiv_rn(acc, (float)size);
      p.y[idx] = p.relu ? fmaxf(v, 0.f) : v;
    }
  }
}

// each input sums the output gradients routed to it, in ascending
// output order (the oracle's scatter order) -- no atomics.  With relu_y the
// in-place ReLU below the pool is back-propagated here too: its
// backward stage disappears.
__global__ void pool_bwd_generic(const __grid_constant__ PoolBwdP p) {
  // thread per input over all planes (grid-stride); each gathers its windows
  // in ascending output order (bit-exact with pool_bwd_plane and the scatter
  // order)
  pdl_enter();
  const int HW = p.H * p.W, HWp = p.Hp * p.Wp;
  const long long total = (long long)p.N * p.C * HW;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long nc = idx / HW;
    const int r = (int)(idx - nc * HW);
    const int h = qdiv(r, p.W), w = r - h * p.W;
    const int a0 = (h + p.ph < p.kh) ? 0 : qdiv(h + p.ph - p.kh, p.sh) + 1;
    const int a1 = min(qdiv(h + p.ph, p.sh), p.Hp - 1);
    const int b0 = (w + p.pw < p.kw) ? 0 : qdiv(w + p.pw - p.kw, p.sw) + 1;
    const int b1 = min(qdiv(w + p.pw, p.sw), p.Wp - 1);
    const float* dyp = p.dy + (size_t)nc * HWp;
    const float y = p.relu_y ? __ldg(p.relu_y + idx) : 1.f;
    float acc = 0.f;
    if (p.method == 0) {
      const int32_t* mp = p.mask + (size_t)nc * HWp;
      for (int a = a0; a <= a1; ++a)
        for (int b = b0; b <= b1; ++b)
          if (__ldg(mp + a * p.Wp + b) == r) acc += __ldg(dyp + a * p.Wp + b);
    } else {
      for (int a = a0; a <= a1; ++a)
        for (int b = b0; b <= b1; ++b) {
          int hs = a * p.sh - p.ph, ws = b * p.sw - p.pw;
          int he = min(hs + p.kh, p.H + p.ph), we = min(ws + p.kw, p.W + p.pw);
          int size = (he - hs) * (we - ws);
          acc += __fdiv_rn(__ldg(dyp + a * p.Wp + b), (float)size);
        }
    }
    if (p.relu_y && !(y > 0.f)) acc = 0.f;
    p.dx[idx] = acc;
  }
}

// Pool backward, a block per group of P = max(1, 1024 / (H W)) consecutive
// (n, c) planes staged in shared memory (small planes -- cifar's 8 x 8 and
// 16 x 16 -- keep every thread busy): the planes' output gradients (divided
// by the window size for AVE, the same IEEE quotient the oracle adds) and
// max-pool origins are read once, coalesced; each input then gathers its
// <= ceil(k/s)^2 windows from shared memory in ascending output order
// (bit-exact with the scatter order).  Window ranges per input row /
// column come from two small tables.
template <int KH, int KW, int SH, int SW>  // window / stride fixed at compile time when nonzero
__global__ void __launch_bounds__(256) pool_bwd_plane(const __grid_constant__ PoolBwdP p) {
  const int kh = KH ? KH : p.kh, kw = KW ? KW : p.kw, sh = SH ? SH : p.sh, sw = SW ? SW : p.sw;
  extern __shared__ __align__(16) uint8_t psm[];
  const int HWp = p.Hp * p.Wp, HW = p.H * p.W, P = pool_bwd_planes(HW);
  float* d = reinterpret_cast<float*>(psm);
  int* m = reinterpret_cast<int*>(d + P * HWp);
  short2* arow = reinterpret_cast<short2*>(m + P * HWp);
  short2* bcol = arow + p.H;
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) {
    const int a0 = (h + p.ph < kh) ? 0 : (h + p.ph - kh) / sh + 1;
    arow[h] = make_short2((short)a0, (short)min((h + p.ph) / sh, p.Hp - 1));
  }
  for (int w = threadIdx.x; w < p.W; w += blockDim.x) {
    const int b0 = (w + p.pw < kw) ? 0 : (w + p.pw - kw) / sw + 1;
    bcol[w] = make_short2((short)b0, (short)min((w + p.pw) / sw, p.Wp - 1));
  }
  pdl_enter();
  const long long NC = (long long)p.N * p.C;
  for (long long nc0 = (long long)blockIdx.x * P; nc0 < NC; nc0 += (long long)gridDim.x * P) {
    const int np = (int)min((long long)P, NC - nc0);
    __syncthreads();
    const float* dyp = p.dy + (size_t)nc0 * HWp;
    for (int o = threadIdx.x; o < np * HWp; o += blockDim.x) {
      float v = __ldg(dyp + o);
      if (p.method == 0) {
        m[o] = __ldg(p.mask + (size_t)nc0 * HWp + o);
      } else {
        const int ol = o % HWp, a = ol / p.Wp, b = ol - a * p.Wp;
        const int hs = a * sh - p.ph, ws = b * sw - p.pw;
        const int he = min(hs + kh, p.H + p.ph), we = min(ws + kw, p.W + p.pw);
        v = __fdiv_rn(v, (float)((he - hs) * (we - ws)));
      }
      d[o] = v;
    }
    __syncthreads();
    // 4 inputs per thread per pass: their ReLU-output loads are issued together
    for (int r0 = threadIdx.x; r0 < np * HW; r0 += 4 * blockDim.x) {
      float y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * blockDim.x;
        y[u] = (p.relu_y && r < np * HW) ? __ldg(p.relu_y + (size_t)nc0 * HW + r) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * blockDim.x;
        if (r >= np * HW) break;
        const int pi = r / HW, rl = r - pi * HW, h = rl / p.W, w = rl - h * p.W;
        const int pb = pi * HWp;
        const short2 ar = arow[h], bc = bcol[w];
        float acc = 0.f;
        if (KH && SH && KW && SW) {  // at most ceil(k/s) windows per dimension: unrolled, ascending
          constexpr int NA = (KH + SH - 1) / (SH ? SH : 1), NB = (KW + SW - 1) / (SW ? SW : 1);
#pragma unroll
          for (int ia = 0; ia < NA; ++ia)
#pragma unroll
            for (int ib = 0; ib < NB; ++ib) {
              const int a = ar.x + ia, b = bc.x + ib;
              if (a <= ar.y && b <= bc.y) {
                const int o = pb + a * p.Wp + b;
                if (p.method != 0 || m[o] == rl) acc += d[o];
              }
            }
        } else {
          for (int a = ar.x; a <= ar.y; ++a)
            for (int b = bc.x; b <= bc.y; ++b) {
              const int o = pb + a * p.Wp + b;
              if (p.method != 0 || m[o] == rl) acc += d[o];
            }
        }
        if (!(y[u] > 0.f)) acc = 0.f;
        p.dx[(size_t)nc0 * HW + r] = acc;
      }
    }
  }
}
template __global__ void pool_bwd_plane<0, 0, 0, 0>(const __grid_constant__ PoolBwdP);
template __global__ void pool_bwd_plane<3, 3, 2, 2>(const __grid_constant__ PoolBwdP);
template __global__ void pool_bwd_plane<2, 2, 2, 2>(const __grid_constant__ PoolBwdP);

// ---------------------------------------------- test-phase blocks (NEXT #3)
// Standalone SoftMax forward: warp per row, stable
// (max-subtracted) exponentials, lane-strided sums.
__global__ void __launch_bounds__(256) softmax_fwd_generic(const __grid_constant__ SoftmaxP p) {
  pdl_enter();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= p.M) return;
  const float* x = p.x + (size_t)row * p.D;
  float* y = p.out + (size_t)row * p.D;
  float m = -INFINITY;
  for (int j = lane; j < p.D; j += 32) m = fmaxf(m, x[j]);
  for (int s = 16; s > 0; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
  float sum = 0.f;
  for (int j = lane; j < p.D; j += 32) sum += expf(x[j] - m);
  for (int s = 16; s > 0; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
  for (int j = lane; j < p.D; j += 32) y[j] = __fdiv_rn(expf(x[j] - m), sum);
}
// SoftMax backward: dx = y (dy - sum_j dy_j y_j)
__global__ void __launch_bounds__(256) softmax_bwd_generic(const __grid_constant__ SoftmaxP p) {
  pdl_enter();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= p.M) return;
  const float* dy = p.x + (size_t)row * p.D;
  const float* y = p.y + (size_t)row * p.D;
  float dot = 0.f;
  for (int j = lane; j < p.D; j += 32) dot = fmaf(dy[j], y[j], dot);
  for (int s = 16; s > 0; s >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s);
  for (int j = lane; j < p.D; j += 32) p.out[(size_t)row * p.D + j] = y[j] * (dy[j] - dot);
}
// Accuracy: warp per row; rank(y) = #{j : x_j > x_y or (x_j == x_y
// and j < y)} (ties by ascending class index, R10), exact compares
__global__ void __launch_bounds__(256) accuracy_generic(const __grid_constant__ AccuracyP p) {
  pdl_enter();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= p.M) return;
  int y = p.labels[row];
  if (y < 0 || y >= p.D) {
    if (lane == 0) atomicOr(p.err, 1u);
    y = 0;
  }
  const float* x = p.x + (size_t)row * p.D;
  const float sy = x[y];
  int rank = 0;
  for (int j0 = 0; j0 < p.D; j0 += 32) {
    const int j = j0 + lane;
    const bool better = j < p.D && (x[j] > sy || (x[j] == sy && j < y));
    rank += __popc(__ballot_sync(0xffffffffu, better));
  }
  if (lane == 0) p.flag[row] = rank < p.k ? 1 : 0;
}
__global__ void __launch_bounds__(256) accuracy_reduce(const __grid_constant__ AccReduceP p) {
  pdl_enter();
  __shared__ int sm[8];
  int c = 0;
  for (int i = threadIdx.x; i < p.M; i += 256) c += p.flag[i];
  for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += sm[w];
    p.out[0] = p.M > 0 ? __fdiv_rn((float)t, (float)p.M) : 0.f;  // = fp32(hits / M)
  }
}

// -------------------------------------------------------------------- GEMM
// 64x64 tile, BK 16, 256 threads x (4x4) outputs; arbitrary strides so one
// kernel serves ip fwd (x W^T), dgrad (dy W) and wgrad (dy^T x).
__global__ void __launch_bounds__(256) gemm_generic(const __grid_constant__ GemmP p) {
  pdl_enter();
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  float acc[4][4] = {};
  // K split over gridDim.z (splits > 1): slice z takes K tiles [nkt z / S, nkt (z+1) / S)
  const int S = max(1, p.splits), nkt = (p.K + 15) / 16;
  const int kt0 = (int)((long long)nkt * blockIdx.z / S), kt1 = (int)((long long)nkt * (blockIdx.z + 1) / S);
  for (int k0 = 16 * kt0; k0 < 16 * kt1; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + 256 * r;
      int mm, kk;
      if (p.sak == 1) { mm = e / 16; kk = e % 16; } else { kk = e / 64; mm = e % 64; }
      int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < p.M && gk < p.K) ? p.A[gm * p.sam + gk * p.sak] : 0.f;
      int nn;
      if (p.sbn == 1) { kk = e / 64; nn = e % 64; } else { nn = e / 16; kk = e % 16; }
      int gn = n0 + nn;
      gk = k0 + kk;
      Bs[kk][nn] = (gn < p.N && gk < p.K) ? p.B[gk * p.sbk + gn * p.sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  if (S > 1) {  // the raw partial of this slice (bias / ReLU in gemm_splitk_reduce)
    float* out = p.part + (size_t)blockIdx.z * p.M * p.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + tm + i;
      if (gm >= p.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (n0 + tn + j < p.N) out[(long long)gm * p.N + n0 + tn + j] = acc[i][j];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + tm + i;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tn + j;
      if (gn >= p.N) continue;
      float v = acc[i][j];
      if (p.bias) v += p.bias[gn];
      if (p.relu) v = v > 0.f ? v : 0.f;
      p.C[(long long)gm * p.N + gn] = v;
    }
  }
}

// Register-tiled fp32 GEMM (the fp32 plans' inner products: LeNet ip1 forward,
// weight and data gradients; the layerwise plans' IP layers).  C = A B as
// gemm_generic, with compile-time operand layouts: AT = 0 A(m,k) at
// A[m*sam + k] (K-contiguous), AT = 1 at A[k*sak + m] (M-contiguous); BT = 0
// B(k,n) at B[n*sbn + k], BT = 1 at B[k*sbk + n].  Tile 64 x 32, K step 16,
// 128 threads x (4 x 4) outputs (float4 shared loads), float4 global loads
// staged through registers one K step ahead into double-buffered shared
// tiles (one barrier per step).  fp32 FMAs in ascending k per output.
template <int AT, int BT>
__global__ void __launch_bounds__(128) gemm_tiled(const __grid_constant__ GemmP p) {
  pdl_enter();
  constexpr int BM = 64, BN = 32, BK = 16;
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tm = (tid >> 3) * 4, tn = (tid & 7) * 4;
  float4 ra[2], rb;
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + 128 * r;  // 256 float4 of A's 64 x 16 tile
      float v[4];
      if (AT == 0) {  // row m = e / 4, k = 4 (e % 4) .. +3
        const int m = m0 + (e >> 2), k = k0 + 4 * (e & 3);
        if (m < p.M && k + 3 < p.K) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p.A + (long long)m * p.sam + k));
          v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (m < p.M && k + q < p.K) ? __ldg(p.A + (long long)m * p.sam + k + q) : 0.f;
        }
      } else {  // k = e / 16, m = 4 (e % 16) .. +3
        const int k = k0 + (e >> 4), m = m0 + 4 * (e & 15);
        if (k < p.K && m + 3 < p.M) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p.A + (long long)k * p.sak + m));
          v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (k < p.K && m + q < p.M) ? __ldg(p.A + (long long)k * p.sak + m + q) : 0.f;
        }
      }
      ra[r] = make_float4(v[0], v[1], v[2], v[3]);
    }
    {
      const int e = tid;  // 128 float4 of B's 16 x 32 tile
      float v[4];
      if (BT == 0) {  // n = e / 4, k = 4 (e % 4) .. +3
        const int n = n0 + (e >> 2), k = k0 + 4 * (e & 3);
        if (n < p.N && k + 3 < p.K) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p.B + (long long)n * p.sbn + k));
          v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (n < p.N && k + q < p.K) ? __ldg(p.B + (long long)n * p.sbn + k + q) : 0.f;
        }
      } else {  // k = e / 8, n = 4 (e % 8) .. +3
        const int k = k0 + (e >> 3), n = n0 + 4 * (e & 7);
        if (k < p.K && n + 3 < p.N) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p.B + (long long)k * p.sbk + n));
          v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = (k < p.K && n + q < p.N) ? __ldg(p.B + (long long)k * p.sbk + n + q) : 0.f;
        }
      }
      rb = make_float4(v[0], v[1], v[2], v[3]);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + 128 * r;
      if (AT == 0) {
        const int m = e >> 2, k = 4 * (e & 3);
        As[buf][k][m] = ra[r].x, As[buf][k + 1][m] = ra[r].y, As[buf][k + 2][m] = ra[r].z, As[buf][k + 3][m] = ra[r].w;
      } else {
        *reinterpret_cast<float4*>(&As[buf][e >> 4][4 * (e & 15)]) = ra[r];
      }
    }
    if (BT == 0) {
      const int n = tid >> 2, k = 4 * (tid & 3);
      Bs[buf][k][n] = rb.x, Bs[buf][k + 1][n] = rb.y, Bs[buf][k + 2][n] = rb.z, Bs[buf][k + 3][n] = rb.w;
    } else {
      *reinterpret_cast<float4*>(&Bs[buf][tid >> 3][4 * (tid & 7)]) = rb;
    }
  };
  float acc[4][4] = {};
  const int nkt = (p.K + BK - 1) / BK, S = p.splits > 1 ? p.splits : 1;  // K steps of this z slice
  const int kt0 = (int)((long long)nkt * blockIdx.z / S), kt1 = (int)((long long)nkt * (blockIdx.z + 1) / S);
  load(kt0 * BK);
  store(0);
  __syncthreads();
#pragma unroll 1
  for (int kt = kt0; kt < kt1; ++kt) {
    const int buf = (kt - kt0) & 1;
    if (kt + 1 < kt1) load((kt + 1) * BK);  // next step's loads in flight under this step's FMAs
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][tm]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][tn]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < kt1) store(buf ^ 1);  // the other buffer: last read one step ago (barrier below)
    __syncthreads();
  }
  if (S > 1) {  // K split: the raw partial of this slice (bias / ReLU in gemm_splitk_reduce)
    float* out = p.part + (size_t)blockIdx.z * p.M * p.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + tm + i;
      if (gm >= p.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (n0 + tn + j < p.N) out[(long long)gm * p.N + n0 + tn + j] = acc[i][j];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + tm + i;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tn + j;
      if (gn >= p.N) continue;
      float v = acc[i][j];
      if (p.bias) v += p.bias[gn];
      if (p.relu) v = v > 0.f ? v : 0.f;
      p.C[(long long)gm * p.N + gn] = v;
    }
  }
}
// C = sum over the K slices (ascending z: a fixed order) + bias, ReLU
__global__ void __launch_bounds__(256) gemm_splitk_reduce(const __grid_constant__ GemmP p) {
  pdl_enter();
  const long long MN = (long long)p.M * p.N;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < MN; i += (long long)gridDim.x * 256) {
    float v = p.part[i];
    for (int z = 1; z < p.splits; ++z) v += p.part[z * MN + i];
    if (p.bias) v += p.bias[i % p.N];
    if (p.relu) v = v > 0.f ? v : 0.f;
    p.C[i] = v;
  }
}
template __global__ void gemm_tiled<0, 0>(const __grid_constant__ GemmP);
template __global__ void gemm_tiled<0, 1>(const __grid_constant__ GemmP);
template __global__ void gemm_tiled<1, 0>(const __grid_constant__ GemmP);
template __global__ void gemm_tiled<1, 1>(const __grid_constant__ GemmP);

// Inner-product forward for few outputs and long K (cifar10_quick ip1/ip2,
// the AlexNet trunk's classifier): block = 4 rows x 8 outputs, its
// 8 warps split K (float4 lanes), warp-shuffle then fixed-order cross-warp
// sums (deterministic), bias + optional ReLU in the epilogue.
__global__ void __launch_bounds__(256) ip_fwd_rows(const __grid_constant__ IpRowsP p) {
  pdl_enter();
  __shared__ float red[8][4][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 4, o0 = blockIdx.y * 8;
  const int k0 = (int)((long long)p.K * warp / 8), k1 = (int)((long long)p.K * (warp + 1) / 8);
  float acc[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[r][o] = 0.f;
  const bool vec = (p.K & 3) == 0 && (k0 & 3) == 0 && (k1 & 3) == 0;
  if (vec) {
    for (int k = k0 + 4 * lane; k < k1; k += 128) {
      float4 xv[4], wv[8];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        xv[r] = m0 + r < p.M ? __ldg(reinterpret_cast<const float4*>(p.x + (long long)(m0 + r) * p.K + k))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int o = 0; o < 8; ++o)
        wv[o] = o0 + o < p.Nout ? __ldg(reinterpret_cast<const float4*>(p.w + (long long)(o0 + o) * p.K + k))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int o = 0; o < 8; ++o)
          acc[r][o] = fmaf(xv[r].w, wv[o].w, fmaf(xv[r].z, wv[o].z, fmaf(xv[r].y, wv[o].y, fmaf(xv[r].x, wv[o].x, acc[r][o]))));
    }
  } else {
    for (int k = k0 + lane; k < k1; k += 32) {
      float xv[4], wv[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) xv[r] = m0 + r < p.M ? __ldg(p.x + (long long)(m0 + r) * p.K + k) : 0.f;
#pragma unroll
      for (int o = 0; o < 8; ++o) wv[o] = o0 + o < p.Nout ? __ldg(p.w + (long long)(o0 + o) * p.K + k) : 0.f;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[r][o] = fmaf(xv[r], wv[o], acc[r][o]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float v = acc[r][o];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
      if (lane == 0) red[warp][r][o] = v;
    }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int r = threadIdx.x >> 3, o = threadIdx.x & 7, m = m0 + r, oo = o0 + o;
    if (m < p.M && oo < p.Nout) {
      float v = red[0][r][o];
#pragma unroll
      for (int w = 1; w < 8; ++w) v += red[w][r][o];
      if (p.b) v += __ldg(p.b + oo);
      if (p.relu) v = v > 0.f ? v : 0.f;
      p.y[(long long)m * p.Nout + oo] = v;
    }
  }
}

// db[n] = sum_m dy[m, n] (InnerProduct bias gradient)
__global__ void __launch_bounds__(256) colsum_generic(const __grid_constant__ ColSumP p) {
  pdl_enter();
  __shared__ float sm[32];
  const int n = blockIdx.x;
  float acc = 0.f;
  for (int m = threadIdx.x; m < p.M; m += blockDim.x) acc += p.a[(long long)m * p.N + n];
  float r = block_sum<256>(acc, sm);
  if (threadIdx.x == 0) p.out[n] = r;
}

// --------------------------------------------------------------------- ReLU
// float4 lanes (blob pointers are 256-B aligned; the tail is scalar)
__global__ void relu_fwd_generic(const __grid_constant__ ReluP p) {
  pdl_enter();
  const long long n4 = p.n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = reinterpret_cast<const float4*>(p.x)[i];  // may alias out (in place)
    v.x = v.x > 0.f ? v.x : __fmul_rn(p.slope, v.x);
    v.y = v.y > 0.f ? v.y : __fmul_rn(p.slope, v.y);
    v.z = v.z > 0.f ? v.z : __fmul_rn(p.slope, v.z);
    v.w = v.w > 0.f ? v.w : __fmul_rn(p.slope, v.w);
    reinterpret_cast<float4*>(p.out)[i] = v;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n; i += stride) {
    float v = p.x[i];
    p.out[i] = v > 0.f ? v : __fmul_rn(p.slope, v);
  }
}
__global__ void relu_bwd_generic(const __grid_constant__ ReluP p) {
  pdl_enter();
  const long long n4 = p.n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 g = reinterpret_cast<const float4*>(p.x)[i];  // may alias out (in place)
    const float4 y = reinterpret_cast<const float4*>(p.y)[i];
    g.x = y.x > 0.f ? g.x : __fmul_rn(g.x, p.slope);
    g.y = y.y > 0.f ? g.y : __fmul_rn(g.y, p.slope);
    g.z = y.z > 0.f ? g.z : __fmul_rn(g.z, p.slope);
    g.w = y.w > 0.f ? g.w : __fmul_rn(g.w, p.slope);
    reinterpret_cast<float4*>(p.out)[i] = g;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n; i += stride) {
    float g = p.x[i];
    p.out[i] = p.y[i] > 0.f ? g : __fmul_rn(g, p.slope);
  }
}

// ----------------------------------------------------------- softmax + loss
// One warp per sample: stable softmax, per-row loss term, lowest-index
// argmax, and the loss gradient (p - onehot) * loss_weight / M.
__global__ void softmax_loss_generic(const __grid_constant__ SoftmaxLossP p) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= p.M) return;
  const float* x = p.logits + (long long)row * p.D;
  float best = -FLT_MAX;
  int arg = 0x7fffffff;
  for (int j = lane; j < p.D; j += 32) {
    float v = x[j];
    if (v > best || arg == 0x7fffffff) { best = v; arg = j; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  float s = 0.f;
  for (int j = lane; j < p.D; j += 32) s += expf(x[j] - best);
  s = warp_sum(s);
  int y = p.labels[row];
  bool bad = (y < 0 || y >= p.D);
  if (bad && lane == 0) atomicOr(p.err, 1u);
  if (bad) y = 0;
  for (int j = lane; j < p.D; j += 32) {
    float pj = __fdiv_rn(expf(x[j] - best), s);
    p.prob[(long long)row * p.D + j] = pj;
    p.dlogits[(long long)row * p.D + j] = __fmul_rn(pj - (j == y ? 1.f : 0.f), p.grad_scale);
  }
  if (lane == 0) {
    float py = __fdiv_rn(expf(x[y] - best), s);
    p.row_loss[row] = -logf(fmaxf(py, FLT_MIN));
    p.pred[row] = arg;
  }
}

// loss = (1/M) sum_i row_loss[i], fixed-order block reduction (one block)
__global__ void __launch_bounds__(256) loss_reduce(const __grid_constant__ LossReduceP p) {
  ST_BEGIN(ST_LOSSRED);
  pdl_enter_k(ST_LOSSRED);
  __shared__ float sm[32];
  float acc = 0.f;
  for (int i = threadIdx.x; i < p.M; i += blockDim.x) acc += p.row_loss[i];
  float r = block_sum<256>(acc, sm);
  if (threadIdx.x == 0) {
    r = r * p.inv_M;
    p.loss_blob[0] = r;
    if (p.loss_out) p.loss_out[0] = r;
  }
  ST_END(ST_LOSSRED);
}

// ------------------------------------------------------------ byte ingest
// NEXT #4 (S:604 MNIST bytes x 1/256; S:613 CIFAR bytes x 1/256 minus the
// per-pixel mean): one fp32 rounding per operation, no FMA (matches the
// harness's numpy float32 arithmetic bit for bit).  4 bytes per thread.
__global__ void ingest_u8(const __grid_constant__ IngestP p) {
  pdl_enter();
  const long long i4 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int q = 0; q < 4; ++q) {
    const long long i = 4 * i4 + q;
    if (i >= p.n) return;
    const float v = __fmul_rn((float)p.x8[i], p.scale);
    p.y[i] = p.mean ? __fsub_rn(v, p.mean[i % p.per]) : v;
  }
}

// ---------------------------------------------------------------------- SGD
// S:536-544 / DESIGN.md R11 (sgd.cuh)

__global__ void sgd_update_kernel(const __grid_constant__ SgdP p) {
  ST_BEGIN(ST_SGD);
  pdl_enter_k(ST_SGD);
  const float lr = p.lr_dev ? __ldg(p.lr_dev) : p.lr;
  long long i4 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long n4 = p.n / 4;
  for (; i4 < n4; i4 += (long long)gridDim.x * blockDim.x) {
    float4 w = reinterpret_cast<float4*>(p.w)[i4];
    float4 v = reinterpret_cast<float4*>(p.v)[i4];
    float4 g = reinterpret_cast<const float4*>(p.g)[i4];
    sgd_one(w.x, g.x, v.x, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.y, g.y, v.y, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.z, g.z, v.z, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.w, g.w, v.w, lr, p.mom, p.decay, p.gscale);
    reinterpret_cast<float4*>(p.w)[i4] = w;
    reinterpret_cast<float4*>(p.v)[i4] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x < (p.n & 3)) {
    long long i = n4 * 4 + threadIdx.x;
    float w = p.w[i], v = p.v[i];
    sgd_one(w, p.g[i], v, lr, p.mom, p.decay, p.gscale);
    p.w[i] = w;
    p.v[i] = v;
  }
  ST_END(ST_SGD);
}

// ----------------------------------------------------- mask representation
// The fused plan stores the max-pool origin as a uint8 offset inside the
// (clipped) window: (h - hs)*kw + (w - ws).  The ABI view is int32 h*W + w.
__global__ void mask_convert(const __grid_constant__ MaskExpandP p) {
  pdl_enter();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = (long long)p.N * p.C * p.Hp * p.Wp;
  if (idx >= total) return;
  int b = idx % p.Wp;
  int a = (idx / p.Wp) % p.Hp;
  int hs = max(a * p.sh - p.ph, 0), ws = max(b * p.sw - p.pw, 0);
  if (p.to32) {
    int off = p.m8[idx];
    p.m32[idx] = (hs + off / p.kw) * p.W + ws + off % p.kw;
  } else {
    int m = p.m32[idx];
    p.m8[idx] = (uint8_t)((m / p.W - hs) * p.kw + (m % p.W - ws));
  }
}

}  // namespace pn

namespace pn {
// TF32-rounded (nearest, ties away) copies of a blob for the tensor-core
// plan's operand buffers; used when a caller overwrites a blob (net_put_blob)
// so the internal operand copies stay consistent with it.
__global__ void tf32_copy(const __grid_constant__ Tf32CopyP p) {
  pdl_enter();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p.R * p.C) return;
  const int r = (int)(idx / p.C), c = (int)(idx % p.C);
  const float v = __uint_as_float((__float_as_uint(p.src[idx]) + 0x1000u) & 0xFFFFE000u);
  if (p.dst) p.dst[idx] = v;
  if (p.dstT) p.dstT[(long long)c * p.ldt + r] = v;
}
PN_STEPTRACE_TU(st_set_generic)

}  // namespace pn
