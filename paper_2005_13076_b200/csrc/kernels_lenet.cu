// kernels_lenet.cu -- fused SIMT fp32 kernels for the LeNet chain
// (conv1 5x5 1->20 on 28x28, pool 2x2/2, conv2 5x5 20->50, pool 2x2/2,
// ip1 800->500 + relu, ip2 500->10 + softmax-loss).
//
// Fusion: conv1+pool1 never stores the 24x24 conv output;
// ip2+softmax+loss+argmax+dlogits is one pass; ip2 backward also applies the
// relu1 derivative; conv1's weight gradient reads the pooled gradient and
// the pool mask directly (the unpooled 24x24 gradient is never stored).
// Max-pool origins are stored as uint8 window offsets.
#include <cfloat>
#include <cstdint>

#include "kernels.h"
#include "solver.cuh"

namespace pn {

// ------------------------------------------------------------ conv1 + pool1
// Items = (image, pooled position q) over the whole batch, split evenly over
// a grid of 2 blocks per SM (each block stages the <= 3 images its contiguous
// item range touches).  Block = 320 threads: warp w owns filters (2w, 2w+1)
// with their 25 weights held in registers as (w_2w, w_2w+1) pairs; lane l
// takes items l, l+32, ...  Per item the four conv values of the 2x2 pool
// window (25 MACs each, tap order i-major, bias added after the sum: S:297
// with P:136) are computed for both filters at once with packed fp32 FMAs
// (FFMA2 = fma.rn.f32x2: two independent round-to-nearest FMAs, the same
// arithmetic as scalar fmaf), the input patch streamed row by row from
// shared memory one row ahead.  Ties: first of (0,0),(0,1),(1,0),(1,1).
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void fma2(unsigned long long& d, float a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(pk2(a, a)), "l"(b));
}
__device__ __forceinline__ float lo32(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }

// the network input element i: the fp32 blob, or a byte normalised on load
// (NEXT #4: x = byte * scale - mean[pixel], two IEEE roundings, no FMA)
__device__ __forceinline__ float in_x(const float* x, const uint8_t* x8, float scale, const float* mean,
                                      long long i) {
  if (!x8) return __ldg(x + i);
  const float v = __fmul_rn((float)__ldg(x8 + i), scale);
  return mean ? __fsub_rn(v, __ldg(mean + i % 784)) : v;
}
// four consecutive values at base (a multiple of 4, pixel base % 784 = pix):
// one 16-B float or 4-B byte load, in_x's per-element normalisation
__device__ __forceinline__ float4 in_x4(const float* x, const uint8_t* x8, float scale, const float* mean,
                                       long long base, int pix) {
  if (!x8) return __ldg(reinterpret_cast<const float4*>(x + base));
  const uchar4 b = __ldg(reinterpret_cast<const uchar4*>(x8 + base));
  float4 v = make_float4(__fmul_rn((float)b.x, scale), __fmul_rn((float)b.y, scale), __fmul_rn((float)b.z, scale),
                         __fmul_rn((float)b.w, scale));
  if (mean) {
    const float4 m = __ldg(reinterpret_cast<const float4*>(mean + pix));
    v = make_float4(__fsub_rn(v.x, m.x), __fsub_rn(v.y, m.y), __fsub_rn(v.z, m.z), __fsub_rn(v.w, m.w));
  }
  return v;
}

constexpr int C1_MAXIMG = 4;  // images a block's item range can touch
constexpr int C1_PAIRS = C1_FPT / 2;    // filter pairs per thread (one FFMA2 lane pair each)
__global__ void __launch_bounds__(C1_THREADS, C1_MINB) lenet_conv1_pool1(const __grid_constant__ Conv1Pool1P p) {
  // everything read here (the batch, conv1's weights from the previous
  // step's SGD) is complete at launch and the predecessor (the TF32 weight
  // packing) touches none of it: run alongside it, wait only at the end
  // (pdl.cuh)
  __shared__ __align__(16) float xs[C1_MAXIMG][28 * 28];
  const int i0 = blockIdx.x * p.per_block, i1 = min(i0 + p.per_block, p.N * 144);
  if (i0 >= i1) {
    pdl_enter();
    return;
  }
  const int nlo = i0 / 144, nimg = (i1 - 1) / 144 - nlo + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f0 = C1_FPT * warp;  // this warp's filters f0 .. f0 + C1_FPT - 1
  {  // every load of the staging issued before the first store (one HBM round
     // trip); 4 values per load when the input is aligned (784 = 196 x 4)
    const bool vec = ((reinterpret_cast<uintptr_t>(p.x8 ? (const void*)p.x8 : (const void*)p.x) &
                       (p.x8 ? 3 : 15)) == 0);
    if (vec) {
      constexpr int PER4 = (C1_MAXIMG * 196 + C1_THREADS - 1) / C1_THREADS;
      float4 v[PER4];
#pragma unroll
      for (int k = 0; k < PER4; ++k) {
        const int i4 = threadIdx.x + C1_THREADS * k;
        v[k] = i4 < nimg * 196 ? in_x4(p.x, p.x8, p.x_scale, p.x_mean, (long long)nlo * 784 + 4 * i4, (4 * i4) % 784)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < PER4; ++k) {
        const int i4 = threadIdx.x + C1_THREADS * k;
        if (i4 < nimg * 196) reinterpret_cast<float4*>(&xs[0][0])[i4] = v[k];
      }
    } else {
      constexpr int PER = (C1_MAXIMG * 784 + C1_THREADS - 1) / C1_THREADS;
      float v[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = threadIdx.x + C1_THREADS * k;
        v[k] = i < nimg * 784 ? in_x(p.x, p.x8, p.x_scale, p.x_mean, (long long)nlo * 784 + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = threadIdx.x + C1_THREADS * k;
        if (i < nimg * 784) xs[i / 784][i % 784] = v[k];
      }
    }
  }
  unsigned long long wp[C1_PAIRS][25];
  float bias[C1_FPT];
#pragma unroll
  for (int g = 0; g < C1_PAIRS; ++g)
#pragma unroll
    for (int t = 0; t < 25; ++t)
      wp[g][t] = pk2(__ldg(p.w + (f0 + 2 * g) * 25 + t), __ldg(p.w + (f0 + 2 * g + 1) * 25 + t));
#pragma unroll
  for (int h = 0; h < C1_FPT; ++h) bias[h] = __ldg(p.b + f0 + h);
  __syncthreads();
#pragma unroll 1
  for (int it = i0 + lane; it < i1; it += 32) {
    const int n = it / 144, q = it - n * 144, im = n - nlo;
    const int ph = q / 12, pw = q - ph * 12;
    const float* xp = &xs[im][(2 * ph) * 28 + 2 * pw];
    unsigned long long acc[C1_PAIRS][2][2];
#pragma unroll
    for (int g = 0; g < C1_PAIRS; ++g) acc[g][0][0] = acc[g][0][1] = acc[g][1][0] = acc[g][1][1] = 0ull;
    float r0[6], r1[6], r2[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      r0[c] = xp[c];
      r1[c] = xp[28 + c];
    }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      if (i < 4) {
#pragma unroll
        for (int c = 0; c < 6; ++c) r2[c] = xp[(i + 2) * 28 + c];
      }
#pragma unroll
      for (int j = 0; j < 5; ++j)
#pragma unroll
        for (int g = 0; g < C1_PAIRS; ++g) {
          fma2(acc[g][0][0], r0[j], wp[g][i * 5 + j]);
          fma2(acc[g][0][1], r0[j + 1], wp[g][i * 5 + j]);
          fma2(acc[g][1][0], r1[j], wp[g][i * 5 + j]);
          fma2(acc[g][1][1], r1[j + 1], wp[g][i * 5 + j]);
        }
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        r0[c] = r1[c];
        r1[c] = r2[c];
      }
    }
    float v[C1_FPT];
#pragma unroll
    for (int h = 0; h < C1_FPT; ++h) {  // filter f0 + h (pair h / 2, lane pair half h % 2)
      const int g = h >> 1;
      const bool hi = h & 1;
      const float bb = bias[h];
      const float c00 = (hi ? hi32(acc[g][0][0]) : lo32(acc[g][0][0])) + bb;
      const float c01 = (hi ? hi32(acc[g][0][1]) : lo32(acc[g][0][1])) + bb;
      const float c10 = (hi ? hi32(acc[g][1][0]) : lo32(acc[g][1][0])) + bb;
      const float c11 = (hi ? hi32(acc[g][1][1]) : lo32(acc[g][1][1])) + bb;
      float best = c00;
      int off = 0;
      if (c01 > best) { best = c01; off = 1; }
      if (c10 > best) { best = c10; off = 2; }
      if (c11 > best) { best = c11; off = 3; }
      // TF32 plan: round to nearest, ties away (the conv2 operand rounding)
      v[h] = p.round_tf32 ? __uint_as_float((__float_as_uint(best) + 0x1000u) & 0xFFFFE000u) : best;
      const long long o = ((long long)n * 20 + f0 + h) * 144 + q;
      p.p1[o] = v[h];
      p.m1[o] = (uint8_t)off;
    }
    if (p.p1c) {  // [pair][cc][h][n][w][4 c]: this thread's channels are adjacent
      float* d = p.p1c + ((size_t)(n >> 1) * 1440 + ((f0 >> 2) * 12 + ph) * 24 + (n & 1) * 12 + pw) * 4 + (f0 & 3);
      if (C1_FPT == 4)
        *reinterpret_cast<float4*>(d) = make_float4(v[0], v[1], v[C1_FPT > 2 ? 2 : 0], v[C1_FPT > 2 ? 3 : 1]);
      else
        *reinterpret_cast<float2*>(d) = make_float2(v[0], v[1]);
    }
  }
  pdl_enter();
}

// ------------------------------------------------------------ conv2 + pool2
// Persistent: each CTA stages all conv2 weights (50x20x25, padded to 28 per
// (f,c)) once, then loops over groups of C2_IMGS images.  Thread = (image,
// filter group of 5, pooled position of 16): 20 accumulators (2x2 window x 5
// filters).  (kC2Imgs = 4, 640 threads, measured 56.5 -> 47.1 µs for this
// kernel alone but 356 -> 430 µs for the fp32 step: two images per CTA.)
constexpr int C2_IMGS = kC2Imgs;
constexpr int C2_THREADS = 160 * C2_IMGS;
__global__ void __launch_bounds__(C2_THREADS, 1) lenet_conv2_pool2_simt(
    const __grid_constant__ Conv2Pool2P p) {
  pdl_enter();
  extern __shared__ __align__(16) float smem[];
  float* ws = smem;                    // [50][20][28]
  float* xs = smem + 50 * 20 * 28;     // [2][20][144]
  __shared__ float bs[50];
  for (int i = threadIdx.x; i < 50 * 20 * 28; i += blockDim.x) {
    int fc = i / 28, t = i % 28;
    ws[i] = t < 25 ? __ldg(p.w + fc * 25 + t) : 0.f;
  }
  if (threadIdx.x < 50) bs[threadIdx.x] = __ldg(p.b + threadIdx.x);
  const int im = threadIdx.x / 160, r = threadIdx.x % 160, g = r / 16, q = r % 16;
  const int ph = q / 4, pw = q % 4;
  for (int n0 = blockIdx.x * C2_IMGS; n0 < p.N; n0 += gridDim.x * C2_IMGS) {
    __syncthreads();
    for (int i = threadIdx.x; i < C2_IMGS * 2880; i += blockDim.x) {
      int ii = i / 2880, e = i % 2880;
      xs[i] = (n0 + ii < p.N) ? __ldg(p.p1 + (long long)(n0 + ii) * 2880 + e) : 0.f;
    }
    __syncthreads();
    const int n = n0 + im;
    float acc[5][4];
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[t][u] = 0.f;
    const float* xi = xs + im * 2880;
#pragma unroll 1
    for (int c = 0; c < 20; ++c) {
      float patch[6][6];
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 6; ++b) patch[a][b] = xi[c * 144 + (2 * ph + a) * 12 + 2 * pw + b];
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const float4* wv4 = reinterpret_cast<const float4*>(ws + ((5 * g + t) * 20 + c) * 28);
        float wv[28];
#pragma unroll
        for (int z = 0; z < 7; ++z) {
          float4 v = wv4[z];
          wv[4 * z] = v.x; wv[4 * z + 1] = v.y; wv[4 * z + 2] = v.z; wv[4 * z + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
          for (int j = 0; j < 5; ++j) {
            const float w = wv[i * 5 + j];
            acc[t][0] = fmaf(w, patch[i][j], acc[t][0]);
            acc[t][1] = fmaf(w, patch[i][j + 1], acc[t][1]);
            acc[t][2] = fmaf(w, patch[i + 1][j], acc[t][2]);
            acc[t][3] = fmaf(w, patch[i + 1][j + 1], acc[t][3]);
          }
      }
    }
    if (n < p.N) {
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const int f = 5 * g + t;
        const float bb = bs[f];
        float best = acc[t][0] + bb;
        int off = 0;
        float v;
        v = acc[t][1] + bb; if (v > best) { best = v; off = 1; }
        v = acc[t][2] + bb; if (v > best) { best = v; off = 2; }
        v = acc[t][3] + bb; if (v > best) { best = v; off = 3; }
        const long long o = ((long long)n * 50 + f) * 16 + q;
        p.p2[o] = best;
        p.m2[o] = (uint8_t)off;
      }
    }
  }
}

// ------------------------------------------- conv2 backward, fp32 (SIMT)
// The fp32 plan's conv2 data and weight gradients, in
// fp32 FMA arithmetic (1e-5 class), specialised to LeNet's geometry (20 ->
// 50 channels, 5x5, 12x12 -> 8x8).  Register-blocked rows so every shared
// load feeds several FMAs (the generic gather kernels did one load per FMA).
//
// Data gradient (gather form of col2im(W^T G)):
//   dp1[n,c,y,x] = sum_f sum_{i,j} W2[f,c,i,j] G2[n,f,y-i,x-j]
// thread = (image of the pair, c, output row y): 12 accumulators; per (f, i)
// the G2 row y-i (8 values; rows outside 0..7 are a zero halo) and the 5
// taps W2[f,c,i,:] -> 40 FMAs.  Persistent blocks of 480 threads over image
// pairs; W2 staged once ([f][c][i][8], taps padded), G2 per pair.
constexpr int C2D_THREADS = 480;
__global__ void __launch_bounds__(C2D_THREADS, 1) lenet_conv2_dgrad_simt(const __grid_constant__ ConvBwdDataP p) {
  extern __shared__ __align__(16) float c2d_smem[];
  float* ws = c2d_smem;                    // [50 f][20 c][5 i][8]
  float* gs = c2d_smem + 50 * 20 * 5 * 8;  // [2][50 f][16 rows: 4 zero + 8 + 4 zero][8]
  pdl_enter();
  for (int u = threadIdx.x; u < 50 * 20 * 5 * 8; u += C2D_THREADS) {
    const int j = u & 7, fci = u >> 3;
    ws[u] = j < 5 ? __ldg(p.w + fci * 5 + j) : 0.f;
  }
  for (int u = threadIdx.x; u < 2 * 50 * 16 * 8; u += C2D_THREADS) gs[u] = 0.f;
  const int im = threadIdx.x / 240, t = threadIdx.x % 240, c = t / 12, y = t % 12;
  for (int n0 = blockIdx.x * 2; n0 < p.N; n0 += gridDim.x * 2) {
    __syncthreads();
    for (int u = threadIdx.x; u < 2 * 3200; u += C2D_THREADS) {
      const int ii = u / 3200, e = u % 3200, f = e >> 6, r = (e >> 3) & 7, x = e & 7;
      gs[((ii * 50 + f) * 16 + 4 + r) * 8 + x] = (n0 + ii < p.N) ? __ldg(p.dy + (size_t)(n0 + ii) * 3200 + e) : 0.f;
    }
    __syncthreads();
    float acc[12];
#pragma unroll
    for (int x = 0; x < 12; ++x) acc[x] = 0.f;
    const float* gb = gs + (im * 50 * 16 + 4 + y) * 8;  // row y - i of filter f: gb + (f*16 - i)*8
    const float* wb = ws + c * 40;                         // W2[f][c][i][:] at wb + f*800 + i*8
#pragma unroll 1
    for (int f = 0; f < 50; ++f) {
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const float4 g0 = *reinterpret_cast<const float4*>(gb + (f * 16 - i) * 8);
        const float4 g1 = *reinterpret_cast<const float4*>(gb + (f * 16 - i) * 8 + 4);
        const float4 w0 = *reinterpret_cast<const float4*>(wb + f * 800 + i * 8);
        const float w4 = wb[f * 800 + i * 8 + 4];
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float w[5] = {w0.x, w0.y, w0.z, w0.w, w4};
#pragma unroll
        for (int j = 0; j < 5; ++j)
#pragma unroll
          for (int x0 = 0; x0 < 8; ++x0) acc[x0 + j] = fmaf(w[j], g[x0], acc[x0 + j]);
      }
    }
    const int n = n0 + im;
    if (n < p.N) {
      float4* d = reinterpret_cast<float4*>(p.dx + ((size_t)n * 20 + c) * 144 + y * 12);
      d[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      d[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      d[2] = make_float4(acc[8], acc[9], acc[10], acc[11]);
    }
  }
}

// Weight gradient  dW2[f,c,i,j] = sum_n sum_{h,w<8} G2[n,f,h,w] p1[n,c,h+i,w+j],
// db2[f] = sum G2[n,f]: one block per split (contiguous images), 512
// threads: thread t < 500 takes filter f = t / 10 and the 10 (c, i) pairs
// q = t % 10 + 10 k; per image and row h, the G2 row (8 values) is loaded
// once and each pair's input row p1[c, h+i, 0..11] feeds 40 FMAs into the
// pair's 5 accumulators.  Split partials, reduced by the conv bucket.
constexpr int C2W_THREADS = 512;
__global__ void __launch_bounds__(C2W_THREADS, 1) lenet_conv2_wgrad_simt(const __grid_constant__ ConvBwdWeightP p) {
  __shared__ __align__(16) float gsm[3200];  // G2[n]: [50 f][8][8]
  __shared__ __align__(16) float psm[2880];  // p1[n]: [20 c][12][12]
  pdl_enter();
  const int s = blockIdx.x;
  const int n0 = (int)((long long)p.N * s / p.splits), n1 = (int)((long long)p.N * (s + 1) / p.splits);
  const int t = threadIdx.x, f = t / 10, q0 = t % 10;
  const bool active = t < 500;
  float acc[10][5], bacc = 0.f;
#pragma unroll
  for (int k = 0; k < 10; ++k)
#pragma unroll
    for (int j = 0; j < 5; ++j) acc[k][j] = 0.f;
  for (int n = n0; n < n1; ++n) {
    __syncthreads();
    for (int u = t; u < 3200 / 4; u += C2W_THREADS)
      reinterpret_cast<float4*>(gsm)[u] = __ldg(reinterpret_cast<const float4*>(p.dy + (size_t)n * 3200) + u);
    for (int u = t; u < 2880 / 4; u += C2W_THREADS)
      reinterpret_cast<float4*>(psm)[u] = __ldg(reinterpret_cast<const float4*>(p.x + (size_t)n * 2880) + u);
    __syncthreads();
    if (!active) continue;
#pragma unroll 1
    for (int h = 0; h < 8; ++h) {
      const float4 g0 = *reinterpret_cast<const float4*>(gsm + f * 64 + h * 8);
      const float4 g1 = *reinterpret_cast<const float4*>(gsm + f * 64 + h * 8 + 4);
      const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      if (q0 == 0) bacc += ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]));
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int q = q0 + 10 * k, c = q / 5, i = q % 5;
        const float4* pr = reinterpret_cast<const float4*>(psm + c * 144 + (h + i) * 12);
        const float4 a0 = pr[0], a1 = pr[1], a2 = pr[2];
        const float a[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
#pragma unroll
        for (int j = 0; j < 5; ++j)
#pragma unroll
          for (int w = 0; w < 8; ++w) acc[k][j] = fmaf(g[w], a[w + j], acc[k][j]);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int q = q0 + 10 * k, c = q / 5, i = q % 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) p.part_w[(size_t)s * p.pstride + ((f * 20 + c) * 5 + i) * 5 + j] = acc[k][j];
  }
  if (q0 == 0) p.part_b[(size_t)s * p.pstride + f] = bacc;
}

// ------------------------------------------------- ip2 + softmax-with-loss
// Warp per sample (4 per block): logits = a1 . W2^T + b2 (W2 staged in smem
// before the PDL wait: it was written by the previous step's SGD), then the
// stable softmax, per-row loss term, lowest-index argmax and the loss
// gradient dz = (p - onehot) * loss_weight / M.  The row's 125
// float4 of a1 are all loaded up front (4 per lane).
__global__ void __launch_bounds__(IP2_SPB * 32) lenet_ip2_loss(const __grid_constant__ Ip2LossP p) {
  constexpr int NT = IP2_SPB * 32, PER = (1250 + NT - 1) / NT;
  __shared__ __align__(16) float ws[10 * 500];
  __shared__ float bs[10];
  ST_BEGIN(ST_IP2);
  {  // W2 as 1250 float4, all loads of a thread in flight together
    float4 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = threadIdx.x + NT * k;
      v[k] = i < 1250 ? __ldg(reinterpret_cast<const float4*>(p.w) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = threadIdx.x + NT * k;
      if (i < 1250) reinterpret_cast<float4*>(ws)[i] = v[k];
    }
  }
  if (threadIdx.x < 10) bs[threadIdx.x] = __ldg(p.b + threadIdx.x);
  pdl_enter_k(ST_IP2);
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * IP2_SPB + (threadIdx.x >> 5);
  float4 av[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int q = lane + 32 * t;
    av[t] = (row < p.N && q < 125) ? __ldg(reinterpret_cast<const float4*>(p.a1 + (long long)row * 500) + q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  if (row >= p.N) return;
  float acc[10];
#pragma unroll
  for (int o = 0; o < 10; ++o) acc[o] = 0.f;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int q = lane + 32 * t;
    if (q < 125) {
#pragma unroll
      for (int o = 0; o < 10; ++o) {
        const float4 w = reinterpret_cast<const float4*>(ws + o * 500)[q];
        acc[o] = fmaf(av[t].x, w.x, fmaf(av[t].y, w.y, fmaf(av[t].z, w.z, fmaf(av[t].w, w.w, acc[o]))));
      }
    }
  }
#pragma unroll
  for (int o = 0; o < 10; ++o) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], s);
    acc[o] += bs[o];
  }
  float best = acc[0];
  int arg = 0;
#pragma unroll
  for (int o = 1; o < 10; ++o)
    if (acc[o] > best) { best = acc[o]; arg = o; }
  float e[10], s = 0.f;
#pragma unroll
  for (int o = 0; o < 10; ++o) { e[o] = expf(acc[o] - best); s += e[o]; }
  int y = p.labels[row];
  bool bad = (y < 0 || y >= 10);
  if (bad) { if (lane == 0) atomicOr(p.err, 1u); y = 0; }
  if (lane < 10) {
    float lo = 0.f, pv = 0.f;
#pragma unroll
    for (int o = 0; o < 10; ++o)
      if (o == lane) { lo = acc[o]; pv = __fdiv_rn(e[o], s); }
    p.logits[(long long)row * 10 + lane] = lo;
    p.prob[(long long)row * 10 + lane] = pv;
    p.dz[(long long)row * 10 + lane] = __fmul_rn(pv - (lane == y ? 1.f : 0.f), p.grad_scale);
  }
  if (lane == 0) {
    float ey = 0.f;
#pragma unroll
    for (int o = 0; o < 10; ++o)
      if (o == y) ey = e[o];
    p.row_loss[row] = -logf(fmaxf(__fdiv_rn(ey, s), FLT_MIN));
    p.pred[row] = arg;
  }
  ST_END(ST_IP2);
}

// ------------------------------------------------ ip2 backward + relu1 bwd
// grid (4 column chunks of 128, splits over samples).  Thread = column k:
// da1[m,k] = (a1[m,k] > 0) * sum_o dz[m,o] W2[o,k]   (S:387 + S:405)
// partial dW2[o,k] = sum_{m in split} dz[m,o] a1[m,k];  partial db2[o].
// Rows go in chunks of 16 with all 16 a1 loads issued together; the TF32
// transpose da1rT[k][m..m+15] is written as 4 x 16 B per thread.
#ifndef IP2B_EARLY_TRIGGER
#define IP2B_EARLY_TRIGGER 0
#endif
__global__ void __launch_bounds__(128) lenet_ip2_bwd(const __grid_constant__ Ip2BwdP p) {
  const int k = blockIdx.x * 128 + threadIdx.x;
  const int s = blockIdx.y;
  const int m0 = (int)((long long)p.N * s / p.splits), m1 = (int)((long long)p.N * (s + 1) / p.splits);
  __shared__ float dzs[16][10];
  ST_BEGIN(ST_IP2B);
  float w2[10], acc[10];
  const bool valid = k < 500;
#pragma unroll
  for (int o = 0; o < 10; ++o) {
    w2[o] = valid ? __ldg(p.w + o * 500 + k) : 0.f;
    acc[o] = 0.f;
  }
  // dz comes from ip2+loss: the immediate predecessor in a whole TF32 step
  // (its loss sum runs on the side branch), two launches back otherwise --
  // wait for it after the weight loads; let the successor launch at the end
  pdl_wait();
  if (IP2B_EARLY_TRIGGER) pdl_trigger();  // ip1's data gradient may launch now (it waits for this kernel)
  if (threadIdx.x == 0) st_mark(ST_IP2B, 1);
  float bacc = 0.f, b1acc = 0.f;
  for (int mb = m0; mb < m1; mb += 16) {
    const int cnt = min(16, m1 - mb);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * 10; i += 128) dzs[i / 10][i % 10] = p.dz[(long long)mb * 10 + i];
    float a[16];
#pragma unroll
    for (int mm = 0; mm < 16; ++mm) a[mm] = (valid && mm < cnt) ? p.a1[(long long)(mb + mm) * 500 + k] : 0.f;
    __syncthreads();
    float r[16];
#pragma unroll
    for (int mm = 0; mm < 16; ++mm) {
      r[mm] = 0.f;
      if (mm < cnt) {
        if (valid) {
          const int m = mb + mm;
          float g = 0.f;
#pragma unroll
          for (int o = 0; o < 10; ++o) {
            const float d = dzs[mm][o];
            g = fmaf(d, w2[o], g);
            acc[o] = fmaf(d, a[mm], acc[o]);
          }
          const float da = a[mm] > 0.f ? g : 0.f;
          p.da1[(long long)m * 500 + k] = da;
          if (p.da1r) {
            r[mm] = __uint_as_float((__float_as_uint(da) + 0x1000u) & 0xFFFFE000u);  // TF32 (RNA)
            p.da1r[(long long)m * 500 + k] = r[mm];
            b1acc += da;
          }
        }
        if (blockIdx.x == 0 && threadIdx.x < 10) bacc += dzs[mm][threadIdx.x];
      }
    }
    if (p.da1rT && valid) {
      float* dst = p.da1rT + (long long)k * p.npad + mb;
      if (cnt == 16 && (mb & 3) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<float4*>(dst)[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
      } else {
        for (int mm = 0; mm < cnt; ++mm) dst[mm] = r[mm];
      }
    }
  }
  if (valid) {
#pragma unroll
    for (int o = 0; o < 10; ++o) p.part_w[(long long)s * p.pstride + o * 500 + k] = acc[o];
    if (p.part_b1) p.part_b1[(long long)s * 500 + k] = b1acc;  // db1 = sum_m da1[m,k]
  }
  if (blockIdx.x == 0 && threadIdx.x < 10) p.part_b[(long long)s * p.pstride + threadIdx.x] = bacc;
  pdl_trigger();
  ST_END(ST_IP2B);
}

// dp2 [N, 50*16] + mask -> dense conv2 output gradient G2 [N,50,8,8]
// (max-pool backward: each gradient goes to its stored origin).
__global__ void lenet_unpool2(const __grid_constant__ Unpool2P p) {
  pdl_enter();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // over N*50*64
  if (idx >= (long long)p.N * 3200) return;
  const int pos = idx % 64;
  const long long nf = idx / 64;
  const int h = pos / 8, w = pos % 8;
  const int q = (h >> 1) * 4 + (w >> 1);
  const int off = (h & 1) * 2 + (w & 1);
  const long long o = nf * 16 + q;
  p.g2[idx] = (p.m2[o] == off) ? p.dp2[o] : 0.f;
}

// ---------------------------------------------------- conv1 weight gradient
// dW1[f,i,j] = sum_n sum_q dp1[n,f,q] * x[n, h_q + i, w_q + j] where (h_q,w_q)
// is the conv1 position pool1 routed gradient q to (P:220-222 composed with
// S:351); db1[f] = sum dp1.  grid = splits over images (<= CW_IMGS images
// per block), block = 320 threads (20 filters x 16 lanes), images staged in
// smem; the (gradient, origin) pairs of two images at a time in registers
// (18 global loads per thread in flight together).
// dp1 comes from conv2's data gradient two launches back (the predecessor,
// conv2's weight gradient, produces nothing read here): the kernel runs
// alongside it and waits only at the end (pdl.cuh).
#ifndef C1W_MINB
#define C1W_MINB 2
#endif
__global__ void __launch_bounds__(320, C1W_MINB) lenet_conv1_wgrad(const __grid_constant__ Conv1WgradP p) {
  __shared__ __align__(16) float xs[CW_IMGS][784];
  ST_BEGIN(ST_CONV1W);
  const int s = blockIdx.x;
  const int n0 = (int)((long long)p.N * s / p.splits), n1 = (int)((long long)p.N * (s + 1) / p.splits);
  const int cnt = min(CW_IMGS, n1 - n0);
  const int f = threadIdx.x / 16, l = threadIdx.x % 16;
  // images in chunks of CH: one chunk's (gradient, origin) pairs in registers
  constexpr int CH = CW_IMGS < 2 ? CW_IMGS : 2;
  float g[CH * 9];
  int off[CH * 9];
  auto load_chunk = [&](int c0) {
#pragma unroll
    for (int im = 0; im < CH; ++im)
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const bool v = c0 + im < cnt;
        const long long idx = ((long long)(n0 + (v ? c0 + im : 0)) * 20 + f) * 144 + l + 16 * t;
        g[im * 9 + t] = v ? __ldg(p.dp1 + idx) : 0.f;
        off[im * 9 + t] = v ? (int)__ldg(p.m1 + idx) : 0;
      }
  };
  load_chunk(0);
  {  // staging loads all in flight together (with the first chunk's); 4
     // values per load when the input is aligned (784 = 196 x 4)
    const bool vec = ((reinterpret_cast<uintptr_t>(p.x8 ? (const void*)p.x8 : (const void*)p.x) &
                       (p.x8 ? 3 : 15)) == 0);
    if (vec) {
      constexpr int PER4 = (CW_IMGS * 196 + 319) / 320;
      float4 v[PER4];
#pragma unroll
      for (int k = 0; k < PER4; ++k) {
        const int i4 = threadIdx.x + 320 * k;
        v[k] = i4 < cnt * 196 ? in_x4(p.x, p.x8, p.x_scale, p.x_mean, (long long)n0 * 784 + 4 * i4, (4 * i4) % 784)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < PER4; ++k) {
        const int i4 = threadIdx.x + 320 * k;
        if (i4 < cnt * 196) reinterpret_cast<float4*>(&xs[0][0])[i4] = v[k];  // xs rows of 784: contiguous
      }
    } else {
      constexpr int PER = (CW_IMGS * 784 + 319) / 320;
      float v[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = threadIdx.x + 320 * k;
        v[k] = i < cnt * 784 ? in_x(p.x, p.x8, p.x_scale, p.x_mean, (long long)n0 * 784 + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = threadIdx.x + 320 * k;
        if (i < cnt * 784) xs[i / 784][i % 784] = v[k];
      }
    }
  }
  __syncthreads();
  float acc[25], bacc = 0.f;
#pragma unroll
  for (int t = 0; t < 25; ++t) acc[t] = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < cnt; c0 += CH) {
    if (c0 > 0) load_chunk(c0);
#pragma unroll
    for (int im = 0; im < CH; ++im) {
      if (c0 + im >= cnt) break;
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const int q = l + 16 * t;
        const float gv = g[im * 9 + t];
        const int o = off[im * 9 + t];
        bacc += gv;
        const int h = 2 * (q / 12) + (o >> 1), w = 2 * (q % 12) + (o & 1);
        const float* xp = &xs[c0 + im][h * 28 + w];
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
          for (int j = 0; j < 5; ++j) acc[i * 5 + j] = fmaf(gv, xp[i * 28 + j], acc[i * 5 + j]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 25; ++t) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) bacc += __shfl_xor_sync(0xffffffffu, bacc, o);
  if (l == 0) {
#pragma unroll
    for (int t = 0; t < 25; ++t) p.part_w[(long long)s * p.pstride + f * 25 + t] = acc[t];
    p.part_b[(long long)s * p.pstride + f] = bacc;
  }
  if (threadIdx.x == 0) st_mark(ST_RED_CONV, 2);  // (step trace: the last block's partials written)
  // dp1 came from two launches back; the predecessor (conv2's weight
  // gradient) runs alongside: wait for it at the end (pdl.cuh)
  pdl_enter_k(ST_CONV1W);
  if (p.tail) {  // a single-GPU whole step: the conv bucket's solver (solver.cuh)
    // (updating conv2's outputs before the barrier -- its partials are final
    // after the PDL wait -- measured slower, statically or claimed: DESIGN §9)
    grid_barrier(p.bar, gridDim.x);
    if (threadIdx.x == 0) st_mark(ST_RED_CONV, 0);  // (step trace: the first block past the barrier)
    solver_tail(p.sp, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, 0, p.sp.nseg);
  }
  ST_END(ST_CONV1W);
}

PN_STEPTRACE_TU(st_set_lenet)

}  // namespace pn
