// tc_conv.cu -- general tcgen05 TF32 convolution for any geometry (kernel,
// stride, padding, channel counts): the tensor-core plan of nets other than
// the fused LeNet chain -- cifar10_quick and the
// AlexNet conv trunk (BASELINE config 5).
//
// It is the paper's own lowering: a convolution is im2col + GEMM,
// its data gradient GEMM + col2im, its weight gradient a GEMM against the
// column matrix.  Each column matrix is materialised once per use as a dense
// TF32 operand (rounded to nearest, ties away, when written) in the layout
// the tensor core reads K-major, and every contraction is one TMA-fed
// tcgen05 kernel (conv_gemm_tma):
//   forward      col[m][k] (im2col_rows)  x  Wf[f][k]          -> y (+b, ReLU)
//   weight grad  colT[k][m] (im2col_t, + ones row for the bias) x Gm[f][m]
//                (gather_gm)  -> split-m partials -> fixed-order sum
//   data grad    col2im(W^T G) = W' (*) G (stride-1 layers, W' the flipped,
//                channel-transposed filter, pad kh-1-p) as an implicit GEMM
//                that gathers G into shared memory (conv_tc_fwd): here the
//                materialised alternative (a K x M column gradient written
//                and re-read, then col2im) measured slower, since the
//                contraction over F is short and the column matrix large
// Round 2 adds, for stride-1 layers where they apply: the
// weight gradient as a tap GEMM over TMA-staged segments of column-shifted
// X copies (conv_wgrad_taps: no column matrix) and, in tc_plane.cu, the
// forward / data gradient over halo-staged channel planes.
// m = (n, ho, wo), k = (c, i, j), f = output channel.  B200 has the HBM (180
// GB, ~7 TB/s) to make the materialisation cheaper than gathering operands
// element by element into shared memory (which measured at 5-35% of the TF32
// pipe: the gather instruction rate, not the bytes, was the limit).
//
// conv_gemm_tma: one CTA = one 128 x BN output tile, 6 warps: warp 0 lane 0
// streams 32-wide K chunks of both operands by TMA (SWIZZLE_128B boxes,
// mbarrier complete_tx) into a STAGES-deep ring, warp 1 lane 0 issues 4 x
// tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) per chunk into a TMEM
// accumulator and commits each stage back, warps 2-5 read TMEM (32x32b, thread
// = tile row) and apply the epilogue.  TMA zero-fills reads outside the
// operand extents, so ragged M / K / F need no padding in memory.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "params.h"
#include "pdl.cuh"
#include "tc_conv.h"
#include "tc_ptx.cuh"

namespace pn {
namespace tcc {
using namespace pn::tc;

__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ int2 lds_i2(uint32_t addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_i2(uint32_t addr, int2 v) {
  asm volatile("st.shared.v2.s32 [%0], {%1,%2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}
// mbarrier arrive (count 1) from a gathering thread
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// K-table entry of patch element k = (c,i,j): {c*H*W + i*W + j, i<<16 | j};
// k >= K gets i = 0x7FFF (always out of bounds -> 0).
__device__ __forceinline__ int2 ktab_entry(int k, int K, int H, int W, int kh, int kw) {
  if (k >= K) return make_int2(0, 0x7FFF << 16);
  const int c = k / (kh * kw), r = k - c * (kh * kw), i = r / kw, j = r - i * kw;
  return make_int2(c * H * W + i * W + j, (i << 16) | j);
}

template <int BN>
struct FwdCfg {
  static constexpr int STAGES = BN > 128 ? 3 : 4;
  static constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int THREADS = 320;
};

// ============================================================ forward / dgrad
template <int BN>
__global__ void __launch_bounds__(320, 1) conv_tc_fwd(const __grid_constant__ ConvTcP p) {
  using Cfg = FwdCfg<BN>;
  constexpr int STAGES = Cfg::STAGES, A_BYTES = Cfg::A_BYTES, STAGE = Cfg::STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem), tab = sbase + STAGES * STAGE;
  const int m0 = blockIdx.x * 128, f0 = blockIdx.y * BN;
  const int HoWo = p.Ho * p.Wo, M = p.N * HoWo;
  // geometry-only setup before the dependency wait
  for (int k = tid; k < p.nk * 32; k += Cfg::THREADS) sts_i2(tab + 8 * k, ktab_entry(k, p.K, p.H, p.W, p.kh, p.kw));
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 256 + 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  pdl_enter();
  const int nk = p.nk;
  if (warp == 0) {
    if (lane == 0) {  // B producer: packed weights, one bulk copy per chunk
      const float* src = p.bpk + (size_t)f0 * 32;
      for (int c = 0; c < nk; ++c) {
        const int st = c % STAGES;
        if (c >= STAGES) mbar_wait(smem_u32(&empty[st]), ((c / STAGES) - 1) & 1);
        const uint32_t bar = smem_u32(&full[st]);
        mbar_expect_tx(bar, Cfg::B_BYTES);
        bulk_g2s(sbase + st * STAGE + A_BYTES, src + (size_t)c * p.Fpad * 32, Cfg::B_BYTES, bar);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = make_idesc(128, BN);
      for (int c = 0; c < nk; ++c) {
        const int st = c % STAGES;
        mbar_wait(smem_u32(&full[st]), (c / STAGES) & 1);
        tc_fence_after();
        const uint32_t As = sbase + st * STAGE, Bs = As + A_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_tf32(tbase, make_desc(As + k * 32), make_desc(Bs + k * 32), idesc, (c | k) != 0);
        mma_commit(smem_u32(&empty[st]));
      }
      mma_commit(smem_u32(&done));
    }
  } else {
    // ---- A gatherers: thread = (row r, half h of the chunk's 32 K values)
    const int g = tid - 64, r = g & 127, h = g >> 7;
    const int m = m0 + r;
    const bool live = m < M;
    int n = 0, pos = 0, ho = 0, wo = 0;
    if (live) {
      n = m / HoWo;
      pos = m - n * HoWo;
      ho = pos / p.Wo;
      wo = pos - ho * p.Wo;
    }
    const int hi0 = ho * p.sh - p.ph, wi0 = wo * p.sw - p.pw;
    const float* xb = p.x + (size_t)n * p.C * p.H * p.W;
    const int base = hi0 * p.W + wi0;
    for (int c = 0; c < nk; ++c) {
      const int st = c % STAGES;
      float v[16];
      const uint32_t t0 = tab + 8 * (c * 32 + h * 16);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int2 e = lds_i2(t0 + 8 * q);
        const int i = e.y >> 16, j = e.y & 0xFFFF;
        const bool ok = live && (unsigned)(hi0 + i) < (unsigned)p.H && (unsigned)(wi0 + j) < (unsigned)p.W;
        v[q] = ok ? __ldg(xb + (base + e.x)) : 0.f;
      }
      if (c >= STAGES) mbar_wait(smem_u32(&empty[st]), ((c / STAGES) - 1) & 1);
      const uint32_t As = sbase + st * STAGE;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        sts128(As + sw_off(r, h * 4 + q),
               f4(tf32f(v[4 * q]), tf32f(v[4 * q + 1]), tf32f(v[4 * q + 2]), tf32f(v[4 * q + 3])));
      fence_proxy_async();
      mbar_arrive(smem_u32(&full[st]));
    }
    // ---- epilogue: TMEM lane quadrant = warp % 4, column half = (warp-2)/4
    const int quad = warp & 3, half = (warp - 2) >> 2, er = quad * 32 + lane, em = m0 + er;
    mbar_wait(smem_u32(&done), 0);
    __syncwarp();
    tc_fence_after();
    const bool elive = em < M;
    int en = 0, epos = 0;
    if (elive) {
      en = em / HoWo;
      epos = em - en * HoWo;
    }
    float* yb = p.y + (size_t)en * p.F * HoWo + epos;
#pragma unroll 1
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + cc, v);
      if (elive && p.relu_y) {  // the ReLU outputs first: 16 independent loads, then the stores
        float y[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          y[t] = f0 + cc + t < p.F ? __ldg(p.relu_y + (yb - p.y) + (size_t)(f0 + cc + t) * HoWo) : 0.f;
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (!(y[t] > 0.f)) v[t] = 0.f;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int f = f0 + cc + t;
        if (elive && f < p.F) {
          float o = v[t];
          if (p.bias) o += __ldg(p.bias + f);
          if (p.relu) o = fmaxf(o, 0.f);
          yb[(size_t)f * HoWo] = o;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, Cfg::TMEM_COLS);
}

// ============================================================ weight packing
// B image of the forward (mode 0: B[f][k] = W[f][k]) or data-gradient
// (mode 1: B[c][(f,i',j')] = W[f][c][kh-1-i'][kw-1-j']) contraction: per
// 32-wide K chunk, rows x 128 B in the SWIZZLE_128B layout, TF32-rounded,
// zero-padded to `rows` rows and nk*32 K values.
__global__ void pack_conv_weights(const __grid_constant__ ConvPackP p) {
  pdl_enter();
  const long long total = (long long)p.rows * p.nk * 32;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    // e enumerates the image in memory order: chunk, row, 16-B slot, word
    const int w = (int)(e & 3), slot = (int)((e >> 2) & 7);
    const long long rc = e >> 5;
    const int row = (int)(rc % p.rows), chunk = (int)(rc / p.rows);
    const int kk = ((slot ^ (row & 7)) << 2) | w, k = chunk * 32 + kk;
    float v = 0.f;
    const int KK = p.kh * p.kw;
    if (p.mode == 0) {
      if (row < p.F && k < p.C * KK) v = p.w[(size_t)row * p.C * KK + k];
    } else {
      if (row < p.C && k < p.F * KK) {
        const int f = k / KK, r = k - f * KK, i = r / p.kw, j = r - i * p.kw;
        v = p.w[(((size_t)f * p.C + row) * p.kh + (p.kh - 1 - i)) * p.kw + (p.kw - 1 - j)];
      }
    }
    p.out[e] = tf32f(v);
  }
}

// ========================================== weight grad, materialised operands
// The paper's own lowering: the column matrix is written out once
// per step -- here transposed, colT[k][m] (k = (c,i,j) plus a ones row k = K
// for the bias, m = (n,ho,wo)), TF32-rounded -- together with the top
// gradient as Gm[f][m].  Both are then dense K-major operands (K = m) that
// TMA streams into the tensor core: D[k, f] = sum_m colT[k, m] Gm[f, m]
// (tile 128 k x BN f, m split over CTAs into fixed-order partials).  This
// replaces the per-element register gather of conv_tc_wgrad, whose gather
// instruction rate capped the weight gradient far below the tensor pipe.
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

// block = 1024 consecutive m (4 per thread: one 16-B store per k row) x a
// group of IM_KROWS k rows; (n, ho, wo) of the thread's 4 positions computed
// once, (c, i, j) from a shared table
constexpr int IM_KROWS = 16;
__global__ void __launch_bounds__(256) im2col_t(const __grid_constant__ Im2colTP p) {
  __shared__ int2 tab[IM_KROWS];
  const int HoWo = p.Ho * p.Wo, M = p.N * HoWo, KK = p.kh * p.kw;
  // grouped layers: Kb rows = G blocks of Kgb rows (the group's K patch rows,
  // then its ones row); row k of block g reads channel g*(C/G) + k/KK
  const int G = max(1, p.G), Kgb = G > 1 ? p.Kgb : p.Kb, Cg = p.C / G;
  const int kb0 = blockIdx.y * IM_KROWS;
  if (threadIdx.x < IM_KROWS) {
    const int k = kb0 + threadIdx.x, g = k / Kgb, kl = k - g * Kgb;
    int2 e = make_int2(0, 0x7FFF << 16);
    if (k < p.Kb && kl < p.K) {
      const int c = g * Cg + kl / KK, r = kl - (kl / KK) * KK, i = r / p.kw, j = r - i * p.kw;
      e = make_int2(c * p.H * p.W + i * p.W + j, (i << 16) | j);
    } else if (k < p.Kb && kl == p.K) {
      e = make_int2(0, -1);  // bias row: ones
    }
    tab[threadIdx.x] = e;
  }
  pdl_enter();
  __syncthreads();
  // unit-stride layers: 4 consecutive m per thread (one 16-B store per k
  // row); strided layers: one m per thread (their loads do not coalesce
  // across the 4 positions anyway)
  const int V = p.sw == 1 ? 4 : 1;
  const int m0 = V * (blockIdx.x * 256 + threadIdx.x);
  if (m0 >= M) return;
  int hi0[4], wi0[4], xoff[4];
  {
    int n = qdiv(m0, HoWo), pos = m0 - n * HoWo, ho = qdiv(pos, p.Wo), wo = pos - ho * p.Wo;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      hi0[u] = ho * p.sh - p.ph;
      wi0[u] = wo * p.sw - p.pw;
      xoff[u] = n * p.C * p.H * p.W + hi0[u] * p.W + wi0[u];
      if (m0 + u >= M || u >= V) hi0[u] = -(1 << 20);  // past the end / unused: zeros
      if (++wo == p.Wo) {
        wo = 0;
        if (++ho == p.Ho) {
          ho = 0;
          ++n;
        }
      }
    }
  }
  const int kend = min(IM_KROWS, p.Kb - kb0);
  const bool full4 = V == 4 && m0 + 4 <= M;
  float* dst = p.col + (size_t)kb0 * p.pitch + m0;
#pragma unroll 2
  for (int t = 0; t < kend; ++t) {
    const int2 e = tab[t];
    float v[4];
    if (e.y == -1) {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = 1.f;
    } else {
      const int i = e.y >> 16, j = e.y & 0xFFFF;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = (u < V && (unsigned)(hi0[u] + i) < (unsigned)p.H && (unsigned)(wi0[u] + j) < (unsigned)p.W)
                   ? tf32f(__ldg(p.x + (xoff[u] + e.x)))
                   : 0.f;
    }
    float* d = dst + (size_t)t * p.pitch;
    if (full4) {
      *reinterpret_cast<float4*>(d) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < V && m0 + u < M) d[u] = v[u];
    }
  }
}

// Gm[f][n*HoWo + pos] = tf32(G[n][f][pos]): flat over G (coalesced reads,
// contiguous runs of HoWo on the write side)
__global__ void __launch_bounds__(256) gather_gm(const __grid_constant__ GmP p) {
  pdl_enter();
  const int total = p.N * p.F * p.HoWo;
  for (int e = blockIdx.x * 256 + threadIdx.x; e < total; e += gridDim.x * 256) {
    const int nf = qdiv(e, p.HoWo), pos = e - nf * p.HoWo, n = qdiv(nf, p.F), f = nf - n * p.F;
    p.gm[(size_t)f * p.pitch + (size_t)n * p.HoWo + pos] = tf32f(__ldg(p.g + e));
  }
}

template <int BN>
struct TwCfg {
  static constexpr int STAGES = BN > 128 ? 4 : 6;
  static constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int THREADS = 192;
};

template <int BN>
static size_t tw_smem() {
  return 1024 + (size_t)TwCfg<BN>::STAGES * TwCfg<BN>::STAGE;
}

// C[r, c] = sum_k A[r, k] B[c, k] over a dense K-major TF32 pair fed by TMA
// (tile 128 x BN, 32-wide K chunks, K range split over blockIdx.z), with the
// epilogue of the conv contraction it serves:
//   EPI_WGRAD  r = k (patch element, K = bias row), c = f -> split partials
//   EPI_FWD    r = m (output position), c = f -> y NCHW + bias (+ ReLU)
enum { EPI_WGRAD = 0, EPI_FWD = 1 };
// Persistent warp-specialized TMA -> tcgen05 GEMM skeleton shared by the
// conv contractions: grid = min(tiles, SMs), CTA b takes tiles b, b+grid, ...
//   warp 0 lane 0  TMA producer, one K chunk per ring stage, running ahead
//                  across tile boundaries
//   warp 1 lane 0  MMA issuer into one of two TMEM accumulators (tile parity)
//   warps 2-5      epilogue of tile t from its accumulator while the MMA
//                  already fills the other one with tile t+1
// Op supplies num_tiles(), tile(t) -> Info (coordinates and chunk count nk),
// issue(info, chunk, A, B, bar) and epilogue(info, tmem, quad, lane).
template <int BN, class Op>
__global__ void __launch_bounds__(192, 1) tc_persistent(const __grid_constant__ typename Op::Params prm) {
  using Cfg = TwCfg<BN>;
  constexpr int STAGES = Cfg::STAGES, A_BYTES = Cfg::A_BYTES, STAGE = Cfg::STAGE, TC = Cfg::TMEM_COLS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  const Op op(prm);
  const int ntiles = op.num_tiles();
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&empty[st]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 128);
    }
    fence_barrier_init();
    op.prefetch();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 2 * TC);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  pdl_enter();
  if (tid == 0) {  // TMA producer (tile decoded once; per chunk only the box coordinates)
    int g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const typename Op::Info t = op.tile(tile);
      for (int c = 0; c < t.nk; ++c, ++g) {
        const int st = g % STAGES;
        if (g >= STAGES) mbar_wait(smem_u32(&empty[st]), ((g / STAGES) - 1) & 1);
        const uint32_t bar = smem_u32(&full[st]), As = sbase + st * STAGE;
        mbar_expect_tx(bar, STAGE);
        op.issue(t, c, As, As + A_BYTES, bar);
      }
    }
  } else if (tid == 32) {  // MMA issuer
    constexpr uint32_t idesc = make_idesc(128, BN);
    int g = 0, it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int buf = it & 1, nk = op.tile(tile).nk;
      if (it >= 2) mbar_wait(smem_u32(&tempty[buf]), ((it >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t acc = tbase + buf * TC;
      for (int c = 0; c < nk; ++c, ++g) {
        const int st = g % STAGES;
        mbar_wait(smem_u32(&full[st]), (g / STAGES) & 1);
        tc_fence_after();
        const uint32_t As = sbase + st * STAGE, Bs = As + A_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_tf32(acc, make_desc(As + k * 32), make_desc(Bs + k * 32), idesc, (c | k) != 0);
        mma_commit(smem_u32(&empty[st]));
      }
      mma_commit(smem_u32(&tfull[buf]));  // (every tile has nk >= 1: the accumulator is always written)
    }
  } else if (warp >= 2) {  // epilogue
    const int quad = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(smem_u32(&tfull[buf]), (it >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      op.template epilogue<BN>(op.tile(tile), tbase + buf * TC + ((uint32_t)(quad * 32) << 16), quad, lane);
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty[buf]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 2 * TC);
}

// C[r, c] = sum_k A[r, k] B[c, k] over a dense K-major TF32 pair by 2-D TMA
// (tile 128 x BN, 32-wide K chunks, K range split into `splits` tiles), with
// the epilogue of the conv contraction it serves:
//   EPI_WGRAD  r = k (patch element, K = bias row), c = f -> split partials
//   EPI_FWD    r = m (output position), c = f -> y NCHW + bias (+ ReLU)
template <int EPI>
struct GemmOp {
  using Params = ConvGemmP;
  const ConvGemmP& p;
  int rt, ct;  // row / column tiles
  __device__ GemmOp(const ConvGemmP& q) : p(q), rt((q.rows + 127) / 128), ct(q.ctiles) {}
  // rows / cols are per group; groups contract disjoint row and column ranges
  __device__ int num_tiles() const { return rt * ct * max(1, p.G) * p.splits; }
  __device__ void prefetch() const { prefetch_tmap(&p.ta); prefetch_tmap(&p.tb); }
  struct Info {
    int r0, q0, g, s, k0, nk;  // group-local row / column origin, group, split, first K element, chunks
  };
  __device__ Info tile(int t) const {
    Info i;
    i.r0 = (t % rt) * 128;
    t /= rt;
    i.q0 = (t % ct) * p.bn;
    t /= ct;
    const int G = max(1, p.G);
    i.g = t % G;
    i.s = t / G;
    const int nc = (p.Kdim + 31) / 32, c0 = (int)((long long)i.s * nc / p.splits),
              c1 = (int)((long long)(i.s + 1) * nc / p.splits);
    // an empty split range (never planned, but safe) reads one chunk past Kdim: zeros
    i.k0 = c1 > c0 ? c0 * 32 : nc * 32;
    i.nk = max(1, c1 - c0);
    return i;
  }
  __device__ void issue(const Info& t, int c, uint32_t As, uint32_t Bs, uint32_t bar) const {
    const int k = t.k0 + c * 32;
    tma2d(As, &p.ta, k, t.g * p.rows + t.r0, bar);
    tma2d(Bs, &p.tb, k, t.g * p.cols + t.q0, bar);
  }
  template <int BN>
  __device__ void epilogue(const Info& t, uint32_t taddr, int quad, int lane) const {
    const int r0 = t.r0, q0 = t.q0, s = t.s, t_g = t.g;
    const int r = r0 + quad * 32 + lane;
    int n = 0, pos = 0;
    if (EPI == EPI_FWD && r < p.rows) {
      n = r / p.HoWo;
      pos = r - n * p.HoWo;
    }
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
      float v[16];
      tmem_ld16(taddr + cc, v);
      if (r >= p.rows) continue;
      float bv[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) bv[t] = (EPI == EPI_FWD && p.bias && q0 + cc + t < p.cols) ? __ldg(p.bias + q0 + cc + t) : 0.f;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int q = q0 + cc + t;
        if (q >= p.cols) break;
        if (EPI == EPI_WGRAD) {  // r = group-local k, q = group-local f
          float* pb = p.out + (size_t)s * p.pstride;
          const int f = t_g * p.cols + q;
          if (r < p.K) pb[(size_t)f * p.K + r] = v[t];
          else if (p.has_bias) pb[(size_t)p.F * p.K + f] = v[t];  // r == K: the ones row
        } else {  // EPI_FWD: r = m, q = f
          float o = v[t] + bv[t];
          if (p.relu) o = fmaxf(o, 0.f);
          p.out[((size_t)n * p.F + q) * p.HoWo + pos] = o;
        }
      }
    }
  }
};

// col[m][k] = tf32(x[n, c, ho*s-p+i, wo*s-p+j]) (row m contiguous in k, pitch
// Kp): threads over k (a register-held (c,i,j) table entry each), a block
// walks IMR_ROWS rows m -- coalesced stores, neighbouring-j loads
constexpr int IMR_ROWS = 16;
__global__ void __launch_bounds__(256) im2col_rows(const __grid_constant__ Im2colTP p) {
  __shared__ int3 rowinfo[IMR_ROWS];  // per row m: input plane base offset, hi0, wi0
  const int k = blockIdx.x * 256 + threadIdx.x, KK = p.kh * p.kw;
  const int HoWo = p.Ho * p.Wo, M = p.N * HoWo, mb = blockIdx.y * IMR_ROWS;
  if (threadIdx.x < IMR_ROWS) {
    const int m = mb + threadIdx.x;
    int3 e = make_int3(0, -(1 << 20), 0);
    if (m < M) {
      const int n = m / HoWo, pos = m - n * HoWo, ho = pos / p.Wo, wo = pos - ho * p.Wo;
      e = make_int3(n * p.C * p.H * p.W, ho * p.sh - p.ph, wo * p.sw - p.pw);
    }
    rowinfo[threadIdx.x] = e;
  }
  int off = 0, i = 0, j = 0;
  if (k < p.K) {
    const int c = k / KK, r = k - c * KK;
    i = r / p.kw;
    j = r - i * p.kw;
    off = c * p.H * p.W + i * p.W + j;
  }
  pdl_enter();
  __syncthreads();
  if (k >= p.K) return;
  const int mend = min(IMR_ROWS, M - mb);
#pragma unroll 4
  for (int t = 0; t < mend; ++t) {
    const int3 e = rowinfo[t];
    const int hi = e.y + i, wi = e.z + j;
    const float v = ((unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W)
                        ? tf32f(__ldg(p.x + (size_t)e.x + (e.y * p.W + e.z) + off))
                        : 0.f;
    p.col[(size_t)(mb + t) * p.pitch + k] = v;
  }
}

// TF32 weight copy of the forward contraction: Wf[f][k] (row pitch Kp)
__global__ void pack_plain(const __grid_constant__ PackPlainP p) {
  pdl_enter();
  const int total = p.F * p.K;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int f = e / p.K, k = e - f * p.K;
    p.out[(size_t)f * p.pitch + k] = tf32f(__ldg(p.w + e));
  }
}

// ================================== stride-1 convolution as a TMA tap GEMM
// With the activation in NHWC (channels innermost, TF32, padded to Cp), the
// A tile of tap (i,j) for a block of 128 output positions is ONE 4-D TMA box
// {32 channels, BW, BH, BNI images} taken at the positions shifted by the tap;
// TMA zero-fills whatever falls outside the image -- the padding -- so the
// convolution is sum over taps and 32-channel chunks of [128 x 32] x [32 x BN]
// with no gather at all:
//   forward    y[n,f,oh,ow]  = sum_{i,j,c} x[n, oh+i-p, ow+j-p, c] W[f,c,i,j]
//   data grad  dx[n,c,h,w]   = sum_{i,j,f} G[n, h-i+p, w-j+p, f] W[f,c,i,j]
// (the same loop with the tap offset negated: s = +1 / -1).  B_t = per-tap
// weight matrix [out channels][in channels] (pack_taps).  Every stride, pitch
// is a multiple of 16 B because Cp is -- unlike NCHW rows of 27 or 13 floats,
// which TMA cannot address.
__device__ __forceinline__ void tma4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                      uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

struct TapOp {
  using Params = ConvTapP;
  const ConvTapP& p;
  int ti;  // position tiles
  __device__ TapOp(const ConvTapP& q) : p(q), ti(q.tiles_w * q.tiles_h * ((q.N + q.bni - 1) / q.bni)) {}
  // tiles: position tile x output-channel tile (ctiles per group) x group
  __device__ int num_tiles() const { return ti * p.ctiles * max(1, p.G); }
  __device__ void prefetch() const { prefetch_tmap(&p.ta); prefetch_tmap(&p.tb); }
  struct Info {
    int n0, oh0, ow0, q0, qend, cbase, nkc, nk;
  };
  __device__ Info tile(int tile) const {
    Info i;
    const int G = max(1, p.G), qt = tile / ti, g = qt / p.ctiles;
    i.q0 = g * p.fg + (qt - g * p.ctiles) * p.bn;  // output channels [q0, qend) of group g
    i.qend = min(p.F, (g + 1) * p.fg);
    i.cbase = g * p.cpg;                              // the group's input-channel slots
    int t = tile % ti;
    i.ow0 = (t % p.tiles_w) * p.bw;
    t /= p.tiles_w;
    i.oh0 = (t % p.tiles_h) * p.bh;
    i.n0 = (t / p.tiles_h) * p.bni;
    i.nkc = (p.cpg + 31) / 32;
    i.nk = p.kh * p.kw * i.nkc;
    (void)G;
    return i;
  }
  __device__ void issue(const Info& t, int c, uint32_t As, uint32_t Bs, uint32_t bar) const {
    const int tap = c / t.nkc, kc = c - tap * t.nkc, i = tap / p.kw, j = tap - i * p.kw;
    tma4d(As, &p.ta, t.cbase + kc * 32, t.ow0 + p.sgn * (j - p.pw), t.oh0 + p.sgn * (i - p.ph), t.n0, bar);
    tma3d(Bs, &p.tb, kc * 32, t.q0, tap, bar);
  }
  template <int BN>
  __device__ void epilogue(const Info& t, uint32_t taddr, int quad, int lane) const {
    const int n0 = t.n0, oh0 = t.oh0, ow0 = t.ow0, q0 = t.q0, qend = t.qend;
    const int r = quad * 32 + lane;
    const int bw = r % p.bw, rr = r / p.bw, bh = rr % p.bh, bi = rr / p.bh;
    const int n = n0 + bi, oh = oh0 + bh, ow = ow0 + bw;
    const bool live = n < p.N && oh < p.Ho && ow < p.Wo;
    const size_t HoWo = (size_t)p.Ho * p.Wo, base = (size_t)n * p.F * HoWo + (size_t)oh * p.Wo + ow;
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
      float v[16];
      tmem_ld16(taddr + cc, v);
      if (!live) continue;
      if (p.relu_y) {  // the ReLU outputs first: 16 independent loads, then the stores
        float y[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          y[u] = q0 + cc + u < qend ? __ldg(p.relu_y + base + (size_t)(q0 + cc + u) * HoWo) : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (!(y[u] > 0.f)) v[u] = 0.f;
      }
      float bv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) bv[u] = (p.bias && q0 + cc + u < qend) ? __ldg(p.bias + q0 + cc + u) : 0.f;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + cc + u;
        if (q >= qend) break;  // (columns past the group's channels belong to the next group's tile)
        float o = v[u] + bv[u];
        if (p.relu) o = fmaxf(o, 0.f);
        p.out[base + (size_t)q * HoWo] = o;
      }
    }
  }
};

// NCHW -> NHWC (channels padded to cp with zeros), TF32: 32 x 32 smem transposes
// Grouped layers (G > 1): group g's channels occupy slots [g*cpg, g*cpg + C/G)
// of the padded channel dimension (cpg a multiple of 32, the rest zeros), so
// no 32-channel chunk of one group reaches into the next.
__global__ void __launch_bounds__(256) to_nhwc(const __grid_constant__ NhwcP p) {
  __shared__ float t[32][33];
  pdl_enter();
  const int n = blockIdx.z, s0 = blockIdx.x * 32, c0 = blockIdx.y * 32, HW = p.H * p.W;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int G = max(1, p.G), Cg = p.C / G, cpg = G > 1 ? p.cpg : p.cp;
  for (int y = ty; y < 32; y += 8) {
    const int slot = c0 + y, g = slot / cpg, cl = slot - g * cpg, sp = s0 + tx;
    const int c = g * Cg + cl;
    t[y][tx] = (g < G && cl < Cg && sp < HW) ? tf32f(__ldg(p.x + ((size_t)n * p.C + c) * HW + sp)) : 0.f;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int sp = s0 + y, c = c0 + tx;
    if (sp < HW && c < p.cp) p.out[((size_t)n * HW + sp) * p.cp + c] = t[tx][y];
  }
}

// per-tap weight matrices, TF32: mode 0 (forward) out[t][f][c] = W[f][c][t],
// mode 1 (data gradient) out[t][c][f] = W[f][c][t]; inner dimension padded to
// ip with zeros (rows beyond the channel count are never read: TMA bounds)
// (grouped: W is [F][C/G][kh][kw]; the inner index is the group-local channel
// (mode 0) or group-local filter (mode 1) of the row's group)
__global__ void pack_taps(const __grid_constant__ PackTapsP p) {
  pdl_enter();
  const int G = max(1, p.G), Cg = p.C / G, Fg = p.F / G;
  const int T = p.kh * p.kw, rows = p.mode == 0 ? p.F : p.C, inner = p.mode == 0 ? Cg : Fg;
  const long long total = (long long)T * rows * p.ip;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % p.ip);
    const long long tr = e / p.ip;
    const int r = (int)(tr % rows), t = (int)(tr / rows);
    float v = 0.f;
    if (k < inner) {
      const int g = p.mode == 0 ? r / Fg : r / Cg;
      const int f = p.mode == 0 ? r : g * Fg + k, cl = p.mode == 0 ? k : r - g * Cg;
      v = tf32f(__ldg(p.w + ((size_t)f * Cg + cl) * T + t));
    }
    p.out[e] = v;
  }
}

// ================================================================ host side
static int pick_bn(int F) {
  if (F <= 32) return 32;
  if (F <= 64) return 64;
  if (F <= 96) return 96;
  if (F <= 128) return 128;
  if (F <= 192) return 192;
  if (F <= 256) return 256;
  // several column tiles: the widest of 256 / 192 / 128 with the least padding
  int best = 256;
  for (int bn : {192, 128})
    if ((F + bn - 1) / bn * bn < (F + best - 1) / best * best) best = bn;
  return best;
}

template <int BN>
static size_t fwd_smem(int nk) {
  return 1024 + (size_t)FwdCfg<BN>::STAGES * FwdCfg<BN>::STAGE + (size_t)nk * 32 * 8;
}

#define PN_BN_LIST(X) X(32) X(64) X(96) X(128) X(192) X(256)

int fwd_rows_pad(int F) {
  const int bn = pick_bn(F);
  return (F + bn - 1) / bn * bn;
}

Launch conv_fwd_launch(const ConvTcP& p) {
  Launch l;
  const int bn = pick_bn(p.F);
  const long long M = (long long)p.N * p.Ho * p.Wo;
  const dim3 grid((unsigned)((M + 127) / 128), (unsigned)((p.F + bn - 1) / bn));
  switch (bn) {
#define CASE(BN) \
  case BN: l.set((const void*)conv_tc_fwd<BN>, grid, dim3(FwdCfg<BN>::THREADS), fwd_smem<BN>(p.nk), p); break;
    PN_BN_LIST(CASE)
#undef CASE
  }
  return l;
}

Launch pack_launch(const ConvPackP& p) {
  Launch l;
  const long long total = (long long)p.rows * p.nk * 32;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 8);
  l.set((const void*)pack_conv_weights, dim3(blocks), dim3(256), 0, p);
  return l;
}

static int pick_tw_bn(int F) {  // F columns per tile: one tile when F <= 256
  if (F <= 32) return 32;
  if (F <= 64) return 64;
  if (F <= 128) return 128;
  if (F <= 256) return (F + 15) / 16 * 16 > 192 ? 256 : 192;
  return (F + 1) / 2 <= 192 ? 192 : 256;
}

ConvTmaPlan conv_tma_plan(int N, int C, int kh, int kw, int F, int Ho, int Wo, int bias, int sms, int G) {
  ConvTmaPlan w;
  const long long M = (long long)N * Ho * Wo;
  w.M = (int)M;
  w.G = std::max(1, G);
  w.K = C / w.G * kh * kw;
  w.F = F;
  w.bias = bias;
  w.howo = Ho * Wo;
  w.pitch_m = (int)((M + 3) / 4 * 4);
  w.kp = (w.K + 3) / 4 * 4;
  w.fp = (F + 3) / 4 * 4;
  w.wg_bn = pick_tw_bn(F / w.G);
  w.wg_kpad = (w.G * (w.K + bias) + 127) / 128 * 128;  // colT rows: G blocks of K + bias
  w.wg_fpad = (F + w.wg_bn - 1) / w.wg_bn * w.wg_bn;
  const long long tiles = (long long)((w.K + bias + 127) / 128) * ((F / w.G + w.wg_bn - 1) / w.wg_bn) * w.G,
                  nc = (M + 31) / 32;
  long long s = std::max(1LL, sms / tiles);  // one wave at one CTA per SM
  w.wg_splits = (int)std::min(s, std::max(1LL, nc / 8));
  w.fw_bn = pick_tw_bn(F);
  const size_t colT = (size_t)w.wg_kpad * w.pitch_m, col = (size_t)M * w.kp;
  w.col_floats = std::max(colT, col);
  w.g_floats = std::max((size_t)w.wg_fpad * w.pitch_m, (size_t)M * w.fp);
  return w;
}

Launch im2col_t_launch(const Im2colTP& p) {
  Launch l;
  const long long M = (long long)p.N * p.Ho * p.Wo;
  const long long per_block = p.sw == 1 ? 1024 : 256;  // (see the kernel)
  l.set((const void*)im2col_t, dim3((unsigned)((M + per_block - 1) / per_block), (unsigned)((p.Kb + IM_KROWS - 1) / IM_KROWS)),
        dim3(256), 0, p);
  return l;
}

Launch im2col_rows_launch(const Im2colTP& p) {
  Launch l;
  const long long M = (long long)p.N * p.Ho * p.Wo;
  l.set((const void*)im2col_rows, dim3((unsigned)((p.K + 255) / 256), (unsigned)((M + IMR_ROWS - 1) / IMR_ROWS)),
        dim3(256), 0, p);
  return l;
}

Launch gm_launch(const GmP& p) {
  Launch l;
  const long long total = (long long)p.N * p.F * p.HoWo;
  l.set((const void*)gather_gm, dim3((unsigned)std::min<long long>((total + 255) / 256, 148 * 16)), dim3(256), 0, p);
  return l;
}

Launch pack_plain_launch(const PackPlainP& p) {
  Launch l;
  const long long total = (long long)p.F * p.K;
  l.set((const void*)pack_plain, dim3((unsigned)std::min<long long>((total + 255) / 256, 148 * 8)), dim3(256), 0, p);
  return l;
}

// ======================================= weight gradient as a tap GEMM
// (tc_conv.h ConvWtapP).  The operands are TF32 copies laid out for it:
//   Xs[n][y][j][c][x] = X[n][c][y][x + j - pw]  (kw column-shifted rows; a TMA
//                       box must start 16-byte aligned in its innermost
//                       dimension, so the column shift is baked into a copy)
//   Gw[n][yo][f][xo]  = G[n][f][yo][xo]
// A CTA takes whole segments of R output rows of one image.  Per segment ONE
// 5-D TMA box brings input rows ys - ph .. ys + R - 1 + kh - ph (R + kh rows,
// zero-filled outside the image) of every copy j and channel c, as blocks of C
// rows x Wo TF32 (row = one swizzle span: Wo = 8 / 16 / 32 -> 32 / 64 / 128 B),
// block index (row - ys + ph) kw + j; and one 4-D box brings G's R rows.
// For output row q of the segment, tap t = (i, j) reads input row q + i, copy
// j: block q kw + t -- so the 128-row accumulator tile m (taps 4m .. 4m+3 when
// C = 32: rows = (tap slot, c)) is the contiguous run of blocks q kw + 4m ..,
// one MMA descriptor, no copy per tap.  (Blocks past tap T - 1 are the next
// row's: their rows of the accumulator are ignored.)  The bias gradient is one
// more tile against a constant all-ones A operand.  TMEM: (MT + 1) x F
// columns.  warp 0 lane 0 TMA (2 segment stages), warp 1 lane 0 MMA, warps 2-5
// write the CTA's split partials at the end.
__device__ __forceinline__ uint64_t make_desc_sw(uint32_t saddr, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46) | (layout << 61);
}
__device__ __forceinline__ void tma5d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                      uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
template <int WO>
__global__ void __launch_bounds__(192, 1) conv_wgrad_taps(const __grid_constant__ ConvWtapP p) {
  constexpr int ROWB = WO * 4;  // bytes of one operand row = the swizzle span
  constexpr uint32_t SBO = 8 * ROWB;
  constexpr uint64_t LAYOUT = WO == 32 ? 2 : (WO == 16 ? 4 : 6);  // SWIZZLE_128B / 64B / 32B
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[2], empty[2], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t ones = sbase + 2 * p.stage_bytes;  // 128 rows of 1.0 (the bias tile's A)
  const int BLK = p.C * ROWB, XB = p.x_bytes;        // one (row, copy) block; X part of a stage
  const int s0 = (int)((long long)p.segs * blockIdx.x / gridDim.x);
  const int ns = (int)((long long)p.segs * (blockIdx.x + 1) / gridDim.x) - s0;
  if (tid == 0) {
    for (int st = 0; st < 2; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&empty[st]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
    prefetch_tmap(&p.tx);
    prefetch_tmap(&p.tg);
  }
  if (warp == 0) tmem_alloc(&tmem_base, p.tmem_cols);
  for (int u = tid; u < 128 * ROWB / 16; u += blockDim.x) sts128(ones + 16 * u, f4(1.f, 1.f, 1.f, 1.f));
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  pdl_enter();
  if (tid == 0) {  // TMA producer: one segment per stage
    for (int g = 0; g < ns; ++g) {
      const int st = g & 1, sg = s0 + g, n = sg / p.seg_per_img, ys = (sg - n * p.seg_per_img) * p.R;
      if (g >= 2) mbar_wait(smem_u32(&empty[st]), ((g >> 1) - 1) & 1);
      const uint32_t bar = smem_u32(&full[st]), As = sbase + st * p.stage_bytes;
      mbar_expect_tx(bar, (uint32_t)p.tx_bytes);  // the two boxes (the pad after X is never written)
      tma5d(As, &p.tx, 0, 0, 0, ys - p.ph, n, bar);
      tma4d(As + XB, &p.tg, 0, 0, ys, n, bar);
    }
  } else if (tid == 32) {  // MMA issuer
    const uint32_t idesc = make_idesc(128, p.F);
    for (int g = 0; g < ns; ++g) {
      const int st = g & 1, sg = s0 + g, n = sg / p.seg_per_img, ys = (sg - n * p.seg_per_img) * p.R;
      const int nq = min(p.R, p.Ho - ys);
      mbar_wait(smem_u32(&full[st]), (g >> 1) & 1);
      tc_fence_after();
      const uint32_t As = sbase + st * p.stage_bytes, Bs = As + XB;
      for (int q = 0; q < nq; ++q) {
#pragma unroll
        for (int k = 0; k < WO / 8; ++k) {
          const uint32_t acc = (g | q | k) != 0;
          const uint64_t bd = make_desc_sw(Bs + q * p.F * ROWB + k * 32, SBO, LAYOUT);
          for (int m = 0; m < p.MT; ++m)
            mma_tf32(tbase + m * p.F, make_desc_sw(As + (q * p.kw + m * p.TPT) * BLK + k * 32, SBO, LAYOUT), bd, idesc,
                     acc);
          mma_tf32(tbase + p.MT * p.F, make_desc_sw(ones + k * 32, SBO, LAYOUT), bd, idesc, acc);
        }
      }
      mma_commit(smem_u32(&empty[st]));
    }
    if (ns > 0) mma_commit(smem_u32(&done));
  } else if (warp >= 2) {  // epilogue: row r of tile m = (tap slot, channel)
    const int quad = warp & 3, r = quad * 32 + lane, sl = r / p.C;  // (channel r % C: the partial's inner index)
    if (ns > 0) {
      mbar_wait(smem_u32(&done), 0);
      __syncwarp();
      tc_fence_after();
    }
    float* pb = p.part + (size_t)blockIdx.x * p.pstride;
    for (int m = 0; m <= p.MT; ++m) {
      const int tap = m * p.TPT + sl;
      for (int f0 = 0; f0 < p.F; f0 += 16) {
        float v[16];
        if (ns > 0) {
          tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + m * p.F + f0, v);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0.f;
        }
        if (m < p.MT && tap < p.T) {  // [f][t][c] = [f][128 m + r]: a warp's 32 rows in one line
#pragma unroll
          for (int q = 0; q < 16; ++q) pb[(size_t)(f0 + q) * p.K + m * 128 + r] = v[q];
        } else if (m == p.MT && p.bias && r == 0) {
#pragma unroll
          for (int q = 0; q < 16; ++q) pb[(size_t)p.F * p.K + f0 + q] = v[q];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, p.tmem_cols);
}

// Xs[n][y][j][c][x] = tf32(X[n][c][y][x + j - pw]) (0 outside the row): a
// block per input row (n, y); W and C powers of two (shifts, no division).
// The row's C x W inputs are staged once in shared memory (16-B loads when
// the rows are 16-B aligned) and each copy is written as 16-B stores.
__global__ void __launch_bounds__(256) tf32_shift_copies(const __grid_constant__ ShiftCopyP p) {
  __shared__ __align__(16) float xs_row[128 * 32];  // C W <= 4096 (wgrad_taps_ok)
  pdl_enter();
  const int lw = __ffs(p.W) - 1, lc = __ffs(p.C) - 1, cw = 1 << (lc + lw), per4 = (p.kw << (lc + lw)) >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.x) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0;
  for (int row = blockIdx.x; row < p.N * p.H; row += gridDim.x) {
    const int n = row / p.H, y = row - n * p.H;
    const float* xr = p.x + ((size_t)n * p.C * p.H + y) * p.W;  // + c H W + x
    __syncthreads();  // the previous row's copies are written
    if (vec) {
      for (int u = threadIdx.x; u < cw >> 2; u += 256) {
        const int c = (u << 2) >> lw, x = (u << 2) & (p.W - 1);
        float4 v = __ldg(reinterpret_cast<const float4*>(xr + (size_t)c * p.H * p.W + x));
        v.x = tf32f(v.x); v.y = tf32f(v.y); v.z = tf32f(v.z); v.w = tf32f(v.w);
        reinterpret_cast<float4*>(xs_row)[u] = v;
      }
    } else {
      for (int u = threadIdx.x; u < cw; u += 256)
        xs_row[u] = tf32f(__ldg(xr + (size_t)(u >> lw) * p.H * p.W + (u & (p.W - 1))));
    }
    __syncthreads();
    float* o = p.out + (size_t)row * (per4 << 2);
    for (int u = threadIdx.x; u < per4; u += 256) {
      const int e = u << 2, x = e & (p.W - 1), c = (e >> lw) & (p.C - 1), j = e >> (lw + lc);
      const float* src = xs_row + (c << lw);
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int xs = x + q + j - p.pw;
        v[q] = (xs >= 0 && xs < p.W) ? src[xs] : 0.f;
      }
      if (vec) reinterpret_cast<float4*>(o)[u] = make_float4(v[0], v[1], v[2], v[3]);
      else {
#pragma unroll
        for (int q = 0; q < 4; ++q) o[e + q] = v[q];
      }
    }
  }
}
// Gw[n][yo][f][xo] = tf32(G[n][f][yo][xo]): a block per output row (n, yo),
// 16-B loads and stores when aligned (Wo a power of two >= 4)
__global__ void __launch_bounds__(256) tf32_gw(const __grid_constant__ GwP p) {
  pdl_enter();
  const int lw = __ffs(p.Wo) - 1, per = p.F << lw;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.g) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0 && p.Wo >= 4;
  for (int row = blockIdx.x; row < p.N * p.Ho; row += gridDim.x) {
    const int n = row / p.Ho, y = row - n * p.Ho;
    const float* g = p.g + ((size_t)n * p.F * p.Ho + y) * p.Wo;  // + f Ho Wo + x
    float* o = p.out + (size_t)row * per;
    if (vec) {
      for (int u = threadIdx.x; u < per >> 2; u += 256) {
        const int e = u << 2;
        float4 v = __ldg(reinterpret_cast<const float4*>(g + (size_t)(e >> lw) * p.Ho * p.Wo + (e & (p.Wo - 1))));
        v.x = tf32f(v.x); v.y = tf32f(v.y); v.z = tf32f(v.z); v.w = tf32f(v.w);
        reinterpret_cast<float4*>(o)[u] = v;
      }
    } else {
      for (int u = threadIdx.x; u < per; u += 256)
        o[u] = tf32f(__ldg(g + (size_t)(u >> lw) * p.Ho * p.Wo + (u & (p.Wo - 1))));
    }
  }
}
Launch shift_copies_launch(const ShiftCopyP& p) {
  Launch l;
  l.set((const void*)tf32_shift_copies, dim3((unsigned)std::min(p.N * p.H, 148 * 8)), dim3(256), 0, p);
  return l;
}
Launch gw_launch(const GwP& p) {
  Launch l;
  l.set((const void*)tf32_gw, dim3((unsigned)std::min(p.N * p.Ho, 148 * 8)), dim3(256), 0, p);
  return l;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}
// [rows][cols] fp32 (row pitch `pitch` floats), box {32 cols, box_rows}, 128B
// swizzle; reads outside [rows) x [cols) return zeros
static bool tmap2d(CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                   uint32_t box_rows) {
  std::memset(m, 0, sizeof(*m));
  EncodeTiledFn fn = encode_fn();
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int g_sms = 148;  // SM count of the device (setup())

template <int EPI>
static bool gemm_launch(int bn, ConvGemmP& p, Launch* out) {
  p.bn = bn;
  p.ctiles = (p.cols + bn - 1) / bn;
  const long long tiles = (long long)((p.rows + 127) / 128) * p.ctiles * std::max(1, p.G) * p.splits;
  const dim3 grid((unsigned)std::min<long long>(tiles, g_sms));
  switch (bn) {
#define CASE(BN)                                                                                              \
  case BN:                                                                                                    \
    out->set((const void*)tc_persistent<BN, GemmOp<EPI>>, grid, dim3(TwCfg<BN>::THREADS), tw_smem<BN>(), p); \
    return true;
    CASE(32) CASE(64) CASE(128) CASE(192) CASE(256)
#undef CASE
  }
  return false;
}

bool gemm_wgrad_launch(const ConvTmaPlan& w, const float* colT, const float* gm, float* part, int pstride,
                       Launch* out) {
  ConvGemmP p{};
  bool ok = tmap2d(&p.ta, colT, (uint64_t)w.wg_kpad, (uint64_t)w.M, (uint64_t)w.pitch_m, 128);
  ok = ok && tmap2d(&p.tb, gm, (uint64_t)w.wg_fpad, (uint64_t)w.M, (uint64_t)w.pitch_m, (uint32_t)w.wg_bn);
  p.out = part;
  p.Kdim = w.M;
  p.G = w.G;
  p.rows = w.K + w.bias;  // per group
  p.cols = w.F / w.G;
  p.splits = w.wg_splits;
  p.K = w.K;
  p.F = w.F;
  p.has_bias = w.bias;
  p.pstride = pstride;
  return gemm_launch<EPI_WGRAD>(w.wg_bn, p, out) && ok;
}

bool gemm_fwd_launch(const ConvTmaPlan& w, const float* col, const float* wf, const float* bias, float* y, int relu,
                     Launch* out) {
  ConvGemmP p{};
  bool ok = tmap2d(&p.ta, col, (uint64_t)w.M, (uint64_t)w.K, (uint64_t)w.kp, 128);
  ok = ok && tmap2d(&p.tb, wf, (uint64_t)w.F, (uint64_t)w.K, (uint64_t)w.kp, (uint32_t)w.fw_bn);
  p.out = y;
  p.bias = bias;
  p.Kdim = w.K;
  p.rows = w.M;
  p.cols = w.F;
  p.splits = 1;
  p.F = w.F;
  p.HoWo = w.howo;
  p.relu = relu;
  return gemm_launch<EPI_FWD>(w.fw_bn, p, out) && ok;
}


// ---- tap GEMM
static int pow2_at_least(int v, int lo) {
  int r = lo;
  while (r < v) r <<= 1;
  return r;
}

bool tap_launch(const float* nhwc, int N, int Hin, int Win, int cp, const float* wtaps, int rows, int ip, int kh,
                int kw, int ph, int pw, int sgn, int Ho, int Wo, int F, const float* bias, int relu,
                const float* relu_y, float* out, Launch* l, int G, int cpg) {
  ConvTapP p{};
  p.G = std::max(1, G);
  p.fg = F / p.G;
  p.cpg = p.G > 1 ? cpg : cp;
  p.bw = std::min(32, pow2_at_least(Wo, 8));
  p.bh = std::min(128 / p.bw, pow2_at_least(Ho, 1));
  p.bni = 128 / (p.bw * p.bh);
  p.tiles_w = (Wo + p.bw - 1) / p.bw;
  p.tiles_h = (Ho + p.bh - 1) / p.bh;
  const int bn = pick_tw_bn(F / std::max(1, G));
  EncodeTiledFn fn = encode_fn();
  bool ok = fn != nullptr;
  {
    cuuint64_t dims[4] = {(cuuint64_t)cp, (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)cp * 4, (cuuint64_t)Win * cp * 4, (cuuint64_t)Hin * Win * cp * 4};
    cuuint32_t box[4] = {32, (cuuint32_t)p.bw, (cuuint32_t)p.bh, (cuuint32_t)p.bni};
    cuuint32_t es[4] = {1, 1, 1, 1};
    ok = ok && fn(&p.ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)nhwc, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)ip, (cuuint64_t)rows, (cuuint64_t)(kh * kw)};
    cuuint64_t strides[2] = {(cuuint64_t)ip * 4, (cuuint64_t)rows * ip * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)bn, 1};
    cuuint32_t es[3] = {1, 1, 1};
    ok = ok && fn(&p.tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)wtaps, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  p.bias = bias;
  p.relu_y = relu_y;
  p.out = out;
  p.N = N;
  p.Ho = Ho;
  p.Wo = Wo;
  p.F = F;
  p.cp = cp;
  p.kh = kh;
  p.kw = kw;
  p.ph = ph;
  p.pw = pw;
  p.sgn = sgn;
  p.relu = relu;
  p.bn = bn;
  p.ctiles = (p.fg + bn - 1) / bn;
  const long long tiles = (long long)p.tiles_w * p.tiles_h * ((N + p.bni - 1) / p.bni) * p.ctiles * p.G;
  const dim3 grid((unsigned)std::min<long long>(tiles, g_sms));
  switch (bn) {
#define CASE(BN) \
  case BN: l->set((const void*)tc_persistent<BN, TapOp>, grid, dim3(TwCfg<BN>::THREADS), tw_smem<BN>(), p); return ok;
    CASE(32) CASE(64) CASE(128) CASE(192) CASE(256)
#undef CASE
  }
  return false;
}

Launch nhwc_launch(const NhwcP& p) {
  Launch l;
  l.set((const void*)to_nhwc, dim3((unsigned)((p.H * p.W + 31) / 32), (unsigned)((p.cp + 31) / 32), (unsigned)p.N),
        dim3(256), 0, p);
  return l;
}

Launch pack_taps_launch(const PackTapsP& p) {
  Launch l;
  const long long total = (long long)p.kh * p.kw * (p.mode == 0 ? p.F : p.C) * p.ip;
  l.set((const void*)pack_taps, dim3((unsigned)std::min<long long>((total + 255) / 256, 148 * 8)), dim3(256), 0, p);
  return l;
}

// ---- weight gradient as a tap GEMM
static constexpr size_t kWtapSmemMax = 220 * 1024;
static int wtap_mt(int C, int T) { return (T + 128 / C - 1) / (128 / C); }
// rows per segment: the largest power of two <= Ho whose two stages (+ the
// ones tile) fit shared memory; 0 if none
// X part of a stage: the R + kh staged input rows' kw C-row blocks, plus the
// blocks the last accumulator tile of the last output row reads past them
// (tap slots >= T: ignored rows, but the reads must stay in the stage)
static size_t wtap_x_bytes(int R, int C, int Wo, int kh, int kw) {
  const int T = kh * kw, MT = wtap_mt(C, T), TPT = 128 / C;
  const int blocks = std::max((R + kh) * kw, (R - 1) * kw + MT * TPT);
  return (size_t)blocks * C * Wo * 4;
}
static int wtap_rows(int C, int Ho, int Wo, int F, int kh, int kw, size_t* stage) {
  for (int R = 1 << 5; R >= 1; R >>= 1) {
    if (R > Ho && R > 1) continue;
    const size_t st = wtap_x_bytes(R, C, Wo, kh, kw) + (size_t)R * F * Wo * 4;
    if (2 * st + 128 * Wo * 4 <= kWtapSmemMax) {
      if (stage) *stage = st;
      return R;
    }
  }
  return 0;
}
bool wgrad_taps_ok(int C, int W, int Wo, int F, int kh, int kw, int sh, int sw, int G) {
  if (getenv("PN_NO_WTAP")) return false;
  if (G != 1 || sh != 1 || sw != 1 || W != Wo) return false;
  // (Wo = 8: 32-byte TMA rows -- measured slower than the materialised
  // column matrix on cifar10_quick conv3, 43 vs 35 us with its copies)
  if (!(C == 16 || C == 32 || C == 64 || C == 128) || !(Wo == 16 || Wo == 32)) return false;
  if (F % 16 || F < 16 || F > 256) return false;
  const int MT = wtap_mt(C, kh * kw);
  return (MT + 1) * F <= 512 && wtap_rows(C, 1 << 5, Wo, F, kh, kw, nullptr) > 0;
}
// CTAs: at least 4 segments each (every CTA writes a whole (C T + 1) F
// partial), at most one per SM
int wgrad_taps_splits(int N, int Ho, int Wo, int C, int F, int kh, int kw, int sms) {
  const int R = wtap_rows(C, Ho, Wo, F, kh, kw, nullptr), segs = N * ((Ho + R - 1) / R);
  return std::max(1, std::min(sms, segs / 4));
}

bool wgrad_taps_launch(const float* xs, const float* gw, int N, int C, int H, int W, int Ho, int Wo, int F, int kh,
                       int kw, int ph, int pw, int bias, float* part, int pstride, int splits, Launch* l) {
  ConvWtapP p{};
  EncodeTiledFn fn = encode_fn();
  const CUtensorMapSwizzle sw = Wo == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                         : (Wo == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  size_t stage = 0;
  p.R = wtap_rows(C, Ho, Wo, F, kh, kw, &stage);
  bool ok = fn != nullptr && p.R > 0;
  {  // Xs [n][y][j][c][x]: box {Wo, C, kw, R + kh, 1}
    cuuint64_t dims[5] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)kw, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[4] = {(cuuint64_t)W * 4, (cuuint64_t)C * W * 4, (cuuint64_t)kw * C * W * 4,
                             (cuuint64_t)H * kw * C * W * 4};
    cuuint32_t box[5] = {(cuuint32_t)Wo, (cuuint32_t)C, (cuuint32_t)kw, (cuuint32_t)(p.R + kh), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    ok = ok && fn(&p.tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void*)xs, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  {  // Gw [n][yo][f][xo]: box {Wo, F, R, 1}
    cuuint64_t dims[4] = {(cuuint64_t)Wo, (cuuint64_t)F, (cuuint64_t)Ho, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)Wo * 4, (cuuint64_t)F * Wo * 4, (cuuint64_t)Ho * F * Wo * 4};
    cuuint32_t box[4] = {(cuuint32_t)Wo, (cuuint32_t)F, (cuuint32_t)p.R, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    ok = ok && fn(&p.tg, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)gw, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  p.part = part;
  p.N = N, p.C = C, p.Ho = Ho, p.Wo = Wo, p.F = F, p.kh = kh, p.kw = kw, p.ph = ph, p.pw = pw;
  p.T = kh * kw, p.K = C * kh * kw, p.bias = bias, p.pstride = pstride;
  p.TPT = 128 / C;
  p.MT = wtap_mt(C, p.T);
  p.x_bytes = (int)wtap_x_bytes(p.R, C, Wo, kh, kw);  // (the X box fills its first (R + kh) kw blocks)
  p.stage_bytes = (int)stage;
  p.tx_bytes = (p.R + kh) * kw * C * Wo * 4 + p.R * F * Wo * 4;
  p.seg_per_img = (Ho + p.R - 1) / p.R;
  p.segs = N * p.seg_per_img;
  p.tmem_cols = pow2_at_least((p.MT + 1) * F, 32);
  const void* f = Wo == 32 ? (const void*)conv_wgrad_taps<32>
                           : (Wo == 16 ? (const void*)conv_wgrad_taps<16> : (const void*)conv_wgrad_taps<8>);
  l->set(f, dim3(std::max(1, splits)), dim3(192), 1024 + 2 * stage + (size_t)128 * Wo * 4, p);
  return ok;
}
cudaError_t setup(int max_nk) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
#define SET(BN)                                                                                         \
  if (e == cudaSuccess)                                                                                 \
    e = cudaFuncSetAttribute((const void*)conv_tc_fwd<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)fwd_smem<BN>(max_nk));
  PN_BN_LIST(SET)
#undef SET
#define SETW(BN)                                                                                            \
  for (const void* f : {(const void*)tc_persistent<BN, GemmOp<EPI_WGRAD>>, (const void*)tc_persistent<BN, GemmOp<EPI_FWD>>}) \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tw_smem<BN>());
  SETW(32) SETW(64) SETW(128) SETW(192) SETW(256)
#undef SETW
#define SETT(BN)      \
  if (e == cudaSuccess) \
    e = cudaFuncSetAttribute((const void*)tc_persistent<BN, TapOp>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tw_smem<BN>());
  SETT(32) SETT(64) SETT(128) SETT(192) SETT(256)
#undef SETT
  if (e == cudaSuccess) e = plane_setup();
  for (const void* f : {(const void*)conv_wgrad_taps<8>, (const void*)conv_wgrad_taps<16>, (const void*)conv_wgrad_taps<32>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kWtapSmemMax + 1024));
  return e;
}

}  // namespace tcc
}  // namespace pn
