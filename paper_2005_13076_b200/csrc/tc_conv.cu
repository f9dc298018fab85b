// tc_conv.cu -- general tcgen05 TF32 implicit-GEMM convolution for any
// geometry (kernel, stride, padding, channel counts): the tensor-core plan of
// nets other than the fused LeNet chain (cifar10_quick, SURVEY §8(a) row a19;
// the AlexNet-shaped conv sweep, BASELINE config 5).
//
// The paper lowers a convolution to im2col + GEMM: a column
// matrix of every (c,i,j) patch element per output position, multiplied by
// the F x (C*kh*kw) weight matrix.  Here the column matrix is never
// materialised: each 128-row tile of it is gathered from the NCHW
// activation straight into the shared-memory operand layout of the tensor
// core (K-major SWIZZLE_128B, 32 fp32 of K per 128-B row), rounded to TF32
// (nearest, ties away) on the way.
//
//   forward   y[m=(n,ho,wo), f]  = sum_k col[m,k] W[f,k] (+ b[f])
//   data grad dx = col2im(W^T G) computed as a stride-1 convolution of G with
//             the spatially flipped, channel-transposed filter
//             W'[c, (f,i',j')] = W[f, c, kh-1-i', kw-1-j'] and padding kh-1-p
//             (identical sums; needs stride 1 -- every non-data conv layer of
//             the configured nets)
//   weight grad dW[f, k] = sum_m G[m,f] col[m,k]; db[f] = sum_m G[m,f] rides
//             along as an extra all-ones column k = K of col; the m range is
//             split over CTAs into fixed-order partials (reduce_partials)
//
// CTA structure (warp-specialized over mbarriers):
//   conv_tc_fwd (fwd and dgrad): warp 0 lane 0 streams the packed TF32 B
//     operand (pack_conv_weights) into a STAGES-deep ring with 1-D bulk
//     copies (complete_tx); warp 1 lane 0 issues 4 x tcgen05.mma (M=128,
//     N=BN, K=8) per 32-wide K chunk into a TMEM accumulator and commits the
//     stage back; warps 2-9 gather the A tile (thread = row, 16 of the 32 K
//     values) and then run the epilogue (tcgen05.ld 32x32b, bias, ReLU,
//     coalesced NCHW stores: lanes = consecutive output positions).
//   conv_tc_wgrad: warp 0 lane 0 = MMA; warps 1-8 gather both operands with
//     lanes over the 32 m values of a chunk (one 128-B swizzle row per warp
//     store, conflict-free) and write the partial tile.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
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
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int f = f0 + cc + t;
        if (elive && f < p.F) {
          float o = v[t];
          if (p.bias) o += __ldg(p.bias + f);
          if (p.relu) o = fmaxf(o, 0.f);
          if (p.relu_y && !(__ldg(p.relu_y + (yb - p.y) + (size_t)f * HoWo) > 0.f)) o = 0.f;
          yb[(size_t)f * HoWo] = o;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, Cfg::TMEM_COLS);
}

// ================================================================ weight grad
template <int BN>
struct WgCfg {
  static constexpr int STAGES = 3;  // BN <= 128: 97 KB, two CTAs per SM
  static constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int THREADS = 288;
};

template <int BN>
__global__ void __launch_bounds__(288, 2) conv_tc_wgrad(const __grid_constant__ ConvTcWgradP p) {
  using Cfg = WgCfg<BN>;
  constexpr int STAGES = Cfg::STAGES, A_BYTES = Cfg::A_BYTES, STAGE = Cfg::STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem), tab = sbase + STAGES * STAGE;
  const int f0 = blockIdx.x * 128, k0 = blockIdx.y * BN, s = blockIdx.z;
  const int HoWo = p.Ho * p.Wo, M = p.N * HoWo, HW = p.H * p.W, CHW = p.C * HW;
  const int nc = (M + 31) / 32, c0 = (int)((long long)s * nc / p.splits),
            c1 = (int)((long long)(s + 1) * nc / p.splits), my = c1 - c0;
  for (int k = tid; k < BN; k += Cfg::THREADS) sts_i2(tab + 8 * k, ktab_entry(k0 + k, p.K, p.H, p.W, p.kh, p.kw));
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(smem_u32(&full[st]), 256);
      mbar_init(smem_u32(&empty[st]), 1);
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
  if (warp == 0) {
    if (lane == 0 && my > 0) {  // MMA issuer: D[f, k] += G^T[f, m] col^T[k, m]
      constexpr uint32_t idesc = make_idesc(128, BN);
      for (int c = 0; c < my; ++c) {
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
    // ---- gatherers: warp gw (0..7) takes rows gw, gw+8, ...; lane = m in chunk.
    // Software-pipelined: the loads of chunk c+1 are in flight while chunk c
    // is rounded and stored (two register sets, loop unrolled by two).
    const int gw = warp - 1;
    const uint32_t lane_off = (uint32_t)((lane & 3) * 4), lane_chunk = (uint32_t)(lane >> 2);
    auto gather = [&](int c, float (&a)[16], float (&b)[BN / 8]) {
      const int m = (c0 + c) * 32 + lane;
      const bool live = m < M;
      int n = 0, pos = 0, ho = 0, wo = 0;
      if (live) {
        n = m / HoWo;
        pos = m - n * HoWo;
        ho = pos / p.Wo;
        wo = pos - ho * p.Wo;
      }
      const int hi0 = ho * p.sh - p.ph, wi0 = wo * p.sw - p.pw;
      const float* gb = p.g + (size_t)n * p.F * HoWo + pos;
      const float* xb = p.x + (size_t)n * CHW + (hi0 * p.W + wi0);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int f = f0 + gw + 8 * t;
        a[t] = (live && f < p.F) ? __ldg(gb + (size_t)f * HoWo) : 0.f;
      }
#pragma unroll
      for (int t = 0; t < BN / 8; ++t) {
        const int kk = gw + 8 * t, k = k0 + kk;
        const int2 e = lds_i2(tab + 8 * kk);
        const int i = e.y >> 16, j = e.y & 0xFFFF;
        const bool ok = live && (unsigned)(hi0 + i) < (unsigned)p.H && (unsigned)(wi0 + j) < (unsigned)p.W;
        float v = ok ? __ldg(xb + e.x) : 0.f;
        if (k == p.K && p.bias_col) v = live ? 1.f : 0.f;
        b[t] = v;
      }
    };
    auto put = [&](int c, const float (&a)[16], const float (&b)[BN / 8]) {
      const int st = c % STAGES;
      if (c >= STAGES) mbar_wait(smem_u32(&empty[st]), ((c / STAGES) - 1) & 1);
      const uint32_t As = sbase + st * STAGE, Bs = As + A_BYTES;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int row = gw + 8 * t;
        sts32(As + row * 128 + ((lane_chunk ^ (row & 7)) << 4) + lane_off, tf32f(a[t]));
      }
#pragma unroll
      for (int t = 0; t < BN / 8; ++t) {
        const int row = gw + 8 * t;
        sts32(Bs + row * 128 + ((lane_chunk ^ (row & 7)) << 4) + lane_off, tf32f(b[t]));
      }
      fence_proxy_async();
      mbar_arrive(smem_u32(&full[st]));
    };
    float a0[16], b0[BN / 8], a1[16], b1[BN / 8];
    if (my > 0) gather(0, a0, b0);
    for (int c = 0; c < my; c += 2) {
      if (c + 1 < my) gather(c + 1, a1, b1);
      put(c, a0, b0);
      if (c + 1 >= my) break;
      if (c + 2 < my) gather(c + 2, a0, b0);
      put(c + 1, a1, b1);
    }
    // ---- epilogue: the partial tile D[f, k] -> part[s][f*K + k] (bias col -> part[s][wcount + f])
    const int quad = warp & 3, half = (warp - 1) >> 2, f = f0 + quad * 32 + lane;
    if (my > 0) {
      mbar_wait(smem_u32(&done), 0);
      __syncwarp();
      tc_fence_after();
    }
    float* pb = p.part + (size_t)s * p.pstride;
    const long long wcount = (long long)p.F * p.K;
#pragma unroll 1
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
      float v[16];
      if (my > 0) {
        tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + cc, v);
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = 0.f;
      }
      if (f < p.F) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int k = k0 + cc + t;
          if (k < p.K) pb[(size_t)f * p.K + k] = v[t];
          else if (k == p.K && p.bias_col) pb[wcount + f] = v[t];
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
// exact a / d for 0 <= a < 2^24, d >= 1 (float estimate + one-step correction)
__device__ __forceinline__ int qdiv(int a, int d) {
  int q = __float2int_rz(__fmul_rn((float)a + 0.5f, __frcp_rn((float)d)));
  q -= (q * d > a);
  q += ((q + 1) * d <= a);
  return q;
}

// block = 256 consecutive m x a group of IM_KROWS k rows: (n, ho, wo) once per
// thread, (c, i, j) from a shared table, one coalesced store per element
constexpr int IM_KROWS = 16;
__global__ void __launch_bounds__(256) im2col_t(const __grid_constant__ Im2colTP p) {
  __shared__ int2 tab[IM_KROWS];
  const int HoWo = p.Ho * p.Wo, M = p.N * HoWo, KK = p.kh * p.kw;
  const int kb0 = blockIdx.y * IM_KROWS;
  if (threadIdx.x < IM_KROWS) {
    const int k = kb0 + threadIdx.x;
    int2 e = make_int2(0, 0x7FFF << 16);
    if (k < p.K) {
      const int c = k / KK, r = k - c * KK, i = r / p.kw, j = r - i * p.kw;
      e = make_int2(c * p.H * p.W + i * p.W + j, (i << 16) | j);
    } else if (k == p.K) {
      e = make_int2(0, -1);  // bias row: ones
    }
    tab[threadIdx.x] = e;
  }
  pdl_enter();
  __syncthreads();
  const int m = blockIdx.x * 256 + threadIdx.x;
  if (m >= M) return;
  const int n = qdiv(m, HoWo), pos = m - n * HoWo, ho = qdiv(pos, p.Wo), wo = pos - ho * p.Wo;
  const int hi0 = ho * p.sh - p.ph, wi0 = wo * p.sw - p.pw;
  const float* xb = p.x + (size_t)n * p.C * p.H * p.W + (hi0 * p.W + wi0);
  const int kend = min(IM_KROWS, p.Kb - kb0);
  float* dst = p.col + (size_t)kb0 * p.pitch + m;
#pragma unroll 4
  for (int t = 0; t < kend; ++t) {
    const int2 e = tab[t];
    float v;
    if (e.y == -1) {
      v = 1.f;
    } else {
      const int i = e.y >> 16, j = e.y & 0xFFFF;
      v = ((unsigned)(hi0 + i) < (unsigned)p.H && (unsigned)(wi0 + j) < (unsigned)p.W) ? tf32f(__ldg(xb + e.x)) : 0.f;
    }
    dst[(size_t)t * p.pitch] = v;
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

template <int BN>
__global__ void __launch_bounds__(192, 1) conv_wgrad_tma(const __grid_constant__ ConvWgTmaP p) {
  using Cfg = TwCfg<BN>;
  constexpr int STAGES = Cfg::STAGES, A_BYTES = Cfg::A_BYTES, STAGE = Cfg::STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  const int k0 = blockIdx.x * 128, f0 = blockIdx.y * BN, s = blockIdx.z;
  const int nc = (p.M + 31) / 32, c0 = (int)((long long)s * nc / p.splits),
            c1 = (int)((long long)(s + 1) * nc / p.splits), my = c1 - c0;
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&empty[st]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
    prefetch_tmap(&p.ta);
    prefetch_tmap(&p.tb);
  }
  if (warp == 0) tmem_alloc(&tmem_base, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  pdl_enter();
  if (tid == 0) {  // TMA producer
    for (int c = 0; c < my; ++c) {
      const int st = c % STAGES;
      if (c >= STAGES) mbar_wait(smem_u32(&empty[st]), ((c / STAGES) - 1) & 1);
      const uint32_t bar = smem_u32(&full[st]), As = sbase + st * STAGE;
      mbar_expect_tx(bar, STAGE);
      tma2d(As, &p.ta, (c0 + c) * 32, k0, bar);
      tma2d(As + A_BYTES, &p.tb, (c0 + c) * 32, f0, bar);
    }
  } else if (tid == 32) {  // MMA issuer
    constexpr uint32_t idesc = make_idesc(128, BN);
    for (int c = 0; c < my; ++c) {
      const int st = c % STAGES;
      mbar_wait(smem_u32(&full[st]), (c / STAGES) & 1);
      tc_fence_after();
      const uint32_t As = sbase + st * STAGE, Bs = As + A_BYTES;
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_tf32(tbase, make_desc(As + k * 32), make_desc(Bs + k * 32), idesc, (c | k) != 0);
      mma_commit(smem_u32(&empty[st]));
    }
    if (my > 0) mma_commit(smem_u32(&done));
  } else if (warp >= 2) {  // epilogue: thread = k row (TMEM lane), columns f
    const int quad = warp & 3, k = k0 + quad * 32 + lane;
    if (my > 0) {
      mbar_wait(smem_u32(&done), 0);
      __syncwarp();
      tc_fence_after();
    }
    float* pb = p.part + (size_t)s * p.pstride;
    const long long wcount = (long long)p.F * p.K;
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
      float v[16];
      if (my > 0) {
        tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + cc, v);
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = 0.f;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int f = f0 + cc + t;
        if (f >= p.F) break;
        if (k < p.K) pb[(size_t)f * p.K + k] = v[t];
        else if (k == p.K && p.bias) pb[wcount + f] = v[t];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, Cfg::TMEM_COLS);
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
template <int BN>
static size_t wg_smem() {
  return 1024 + (size_t)WgCfg<BN>::STAGES * WgCfg<BN>::STAGE + (size_t)BN * 8;
}

#define PN_BN_LIST(X) X(32) X(64) X(96) X(128) X(192) X(256)

cudaError_t setup(int max_nk) {
  cudaError_t e = cudaSuccess;
#define SET(BN)                                                                                            \
  if (e == cudaSuccess)                                                                                    \
    e = cudaFuncSetAttribute((const void*)conv_tc_fwd<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                             (int)fwd_smem<BN>(max_nk));                                                   \
  if (e == cudaSuccess)                                                                                    \
    e = cudaFuncSetAttribute((const void*)conv_tc_wgrad<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)wg_smem<BN>());
  PN_BN_LIST(SET)
#undef SET
#define SETW(BN)                                                                                            \
  if (e == cudaSuccess)                                                                                     \
    e = cudaFuncSetAttribute((const void*)conv_wgrad_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)tw_smem<BN>());
  SETW(32) SETW(64) SETW(128) SETW(192) SETW(256)
#undef SETW
  return e;
}

int fwd_rows_pad(int F) {
  const int bn = pick_bn(F);
  return (F + bn - 1) / bn * bn;
}

size_t fwd_smem_bytes(int F, int nk) {
  switch (pick_bn(F)) {
#define CASE(BN) \
  case BN: return fwd_smem<BN>(nk);
    PN_BN_LIST(CASE)
#undef CASE
  }
  return 0;
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

static int pick_wbn(int Kb) {  // columns of the weight-gradient tile (K + bias column)
  if (Kb <= 32) return 32;
  if (Kb <= 64) return 64;
  return 128;
}

int wgrad_splits(int N, int Ho, int Wo, int F, int K, int bias, int sms) {
  // one wave at two CTAs per SM: splits = floor(2 sms / tiles), at least ~8
  // chunks per split
  const int bn = pick_wbn(K + bias);
  const long long tiles = (long long)((F + 127) / 128) * ((K + bias + bn - 1) / bn);
  const long long nc = ((long long)N * Ho * Wo + 31) / 32;
  long long s = std::max(1LL, 2 * sms / tiles);
  s = std::min(s, std::max(1LL, nc / 8));
  return (int)s;
}

Launch conv_wgrad_launch(const ConvTcWgradP& p) {
  Launch l;
  const int bn = pick_wbn(p.K + p.bias_col);
  const dim3 grid((unsigned)((p.F + 127) / 128), (unsigned)((p.K + p.bias_col + bn - 1) / bn), (unsigned)p.splits);
  switch (bn) {
#define CASE(BN) \
  case BN: l.set((const void*)conv_tc_wgrad<BN>, grid, dim3(WgCfg<BN>::THREADS), wg_smem<BN>(), p); break;
    CASE(32) CASE(64) CASE(128)
#undef CASE
  }
  return l;
}

// ---- materialised-operand weight gradient
static int pick_tw_bn(int F) {  // F columns per tile: one tile when F <= 256
  if (F <= 32) return 32;
  if (F <= 64) return 64;
  if (F <= 128) return 128;
  if (F <= 256) return (F + 15) / 16 * 16 > 192 ? 256 : 192;
  return (F + 1) / 2 <= 192 ? 192 : 256;
}

WgTmaPlan wgrad_tma_plan(int N, int Ho, int Wo, int F, int K, int bias, int sms) {
  WgTmaPlan w;
  w.bn = pick_tw_bn(F);
  w.kpad = (K + bias + 127) / 128 * 128;
  w.fpad = (F + w.bn - 1) / w.bn * w.bn;
  const long long M = (long long)N * Ho * Wo;
  w.pitch = (int)((M + 3) / 4 * 4);
  const long long tiles = (long long)(w.kpad / 128) * (w.fpad / w.bn), nc = (M + 31) / 32;
  long long s = std::max(1LL, sms / tiles);  // one wave at one CTA per SM
  s = std::min(s, std::max(1LL, nc / 8));
  w.splits = (int)s;
  return w;
}

Launch im2col_t_launch(const Im2colTP& p) {
  Launch l;
  const long long M = (long long)p.N * p.Ho * p.Wo;
  l.set((const void*)im2col_t, dim3((unsigned)((M + 255) / 256), (unsigned)((p.Kb + IM_KROWS - 1) / IM_KROWS)),
        dim3(256), 0, p);
  return l;
}

Launch gm_launch(const GmP& p) {
  Launch l;
  const long long total = (long long)p.N * p.F * p.HoWo;
  l.set((const void*)gather_gm, dim3((unsigned)std::min<long long>((total + 255) / 256, 148 * 16)), dim3(256), 0, p);
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
// [rows][cols] fp32 (row pitch `pitch` floats), box {32 cols, box_rows}, 128B swizzle
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

bool wgrad_tma_launch(const WgTmaPlan& w, const float* col, const float* gm, float* part, int M, int K, int F,
                      int bias, int pstride, Launch* out) {
  ConvWgTmaP p;
  bool ok = tmap2d(&p.ta, col, (uint64_t)w.kpad, (uint64_t)M, (uint64_t)w.pitch, 128);
  ok = ok && tmap2d(&p.tb, gm, (uint64_t)w.fpad, (uint64_t)M, (uint64_t)w.pitch, (uint32_t)w.bn);
  p.part = part;
  p.M = M;
  p.K = K;
  p.F = F;
  p.bias = bias;
  p.splits = w.splits;
  p.pstride = pstride;
  const dim3 grid((unsigned)(w.kpad / 128), (unsigned)(w.fpad / w.bn), (unsigned)w.splits);
  switch (w.bn) {
#define CASE(BN) \
  case BN: out->set((const void*)conv_wgrad_tma<BN>, grid, dim3(TwCfg<BN>::THREADS), tw_smem<BN>(), p); break;
    CASE(32) CASE(64) CASE(128) CASE(192) CASE(256)
#undef CASE
    default: return false;
  }
  return ok;
}

Launch pack_launch(const ConvPackP& p) {
  Launch l;
  const long long total = (long long)p.rows * p.nk * 32;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 8);
  l.set((const void*)pack_conv_weights, dim3(blocks), dim3(256), 0, p);
  return l;
}

}  // namespace tcc
}  // namespace pn
