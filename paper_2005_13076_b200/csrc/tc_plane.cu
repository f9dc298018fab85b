// tc_plane.cu -- stride-1 convolution (forward, and data gradient as the
// convolution of G with the flipped, channel-transposed filter) as a tap GEMM
// over halo-staged activation blocks, for the layerwise TF32 plan
// (cifar10_quick: conv1 -- the stem's forward --, conv2 forward and data
// gradient, conv3 forward).  The LeNet conv2 forward's
// scheme (tc.cu conv2_fwd_persistent) for any stride-1 layer whose output
// rows are a multiple of 8 wide:
//   * an output tile is 128 positions = TY rows x TN images x 8 columns
//     (rows r = (y, n, x), x fastest); its input block with halo, HY = TY +
//     kh - 1 rows x TN x HX = 8 + kw - 1 columns, is packed once per step by
//     plane_pack as 4-channel planes [cq][hy][n][hx][4 c] (TF32, zeros in the
//     halo outside the image): ONE contiguous bulk copy per tile;
//   * in the UMMA K-major no-swizzle layout (core matrix = 8 rows x 16 B) the
//     A operand of tap (i, j) is a descriptor into that block: 8-row group
//     (y, n) at SBO = HX * 16 B, channel quad at LBO = one plane, start shifted
//     by (i TN HX + j) * 16 B -- no im2col, no per-tap load;
//   * B = every tap's weights [t][cq][o][4 c], staged once per CTA (no-swizzle,
//     LBO = Nout * 16 B, SBO = 128 B), packed once per step by plane_wpack;
//     when they do not fit beside the ring, the output channels go in two
//     splits (CTA b computes split b % 2 and stages only its weights);
//   * persistent over tiles: warp 0 lane 0 bulk copies (weights, then an
//     A-block ring), warp 1 lane 0 issues T x Kc/8 tcgen05.mma (M = 128,
//     N = Nout, K = 8) per tile into one of two TMEM accumulators, warps 2-5
//     drain the other: + bias, ReLU (forward) or the in-place ReLU's mask
//     (data gradient), NCHW stores.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "params.h"
#include "pdl.cuh"
#include "tc_conv.h"
#include "tc_ptx.cuh"

namespace pn {
namespace tcc {
using namespace pn::tc;

constexpr int PL_MAX_STAGES = 4;
constexpr size_t kPlaneSmemMax = 220 * 1024;

// A blocks: element (tile, cq, hy, n, hx, c4) = tf32(src[n0 + n][4 cq + c4][y0 + hy - ph][x0 + hx - pw])
__global__ void __launch_bounds__(256) plane_pack(const __grid_constant__ PlanePackP p) {
  // a block per tile (grid-stride); thread = one halo position (hy, n, hx),
  // all its channel quads (loads in flight together, one float4 store per plane)
  pdl_enter();
  const int pos = p.HY * p.TN * p.HX, HW = p.H * p.W;
  for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const int tx = tile % p.tiles_x, t2 = tile / p.tiles_x, ty = t2 % p.tiles_y, nb = t2 / p.tiles_y;
    float4* o = reinterpret_cast<float4*>(p.out) + (size_t)tile * p.Kq * pos;
    for (int r = threadIdx.x; r < pos; r += 256) {
      const int hx = r % p.HX, r2 = r / p.HX, nn = r2 % p.TN, hy = r2 / p.TN;
      const int n = nb * p.TN + nn, y = ty * p.TY + hy - p.ph, x = tx * 8 + hx - p.pw;
      const bool in = n < p.N && y >= 0 && y < p.H && x >= 0 && x < p.W;
      const float* s = p.src + (((size_t)n * p.C) * p.H + y) * p.W + x;
      for (int cq0 = 0; cq0 < p.Kq; cq0 += 4) {
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int c = 4 * cq0 + q;
          v[q] = (in && c < p.C) ? tf32f(__ldg(s + (size_t)c * HW)) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (cq0 + k < p.Kq) o[(size_t)(cq0 + k) * pos + r] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      }
    }
  }
}

// B: [split][t][cq][o][4 c] (output channels in ns splits of Nout / ns);
// mode 0 (forward) = W[o][c][i][j]; mode 1 (data
// gradient) = W[c][o][kh-1-i][kw-1-j] (rows o = the layer's input channels,
// inner c = its output channels)
__global__ void __launch_bounds__(256) plane_wpack(const __grid_constant__ PlaneWpackP p) {
  pdl_enter();
  const int T = p.kh * p.kw, nos = p.Nout / p.ns;
  const long long total = (long long)T * p.Kq * p.Nout * 4;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < total; e += (long long)gridDim.x * 256) {
    int r = (int)e;
    const int c4 = r & 3;
    r >>= 2;
    const int ol = r % nos;
    r /= nos;
    const int cq = r % p.Kq;
    r /= p.Kq;
    const int t = r % T, o = (r / T) * nos + ol, i = t / p.kw, j = t - i * p.kw, c = 4 * cq + c4;
    float v = 0.f;
    if (p.mode == 0) {
      if (c < p.Cin) v = p.w[(((size_t)o * p.Cin + c) * p.kh + i) * p.kw + j];
    } else {
      if (c < p.Cin) v = p.w[(((size_t)c * p.Nout + o) * p.kh + (p.kh - 1 - i)) * p.kw + (p.kw - 1 - j)];
    }
    p.out[e] = tf32f(v);
  }
}

// KH, KW, KQH > 0: taps and channel steps (Kq / 2) fixed at compile time, the
// whole tile's MMAs unrolled with immediate accumulate flags and descriptor
// offsets (single-thread issue: ~45 cycles per MMA instead of ~115-200 in a
// rolled loop); 0: runtime geometry
template <int KH, int KW, int KQH>
__global__ void __launch_bounds__(192, 1) conv_plane_taps(const __grid_constant__ PlaneConvP p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t W_s = smem_u32(smem), A_s = W_s + (uint32_t)((p.w_bytes + 1023) & ~1023);
  __shared__ __align__(8) uint64_t wbar, full[PL_MAX_STAGES], empty[PL_MAX_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float bias_s[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, S = p.stages;
  // output-channel split: this CTA's channels [half nos, + nos), tiles cta, cta + nct, ...
  const int half = blockIdx.x % p.ns, cta = blockIdx.x / p.ns, nct = gridDim.x / p.ns, nos = p.Nout / p.ns;
  for (int o = tid; o < nos; o += blockDim.x) bias_s[o] = p.bias ? __ldg(p.bias + half * nos + o) : 0.f;
  const int mine = p.tiles > cta ? (p.tiles - 1 - cta) / nct + 1 : 0;
  if (tid == 0) {
    mbar_init(smem_u32(&wbar), 1);
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    // the packed weights (two or more launches back: readable before the PDL
    // wait), then -- once the predecessor (the A-block pack) is done -- the ring
    if (mine > 0) {
      mbar_expect_tx(smem_u32(&wbar), (uint32_t)p.w_bytes);
      for (int off = 0; off < p.w_bytes; off += 32768)
        bulk_g2s(W_s + off, (const uint8_t*)p.wts + (size_t)half * p.w_bytes + off,
                 (uint32_t)min(32768, p.w_bytes - off), smem_u32(&wbar));
    }
    pdl_enter();
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int s = it % S, tile = cta + it * nct;
      if (it >= S) mbar_wait(smem_u32(&empty[s]), ((it / S) - 1) & 1);
      mbar_expect_tx(smem_u32(&full[s]), (uint32_t)p.a_bytes);
      bulk_g2s(A_s + s * p.a_bytes, (const uint8_t*)p.src + (size_t)tile * p.a_bytes, (uint32_t)p.a_bytes,
               smem_u32(&full[s]));
    }
  } else if (tid == 32) {
    const uint32_t idesc = make_idesc(128, nos);
    const uint32_t plane = (uint32_t)(p.HY * p.TN * p.HX * 16), lbo_b = (uint32_t)(nos * 16);
    const uint32_t tap_b = (uint32_t)p.Kq * lbo_b;
    const uint64_t bd0 = make_desc_ns(W_s, lbo_b, 128);
    if (mine > 0) {
      mbar_wait(smem_u32(&wbar), 0);
      tc_fence_after();
    }
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int s = it % S, b = it & 1;
      mbar_wait(smem_u32(&full[s]), (it / S) & 1);
      if (it >= 2) mbar_wait(smem_u32(&tempty[b]), ((it >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tbase + b * nos;
      const uint64_t ad0 = make_desc_ns(A_s + s * p.a_bytes, plane, (uint32_t)(p.HX * 16));
      if constexpr (KH > 0) {
        const uint32_t row = (uint32_t)(p.TN * p.HX * 16);
#pragma unroll
        for (int i = 0; i < KH; ++i)
#pragma unroll
          for (int j = 0; j < KW; ++j)
#pragma unroll
            for (int ks = 0; ks < KQH; ++ks) {
              const uint64_t a = ad0 + (uint64_t)((i * row + j * 16 + ks * 2 * plane) >> 4);
              const uint64_t bq = bd0 + (uint64_t)(((i * KW + j) * tap_b + ks * 2 * lbo_b) >> 4);
              if (i == 0 && j == 0 && ks == 0) mma_tf32_c<0>(d, a, bq, idesc);
              else mma_tf32_c<1>(d, a, bq, idesc);
            }
      } else {
        for (int i = 0; i < p.kh; ++i)
          for (int j = 0; j < p.kw; ++j) {
            const uint32_t sh = (uint32_t)((i * p.TN * p.HX + j) * 16), tb = (uint32_t)(i * p.kw + j) * tap_b;
            for (int ks = 0; ks < p.Kq / 2; ++ks)
              mma_tf32(d, ad0 + (uint64_t)((sh + ks * 2 * plane) >> 4), bd0 + (uint64_t)((tb + ks * 2 * lbo_b) >> 4),
                       idesc, (i | j | ks) != 0);
          }
      }
      mma_commit(smem_u32(&empty[s]));
      mma_commit(smem_u32(&tfull[b]));
    }
  } else if (warp >= 2) {
    const int quad = warp & 3, r = quad * 32 + lane;
    const int x = r & 7, g = r >> 3, nn = g % p.TN, y = g / p.TN;
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int b = it & 1, tile = cta + it * nct;
      const int tx = tile % p.tiles_x, t2 = tile / p.tiles_x, ty = t2 % p.tiles_y, nb = t2 / p.tiles_y;
      const int n = nb * p.TN + nn, oy = ty * p.TY + y, ox = tx * 8 + x;
      const bool live = n < p.N && oy < p.Ho && ox < p.Wo;
      mbar_wait(smem_u32(&tfull[b]), (it >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const size_t HW = (size_t)p.Ho * p.Wo;
      const size_t base = ((size_t)n * p.Nout + half * nos) * HW + (size_t)oy * p.Wo + ox;
      for (int o0 = 0; o0 < nos; o0 += 16) {
        float v[16], m[16];
        tmem_ld16_nowait(tbase + ((uint32_t)(quad * 32) << 16) + b * nos + o0, v);
        // the in-place ReLU's outputs of these 16 channels: every load in flight together
#pragma unroll
        for (int q = 0; q < 16; ++q) m[q] = (p.relu_y && live) ? __ldg(p.relu_y + base + (size_t)(o0 + q) * HW) : 1.f;
        tmem_ld_wait();
        if (!live) continue;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float o = v[q] + bias_s[o0 + q];
          if (p.relu) o = fmaxf(o, 0.f);
          if (!(m[q] > 0.f)) o = 0.f;
          p.out[base + (size_t)(o0 + q) * HW] = o;
        }
      }
      tc_fence_before();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, p.tmem_cols);
}

// ---------------------------------------------------------------- host side
static int pow2_ge(int v, int lo) {
  int r = lo;
  while (r < v) r <<= 1;
  return r;
}
// tile geometry of a stride-1 convolution producing Nout channels of Ho x Wo
// from Cin channels (kh x kw taps); false if the scheme does not apply
bool plane_plan(int N, int Cin, int Ho, int Wo, int Nout, int kh, int kw, PlanePlan* pl) {
  if (getenv("PN_NO_PLANE")) return false;
  if (Wo % 8 || Nout % 16 || Nout < 16 || Nout > 256) return false;
  PlanePlan q{};
  if (Ho % 16 == 0) q.TY = 16, q.TN = 1;
  else if (16 % Ho == 0) q.TY = Ho, q.TN = 16 / Ho;
  else return false;
  q.HY = q.TY + kh - 1, q.HX = 8 + kw - 1;
  q.Kq = (Cin + 7) / 8 * 2;
  q.a_bytes = q.Kq * q.HY * q.TN * q.HX * 16;
  // the output channels in one or two splits (each CTA stages one split's weights)
  size_t wpad = 0;
  for (q.ns = 1; q.ns <= 2; ++q.ns) {
    if (Nout % q.ns || (Nout / q.ns) % 16) continue;
    q.w_bytes = kh * kw * q.Kq * (Nout / q.ns) * 16;
    wpad = ((size_t)q.w_bytes + 1023) & ~(size_t)1023;
    if (wpad + 2 * (size_t)q.a_bytes <= kPlaneSmemMax) break;
  }
  if (q.ns > 2) return false;
  q.stages = (int)std::min<size_t>(PL_MAX_STAGES, (kPlaneSmemMax - wpad) / q.a_bytes);
  q.tiles_x = Wo / 8, q.tiles_y = Ho / q.TY;
  q.tiles = (N + q.TN - 1) / q.TN * q.tiles_y * q.tiles_x;
  q.smem = 1024 + wpad + (size_t)q.stages * q.a_bytes;
  *pl = q;
  return true;
}
Launch plane_pack_launch(const PlanePlan& pl, const float* src, float* out, int N, int C, int H, int W, int ph,
                         int pw) {
  PlanePackP p{src, out, N, C, H, W, ph, pw, pl.Kq, pl.HY, pl.HX, pl.TY, pl.TN, pl.tiles, pl.tiles_x, pl.tiles_y};
  Launch l;
  l.set((const void*)plane_pack, dim3((unsigned)std::min(pl.tiles, 148 * 8)), dim3(256), 0, p);
  return l;
}
Launch plane_wpack_launch(const PlanePlan& pl, const float* w, float* out, int Cin, int Nout, int kh, int kw,
                          int mode) {
  PlaneWpackP p{w, out, Cin, Nout, kh, kw, pl.Kq, mode, pl.ns};
  Launch l;
  const long long total = (long long)kh * kw * pl.Kq * Nout * 4;
  l.set((const void*)plane_wpack, dim3((unsigned)std::min<long long>((total + 255) / 256, 148LL * 8)), dim3(256), 0, p);
  return l;
}
Launch plane_conv_launch(const PlanePlan& pl, const float* src, const float* wts, const float* bias,
                         const float* relu_y, float* out, int N, int Ho, int Wo, int Nout, int kh, int kw, int relu,
                         int sms) {
  PlaneConvP p{src, wts, bias, relu_y, out, N, Ho, Wo, Nout, pl.Kq, kh, kw, pl.TY, pl.TN, pl.HY, pl.HX,
               pl.tiles, pl.tiles_x, pl.tiles_y, pl.a_bytes, pl.w_bytes, relu, pl.stages,
               pow2_ge(2 * Nout / pl.ns, 32), pl.ns};
  Launch l;
  const void* f = (kh == 5 && kw == 5 && pl.Kq == 2)   ? (const void*)conv_plane_taps<5, 5, 1>
                  : (kh == 5 && kw == 5 && pl.Kq == 8)  ? (const void*)conv_plane_taps<5, 5, 4>
                  : (kh == 5 && kw == 5 && pl.Kq == 16) ? (const void*)conv_plane_taps<5, 5, 8>
                  : (kh == 3 && kw == 3 && pl.Kq == 8)  ? (const void*)conv_plane_taps<3, 3, 4>
                                                        : (const void*)conv_plane_taps<0, 0, 0>;
  int grid = std::max(pl.ns, std::min(pl.tiles * pl.ns, sms) / pl.ns * pl.ns);  // a multiple of ns
  if (const char* e = getenv("PN_PLANE_CTAS"))  // test hook: fewer CTAs, so small batches wrap the ring
    grid = std::max(1, std::min(grid / pl.ns, atoi(e))) * pl.ns;
  l.set(f, dim3((unsigned)grid), dim3(192), pl.smem, p);
  return l;
}
cudaError_t plane_setup() {
  cudaError_t e = cudaSuccess;
  for (const void* f : {(const void*)conv_plane_taps<5, 5, 1>, (const void*)conv_plane_taps<5, 5, 4>, (const void*)conv_plane_taps<5, 5, 8>,
                        (const void*)conv_plane_taps<3, 3, 4>, (const void*)conv_plane_taps<0, 0, 0>})
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kPlaneSmemMax + 1024));
  return e;
}

}  // namespace tcc
}  // namespace pn
