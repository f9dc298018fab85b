// tc_conv1.cu -- conv1 + pool1 of the fused LeNet TF32 plan on the tensor
// cores (SURVEY §8(a) rows a1 + a2; P:118-122 im2col + GEMM
// max pooling with stored origins).
//
// Implicit GEMM  D[m, f] = sum_k A[m, k] W[f, k]  over 128-row tiles:
//   m = 32 q + k for window slot q = 2*dh + dw of pooled position
//       P = 32 t + k = n*144 + ph*12 + pw -- the four conv outputs of one
//       2x2 pooling window sit in the four TMEM lane quadrants;
//   k = 5*i + j (25 taps, padded to 32), A[m, k] = x[n, 2ph+dh+i, 2pw+dw+j]:
//       the im2col row of P:122, written straight into TENSOR MEMORY by the
//       builder warps (tcgen05.st; the MMA reads A from TMEM) from the CTA's
//       images staged once in shared memory -- no shared-memory operand and
//       no proxy fence on the build path (a shared-memory A tile costs 16 KB
//       of stores + a fence per tile, which bounded the first version);
//   f = 20 filters padded to N = 32 (B = the TF32 weights, resident in
//       shared memory, SWIZZLE_128B K-major).
// Per tile 4 x tcgen05.mma M=128 N=32 K=8 (TF32); tiles go in batches of SUP
// with ONE commit per batch (a commit waits for the MMAs before it: ~300
// cycles, tools/mma_lat.cu), two batches in flight.  x and W are rounded to
// TF32 (nearest, ties away) once, when staged.  Bias is added after the sum
// (P:160-167), the 2x2 max keeps the first maximum in window scan order
// (strict >) and stores it TF32 rounded (its only consumers are
// conv2's contractions) with its uint8 window offset, NCHW (p1) and in
// conv2's tap-GEMM layout (p1c).
//
// Persistent CTAs over contiguous ranges of <= 16 tiles (<= 5 images):
//   all warps   prologue: stage the range's images (TF32) and W1 (B tile)
//   warp 0      MMA issuer (one thread)
//   warps 1-8   builders, two groups of 4 (warp w writes TMEM lane quadrant
//               w % 4 = window slot q of every position of its tiles): 25
//               shared loads + one tcgen05.st.32x32b.x32 per tile
//   warps 9-16  epilogue, two groups of 4 taking alternate batches:
//               TMEM -> bias -> shared staging -> 2x2 max / argmax -> stores
// TMEM: A tiles in columns [0, 32 ABUF), accumulators after them (256 columns at
// SUP 1 x NSET 4: conv2's forward CTAs then fit beside it and stage their
// weights during its tail -- 85.5 -> 84.6 µs/step vs 512 columns)
// Everything it reads was written two or more launches back (the input, the
// weights of the previous step's solver) and its immediate predecessor reads
// none of its outputs: the whole kernel runs before the PDL wait (pdl.cuh).
#include <algorithm>
#include <cstdint>

#include "kernels.h"
#include "pdl.cuh"
#include "tc.h"
#include "tc_ptx.cuh"

namespace pn {
namespace tc {
namespace c1 {
// warp 0: MMA issuer; warps 1-8: two builder groups; warps 9-16: two
// epilogue groups (group g takes the tiles it = g mod 2)
constexpr int WARPS = 17, THREADS = WARPS * 32;
#ifndef C1_SUP
#define C1_SUP 1
#endif
#ifndef C1_EARLY_TRIGGER
#define C1_EARLY_TRIGGER 1
#endif
#ifndef C1_NSET
#define C1_NSET 4
#endif
constexpr int SUP = C1_SUP;                 // tiles per MMA batch (one commit per batch)
constexpr int NSET = C1_NSET;               // batches in flight (A tiles and TMEM accumulators)
static_assert(SUP * NSET <= 8, "TMEM: A and D columns of SUP x NSET tiles");
constexpr int ABUF = SUP * NSET;            // A tiles in TMEM (32 columns each); as many accumulators
constexpr int D_OFF = 32 * ABUF;            // accumulator columns follow the A tiles
constexpr int TMEM_COLS = 2 * D_OFF <= 32 ? 32 : 2 * D_OFF <= 64 ? 64 : 2 * D_OFF <= 128 ? 128 : 2 * D_OFF <= 256 ? 256 : 512;
constexpr int B_BYTES = 32 * 128;           // 32 filter rows x 32 TF32
constexpr int MAXT = 16;                    // tiles per CTA
constexpr int MAXIMG = 5;                   // images a range of MAXT tiles can touch
constexpr int XS_FLOATS = MAXIMG * 784;
constexpr int S_PITCH = 128;                // epilogue staging S[tile][f][row] (floats)
constexpr int S_BYTES = 20 * S_PITCH * 4;   // one tile
constexpr int SMEM = B_BYTES + XS_FLOATS * 4 + 2 * 2 * SUP * S_BYTES + 1024;  // 2 groups x 2 sets x SUP tiles
static_assert(SMEM <= 227 * 1024, "shared memory");
}  // namespace c1

__device__ __forceinline__ float c1_in(const Conv1Pool1P& p, long long i) {
  if (!p.x8) return __ldg(p.x + i);
  const float v = __fmul_rn((float)__ldg(p.x8 + i), p.x_scale);
  return p.x_mean ? __fsub_rn(v, __ldg(p.x_mean + i % 784)) : v;
}
// four consecutive input values at base (a multiple of 4; pixel base % 784 =
// pix): one 16-B float load or one 4-B byte load, the same per-element
// normalisation as c1_in
__device__ __forceinline__ float4 c1_in4(const Conv1Pool1P& p, long long base, int pix) {
  if (!p.x8) return __ldg(reinterpret_cast<const float4*>(p.x + base));
  const uchar4 b = __ldg(reinterpret_cast<const uchar4*>(p.x8 + base));
  float4 v = make_float4(__fmul_rn((float)b.x, p.x_scale), __fmul_rn((float)b.y, p.x_scale),
                         __fmul_rn((float)b.z, p.x_scale), __fmul_rn((float)b.w, p.x_scale));
  if (p.x_mean) {
    const float4 m = __ldg(reinterpret_cast<const float4*>(p.x_mean + pix));
    v = make_float4(__fsub_rn(v.x, m.x), __fsub_rn(v.y, m.y), __fsub_rn(v.z, m.z), __fsub_rn(v.w, m.w));
  }
  return v;
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 ld_shared_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ bool r_epi_done(int warp, int lane) { return warp == 9 && lane == 0; }

__global__ void __launch_bounds__(c1::THREADS, 1) conv1_pool1_tc(const __grid_constant__ Conv1Pool1P p) {
  using namespace c1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  ST_BEGIN(ST_CONV1);
  // the step's first kernel: no programmatic predecessor (its wait below is
  // trivial), so let conv2's forward launch at once -- its CTAs take the SMs
  // these CTAs leave and stage W2 while the last conv1 tiles finish
  if (C1_EARLY_TRIGGER) pdl_trigger();
  const uint32_t B_s = smem_u32(smem), X_s = B_s + B_BYTES, S_s = X_s + XS_FLOATS * 4;
  // afull[set]: the batch's SUP tiles built (SUP warps arrive); mdone[set]:
  // its MMAs retired (one commit: frees the A tiles and fills the
  // accumulators -- each commit waits for the MMAs before it, so one per
  // batch of SUP x 4 MMAs); accfree[set]: the epilogue group has read them
  __shared__ __align__(8) uint64_t afull[NSET], mdone[NSET], accfree[NSET];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P_total = p.N * 144;  // (N < 2^24)
  const int T = (P_total + 31) / 32;
  const int t0 = blockIdx.x * p.per_block, mine = max(0, min(p.per_block, T - t0));
  const int n_lo = t0 * 32 / 144;
  const int n_hi = mine > 0 ? (min((t0 + mine) * 32, P_total) - 1) / 144 : n_lo - 1;
  if (tid == 0) {
    for (int s = 0; s < NSET; ++s) {
      mbar_init(smem_u32(&afull[s]), 4 * SUP);  // one arrival per builder warp and tile
      mbar_init(smem_u32(&mdone[s]), 1);
      mbar_init(smem_u32(&accfree[s]), 128);
    }
    fence_barrier_init();
  }
  if (tid == 0) stamp(0);
  if (warp == 0) tmem_alloc(&tmem_base, TMEM_COLS);
  // ---- prologue: the range's images (TF32) and the weight tile
  {
    const int nimg = n_hi - n_lo + 1, total = nimg * 784;
    const bool vec = ((reinterpret_cast<uintptr_t>(p.x8 ? (const void*)p.x8 : (const void*)p.x) &
                       (p.x8 ? 3 : 15)) == 0);
    if (vec) {  // 4 values per load (784 = 196 x 4: a group never straddles images)
      constexpr int PER4 = (MAXIMG * 196 + THREADS - 1) / THREADS;
      float4 v[PER4];
#pragma unroll
      for (int u = 0; u < PER4; ++u) {
        const int i4 = tid + THREADS * u;
        v[u] = 4 * i4 < total ? c1_in4(p, (long long)n_lo * 784 + 4 * i4, (4 * i4) % 784) : zero4();
      }
#pragma unroll
      for (int u = 0; u < PER4; ++u) {
        const int i4 = tid + THREADS * u;
        if (4 * i4 < total) sts128(X_s + 16 * i4, f4(tf32f(v[u].x), tf32f(v[u].y), tf32f(v[u].z), tf32f(v[u].w)));
      }
    } else {
      constexpr int PER = (MAXIMG * 784 + THREADS - 1) / THREADS;
      float v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = tid + THREADS * u;
        v[u] = i < total ? c1_in(p, (long long)n_lo * 784 + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = tid + THREADS * u;
        if (i < total) stsf(X_s + 4 * i, tf32f(v[u]));
      }
    }
    // B[f][k] = W[f, k] for f < 20, k < 25, else 0 (SW128, K-major)
    for (int u = tid; u < 32 * 8; u += THREADS) {
      const int f = u >> 3, kc = u & 7;
      float w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = 4 * kc + e;
        w[e] = (f < 20 && k < 25) ? tf32f(__ldg(p.w + f * 25 + k)) : 0.f;
      }
      sts128(B_s + sw_off(f, kc), f4(w[0], w[1], w[2], w[3]));
    }
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) stamp(1);
  if (tid == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = make_idesc(128, 32);
    const uint64_t bd0 = make_desc(B_s);  // K step of 8 TF32 = +32 B = +2 in the descriptor
    const int nb = (mine + SUP - 1) / SUP;
#pragma unroll 1
    for (int bt = 0; bt < nb; ++bt) {
      const int set = bt % NSET;
      mbar_wait(smem_u32(&afull[set]), (bt / NSET) & 1);
      if (bt >= NSET) mbar_wait(smem_u32(&accfree[set]), ((bt / NSET) - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < SUP; ++j) {  // tile j of the batch: A columns 32*(set*SUP + j), D 256 + the same
        const uint32_t a = tbase + (set * SUP + j) * 32, d = a + D_OFF;
        mma_tf32_ts<0>(d, a, bd0, idesc);
        mma_tf32_ts<1>(d, a + 8, bd0 + 2, idesc);
        mma_tf32_ts<1>(d, a + 16, bd0 + 4, idesc);
        mma_tf32_ts<1>(d, a + 24, bd0 + 6, idesc);
      }
      mma_commit(smem_u32(&mdone[set]));
      if (bt == 0) stamp(3);
    }
    stamp(5);
  } else if (warp >= 1 && warp < 9) {
    // ---- builders: group gb = (warp - 1) / 4 builds tiles j = gb, gb + 2 of
    // every batch; warp w writes lane quadrant q = w % 4 (window slot q =
    // (dh, dw)) for the 32 positions k = lane: the 5x5 window (25 shared
    // loads) + 7 zeros as one 32-column TMEM row
    const int q = warp & 3, dh = q >> 1, dw = q & 1, gb = (warp - 1) >> 2;
    const int nb = (mine + SUP - 1) / SUP;
#pragma unroll 1
    for (int it = gb; it < nb * SUP; it += 2) {  // group gb: tiles it = gb (mod 2) (a short last batch: arrive only)
      const int bt = it / SUP, set = bt % NSET, j = it % SUP;
      if (bt >= NSET) mbar_wait(smem_u32(&mdone[set]), ((bt / NSET) - 1) & 1);  // batch bt - NSET is done with A
      {
        const int P = (t0 + it) * 32 + lane;
        uint32_t a[32];
        if (it < mine && P < P_total) {
          const int n = P / 144, pq = P - n * 144, ph = pq / 12, pw = pq - 12 * ph;
          const uint32_t xb = X_s + 4 * ((n - n_lo) * 784 + (2 * ph + dh) * 28 + 2 * pw + dw);
#pragma unroll
          for (int k = 0; k < 25; ++k) a[k] = __float_as_uint(ldsf_nc(xb + 4 * ((k / 5) * 28 + k % 5)));
        } else {
#pragma unroll
          for (int k = 0; k < 25; ++k) a[k] = 0u;
        }
#pragma unroll
        for (int k = 25; k < 32; ++k) a[k] = 0u;
        tmem_st32(tbase + ((uint32_t)(q * 32) << 16) + (set * SUP + j) * 32, a);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[set])) : "memory");
        if (lane == 0 && it == 0) stamp(2);
      }
    }
    if (lane == 0 && warp == 1) stamp(4);
  } else if (warp >= 9) {
    // ---- epilogue, per batch (one TMEM wait and one named barrier for its
    // SUP tiles): (1) thread = TMEM lane (tile row r) of its quadrant: the
    // row's 20 biased conv values of every tile -> S[tile][f][r] (two sets
    // per group); (2) the same thread (quadrant q, lane k) takes position k
    // and filters 5q .. 5q+4 of each tile: the four window values of each
    // (rows k, 32+k, 64+k, 96+k), the first maximum in window scan order
    // (strict >) -> p1 / m1 (lanes: consecutive positions) and p1c.
    const int quad = warp & 3, r = quad * 32 + lane, g = (warp - 9) >> 2;
    float bias[20];
#pragma unroll
    for (int f = 0; f < 20; ++f) bias[f] = __ldg(p.b + f);
    const int nb = (mine + SUP - 1) / SUP;
    int step = 0;
#pragma unroll 1
    for (int bt = g; bt < nb; bt += 2, ++step) {
      const int set = bt % NSET;
      mbar_wait(smem_u32(&mdone[set]), (bt / NSET) & 1);
      if (r == 0 && bt == 0) stamp(6);
      __syncwarp();
      tc_fence_after();
      // the batch's SUP accumulators (20 columns each), one wait, then free them
      float v[SUP][20];
#pragma unroll
      for (int j = 0; j < SUP; ++j) {
        const uint32_t ta = tbase + ((uint32_t)(quad * 32) << 16) + D_OFF + (set * SUP + j) * 32;
        tmem_ld16_nowait(ta, *reinterpret_cast<float(*)[16]>(&v[j][0]));
        tmem_ld4_nowait(ta + 16, *reinterpret_cast<float(*)[4]>(&v[j][16]));
      }
      tmem_ld_wait();
      tc_fence_before();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[set])) : "memory");
      const uint32_t Sg = S_s + (2 * g + (step & 1)) * SUP * S_BYTES;  // [tile][f][row], two sets per group
#pragma unroll
      for (int j = 0; j < SUP; ++j)
#pragma unroll
        for (int f = 0; f < 20; ++f) stsf(Sg + 4 * ((j * 20 + f) * S_PITCH + r), v[j][f] + bias[f]);
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
      // thread (quadrant q, lane k): position k of each tile, filters 5q .. 5q+4
#pragma unroll 1
      for (int j = 0; j < SUP; ++j) {
        const int it = bt * SUP + j, P = (t0 + it) * 32 + lane;
        if (it >= mine || P >= P_total) continue;
        const int n = P / 144, pq = P - n * 144, ph = pq / 12, pw = pq - 12 * ph;
        float* p1o = p.p1 + (size_t)(n * 20) * 144 + pq;
        uint8_t* m1o = p.m1 + (size_t)(n * 20) * 144 + pq;
        float* pco = p.p1c ? p.p1c + ((size_t)(n >> 1) * 1440 + ph * 24 + (n & 1) * 12 + pw) * 4 : nullptr;
        const uint32_t Sb = Sg + 4 * (j * 20 * S_PITCH + lane);
#pragma unroll
        for (int e = 0; e < 5; ++e) {
          const int f = 5 * quad + e;
          // window slots 0..3 are rows k, 32+k, 64+k, 96+k; first maximum in scan order
          const float w0 = ldsf_nc(Sb + 4 * (f * S_PITCH)), w1 = ldsf_nc(Sb + 4 * (f * S_PITCH + 32));
          const float w2 = ldsf_nc(Sb + 4 * (f * S_PITCH + 64)), w3 = ldsf_nc(Sb + 4 * (f * S_PITCH + 96));
          float best = w0;
          int off = 0;
          if (w1 > best) { best = w1; off = 1; }
          if (w2 > best) { best = w2; off = 2; }
          if (w3 > best) { best = w3; off = 3; }
          if (p.round_tf32) best = tf32f(best);
          p1o[f * 144] = best;
          m1o[f * 144] = (uint8_t)off;
          if (pco) pco[(f >> 2) * 12 * 24 * 4 + (f & 3)] = best;  // [pair][cc][h][n][w][4 c]
        }
      }
    }
  }
  if (r_epi_done(warp, lane)) stamp(7);
  tc_fence_before();
  __syncthreads();
  if (tid == 0) stamp(8);
  pdl_enter_k(ST_CONV1);
  ST_END(ST_CONV1);
  if (warp == 0) tmem_dealloc(tbase, TMEM_COLS);
}

PN_STEPTRACE_TU(st_set_c1)

cudaError_t conv1_setup() {
  return cudaFuncSetAttribute((const void*)conv1_pool1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, c1::SMEM);
}

Launch conv1_pool1_tc_launch(const Conv1Pool1P& p0, int sms) {
  Conv1Pool1P p = p0;
  const long long T = ((long long)p.N * 144 + 31) / 32;
  int grid = (int)std::min<long long>(T, sms);
  int per = (int)((T + grid - 1) / grid);
  if (per > c1::MAXT) {
    per = c1::MAXT;
    grid = (int)((T + per - 1) / per);
  }
  p.per_block = per;
  Launch l;
  l.set((const void*)conv1_pool1_tc, dim3(grid), dim3(c1::THREADS), c1::SMEM, p);
  return l;
}

}  // namespace tc
}  // namespace pn
