// tc.cu -- tcgen05 TF32 kernels for the GEMM-shaped LeNet layers (SURVEY
// §8(a) rows a3/a4, a5/a6, a12/a13, a14) and the per-step TF32 weight packing.
//
// Common ground (the kernels below are warp-specialised variations on it):
//   * every operand lives in shared memory in a UMMA K-major layout: the
//     canonical SWIZZLE_128B one (row = 128 B of K, 16-B chunk index XOR
//     row%8, 8-row atoms of 1 KB; SBO = 1 KB, K step of 8 = +32 B) when TMA
//     delivers it, or the no-swizzle core-matrix one (8 rows x 16 B; LBO /
//     SBO free) when a shifted descriptor must address a tap of a staged
//     image (conv2's forward and data gradient).  MN-major TF32 descriptors
//     were measured to produce zeros on this part (tools/umma_probe.cu);
//   * operands are already TF32 in memory: packed weight copies
//     (pack_weights) and activations rounded to nearest by their producers
//      -- the tensor core never truncates;
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::tf32 (M=128,
//     K=8) into TMEM accumulators and tcgen05.commit's stages back through
//     mbarriers; TMA / bulk-copy producers, gather / build warps and TMEM
//     epilogue warps (tcgen05.ld 32x32b, thread = tile row) run beside it;
//   * kernels launch with programmatic dependent launch (pdl.cuh): inputs
//     from two or more launches back are requested before the dependency
//     wait.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "pdl.cuh"
#include "reduce.cuh"
#include "sgd.cuh"
#include "solver.cuh"
#include "tc.h"
#include "tc_ptx.cuh"

namespace pn {
namespace tc {

// ================================================= ip1 GEMMs: 128 x 32 tiles, K split in two
// C[M,N] = A[M,K] B[N,K]^T (both K-major TF32 by TMA, SW128).  One cluster
// of two CTAs per 128 x 32 tile, CTA r taking half of K:
//   warp 0      TMA producer: a STAGES-deep ring -- operands produced two or
//               more launches back are requested before the PDL wait, the
//               rest after it
//   warp 1      MMA: 4 x tcgen05.mma (M=128, N=32, K=8) per chunk into TMEM
//   warps 2-5   TMEM -> shared-memory partial tile C[128][33]
// then (cluster barrier) CTA r owns rows [64r, 64r+64): partial 0 + partial 1
// (fixed order; the peer's half read over DSMEM: 8 KB) and applies the
// layer's epilogue (bias+ReLU / dW / pool2 backward) to them, two threads per
// row.  Few tiles (M = 512 images, N <= 800) and an L2 ingest of ~40 B/clk
// per SM (B300_MICROARCH: LTS cap ~6300 B/clk over 148 SMs) make the per-CTA
// operand bytes the cost: the split halves them, and the 8-KB exchange is
// the cheapest reduction (a 128 x 128 split-K tile over DSMEM at ~20 B/clk
// was the bottleneck of the previous design).
// ring depths (compile-time knobs for A/B builds, tools/ab_build.sh)
#ifndef IPF_STAGES
#define IPF_STAGES 4
#endif
#ifndef IPG_STAGES
#define IPG_STAGES 5
#endif
#ifndef IPD_STAGES
#define IPD_STAGES 4  // (5 -> 4 with the 64-wide weight-gradient tiles: a data- and a weight-gradient CTA then share an SM; 80.7 -> 80.1 us/step)
#endif
#ifndef WG_SLOTS
#define WG_SLOTS 6
#endif
#ifndef WG_ABUF
#define WG_ABUF 2  // conv2 weight gradient: A tiles in flight (A/B: 3-4 with fewer image slots measured slower)
#endif
#ifndef PACK_GRID
#define PACK_GRID 0  // weight-pack blocks (0: one per W1 tile)
#endif
#ifndef IPF_SPLIT
#define IPF_SPLIT 4
#endif
#ifndef IPF_BN
#define IPF_BN 64
#endif
#ifndef IPD_SPLIT
#define IPD_SPLIT 1
#endif
#ifndef IPD_BN
#define IPD_BN 32
#endif
#ifndef IPG_SPLIT
#define IPG_SPLIT 1
#endif
// column tiles per cluster sharing (TMA multicast) each A chunk of the ip1
// weight / data gradients (1: every CTA loads its own)
#ifndef IPG_MC
#define IPG_MC 1
#endif
#ifndef IPD_MC
#define IPD_MC 1
#endif
#ifndef IPG_BN
#define IPG_BN 64  // (32 -> 64: 82.1 -> 80.6 us/step, same-box A/B x4: half the weight-gradient CTAs beside the data gradient)
#endif
namespace ipk {
constexpr int THREADS = 192;
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_cluster4(uint32_t local_addr, uint32_t rank) {
  uint32_t a;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local_addr), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// TMA 2-D box multicast to the CTAs of `mask` in the cluster (same smem
// offset, complete_tx on each one's mbarrier at the same offset)
__device__ __forceinline__ void tma2d_mc(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar,
                                         uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
      : "memory");
}
// tcgen05.commit arriving on the mbarrier at `bar`'s offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   bar),
               "h"(mask)
               : "memory");
}
}  // namespace ipk

template <class Op>
__global__ void __launch_bounds__(ipk::THREADS, 1) ip_tile(const __grid_constant__ typename Op::Params prm) {
  using namespace ipk;
  constexpr int BN = Op::BN, CPB = BN + 4;  // tile width, C pitch (floats; rows 16-B aligned)
  // Op::X3 (3xTF32): each operand chunk staged as hi and lo copies (A_hi A_lo B_hi B_lo)
  constexpr int X = Op::X3 ? 2 : 1;
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = X * (A_BYTES + B_BYTES), STAGES = Op::STAGES;
  static_assert(128 * CPB * 4 <= STAGES * STAGE, "C fits the ring");
  static_assert(BN == 32 || BN == 64 || BN == 128, "tile width");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  __shared__ float red[Op::RED_FLOATS + 1];
  __shared__ __align__(16) uint8_t epi_s[Op::EPI_BYTES + 16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int SPLIT = Op::SPLIT, ROWS = 128 / SPLIT;  // K split over a cluster of SPLIT CTAs, or the whole K
  const uint32_t rank = SPLIT > 1 ? cluster_rank() : 0u;  // cluster = (SPLIT, 1, 1): blockIdx.x = SPLIT * column + rank
  // Op::MC > 1: a cluster of MC column tiles (same rows) shares each A chunk --
  // chunk c loaded by CTA c % MC and multicast to all; each stage is freed by
  // all MC consumers (their MMA commits arrive on every CTA's empty barrier)
  constexpr int MC = Op::MC;
  static_assert(MC == 1 || SPLIT == 1, "A multicast with a split K cluster");
  const uint32_t mrank = MC > 1 ? cluster_rank() : 0u;
  constexpr uint16_t MMASK = (uint16_t)((1u << MC) - 1);
  Op op(prm);
  const int nk = op.num_k_chunks(), c0 = (int)rank * nk / SPLIT, my = ((int)rank + 1) * nk / SPLIT - c0;
  const uint32_t sbase = smem_u32(smem);
  ST_BEGIN(Op::ST);
  if (tid == 0) {
    for (int c = 0; c < STAGES; ++c) {
      mbar_init(smem_u32(&full[c]), 1);
      mbar_init(smem_u32(&empty[c]), MC);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
    op.prefetch();
  }
  if (warp == 0) tmem_alloc(&tmem_base, BN);
  op.stage_epilogue(tid, epi_s, (int)rank);  // epilogue inputs from >= 2 launches back
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync();  // every CTA's barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) stamp(0);
  if (tid == 0) {
    const int pre = min(my, STAGES);
    for (int c = 0; c < pre; ++c) {
      const uint32_t As = sbase + c * STAGE, bar = smem_u32(&full[c]);
      mbar_expect_tx(bar, STAGE);
      if (Op::A_EARLY && (MC == 1 || (c0 + c) % MC == (int)mrank)) op.issue_a_mc(c0 + c, As, bar, MMASK);
      if (Op::B_EARLY) op.issue_b(c0 + c, As + X * A_BYTES, bar);
    }
    pdl_enter_k(Op::ST);
    stamp(1);
    for (int c = 0; c < pre; ++c) {
      const uint32_t As = sbase + c * STAGE, bar = smem_u32(&full[c]);
      if (!Op::A_EARLY && (MC == 1 || (c0 + c) % MC == (int)mrank)) op.issue_a_mc(c0 + c, As, bar, MMASK);
      if (!Op::B_EARLY) op.issue_b(c0 + c, As + X * A_BYTES, bar);
    }
    for (int c = STAGES; c < my; ++c) {
      const int st = c % STAGES;
      mbar_wait(smem_u32(&empty[st]), ((c / STAGES) - 1) & 1);
      const uint32_t As = sbase + st * STAGE, bar = smem_u32(&full[st]);
      mbar_expect_tx(bar, STAGE);
      if (MC == 1 || (c0 + c) % MC == (int)mrank) op.issue_a_mc(c0 + c, As, bar, MMASK);
      op.issue_b(c0 + c, As + X * A_BYTES, bar);
    }
  } else if (tid == 32) {
    constexpr uint32_t idesc = make_idesc(128, BN);
    for (int c = 0; c < my; ++c) {
      const int st = c % STAGES;
      mbar_wait(smem_u32(&full[st]), (c / STAGES) & 1);
      tc_fence_after();
      const uint32_t As = sbase + st * STAGE, Bs = As + X * A_BYTES;
      if constexpr (Op::X3) {  // A_lo B_hi + A_hi B_lo + A_hi B_hi (the A_lo B_lo term dropped)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mma_tf32(tbase, make_desc(As + A_BYTES + k * 32), make_desc(Bs + k * 32), idesc, (c | k) != 0);
          mma_tf32_c<1>(tbase, make_desc(As + k * 32), make_desc(Bs + B_BYTES + k * 32), idesc);
          mma_tf32_c<1>(tbase, make_desc(As + k * 32), make_desc(Bs + k * 32), idesc);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_tf32(tbase, make_desc(As + k * 32), make_desc(Bs + k * 32), idesc, (c | k) != 0);
      }
      if (MC > 1) mma_commit_mc(smem_u32(&empty[st]), MMASK);
      else mma_commit(smem_u32(&empty[st]));
    }
    if (my > 0) mma_commit(smem_u32(&done));
  } else if (warp >= 2) {
    // TMEM -> C over the drained ring (all MMAs retired)
    const int quad = warp & 3, row = quad * 32 + lane;
    if (my > 0) {
      mbar_wait(smem_u32(&done), 0);
      if (warp == 2 && lane == 0) stamp(2);
      __syncwarp();
      tc_fence_after();
    }
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if (my > 0) {
        tmem_ld16_nowait(tbase + ((uint32_t)(quad * 32) << 16) + c0, *reinterpret_cast<float(*)[16]>(v));
        tmem_ld16_nowait(tbase + ((uint32_t)(quad * 32) << 16) + c0 + 16, *reinterpret_cast<float(*)[16]>(v + 16));
        tmem_ld_wait();
      } else {  // an empty K slice (tiny K): a zero partial
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 4) sts128(sbase + 4 * (row * CPB + c0 + j), f4(v[j], v[j + 1], v[j + 2], v[j + 3]));
    }
  }
  tc_fence_before();
  if (SPLIT > 1) {
    cluster_sync();  // every partial tile of the cluster complete
    if (tid == 0) stamp(3);
    // rows [ROWS rank, +ROWS): the SPLIT partials summed in rank order, in
    // place in the local C (no other CTA reads this CTA's own rows); float4
    // DSMEM loads, every source of an item in flight together
    for (int u = tid; u < ROWS * BN / 4; u += THREADS) {
      const int r = ROWS * (int)rank + u / (BN / 4), col = 4 * (u % (BN / 4));
      const uint32_t addr = sbase + 4 * (r * CPB + col);
      float4 t[SPLIT];
#pragma unroll
      for (int q = 0; q < SPLIT; ++q) t[q] = ld_cluster4(addr, (uint32_t)q);  // (the own rank: a local address)
      float4 acc = t[0];
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) acc.x += t[q].x, acc.y += t[q].y, acc.z += t[q].z, acc.w += t[q].w;
      sts128(addr, acc);
    }
    cluster_sync();  // the other CTAs' reads of this CTA's C are done; local sums visible
  } else {
    __syncthreads();
  }
  // the layer's epilogue: BN / 16 threads per owned row, 16 columns each
  for (int u = tid; u < (BN / 16) * ROWS; u += THREADS) {
    const int rr = u % ROWS, half = u / ROWS, r = ROWS * (int)rank + rr;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = ldsf_nc(sbase + 4 * (r * CPB + 16 * half + j));
    op.store(r, rr, half, v, red, epi_s);
  }
  __syncthreads();
  if (tid == 0) stamp(4);
  op.finish(tid, red, (int)rank);
  ST_END(Op::ST);
  if (MC > 1) cluster_sync();  // no CTA leaves while a peer's MMA commits may still arrive on its barriers
  if (warp == 0) tmem_dealloc(tbase, BN);
}

// y[n,o] = relu(sum_k p2[n,k] W1[o,k] + b[o]): rows n, cols o (16 tiles of
// 32), K = 800 (25 chunks).  A = p2 (TF32, from conv2 -- the immediate
// predecessor), B = W1f (packed at the start of the step).
struct IpFwd {
  struct Params {
    CUtensorMap ta, tb;
    const float* b;
    float* y;
    int M, K, Nout;
  };
  static constexpr int RED_FLOATS = 0, STAGES = IPF_STAGES, EPI_BYTES = 0, SPLIT = IPF_SPLIT, BN = IPF_BN;
  static constexpr bool A_EARLY = false, B_EARLY = true, X3 = false;
  static constexpr int ST = ST_IPF;
  const Params& p;
  int m0, o0;
  __device__ IpFwd(const Params& q) : p(q), m0(blockIdx.y * 128), o0((blockIdx.x / SPLIT) * BN) {}
  __device__ int num_k_chunks() const { return (p.K + BK - 1) / BK; }
  __device__ void prefetch() { prefetch_tmap(&p.ta); prefetch_tmap(&p.tb); }
  static constexpr int MC = 1;
  __device__ void issue_a_mc(int c, uint32_t s, uint32_t bar, uint16_t) { tma2d(s, &p.ta, c * BK, m0, bar); }
  __device__ void issue_b(int c, uint32_t s, uint32_t bar) { tma2d(s, &p.tb, c * BK, o0, bar); }
  __device__ void stage_epilogue(int, uint8_t*, int) {}
  __device__ void store(int row, int, int half, const float (&v)[16], float*, const uint8_t*) const {
    const int m = m0 + row;
    if (m >= p.M) return;
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      const int o = o0 + 16 * half + c;
      if (o >= p.Nout) break;  // Nout % 4 == 0
      float4 r = f4(v[c] + __ldg(p.b + o), v[c + 1] + __ldg(p.b + o + 1), v[c + 2] + __ldg(p.b + o + 2),
                    v[c + 3] + __ldg(p.b + o + 3));
      r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f); r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
      *reinterpret_cast<float4*>(p.y + (size_t)m * p.Nout + o) = r;
    }
  }
  __device__ void finish(int, const float*, int) const {}
};

// dW1[o,k] = sum_n da1[n,o] p2[n,k]: rows o (4 tiles), cols k (25 tiles of
// 32), K = batch.  A = da1^T (da1rT [500][npad], TF32, from ip2 backward =
// the immediate predecessor), B = p2^T (p2T, from conv2).  The bias gradient
// comes from the ip2 backward kernel (exact fp32).
struct IpWgrad {
  struct Params {
    CUtensorMap ta, tb;
    float* dw;
    int M, K, Nout;  // M = batch (contraction), K = 800 (cols), Nout = 500 (rows)
  };
  static constexpr int RED_FLOATS = 0, STAGES = IPG_STAGES, EPI_BYTES = 0, SPLIT = IPG_SPLIT, BN = IPG_BN;
  static constexpr bool A_EARLY = false, B_EARLY = true, X3 = false;
  static constexpr int ST = ST_IPG;
  const Params& p;
  int o0, k0;
  __device__ IpWgrad(const Params& q) : p(q), o0(blockIdx.y * 128), k0((blockIdx.x / SPLIT) * BN) {}
  __device__ int num_k_chunks() const { return (p.M + BK - 1) / BK; }
  __device__ void prefetch() { prefetch_tmap(&p.ta); prefetch_tmap(&p.tb); }
  static constexpr int MC = IPG_MC;
  __device__ void issue_a_mc(int c, uint32_t s, uint32_t bar, uint16_t mask) {
    if (MC > 1) ipk::tma2d_mc(s, &p.ta, c * BK, o0, bar, mask);
    else tma2d(s, &p.ta, c * BK, o0, bar);
  }
  __device__ void issue_b(int c, uint32_t s, uint32_t bar) { tma2d(s, &p.tb, c * BK, k0, bar); }
  __device__ void stage_epilogue(int, uint8_t*, int) {}
  __device__ void store(int row, int, int half, const float (&v)[16], float*, const uint8_t*) const {
    const int o = o0 + row;
    if (o >= p.Nout) return;
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      const int k = k0 + 16 * half + c;
      if (k < p.K) *reinterpret_cast<float4*>(p.dw + (size_t)o * p.K + k) = f4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
  }
  __device__ void finish(int, const float*, int) const {}
};

// dp2[n,k] = sum_o da1[n,o] W1[o,k]: rows n, cols k (25 tiles of 32 = 2
// filters x 16 pooled outputs), K = o (500 -> 512).  A = da1 (TF32 copy
// [N][500]), B = W1t [800][512] -- neither comes from the immediate
// predecessor (the ip bucket reduce), so all loads precede the PDL wait.
// Epilogue (thread = (image n, filter)): the filter's 16 dp2 values go to
// their pool2 origins in the dense conv2 gradient G2[n,f,8,8] (zeros
// elsewhere), stored TF32-rounded (its only consumers are conv2's
// contractions); the exact dp2 sum per filter over the CTA's 64 rows (fixed
// order) is the conv2 bias-gradient partial part_db2[row tile * 2 + rank][f].
struct IpDgradUnpool {
  struct Params {
    CUtensorMap ta, tb;
    const uint8_t* m2;  // [N,800]
    float* g2;          // [N,50,8,8]
    float* part_db2;    // [row tiles * 2][50]
    int N;
  };
  static constexpr int SPLIT = IPD_SPLIT, ROWS = 128 / SPLIT, STAGES = IPD_STAGES, BN = IPD_BN, FT = BN / 16;
  static constexpr int RED_FLOATS = FT * ROWS;  // red: [filter in tile][owned row]
  static constexpr int EPI_BYTES = ROWS * BN;   // the owned rows' pool2 origins [row][FT x 16]
  static constexpr bool A_EARLY = !FORK_PDL, B_EARLY = true, X3 = false;  // (FORK_PDL: da1r from the immediate predecessor)
  static constexpr int ST = ST_IPD;
  const Params& p;
  int m0, k0;
  __device__ IpDgradUnpool(const Params& q) : p(q), m0(blockIdx.y * 128), k0((blockIdx.x / SPLIT) * BN) {}
  __device__ int num_k_chunks() const { return 16; }  // 500 -> 512
  __device__ void prefetch() { prefetch_tmap(&p.ta); prefetch_tmap(&p.tb); }
  static constexpr int MC = IPD_MC;
  __device__ void issue_a_mc(int c, uint32_t s, uint32_t bar, uint16_t mask) {
    if (MC > 1) ipk::tma2d_mc(s, &p.ta, c * BK, m0, bar, mask);
    else tma2d(s, &p.ta, c * BK, m0, bar);
  }
  __device__ void issue_b(int c, uint32_t s, uint32_t bar) { tma2d(s, &p.tb, c * BK, k0, bar); }
  __device__ void stage_epilogue(int tid, uint8_t* es, int rank) {  // conv2's forward wrote them, many launches back
    for (int u = tid; u < FT * ROWS; u += ipk::THREADS) {
      const int rr = u % ROWS, half = u / ROWS, n = m0 + ROWS * rank + rr;
      uint4 m = make_uint4(0, 0, 0, 0);
      if (n < p.N && k0 + 16 * half < 800) m = __ldg(reinterpret_cast<const uint4*>(p.m2 + (size_t)n * 800 + k0) + half);
      reinterpret_cast<uint4*>(es)[rr * FT + half] = m;
    }
  }
  __device__ void store(int row, int rr, int half, const float (&v)[16], float* red, const uint8_t* es) const {
    const int n = m0 + row, f = (k0 >> 4) + half;
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) sum += v[q];
    red[half * ROWS + rr] = n < p.N ? sum : 0.f;
    if (n >= p.N || f >= 50) return;
    const uint4 mk = reinterpret_cast<const uint4*>(es)[rr * FT + half];
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
    float* g = p.g2 + ((size_t)n * 50 + f) * 64;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      float o8[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int q = (h >> 1) * 4 + (w >> 1);
        const int off = (mw[q >> 2] >> (8 * (q & 3))) & 0xff;
        o8[w] = (off == ((h & 1) * 2 + (w & 1))) ? tf32f(v[q]) : 0.f;
      }
      *reinterpret_cast<float4*>(g + h * 8) = f4(o8[0], o8[1], o8[2], o8[3]);
      *reinterpret_cast<float4*>(g + h * 8 + 4) = f4(o8[4], o8[5], o8[6], o8[7]);
    }
  }
  __device__ void finish(int tid, const float* red, int rank) const {
    const int f = (k0 >> 4) + tid;
    if (tid < FT && f < 50) {  // fixed-order sum over the CTA's rows
      float s = 0.f;
      for (int r = 0; r < ROWS; ++r) s += red[tid * ROWS + r];
      p.part_db2[((size_t)blockIdx.y * SPLIT + rank) * 50 + f] = s;
    }
  }
};

// ---------------------------- ip1 at fp32 class: 3xTF32 on the tensor cores
// The fp32 plan's PN_3XTF32 variant of the three ip1 contractions: every
// operand x is split once per step (split3) into hi = x with its 13 low
// mantissa bits cleared (exact in TF32) and lo = TF32(x - hi) (x - hi is
// exact in fp32), and the tile accumulates A_lo B_hi + A_hi B_lo + A_hi B_hi
// in TMEM (fp32); the dropped A_lo B_lo and the rounding of lo are below
// 2^-20 |a b| per product, the fp32 class (R21).  Same tiles,
// rings and epilogues as the TF32 Ops, each chunk staged as hi + lo copies.
struct Ip3Fwd {  // y = relu(p2 W1^T + b): IpFwd's tiles (K split over a cluster)
  struct Params {
    CUtensorMap ta, tal, tb, tbl;
    const float* b;
    float* y;
    int M, K, Nout;
  };
  static constexpr int RED_FLOATS = 0, STAGES = 4, EPI_BYTES = 0, SPLIT = IPF_SPLIT, BN = IPF_BN;
  static constexpr bool A_EARLY = false, B_EARLY = true, X3 = true;
  static constexpr int ST = ST_IPF;
  const Params& p;
  int m0, o0;
  __device__ Ip3Fwd(const Params& q) : p(q), m0(blockIdx.y * 128), o0((blockIdx.x / SPLIT) * BN) {}
  __device__ int num_k_chunks() const { return (p.K + BK - 1) / BK; }
  __device__ void prefetch() { prefetch_tmap(&p.ta); prefetch_tmap(&p.tal); prefetch_tmap(&p.tb); prefetch_tmap(&p.tbl); }
  static constexpr int MC = 1;
  __device__ void issue_a_mc(int c, uint32_t s, uint32_t bar, uint16_t) {
    tma2d(s, &p.ta, c * BK, m0, bar);
    tma2d(s + 128 * 128, &p.tal, c * BK, m0, bar);
  }
  __device__ void issue_b(int c, uint32_t s, uint32_t bar) {
    tma2d(s, &p.tb, c * BK, o0, bar);
    tma2d(s + BN * 128, &p.tbl, c * BK, o0, bar);
  }
  __device__ void stage_epilogue(int, uint8_t*, int) {}
  __device__ void store(int row, int, int half, const float (&v)[16], float*, const uint8_t*) const {
    const int m = m0 + row;
    if (m >= p.M) return;
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      const int o = o0 + 16 * half + c;
      if (o >= p.Nout) break;
      float4 r = f4(v[c] + __ldg(p.b + o), v[c + 1] + __ldg(p.b + o + 1), v[c + 2] + __ldg(p.b + o + 2),
                    v[c + 3] + __ldg(p.b + o + 3));
      r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f); r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
      *reinterpret_cast<float4*>(p.y + (size_t)m * p.Nout + o) = r;
    }
  }
  __device__ void finish(int, const float*, int) const {}
};
// dW1 = da1^T p2 (K = batch) and dp2 = da1 W1 (K = 500 -> 512): rows r0 + row,
// 16 columns per call, out[r][c] fp32 (row pitch ldo)
struct Ip3Grad {
  struct Params {
    CUtensorMap ta, tal, tb, tbl;
    float* out;
    int rows, cols, ldo, nk;  // output rows / cols, K chunks of 32
  };
  static constexpr int RED_FLOATS = 0, STAGES = 5, EPI_BYTES = 0, SPLIT = 1, BN = 32;
  static constexpr bool A_EARLY = false, B_EARLY = false, X3 = true;
  static constexpr int ST = ST_IPG;
  const Params& p;
  int r0, c0;
  __device__ Ip3Grad(const Params& q) : p(q), r0(blockIdx.y * 128), c0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return p.nk; }
  __device__ void prefetch() { prefetch_tmap(&p.ta); prefetch_tmap(&p.tal); prefetch_tmap(&p.tb); prefetch_tmap(&p.tbl); }
  static constexpr int MC = 1;
  __device__ void issue_a_mc(int c, uint32_t s, uint32_t bar, uint16_t) {
    tma2d(s, &p.ta, c * BK, r0, bar);
    tma2d(s + 128 * 128, &p.tal, c * BK, r0, bar);
  }
  __device__ void issue_b(int c, uint32_t s, uint32_t bar) {
    tma2d(s, &p.tb, c * BK, c0, bar);
    tma2d(s + BN * 128, &p.tbl, c * BK, c0, bar);
  }
  __device__ void stage_epilogue(int, uint8_t*, int) {}
  __device__ void store(int row, int, int half, const float (&v)[16], float*, const uint8_t*) const {
    const int r = r0 + row;
    if (r >= p.rows) return;
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      const int k = c0 + 16 * half + c;
      if (k < p.cols) *reinterpret_cast<float4*>(p.out + (size_t)r * p.ldo + k) = f4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
  }
  __device__ void finish(int, const float*, int) const {}
};
// hi / lo copies of src [R][C] (and transposed [C][ldt]); null outputs
// skipped.  32 x 32 tiles: coalesced reads and row-major writes, the
// transposes through a padded shared tile (coalesced writes too).
__global__ void __launch_bounds__(256) split3(const __grid_constant__ Split3P p) {
  __shared__ float th[32][33], tl[32][33];
  pdl_enter();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = r0 + ty + 8 * k, c = c0 + tx;
    float hi = 0.f, lo = 0.f;
    if (r < p.R && c < p.C) {
      const float x = __ldg(p.src + (size_t)r * p.C + c);
      hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      lo = tf32f(x - hi);
      if (p.hi) p.hi[(size_t)r * p.C + c] = hi, p.lo[(size_t)r * p.C + c] = lo;
    }
    th[ty + 8 * k][tx] = hi, tl[ty + 8 * k][tx] = lo;
  }
  if (!p.hiT) return;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c0 + ty + 8 * k, r = r0 + tx;
    if (c < p.C && r < p.R) {
      p.hiT[(size_t)c * p.ldt + r] = th[tx][ty + 8 * k];
      p.loT[(size_t)c * p.ldt + r] = tl[tx][ty + 8 * k];
    }
  }
}

// ------------------------- conv2 + bias + pool2 (+mask), persistent tap GEMM
// conv2 as 25 tap GEMMs accumulated in TMEM, with NO im2col:
//   D[(ho,n,wo), f] = sum_{i,j} sum_c p1[n,c,ho+i,wo+j] W2[f,c,i,j]
// The pooled layer-1 output of an image pair is stored (by conv1+pool1, TF32)
// as p1c[pair][cc 5][h 12][n 2][w 12][4 c]: 4-channel planes of 16-B pixels.
// In the UMMA K-major no-swizzle layout (core matrix = 8 rows x 16 B,
// LBO = K-direction core-matrix stride, SBO = 8-row-group stride) the A
// operand of tap (i,j) is then just a descriptor into that staged pair:
//   rows r = (ho, n, wo) (8-row group = (ho, n), SBO = 192 B = one (h, n) row
//   of 12 pixels), K = 24 channels (5 stored planes + 1 zero plane,
//   LBO = 4608 B = one plane), start = pair + (i*24 + j)*16 B.
// B = all 25 taps of W2 resident in shared memory as w2c[tap][cc 5][f 50][4 c]
// (exactly W2's 25000 values, 100 KB, loaded once per CTA): rows f at 16 B
// (SBO 128), planes at LBO = 800 B.  The N = 64 MMA also reads rows 50..63
// (the next plane's first rows: finite values into ignored columns) and a 6th
// plane (the next tap's first plane, or a zero pad) against A's zero plane.
// Per pair: 25 taps x 3 MMAs (M=128, N=64, K=8).
// Persistent, pairs split evenly over the CTAs: warp 0 = bulk-copy producer
// (weights in 5 pieces, then a 3-stage pair ring), warp 1 = MMA issuer (2
// TMEM accumulators), warps 2-5 = epilogue: TMEM -> smem tile C[row][f] (bank
// skewed), then one thread per pooled (f, ph, pw) for both images: bias,
// 2x2 max with the first-max mask, TF32 p2, its transpose p2T, the mask.
#ifndef CF_STAGES
#define CF_STAGES 2  // pair stages of conv2's forward (2: fits beside a conv1+pool1 block)
#endif
namespace cf {
constexpr int PLANE = 12 * 2 * 12 * 16;        // [h][n][w][4 c] of one pair = 4608 B
constexpr int A_BYTES = 6 * PLANE;             // 24 channels per stage
constexpr int A_GLOBAL = 5 * PLANE;            // 20 channels stored per pair
constexpr int TAP_BYTES = 5 * 800;             // [cc 5][f 50][4 c]
constexpr int B_BYTES = 99 * 1024;             // 25 taps + >= 1024 B zero pad
constexpr int C_PITCH = 50;                    // floats per C row (+ skew below)
constexpr int C_BYTES = 25 * 1024 + 1024;      // 128 x 50 floats + max skew
constexpr int STAGES = CF_STAGES;
#ifndef CF_POOL_WARPS
#define CF_POOL_WARPS 4  // extra warps that join the pooling phase of the epilogue
#endif
constexpr int POOLW = CF_POOL_WARPS;
constexpr int THREADS_F = 192 + 32 * POOLW;
constexpr int EPI_T = 128 + 32 * POOLW;  // threads of the pooling phase
constexpr int SMEM = B_BYTES + STAGES * A_BYTES + C_BYTES + 1024;
static_assert(25 * TAP_BYTES + 1024 <= B_BYTES, "B pad");
struct Params {
  const float* w2c;
  const float* p1c;
  const float* b;
  float* p2;
  float* p2T;  // [800][npad]
  uint8_t* m2;
  int N, npad, per_cta;  // pairs [blockIdx.x * per_cta, + per_cta)
};
// C tile address of (row r, col f): rows of 50 floats, skewed by the pooled
// row ph = r / 32 so that both the row-per-lane 8-B stores and the pooling
// reads (lanes = 2 f x 4 ph x 4 pw) are bank-conflict free
__device__ __forceinline__ uint32_t c_addr(uint32_t C_s, int r, int f) {
  const int ph = r >> 5;
  return C_s + 4 * (r * C_PITCH + f + 2 * (ph & 1) + 16 * (ph >> 1));
}
}  // namespace cf



__global__ void __launch_bounds__(cf::THREADS_F, 1) conv2_fwd_persistent(const __grid_constant__ cf::Params p) {
  using namespace cf;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t B_s = smem_u32(smem), A_s = B_s + B_BYTES, C_s = A_s + STAGES * A_BYTES;
  __shared__ __align__(8) uint64_t wbar[5], full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float bias_s[50];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int npairs = (p.N + 1) / 2;
  const int pair0 = blockIdx.x * p.per_cta;
  ST_BEGIN(ST_CONV2F);
  if (tid < 50) bias_s[tid] = p.b[tid];
  const int mine = max(0, min(p.per_cta, npairs - pair0));
  if (tid == 0) stamp(0);
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(smem_u32(&wbar[i]), 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 128);
  // zero channel plane 5 of every stage and the pad after the last tap (the
  // copies never write them); generic stores -> async proxy before the MMAs
  for (int i = tid; i < STAGES * (PLANE / 16); i += THREADS_F)
    sts128(A_s + (i / (PLANE / 16)) * A_BYTES + 5 * PLANE + (i % (PLANE / 16)) * 16, zero4());
  for (int i = tid; i < (B_BYTES - 25 * TAP_BYTES) / 16; i += THREADS_F)
    sts128(B_s + 25 * TAP_BYTES + 16 * i, zero4());
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    // ---- producer: the weights in 5 pieces (taps of one kernel row each;
    // packed two launches back, so readable before the PDL wait), then -- once
    // conv1+pool1 has completed -- the pairs
    if (mine > 0)
      for (int i = 0; i < 5; ++i) {
        mbar_expect_tx(smem_u32(&wbar[i]), 5 * TAP_BYTES);
        bulk_g2s(B_s + i * 5 * TAP_BYTES, (const uint8_t*)p.w2c + i * 5 * TAP_BYTES, 5 * TAP_BYTES,
                 smem_u32(&wbar[i]));
      }
    pdl_enter_k(ST_CONV2F);
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(smem_u32(&empty[s]), ((it / STAGES) - 1) & 1);
      mbar_expect_tx(smem_u32(&full[s]), A_GLOBAL);
      bulk_g2s(A_s + s * A_BYTES, (const uint8_t*)p.p1c + (size_t)(pair0 + it) * A_GLOBAL, A_GLOBAL,
               smem_u32(&full[s]));
    }
  } else if (tid == 32) {
    // ---- MMA issuer
    constexpr uint32_t idesc = make_idesc(128, 64);
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int s = it % STAGES, b = it & 1;
      mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
      if (it >= 2) mbar_wait(smem_u32(&tempty[b]), ((it >> 1) - 1) & 1);
      tc_fence_after();
      if (it < 4) stamp(1 + it);  // pair landed
      const uint32_t d = tbase + b * 64;
      // descriptors of tap (0,0), k step 0; every other MMA adds a
      // compile-time offset to the 14-bit start-address field (no carry:
      // shared addresses < 256 KB)
      const uint64_t ad0 = make_desc_ns(A_s + s * A_BYTES, PLANE, 192), bd0 = make_desc_ns(B_s, 800, 128);
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (it == 0) {
          mbar_wait(smem_u32(&wbar[i]), 0);
          tc_fence_after();
          if (i == 0) stamp(14);  // first weight piece landed
          if (i == 4) stamp(5);   // weights landed
        }
#pragma unroll
        for (int j = 0; j < 5; ++j)
#pragma unroll
          for (int ks = 0; ks < 3; ++ks)
            mma_tf32(d, ad0 + (uint64_t)(((i * 24 + j) * 16 + ks * 2 * PLANE) >> 4),
                     bd0 + (uint64_t)(((i * 5 + j) * TAP_BYTES + ks * 1600) >> 4), idesc, (i | j | ks) != 0);
      }
      mma_commit(smem_u32(&empty[s]));
      mma_commit(smem_u32(&tfull[b]));
    }
  } else if (warp >= 2) {
    // ---- epilogue: warps 2-5 (TMEM lane quadrant q = warp % 4 = rows 32q..)
    // drain the accumulator into the shared C tile; they and POOLW more warps
    // then pool it (800 pooled outputs per pair over EPI_T threads)
    const bool drains = warp < 6;
    const int quad = warp & 3, row = quad * 32 + lane, et = tid - 64;
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int b = it & 1, pair = pair0 + it;
      if (drains) {
        mbar_wait(smem_u32(&tfull[b]), (it >> 1) & 1);
        if (warp == 2 && lane == 0 && it < 4) stamp(6 + it);  // accumulator ready
        __syncwarp();
        tc_fence_after();
      }
      float v[64];
      if (drains) {
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16)
          tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + b * 64 + c0, *reinterpret_cast<float(*)[16]>(v + c0));
        tc_fence_before();
        if (warp == 2 && lane == 0 && it == 0) stamp(11);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"r"(EPI_T) : "memory");  // C free (previous pair pooled)
      if (drains) {
#pragma unroll
        for (int f = 0; f < 50; f += 2)
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(c_addr(C_s, row, f)), "f"(v[f]), "f"(v[f + 1])
                       : "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"r"(EPI_T) : "memory");  // C complete
      if (warp == 2 && lane == 0 && it == 0) stamp(12);
      const int n0 = 2 * pair;
#pragma unroll
      for (int q = 0; q < (800 + EPI_T - 1) / EPI_T; ++q) {  // 800 pooled (f, ph, pw) over EPI_T threads
        const int k = et + EPI_T * q;
        if (k >= 800) break;
        const int f = k >> 4, ph = (k >> 2) & 3, pw = k & 3;
        const float bias = bias_s[f];
        float out[2];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int r = ph * 32 + n * 8 + pw * 2;  // window rows r, r+1, r+16, r+17
          const float v00 = ldsf_nc(c_addr(C_s, r, f)) + bias, v01 = ldsf_nc(c_addr(C_s, r + 1, f)) + bias;
          const float v10 = ldsf_nc(c_addr(C_s, r + 16, f)) + bias, v11 = ldsf_nc(c_addr(C_s, r + 17, f)) + bias;
          float best = v00;
          int arg = 0;  // first maximum in window order (0,0),(0,1),(1,0),(1,1)
          if (v01 > best) { best = v01; arg = 1; }
          if (v10 > best) { best = v10; arg = 2; }
          if (v11 > best) { best = v11; arg = 3; }
          out[n] = tf32f(best);
          if (n0 + n < p.N) {
            p.p2[(size_t)(n0 + n) * 800 + k] = out[n];
            p.m2[(size_t)(n0 + n) * 800 + k] = (uint8_t)arg;
          }
        }
        if (n0 + 1 < p.N)
          *reinterpret_cast<float2*>(p.p2T + (size_t)k * p.npad + n0) = make_float2(out[0], out[1]);
        else
          p.p2T[(size_t)k * p.npad + n0] = out[0];
      }
      if (warp == 2 && lane == 0 && it == 0) stamp(13);
    }
    if (warp == 2 && lane == 0) stamp(15);
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) stamp(10);
  ST_END(ST_CONV2F);
  if (warp == 0) tmem_dealloc(tbase, 128);
}

// ------------------------------ conv2 data gradient, persistent pipeline
// dp1 = col2im(W2^T G2).  Half of col2im is folded into the
// contraction: with M = (c, j) (100 rows), K = (i, f), N = (n, h, w),
//   Y[(c,j), (n,h,w)] = sum_{i,f} W2[f,c,i,j] G2[n,f,h-i,w]      (h in 0..11)
//   dp1[n,c,h,w]       = sum_j Y[(c,j), (n,h,w-j)]               (0 <= w-j < 8)
// (the same products as col2im of W2^T G2, summed over i inside the tensor
// core and over j in the epilogue: 5 terms per output instead of 25).
// The B operand of kernel row i is G2 shifted by i image rows, and in the
// UMMA K-major no-swizzle layout (core matrix = 8 rows x 16 B) a shift by one
// image row is a shift of the descriptor start by one 8-row group: each image
// pair is staged once as Gs[plane f/4][slot][w][4 f], slot = 4 + 12 n + h
// (slots 0-3, 12-15, 24-27 stay zero: the out-of-image rows), so
//   B_i = descriptor(Gs + (4 - i) * 128 B), N = 192 = (n, h 0..11, w 0..7),
// SBO = 128 B, LBO = one plane.  A = W2 as W2d[i][plane][(c,j)][4 f] (packed
// per step), resident: 5 taps x 7 K steps of tcgen05.mma M=128 N=192 K=8 per
// pair.  The remaining column sum (5 terms per output) runs in the epilogue.
//   warp 0      producer: W2d (bulk copies, once)
//   warp 1      MMA issuer, 2 TMEM accumulators (192 columns each)
//   warps 2-5   B builders: G2[n,f,h,w] (global/L2, coalesced along (h,w))
//               -> Gs (one buffer)
//   warps 6-13  epilogue, one group of 4 per image of the pair: per chunk
//               of 4 image rows, TMEM -> smem scratch -> the j-sum -> dp1
//               (NCHW)
// (one G buffer: the builders hold the next pair in registers and store it
// as soon as the MMAs have read the previous one; the freed shared memory
// holds the second epilogue group's scratch)
#ifndef DG_RESTRICT
#define DG_RESTRICT 1
#endif
namespace dg {
constexpr int PLANES = 14;
static_assert(PLANES == kW2dPlanes, "W2d layout (solver.cuh)");                          // 56 f (50 + zeros), 7 K steps of 8
constexpr int AROWS = 104;                          // (c,j) rows 0..99 + 4 zero rows
static_assert(AROWS == kW2dRows, "W2d layout (solver.cuh)");
constexpr int A_PLANE = AROWS * 16;                 // 1664 B
constexpr int A_TAP = PLANES * A_PLANE;             // 23296 B
constexpr int A_BYTES = 5 * A_TAP + 384;            // + the rows 104..127 the M=128 MMA over-reads
constexpr int G_PLANE = 28 * 128;                   // 28 slots x 8 w x 16 B
constexpr int G_BYTES = PLANES * G_PLANE;           // 50176 B per buffer
constexpr int RCH = 4;                              // epilogue: output rows per staged chunk
constexpr int SP = RCH * 8 + 4;                     // scratch pitch (floats): conflict-free 16-B stores
constexpr int S_BYTES = 128 * SP * 4;               // per epilogue group
constexpr int WARPS = 14, THREADS_D = WARPS * 32;   // producer, MMA, 4 builders, 2 x 4 epilogue
constexpr int SMEM = A_BYTES + G_BYTES + 2 * S_BYTES + 1024;
constexpr int W2D_FLOATS = A_BYTES / 4;
struct Params {
  const float* w2d;  // packed A (W2D_FLOATS)
  const float* g2;   // [N][50][64] TF32
  float* dp1;        // [N][20][144]
  int N, per_cta;    // pairs [blockIdx.x * per_cta, + per_cta)
};
}  // namespace dg

__global__ void __launch_bounds__(dg::THREADS_D, 1) conv2_dgrad_persistent(const __grid_constant__ dg::Params p) {
  using namespace dg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t A_s = smem_u32(smem), G_s = A_s + A_BYTES, S_s = G_s + G_BYTES;
  __shared__ __align__(8) uint64_t afull, gfull, gfree, accfull[2], accfree[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int npairs = (p.N + 1) / 2, pair0 = blockIdx.x * p.per_cta;
  const int mine = max(0, min(p.per_cta, npairs - pair0));
  ST_BEGIN(ST_CONV2D);
  if (tid == 0) {
    mbar_init(smem_u32(&afull), 1);
    mbar_init(smem_u32(&gfull), 128);
    mbar_init(smem_u32(&gfree), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&accfull[b]), 1);
      mbar_init(smem_u32(&accfree[b]), 256);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  // zero the G buffer once: the builders only ever write the in-image slots
  // of planes 0..12, so the halo slots and plane 13 stay zero
  for (int i = tid; i < G_BYTES / 16; i += THREADS_D) sts128(G_s + 16 * i, zero4());
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) stamp(0);
  if (tid == 0) {
    // ---- producer: the packed weights (written by the step's first launch,
    // so readable before the PDL wait), then let the successor launch
    if (mine > 0) {
      mbar_expect_tx(smem_u32(&afull), A_BYTES);
      for (int i = 0; i < 5; ++i) {
        const uint32_t bytes = i < 4 ? A_TAP : A_TAP + 384;
        bulk_g2s(A_s + i * A_TAP, (const uint8_t*)p.w2d + i * A_TAP, bytes, smem_u32(&afull));
      }
    }
    pdl_enter();
  } else if (tid == 32) {
    // ---- MMA issuer
    constexpr uint32_t idesc = make_idesc(128, 192);
    if (mine > 0) mbar_wait(smem_u32(&afull), 0);
    stamp(1);
    const uint64_t ad0 = make_desc_ns(A_s, A_PLANE, 128);
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int b = it & 1;
      mbar_wait(smem_u32(&gfull), it & 1);
      if (it < 2) stamp(2 + 2 * it);  // pair built
      if (it >= 2) mbar_wait(smem_u32(&accfree[b]), ((it >> 1) - 1) & 1);
      tc_fence_after();
      const uint64_t bd0 = make_desc_ns(G_s, G_PLANE, 128);
#if DG_RESTRICT
      // kernel row 2 over all 12 output rows of both images (N = 192; its
      // zero halo rows make it exact everywhere, and it initialises the
      // accumulator), then rows 0, 1, 3, 4 only over the 8 output rows they
      // reach, one image at a time (N = 64: B = the image's 8 real G2 rows,
      // D columns from output row i): 27% fewer MMA cycles (floor ~ N)
      constexpr uint32_t idesc64 = make_idesc(128, 64);
#pragma unroll
      for (int ks = 0; ks < PLANES / 2; ++ks)
        mma_tf32(tbase + b * 256, ad0 + (uint64_t)((2 * A_TAP + ks * 2 * A_PLANE) >> 4),
                 bd0 + (uint64_t)((2 * 128 + ks * 2 * G_PLANE) >> 4), idesc, ks != 0);
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i == 2) continue;
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int ks = 0; ks < PLANES / 2; ++ks)
            mma_tf32(tbase + b * 256 + (n * 12 + i) * 8, ad0 + (uint64_t)((i * A_TAP + ks * 2 * A_PLANE) >> 4),
                     bd0 + (uint64_t)(((4 + 12 * n) * 128 + ks * 2 * G_PLANE) >> 4), idesc64, 1u);
      }
#else
#pragma unroll
      for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int ks = 0; ks < PLANES / 2; ++ks)
          mma_tf32(tbase + b * 256, ad0 + (uint64_t)((i * A_TAP + ks * 2 * A_PLANE) >> 4),
                   bd0 + (uint64_t)(((4 - i) * 128 + ks * 2 * G_PLANE) >> 4), idesc, (i | ks) != 0);
#endif
      mma_commit(smem_u32(&gfree));
      mma_commit(smem_u32(&accfull[b]));
      if (it < 2) stamp(3 + 2 * it);  // MMAs issued
    }
  } else if (warp >= 2 && warp < 6) {
    // ---- B builders: thread = (image n, position h*8+w); 13 planes of 4 f
    pdl_enter_k(ST_CONV2D);  // G2 comes from the immediate predecessor
    if (tid == 64) stamp(11);
    const int t = tid - 64, n = t >> 6, pos = t & 63, h = pos >> 3, w = pos & 7;
    const uint32_t dst0 = (uint32_t)((4 + 12 * n + h) * 128 + w * 16);
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int img = 2 * (pair0 + it) + n;
      float v[52];
      if (img < p.N) {
        const float* g = p.g2 + (size_t)img * 3200 + pos;
#pragma unroll
        for (int f = 0; f < 50; ++f) v[f] = __ldcg(g + f * 64);
      } else {
#pragma unroll
        for (int f = 0; f < 50; ++f) v[f] = 0.f;
      }
      v[50] = v[51] = 0.f;
      // one G buffer: its next pair is stored (from registers, loaded above)
      // as soon as the previous pair's MMAs have read it
      if (it >= 1) mbar_wait(smem_u32(&gfree), (it - 1) & 1);
      const uint32_t dst = G_s + dst0;
#pragma unroll
      for (int q = 0; q < 13; ++q) sts128(dst + q * G_PLANE, f4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      fence_proxy_async();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&gfull)) : "memory");
    }
  } else if (warp >= 6) {
    // ---- epilogue: two groups of 4 warps, group g = image n of the pair
    // (its 96 accumulator columns); TMEM lane quadrant q = warp % 4 holds
    // rows (c,j) 32q..  Per chunk of RCH output rows: the 8 columns w of
    // every row and chunk row go through the group's scratch tile (one
    // barrier to publish, one before it is rewritten), then thread ->
    // outputs (c, h, w): the 5-term column sum in fixed j order.
    const int quad = warp & 3, row = quad * 32 + lane, g = (warp - 6) >> 2, et = (tid - 192) & 127;
    const uint32_t S = S_s + g * S_BYTES;
#pragma unroll 1
    for (int it = 0; it < mine; ++it) {
      const int b = it & 1, img = 2 * (pair0 + it) + g;
      mbar_wait(smem_u32(&accfull[b]), (it >> 1) & 1);
      if (et == 0 && g == 0 && it < 2) stamp(6 + 2 * it);  // accumulator ready
      __syncwarp();
      tc_fence_after();
#pragma unroll 1
      for (int h0 = 0; h0 < 12; h0 += RCH) {
        float v[RCH * 8];
#pragma unroll
        for (int u = 0; u < RCH / 2; ++u)
          tmem_ld16_nowait(tbase + ((uint32_t)(quad * 32) << 16) + b * 256 + (g * 12 + h0 + 2 * u) * 8,
                           *reinterpret_cast<float(*)[16]>(v + 16 * u));
        tmem_ld_wait();
        if (h0 + RCH == 12) {  // every column of this image is in registers
          tc_fence_before();
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[b])) : "memory");
        }
#pragma unroll
        for (int u = 0; u < RCH * 2; ++u) sts128(S + 4 * (row * SP + 4 * u), f4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
        if (img < p.N) {
          // all shared loads of the thread's outputs first (no memory clobber:
          // the compiler may hoist them above the previous outputs' global
          // stores), then the fixed-order sums
          constexpr int NO = (RCH * 240 + 127) / 128;
          float t[NO][5];
#pragma unroll
          for (int k = 0; k < NO; ++k) {
            const int o = et + 128 * k;
            const int hh = o / 240, r2 = o - 240 * hh, c = r2 / 12, w = r2 - 12 * c;
#pragma unroll
            for (int jj = 0; jj < 5; ++jj)
              t[k][jj] = (o < RCH * 240 && (unsigned)(w - jj) < 8u)
                             ? ldsf_nc(S + 4 * ((c * 5 + jj) * SP + hh * 8 + w - jj)) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < NO; ++k) {
            const int o = et + 128 * k;
            if (o >= RCH * 240) break;
            const int hh = o / 240, r2 = o - 240 * hh, c = r2 / 12, w = r2 - 12 * c;
            float acc = 0.f;  // j ascending over the valid taps (the first valid term initialises it)
#pragma unroll
            for (int jj = 0; jj < 5; ++jj)
              if ((unsigned)(w - jj) < 8u) acc += t[k][jj];
            p.dp1[(size_t)img * 2880 + c * 144 + (h0 + hh) * 12 + w] = acc;
          }
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // the scratch is read before it is rewritten
      }
      if (et == 0 && g == 0 && it < 2) stamp(7 + 2 * it);  // pair stored
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) stamp(10);
  ST_END(ST_CONV2D);
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// ------------------------------------- conv2 weight gradient, persistent
// dW2[f,(c,i,j)] = sum_{n,p} G2[n,f,p] p1[n,c,ho+i,wo+j] as the GEMM
//   D[(c,i,j), f] = sum_K A[(c,i,j), K] G2[f, K],  K = (image n, position p)
// rows (c,i,j) 500 in 4 tiles of 128, N = 64 (f 50 + TMA zero fill), split
// over images: grid (4 row tiles, S image ranges), one CTA per SM.  The
// sliding window runs along the contraction (K-major only for TF32), so A is
// materialised per image -- but from registers: one thread per (c, i, ho)
// loads the input row p1[n,c,ho+i,0..11] (3 x 16 B) and writes the 5 j-shifted
// 8-wide windows (10 x 16 B) into the SW128 K-major A tile.
//   warp 0      producer: per image, the tile's <= 6 input channels (bulk
//               copy) and G2[n] (TMA 3D, 2 x {32 p, 64 f}), 3-slot ring
//   warp 1      MMA: 8 x tcgen05.mma (M=128, N=64, K=8) per image, one TMEM
//               accumulator over the CTA's images
//   warps 2-9   A builders (2 A buffers); warps 2-5 then drain TMEM into the
//               split's partial sums part[split][f*500 + (c,i,j)]
namespace wg {
constexpr int WARPS = 10, THREADS_W = WARPS * 32, NB = 256;  // A builder threads
constexpr int A_BYTES = 2 * 128 * 128;   // 2 K-chunks (32 positions each) x 128 rows x 128 B
constexpr int G_BYTES = 2 * 64 * 128;    // 2 K-chunks x 64 f rows x 128 B
constexpr int P_BYTES = 6 * 144 * 4;     // <= 6 input channels of one image
constexpr int SLOTS = WG_SLOTS;  // images in flight
constexpr int NA = WG_ABUF;      // A tiles in flight (builders vs MMAs)
constexpr int SMEM = NA * A_BYTES + SLOTS * G_BYTES + SLOTS * P_BYTES + 1024;
static_assert(SMEM <= 227 * 1024, "shared memory");
struct Params {
  CUtensorMap tg;  // G2 as {64 p, 50 f, N n}
  const float* p1;
  float* part;
  int N, splits, pstride;
};
}  // namespace wg


__global__ void __launch_bounds__(wg::THREADS_W, 1) conv2_wgrad_persistent(const __grid_constant__ wg::Params p) {
  using namespace wg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t A_s = smem_u32(smem), G_s = A_s + NA * A_BYTES, P_s = G_s + SLOTS * G_BYTES;
  __shared__ __align__(8) uint64_t full[SLOTS], sfree[SLOTS], afull[NA], afree[NA], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = blockIdx.x, split = blockIdx.y;
  const int n0 = (int)((long long)p.N * split / p.splits), n1 = (int)((long long)p.N * (split + 1) / p.splits);
  const int nimg = n1 - n0;
  ST_BEGIN(ST_CONV2W);
  // (c,i) pairs and input channels this row tile touches
  const int R0 = 128 * m, P_lo = R0 / 5, P_hi = min(R0 + 127, 499) / 5, NP = P_hi - P_lo + 1;
  const int c_lo = P_lo / 5, nch = P_hi / 5 - c_lo + 1;
  if (tid == 0) {
    for (int s = 0; s < SLOTS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&sfree[s]), NB + 1);  // builders done with P + MMA done with G
    }
    for (int b = 0; b < NA; ++b) {
      mbar_init(smem_u32(&afull[b]), NB);
      mbar_init(smem_u32(&afree[b]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
    prefetch_tmap(&p.tg);
  }
  if (warp == 0) tmem_alloc(&tmem_base, 64);
  // rows no builder writes (tile 3 beyond row 499) stay zero
  for (int i = tid; i < NA * A_BYTES / 16; i += THREADS_W) sts128(A_s + 16 * i, zero4());
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) stamp(0);
  if (tid == 0) {
    // ---- producer (G2 and p1 come from the two preceding launches' producers:
    // wait for the immediate predecessor first)
    pdl_enter_k(ST_CONV2W);
    const uint32_t bytes = nch * 576 + G_BYTES;
#pragma unroll 1
    for (int t = 0; t < nimg; ++t) {
      const int s = t % SLOTS, n = n0 + t;
      if (t >= SLOTS) mbar_wait(smem_u32(&sfree[s]), ((t / SLOTS) - 1) & 1);
      const uint32_t bar = smem_u32(&full[s]);
      mbar_expect_tx(bar, bytes);
      bulk_g2s(P_s + s * P_BYTES, p.p1 + (size_t)n * 2880 + c_lo * 144, nch * 576, bar);
      tma3d(G_s + s * G_BYTES, &p.tg, 0, 0, n, bar);
      tma3d(G_s + s * G_BYTES + 64 * 128, &p.tg, 32, 0, n, bar);
    }
  } else if (tid == 32) {
    // ---- MMA issuer
    constexpr uint32_t idesc = make_idesc(128, 64);
#pragma unroll 1
    for (int t = 0; t < nimg; ++t) {
      const int s = t % SLOTS, b = t % NA;
      mbar_wait(smem_u32(&full[s]), (t / SLOTS) & 1);
      if (t < 4) stamp(1 + t);  // image t landed
      mbar_wait(smem_u32(&afull[b]), (t / NA) & 1);
      if (t < 4) stamp(5 + t);  // A tile t built
      tc_fence_after();
      const uint32_t Ab = A_s + b * A_BYTES, Gb = G_s + s * G_BYTES;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_tf32(tbase, make_desc(Ab + kc * 16384 + k * 32), make_desc(Gb + kc * 8192 + k * 32), idesc,
                   (t | kc | k) != 0);
      mma_commit(smem_u32(&afree[b]));
      mma_commit(smem_u32(&sfree[s]));
    }
    mma_commit(smem_u32(&done));
  } else if (warp >= 2) {
    // ---- A builders: item g = (pair P_lo + g % NP, ho = g / NP); lanes with
    // consecutive pairs write rows 5 apart (distinct swizzle phases)
    const int g = tid - 64;
    const bool active = g < NP * 8;
    const int P = P_lo + g % NP, ho = g / NP, c = P / 5, i = P - 5 * (P / 5);
    const uint32_t src_off = 4 * ((c - c_lo) * 144 + (ho + i) * 12);
    const int r0 = 5 * P - R0;  // tile row of j = 0
    const uint32_t dst_off = (ho >> 2) * 16384;
    const int q0 = (ho & 3) * 2;
#pragma unroll 1
    for (int t = 0; t < nimg; ++t) {
      const int s = t % SLOTS, b = t % NA;
      mbar_wait(smem_u32(&full[s]), (t / SLOTS) & 1);
      if (t >= NA) mbar_wait(smem_u32(&afree[b]), ((t / NA) - 1) & 1);
      if (active) {
        float x[12];
        const uint32_t src = P_s + s * P_BYTES + src_off;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int4 v = lds_i4(src + 16 * u);
          x[4 * u] = __int_as_float(v.x);
          x[4 * u + 1] = __int_as_float(v.y);
          x[4 * u + 2] = __int_as_float(v.z);
          x[4 * u + 3] = __int_as_float(v.w);
        }
        const uint32_t Ab = A_s + b * A_BYTES + dst_off;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const int r = r0 + j;
          if (r >= 0 && r < 128 && 5 * P + j < 500) {
            sts128(Ab + sw_off(r, q0), f4(x[j], x[j + 1], x[j + 2], x[j + 3]));
            sts128(Ab + sw_off(r, q0 + 1), f4(x[j + 4], x[j + 5], x[j + 6], x[j + 7]));
          }
        }
      }
      fence_proxy_async();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sfree[s])) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[b])) : "memory");
    }
    // ---- epilogue (warps 2-5): TMEM lane quadrant warp % 4 -> rows; the
    // split's partial dW2[f][(c,i,j)] (coalesced over rows)
    if (warp < 6) {
      const int quad = warp & 3, row = quad * 32 + lane, R = R0 + row;
      float* dst = p.part + (size_t)split * p.pstride;
      if (nimg > 0) {
        mbar_wait(smem_u32(&done), 0);
        if (warp == 2 && lane == 0) stamp(9);  // accumulation done
        __syncwarp();
        tc_fence_after();
      }
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        float v[16];
        if (nimg > 0) {
          tmem_ld16(tbase + ((uint32_t)(quad * 32) << 16) + c0, v);
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = 0.f;
        }
        if (R < 500) {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (c0 + u < 50) dst[(c0 + u) * 500 + R] = v[u];
        }
      }
    }
  }
  if (warp == 2 && lane == 0) stamp(10);  // partials written
  tc_fence_before();
  __syncthreads();
  ST_END(ST_CONV2W);
  if (warp == 0) tmem_dealloc(tbase, 64);
}

// --------------------------------------------------------- weight packing
// Once per forward (weights change only in SGD), TF32-rounded copies of the
// weights in the layouts the GEMMs consume, zero padded:
//   W1f [500][800]  = W1                      (ip1 fwd B)
//   W2c [25 taps][5 cc][50 f][4 c] = W2[f, 4cc + c, tap]   (conv2 fwd B)
//   W2d [5 i][14 planes][104 (c,j)][4 f] = W2[4 plane + q, c, i, j] (conv2 dgrad A, see dg)
//   W1t [800][512]  = W1^T                    (ip1 dgrad B; tiled transpose)
constexpr int W2C_N = 25 * 5 * 50 * 4, W2T_N = dg::W2D_FLOATS;
static_assert(W2T_N == kW2tFloats, "W2d size");
constexpr int W1_TILES = (800 / 32) * (512 / 32);  // 32 x 32 tiles of W1 (o padded to 512)
// One launch: blocks [0, W1_TILES) copy + transpose a 32 x 32 tile of W1
// through shared memory (W1f rows and W1t rows both coalesced); the rest pack
// W2c and W2d element-wise.
__global__ void pack_weights(const __grid_constant__ PackP p) {
  ST_BEGIN(ST_PACK);
  pdl_enter_k(ST_PACK);
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  // W1 tiles (grid-stride: PACK_GRID > 0 runs the pack in fewer, longer blocks)
#pragma unroll 1
  for (int tile = blockIdx.x; tile < W1_TILES; tile += gridDim.x) {
    const int k0 = (tile % 25) * 32, o0 = (tile / 25) * 32;
    float v[4];  // the tile's four rows per thread loaded together
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = o0 + ty + 8 * u;
      v[u] = o < 500 ? tf32f(p.w1[(size_t)o * 800 + k0 + tx]) : 0.f;
    }
    __syncthreads();  // the previous tile's transpose reads are done
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = o0 + ty + 8 * u;
      t[ty + 8 * u][tx] = v[u];
      if (o < 500) p.w1f[(size_t)o * 800 + k0 + tx] = v[u];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) p.w1t[(size_t)(k0 + ty + 8 * u) * 512 + o0 + tx] = t[tx][ty + 8 * u];
  }
  // W2c and W2d element-wise, over all blocks
  const int nb = gridDim.x, bx = blockIdx.x;
#pragma unroll 1
  for (int idx = bx * blockDim.x + threadIdx.x; idx < W2C_N + W2T_N; idx += nb * blockDim.x) {
    if (idx < W2C_N) {
      const int c4 = idx & 3, f = (idx >> 2) % 50, cc = (idx / 200) % 5, tap = idx / 1000;
      p.w2c[idx] = tf32f(p.w2[f * 500 + (cc * 4 + c4) * 25 + tap]);
    } else {  // W2d[i][plane][(c,j)][4 f] (conv2 dgrad A), zero rows / filters / tail pad
      const int e = idx - W2C_N;
      const int q = e & 3, r = (e >> 2) % dg::AROWS, pl = (e / (4 * dg::AROWS)) % dg::PLANES;
      const int i = e / (4 * dg::AROWS * dg::PLANES), f = 4 * pl + q, c = r / 5, j = r % 5;
      float v = 0.f;
      if (i < 5 && f < 50 && r < 100) v = p.w2[f * 500 + c * 25 + i * 5 + j];
      p.w2t[e] = tf32f(v);
    }
  }
  ST_END(ST_PACK);
}
// ---------------------------------------------------------- fused solver
// The TF32 plan's solver (a17, S:536-544 / R11): one launch that, per
// parameter, takes the gradient (conv bucket: the fixed-order sum of the
// weight-gradient partials, the same order as reduce_partials_multi, written
// back to the gradient blob; ip bucket: already reduced), applies the SGD
// update (sgd_one) and writes the TF32 copies the next step's contractions
// read (W1f, W1t, W2c, W2d -- the weight pack, so no packing launch opens the
// next step).  Blocks [0, W1_TILES): a 32 x 32 tile of ip1's weights (W1t
// through a shared-memory transpose); then 32-output blocks over the reduce
// segments (8 warps over the splits, warp 0 sums the 8 in order and updates);
// then grid-stride blocks over the plain ranges.  A single-GPU whole step
// splits it: the ip layers' part on the backward's side branch (their
// gradients are final after ip1's weight gradient; it overlaps the conv
// backward), the conv bucket's at the end.  w1_tiles = 0: no ip1 weights.
__global__ void __launch_bounds__(256) lenet_solver(const __grid_constant__ SolverP p) {
  const int stk = p.w1_tiles ? ST_OTHER : ST_SGD;  // (step trace: the ip part / the rest)
  ST_BEGIN(stk);
  pdl_enter_k(stk);
  const float lr = p.lr_dev ? __ldg(p.lr_dev) : p.lr;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  if ((int)blockIdx.x < p.w1_tiles) {
    __shared__ float t[32][33];
    const int tile = blockIdx.x, k0 = (tile % 25) * 32, o0 = (tile / 25) * 32;
    float w[4], v[4], g[4];  // the tile's four rows per thread: all loads in flight together
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = o0 + wp + 8 * u;
      const long long i = p.w1_off + (long long)min(o, 499) * 800 + k0 + lane;
      w[u] = __ldcg(p.w + i), v[u] = __ldcg(p.v + i), g[u] = __ldcg(p.g + i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = o0 + wp + 8 * u;
      float wf = 0.f;
      if (o < 500) {
        const long long i = p.w1_off + (long long)o * 800 + k0 + lane;
        sgd_one(w[u], g[u], v[u], lr, p.mom, p.decay, p.gscale);
        p.w[i] = w[u];
        p.v[i] = v[u];
        wf = tf32f(w[u]);
        p.w1f[(size_t)o * 800 + k0 + lane] = wf;
      }
      t[wp + 8 * u][lane] = wf;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) p.w1t[(size_t)(k0 + wp + 8 * u) * 512 + o0 + lane] = t[lane][wp + 8 * u];
  } else if ((int)blockIdx.x < p.w1_tiles + p.seg_blocks) {
    __shared__ float sm[8][33];
    int b = blockIdx.x - p.w1_tiles, k = 0;
    while (k < p.nseg - 1 && b >= (p.seg[k].n + 31) / 32) b -= (p.seg[k++].n + 31) / 32;
    const ReduceP& s = p.seg[k];
    const int i = b * 32 + lane;
    sm[wp][lane] = split_sum_warp(s, i, wp);  // reduce_partials_multi's order (reduce.cuh)
    __syncthreads();
    if (wp == 0 && i < s.n) {
      float r = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) r += sm[q][lane];
      if (s.part != s.out) s.out[i] = r;  // the reduced gradient stays readable
      const long long e = (s.out - p.g) + i;
      float w = p.w[e], v = p.v[e];
      sgd_one(w, r, v, lr, p.mom, p.decay, p.gscale);
      p.w[e] = w;
      p.v[e] = v;
      const long long q2 = e - p.w2_off;
      if (q2 >= 0 && q2 < 25000) {  // conv2 weight (f, c, i, j): its W2c and W2d slots
        const int f = (int)q2 / 500, c = ((int)q2 / 25) % 20, ii = ((int)q2 / 5) % 5, jj = (int)q2 % 5;
        const float wf = tf32f(w);
        p.w2c[(ii * 5 + jj) * 1000 + (c >> 2) * 200 + f * 4 + (c & 3)] = wf;
        p.w2t[((ii * dg::PLANES + (f >> 2)) * dg::AROWS + c * 5 + jj) * 4 + (f & 3)] = wf;
      }
    }
  } else {
    const int nb = gridDim.x - p.w1_tiles - p.seg_blocks;
    const int t0 = (blockIdx.x - p.w1_tiles - p.seg_blocks) * 256 + tid;
    for (int r = 0; r < p.nplain; ++r)
      for (long long e = p.plain_lo[r] + t0; e < p.plain_hi[r]; e += (long long)nb * 256) {
        float w = p.w[e], v = p.v[e];
        sgd_one(w, p.g[e], v, lr, p.mom, p.decay, p.gscale);
        p.w[e] = w;
        p.v[e] = v;
      }
  }
  ST_END(stk);
}

// p1c (conv2 forward operand, see conv2_fwd_persistent) from an NCHW pool1
// blob, TF32-rounded: used when pool1 is overwritten through the ABI (the
// forward pass writes p1c directly from conv1+pool1).
struct PackP1cArgs {
  const float* p1;
  float* p1c;
  int N;
};
__global__ void pack_p1c_k(const __grid_constant__ PackP1cArgs a) {
  pdl_enter();
  const float* p1 = a.p1;
  float* p1c = a.p1c;
  const int N = a.N;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // one 4-channel pixel
  const long long npairs = (N + 1) / 2;
  if (idx >= npairs * 5 * 288) return;
  const int pair = (int)(idx / 1440), rem = (int)(idx % 1440);
  const int cc = rem / 288, hnw = rem % 288, h = hnw / 24, nw = hnw % 24, nin = nw / 12, w = nw % 12;
  const int n = 2 * pair + nin;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  if (n < N)
    for (int t = 0; t < 4; ++t) v[t] = tf32f(p1[((size_t)n * 20 + cc * 4 + t) * 144 + h * 12 + w]);
  reinterpret_cast<float4*>(p1c)[idx] = make_float4(v[0], v[1], v[2], v[3]);
}

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PN_STEPTRACE_TU(st_set_tc)

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
static bool g_tmap_ok = true;
// row-major fp32 [rows][cols] (row pitch `pitch` floats): box {32 cols, box_rows}, 128B swizzle
static CUtensorMap tmap2d(const float* base, uint64_t rows, uint64_t cols, uint64_t pitch, uint32_t box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  EncodeTiledFn fn = encode_fn();
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  if (!fn || fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    g_tmap_ok = false;
  return m;
}
// G2 [N][50][64] as {64 p, 50 f, N n}: box {32, 64, 1}, 128B swizzle
static CUtensorMap tmap_g2(const float* base, uint64_t N) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  EncodeTiledFn fn = encode_fn();
  cuuint64_t dims[3] = {64, 50, N};
  cuuint64_t strides[2] = {64 * 4, 3200 * 4};
  cuuint32_t box[3] = {32, 64, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (!fn || fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    g_tmap_ok = false;
  return m;
}

template <class Op>
static constexpr size_t ip_smem() {  // the ring + 1 KB alignment slack
  return (size_t)Op::STAGES * (Op::X3 ? 2 : 1) * (128 * 128 + Op::BN * 128) + 1024;
}
template <class Op>
static cudaError_t opt_in() {
  return cudaFuncSetAttribute((const void*)ip_tile<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ip_smem<Op>());
}

cudaError_t setup() {
  if (!encode_fn()) return cudaErrorNotSupported;
  cudaError_t e;
  if ((e = opt_in<IpFwd>()) != cudaSuccess) return e;
  if ((e = opt_in<IpWgrad>()) != cudaSuccess) return e;
  if ((e = opt_in<IpDgradUnpool>()) != cudaSuccess) return e;
  if ((e = opt_in<Ip3Fwd>()) != cudaSuccess) return e;
  if ((e = opt_in<Ip3Grad>()) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute((const void*)conv2_wgrad_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                wg::SMEM)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute((const void*)conv2_dgrad_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                dg::SMEM)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute((const void*)conv2_fwd_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                cf::SMEM)) != cudaSuccess)
    return e;
  return conv1_setup();
}

bool tensor_maps_ok() { return g_tmap_ok; }

static unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

Launch lenet_solver_launch(const SolverP& p0) {
  SolverP p = p0;
  p.seg_blocks = 0;
  for (int k = 0; k < p.nseg; ++k) p.seg_blocks += (p.seg[k].n + 31) / 32;
  Launch l;
  l.set((const void*)lenet_solver, dim3(p.w1_tiles + p.seg_blocks + (p.nplain ? 8 : 0)), dim3(256), 0, p);
  return l;
}

Launch pack_weights_launch(const PackP& p) {
  Launch l;
  l.set((const void*)pack_weights, dim3(PACK_GRID > 0 ? PACK_GRID : W1_TILES), dim3(256), 0, p);
  return l;
}

Launch conv2_pool2_launch(const float* w2c, const float* b, const float* p1c, float* p2, float* p2T, uint8_t* m2,
                          int N, int npad, int sms) {
  Launch l;
  // pairs split evenly: ceil(pairs / sms) per CTA, as few CTAs as that needs
  // (every CTA loads the 100 KB of weights once)
  const int pairs = (N + 1) / 2, per = std::max(1, (pairs + sms - 1) / sms);
  cf::Params p{w2c, p1c, b, p2, p2T, m2, N, npad, per};
  l.set((const void*)conv2_fwd_persistent, dim3(std::max(1, (pairs + per - 1) / per)), dim3(cf::THREADS_F), cf::SMEM,
        p);
  return l;
}

Launch pack_p1c_launch(const float* p1, float* p1c, int N) {
  Launch l;
  PackP1cArgs a{p1, p1c, N};
  l.set((const void*)pack_p1c_k, dim3(cdiv((long long)((N + 1) / 2) * 1440, 256)), dim3(256), 0, a);
  return l;
}

Launch ip1_fwd_launch(const float* p2, const float* w1f, const float* b, float* y, int N) {
  Launch l;
  IpFwd::Params p{tmap2d(p2, N, 800, 800, 128), tmap2d(w1f, 500, 800, 800, IpFwd::BN), b, y, N, 800, 500};
  l.set((const void*)ip_tile<IpFwd>, dim3(IpFwd::SPLIT * cdiv(500, IpFwd::BN), cdiv(N, 128)), dim3(ipk::THREADS),
        ip_smem<IpFwd>(), p);
  l.cluster = dim3(IpFwd::SPLIT, 1, 1);
  return l;
}

Launch split3_launch(const Split3P& p) {
  Launch l;
  l.set((const void*)split3, dim3(cdiv(p.C, 32), cdiv(p.R, 32)), dim3(256), 0, p);
  return l;
}
Launch ip1_fwd3_launch(const float* p2h, const float* p2l, const float* w1h, const float* w1l, const float* b, float* y,
                       int N) {
  Launch l;
  Ip3Fwd::Params p{tmap2d(p2h, N, 800, 800, 128), tmap2d(p2l, N, 800, 800, 128), tmap2d(w1h, 500, 800, 800, Ip3Fwd::BN),
                   tmap2d(w1l, 500, 800, 800, Ip3Fwd::BN), b, y, N, 800, 500};
  l.set((const void*)ip_tile<Ip3Fwd>, dim3(Ip3Fwd::SPLIT * cdiv(500, Ip3Fwd::BN), cdiv(N, 128)), dim3(ipk::THREADS),
        ip_smem<Ip3Fwd>(), p);
  l.cluster = dim3(Ip3Fwd::SPLIT, 1, 1);
  return l;
}
// out[rows][cols] = A B^T with A = [rows][K] (hi / lo, pitch lda), B = [cols][K] (pitch ldb)
Launch ip1_grad3_launch(const float* ah, const float* al, int rows, int K, int lda, const float* bh, const float* bl,
                        int cols, int ldb, float* out, int ldo) {
  Launch l;
  Ip3Grad::Params p{tmap2d(ah, rows, K, lda, 128), tmap2d(al, rows, K, lda, 128), tmap2d(bh, cols, K, ldb, Ip3Grad::BN),
                    tmap2d(bl, cols, K, ldb, Ip3Grad::BN), out, rows, cols, ldo, (int)cdiv(K, 32)};
  l.set((const void*)ip_tile<Ip3Grad>, dim3(cdiv(cols, Ip3Grad::BN), cdiv(rows, 128)), dim3(ipk::THREADS),
        ip_smem<Ip3Grad>(), p);
  return l;
}

Launch ip1_wgrad_launch(const float* da1T, const float* p2T, float* dw, int N, int npad) {
  Launch l;
  IpWgrad::Params p{tmap2d(da1T, 500, N, npad, 128), tmap2d(p2T, 800, N, npad, IpWgrad::BN), dw, N, 800, 500};
  l.set((const void*)ip_tile<IpWgrad>, dim3(IpWgrad::SPLIT * cdiv(800, IpWgrad::BN), cdiv(500, 128)), dim3(ipk::THREADS),
        ip_smem<IpWgrad>(), p);
  l.cluster = dim3(IpWgrad::SPLIT * IpWgrad::MC, 1, 1);
  return l;
}

Launch ip1_dgrad_unpool_launch(const float* da1r, const float* w1t, const uint8_t* m2, float* g2, float* part_db2,
                               int N) {
  Launch l;
  IpDgradUnpool::Params p{tmap2d(da1r, N, 500, 500, 128), tmap2d(w1t, 800, 512, 512, IpDgradUnpool::BN), m2, g2,
                          part_db2, N};
  l.set((const void*)ip_tile<IpDgradUnpool>, dim3(IpDgradUnpool::SPLIT * cdiv(800, IpDgradUnpool::BN), cdiv(N, 128)),
        dim3(ipk::THREADS), ip_smem<IpDgradUnpool>(), p);
  l.cluster = dim3(IpDgradUnpool::SPLIT * IpDgradUnpool::MC, 1, 1);
  return l;
}

int db2_partials(int N) { return (int)cdiv(N, 128) * IpDgradUnpool::SPLIT; }

Launch conv2_dgrad_launch(const float* g2, const float* w2d, float* dp1, int N, int sms) {
  Launch l;
  // persistent: pairs split evenly, ceil(pairs / sms) per CTA
  const int pairs = (N + 1) / 2, per = std::max(1, (pairs + sms - 1) / sms);
  dg::Params p{w2d, g2, dp1, N, per};
  l.set((const void*)conv2_dgrad_persistent, dim3(std::max(1, (pairs + per - 1) / per)), dim3(dg::THREADS_D), dg::SMEM,
        p);
  return l;
}

Launch conv2_wgrad_launch(const float* g2, const float* p1, float* part, int splits, int N) {
  Launch l;
  wg::Params p{tmap_g2(g2, N), p1, part, N, splits, 25050};
  l.set((const void*)conv2_wgrad_persistent, dim3(4, splits), dim3(wg::THREADS_W), wg::SMEM, p);
  return l;
}

}  // namespace tc
}  // namespace pn
