// tc.cu -- tcgen05 TF32 implicit-GEMM kernels for the GEMM-shaped LeNet
// layers.
//
// Engine (one CTA = one 128-row output tile, 4 warps):
//   * every thread is a producer: it gathers its share of the A (128 x 32)
//     and B (BN x 32) K-chunk straight from global memory -- the implicit
//     im2col / col2im index math of the layer -- rounds each value to TF32
//     with cvt.rna (round to nearest), and stores 16-byte
//     core-matrix rows into shared memory in the UMMA canonical K-major
//     no-swizzle layout (8 rows x 16 B core matrices; LBO = 128 B between
//     the two K halves of one MMA, SBO = 1024 B between 8-row groups);
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::tf32
//     (M = 128, N = BN, K = 8) x 4 per chunk, accumulating in TMEM, and
//     tcgen05.commit's the chunk's stage back to the producers (mbarrier);
//   * a 3-stage smem ring lets the gather of chunk k+1.. overlap the MMAs
//     of chunk k;
//   * the epilogue reads TMEM with tcgen05.ld 32x32b (thread = tile row)
//     and applies the layer's fused tail: bias + 2x2 max-pool + origin mask
//     (conv2), bias + ReLU (ip1), max-pool backward scatter (ip1 dgrad),
//     plain stores (conv2 dgrad), split-K partial stores + bias gradient
//     (conv2 / ip1 weight gradients).
#include <cstdint>

#include "tc.h"

namespace pn {
namespace tc {

constexpr int BM = 128;     // tile rows = UMMA M
constexpr int BK = 32;      // K elements per chunk (4 MMAs of K = 8)
constexpr int STAGES = 3;
constexpr int THREADS = 128;

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(to_tf32(v.x)), "r"(to_tf32(v.y)),
               "r"(to_tf32(v.z)), "r"(to_tf32(v.w))
               : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle (sm_100 "version" 1).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);       // start address
  d |= (uint64_t)(128 >> 4) << 16;               // LBO: next 16-B K chunk
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO: next 8-row group
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  return d;                                      // layout type 0 = SWIZZLE_NONE
}
// Instruction descriptor: kind::tf32, D = F32, A = B = TF32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t core_off(int r, int kc) {  // byte offset of (row, 16-B K chunk)
  return (uint32_t)((r >> 3) * 1024 + kc * 128 + (r & 7) * 16);
}

// ------------------------------------------------------------------ engine
template <class Op>
__global__ void __launch_bounds__(THREADS) tc_gemm(const __grid_constant__ typename Op::Params prm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[STAGES + 1];
  __shared__ uint32_t tmem_base;
  constexpr int BN = Op::BN;
  constexpr int A_BYTES = BM * BK * 4;
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = A_BYTES + B_BYTES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Op op(prm);
  if (tid == 0) {
    for (int s = 0; s <= STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, Op::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t sbase = smem_u32(smem);
  constexpr uint32_t idesc = make_idesc(BM, BN);
  const int nk = op.num_k_chunks();
  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % STAGES, fill = kb / STAGES;
    if (fill > 0) mbar_wait(&bars[s], (fill - 1) & 1);
    const uint32_t As = sbase + s * STAGE, Bs = As + A_BYTES;
    const int k0 = kb * BK;
#pragma unroll 2
    for (int u = tid; u < BM * (BK / 4); u += THREADS) {
      const int r = u & (BM - 1), kc = u >> 7;
      sts128(As + core_off(r, kc), op.a4(r, k0 + kc * 4));
    }
#pragma unroll 2
    for (int u = tid; u < BN * (BK / 4); u += THREADS) {
      const int c = u % BN, kc = u / BN;
      sts128(Bs + core_off(c, kc), op.b4(c, k0 + kc * 4));
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < BK / 8; ++k)
        mma_tf32(tbase, make_desc(As + k * 256), make_desc(Bs + k * 256), idesc, (kb | k) != 0);
      mma_commit(&bars[s]);
      if (kb == nk - 1) mma_commit(&bars[STAGES]);
    }
  }
  const int row = warp * 32 + lane;
  if (nk > 0) {
    mbar_wait(&bars[STAGES], 0);
    tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
      op.epilogue(row, c0, v, lane);
    }
  } else {  // empty K range (e.g. a weight-gradient split with no images)
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
      op.epilogue(row, c0, v, lane);
    }
  }
  op.finish(row);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, Op::TMEM_COLS);
}

__device__ __forceinline__ float4 f4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }
__device__ __forceinline__ float ld(const float* p) { return __ldg(p); }

// ------------------------------------------- conv2 + bias + pool2 (+mask)
// rows r = (image n = 2*tile + r/64, position p = ho*8+wo), cols f (50 of 64),
// K = (c,i,j) 500 (+12 zero pad).  A(r,k) = p1[n,c,ho+i,wo+j], B(f,k) = W2[f,k].
struct Conv2Fwd {
  struct Params {
    const float* p1;
    const float* w;
    const float* b;
    float* p2;
    uint8_t* m2;
    int N;
  };
  static constexpr int BN = 64, TMEM_COLS = 64;
  const Params& p;
  int n0;
  __device__ Conv2Fwd(const Params& q) : p(q), n0(blockIdx.x * 2) {}
  __device__ int num_k_chunks() const { return 16; }
  __device__ float a1(int r, int k) const {
    const int n = n0 + (r >> 6);
    if (k >= 500 || n >= p.N) return 0.f;
    const int pos = r & 63, ho = pos >> 3, wo = pos & 7;
    const int c = k / 25, rem = k - c * 25, i = rem / 5, j = rem - i * 5;
    return ld(p.p1 + (size_t)n * 2880 + c * 144 + (ho + i) * 12 + wo + j);
  }
  __device__ float4 a4(int r, int k) const { return f4(a1(r, k), a1(r, k + 1), a1(r, k + 2), a1(r, k + 3)); }
  __device__ float4 b4(int f, int k) const {
    if (f >= 50 || k >= 500) return f4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(p.w + f * 500 + k));  // 500*4 B rows, k % 4 == 0
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int lane) const {
    const int n = n0 + (row >> 6), pos = row & 63, ho = pos >> 3, wo = pos & 7;
    const int off = (ho & 1) * 2 + (wo & 1);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int f = c0 + j;
      if (f >= 50) break;
      float best = v[j] + __ldg(p.b + f);
      int arg = off;
#pragma unroll
      for (int x = 1; x <= 8; x <<= 3) {  // xor 1 (wo pair), xor 8 (ho pair)
        const float ov = __shfl_xor_sync(0xffffffffu, best, x);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, x);
        if (ov > best || (ov == best && oa < arg)) { best = ov; arg = oa; }
      }
      if (off == 0 && n < p.N) {
        const size_t o = ((size_t)n * 50 + f) * 16 + (ho >> 1) * 4 + (wo >> 1);
        p.p2[o] = best;
        p.m2[o] = (uint8_t)arg;
      }
    }
  }
  __device__ void finish(int) const {}
};

// ------------------------------------------------------ ip fwd + bias + relu
// rows n, cols o (BN 64 per CTA column tile), K = 800.
struct IpFwd {
  struct Params {
    const float* x;
    const float* w;
    const float* b;
    float* y;
    int M, K, Nout, relu;
  };
  static constexpr int BN = 64, TMEM_COLS = 64;
  const Params& p;
  int m0, o0;
  __device__ IpFwd(const Params& q) : p(q), m0(blockIdx.y * BM), o0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return (p.K + BK - 1) / BK; }
  __device__ float4 a4(int r, int k) const {
    const int m = m0 + r;
    if (m >= p.M || k >= p.K) return f4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(p.x + (size_t)m * p.K + k));
  }
  __device__ float4 b4(int c, int k) const {
    const int o = o0 + c;
    if (o >= p.Nout || k >= p.K) return f4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(p.w + (size_t)o * p.K + k));
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int) const {
    const int m = m0 + row;
    if (m >= p.M) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int o = o0 + c0 + j;
      if (o >= p.Nout) break;
      float4 r;
      r.x = v[j] + __ldg(p.b + o);
      r.y = v[j + 1] + __ldg(p.b + o + 1);
      r.z = v[j + 2] + __ldg(p.b + o + 2);
      r.w = v[j + 3] + __ldg(p.b + o + 3);
      if (p.relu) {
        r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f); r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
      }
      *reinterpret_cast<float4*>(p.y + (size_t)m * p.Nout + o) = r;
    }
  }
  __device__ void finish(int) const {}
};

// --------------------------------------------- ip weight gradient (+ bias)
// dW[o,k] = sum_n dy[n,o] x[n,k]: rows o, cols k (BN 160), K = n (batch).
struct IpWgrad {
  struct Params {
    const float* dy;
    const float* x;
    float* dw;
    float* db;
    int M, K, Nout;
  };
  static constexpr int BN = 160, TMEM_COLS = 256;
  const Params& p;
  int o0, k0;
  __device__ IpWgrad(const Params& q) : p(q), o0(blockIdx.y * BM), k0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return (p.M + BK - 1) / BK; }
  __device__ float4 a4(int r, int n) const {
    const int o = o0 + r;
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = (o < p.Nout && n + t < p.M) ? ld(p.dy + (size_t)(n + t) * p.Nout + o) : 0.f;
    return f4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 b4(int c, int n) const {
    const int k = k0 + c;
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = (k < p.K && n + t < p.M) ? ld(p.x + (size_t)(n + t) * p.K + k) : 0.f;
    return f4(v[0], v[1], v[2], v[3]);
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int) const {
    const int o = o0 + row;
    if (o >= p.Nout) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int k = k0 + c0 + j;
      if (k >= p.K) break;
      *reinterpret_cast<float4*>(p.dw + (size_t)o * p.K + k) = f4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  __device__ void finish(int row) const {  // db[o] = sum_n dy[n,o], fp32, ascending n
    const int o = o0 + row;
    if (blockIdx.x != 0 || o >= p.Nout || !p.db) return;
    float acc = 0.f;
    for (int n = 0; n < p.M; ++n) acc += ld(p.dy + (size_t)n * p.Nout + o);
    p.db[o] = acc;
  }
};

// ------------------------------- ip1 data gradient + pool2 backward (LeNet)
// dp2[n,k] = sum_o dy[n,o] W1[o,k]; rows n, cols k (BN 160 = 10 filters x 16),
// K = o (500).  Epilogue scatters each dp2 value to its pool2 origin in the
// dense conv2 gradient G2[n,f,8,8] (zeros elsewhere).
struct IpDgradUnpool {
  struct Params {
    const float* dy;   // [N,500]
    const float* w;    // [500,800]
    const uint8_t* m2; // [N,800]
    float* g2;         // [N,50,8,8]
    int N;
  };
  static constexpr int BN = 160, TMEM_COLS = 256;
  const Params& p;
  int m0, k0;
  __device__ IpDgradUnpool(const Params& q) : p(q), m0(blockIdx.y * BM), k0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return 16; }  // 500 -> 512
  __device__ float4 a4(int r, int o) const {
    const int n = m0 + r;
    if (n >= p.N || o >= 500) return f4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(p.dy + (size_t)n * 500 + o));
  }
  __device__ float4 b4(int c, int o) const {
    const int k = k0 + c;
    if (o >= 500) return f4(0.f, 0.f, 0.f, 0.f);
    return f4(ld(p.w + (size_t)o * 800 + k), ld(p.w + (size_t)(o + 1) * 800 + k), ld(p.w + (size_t)(o + 2) * 800 + k),
              ld(p.w + (size_t)(o + 3) * 800 + k));
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int) const {
    const int n = m0 + row;
    if (n >= p.N) return;
    const int f = (k0 + c0) >> 4;  // the 16 columns are filter f's 4x4 pooled outputs
    const uint8_t* m = p.m2 + (size_t)n * 800 + f * 16;
    float* g = p.g2 + ((size_t)n * 50 + f) * 64;
    uint32_t mw[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) mw[t] = __ldg(reinterpret_cast<const uint32_t*>(m) + t);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      float o8[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int q = (h >> 1) * 4 + (w >> 1);
        const int off = (mw[q >> 2] >> (8 * (q & 3))) & 0xff;
        o8[w] = (off == ((h & 1) * 2 + (w & 1))) ? v[q] : 0.f;
      }
      *reinterpret_cast<float4*>(g + h * 8) = f4(o8[0], o8[1], o8[2], o8[3]);
      *reinterpret_cast<float4*>(g + h * 8 + 4) = f4(o8[4], o8[5], o8[6], o8[7]);
    }
  }
  __device__ void finish(int) const {}
};

// ------------------------------------------------- conv2 data gradient
// dp1[n,c,h,w] = sum_{f,i,j} W2[f,c,i,j] G2[n,f,h-i,w-j] (col2im of W^T G,
// gather form).  rows r = n*144 + h*12 + w, cols c (20 of 32),
// K = (f,i,j) 1250 (+30 pad).
struct Conv2Dgrad {
  struct Params {
    const float* g2;
    const float* w;
    float* dp1;
    int N;
  };
  static constexpr int BN = 32, TMEM_COLS = 32;
  const Params& p;
  int r0;
  __device__ Conv2Dgrad(const Params& q) : p(q), r0(blockIdx.x * BM) {}
  __device__ int num_k_chunks() const { return 40; }
  __device__ float a1(int n, int h, int w, int k) const {
    if (k >= 1250) return 0.f;
    const int f = k / 25, rem = k - f * 25, i = rem / 5, j = rem - i * 5;
    const int ho = h - i, wo = w - j;
    if ((unsigned)ho >= 8u || (unsigned)wo >= 8u) return 0.f;
    return ld(p.g2 + (size_t)n * 3200 + f * 64 + ho * 8 + wo);
  }
  __device__ float4 a4(int r, int k) const {
    const int gr = r0 + r;
    if (gr >= p.N * 144) return f4(0.f, 0.f, 0.f, 0.f);
    const int n = gr / 144, hw = gr - n * 144, h = hw / 12, w = hw - h * 12;
    return f4(a1(n, h, w, k), a1(n, h, w, k + 1), a1(n, h, w, k + 2), a1(n, h, w, k + 3));
  }
  __device__ float b1(int c, int k) const {
    if (k >= 1250) return 0.f;
    const int f = k / 25, rem = k - f * 25;
    return ld(p.w + f * 500 + c * 25 + rem);
  }
  __device__ float4 b4(int c, int k) const {
    if (c >= 20) return f4(0.f, 0.f, 0.f, 0.f);
    return f4(b1(c, k), b1(c, k + 1), b1(c, k + 2), b1(c, k + 3));
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int) const {
    const int gr = r0 + row;
    if (gr >= p.N * 144) return;
    const int n = gr / 144, hw = gr - n * 144;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = c0 + j;
      if (c >= 20) break;
      p.dp1[(size_t)n * 2880 + c * 144 + hw] = v[j];
    }
  }
  __device__ void finish(int) const {}
};

// ------------------------------------------------ conv2 weight gradient
// dW2[f,(c,i,j)] = sum_{n,p} G2[n,f,p] p1[n,c,ho+i,wo+j]; rows (c,i,j) 500 of
// 512 (4 tiles), cols f (50 of 64), K = (n in split, p).  Writes split
// partials [split][f*500 + k]; bias partial db2[f] = sum G2 (row tile 0).
struct Conv2Wgrad {
  struct Params {
    const float* g2;
    const float* p1;
    float* part;
    int N, splits, pstride;
  };
  static constexpr int BN = 64, TMEM_COLS = 64;
  const Params& p;
  int kw0, n0, n1;
  __device__ Conv2Wgrad(const Params& q) : p(q), kw0(blockIdx.x * BM) {
    n0 = (int)((long long)q.N * blockIdx.y / q.splits);
    n1 = (int)((long long)q.N * (blockIdx.y + 1) / q.splits);
  }
  __device__ int num_k_chunks() const { return (n1 - n0) * 2; }  // 64 positions = 2 chunks per image
  __device__ float4 a4(int r, int kk) const {
    const int kw = kw0 + r;
    if (kw >= 500) return f4(0.f, 0.f, 0.f, 0.f);
    const int n = n0 + (kk >> 6), pos = kk & 63, ho = pos >> 3, wo = pos & 7;
    const int c = kw / 25, rem = kw - c * 25, i = rem / 5, j = rem - i * 5;
    const float* src = p.p1 + (size_t)n * 2880 + c * 144 + (ho + i) * 12 + wo + j;
    return f4(ld(src), ld(src + 1), ld(src + 2), ld(src + 3));
  }
  __device__ float4 b4(int f, int kk) const {
    if (f >= 50) return f4(0.f, 0.f, 0.f, 0.f);
    const int n = n0 + (kk >> 6), pos = kk & 63;
    return __ldg(reinterpret_cast<const float4*>(p.g2 + (size_t)n * 3200 + f * 64 + pos));
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16], int) const {
    const int kw = kw0 + row;
    if (kw >= 500) return;
    float* dst = p.part + (size_t)blockIdx.y * p.pstride;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int f = c0 + j;
      if (f >= 50) break;
      dst[f * 500 + kw] = v[j];
    }
  }
  __device__ void finish(int row) const {  // bias partial: fp32, ascending (n, p)
    if (blockIdx.x != 0 || row >= 50) return;
    float acc = 0.f;
    for (int n = n0; n < n1; ++n) {
      const float* g = p.g2 + (size_t)n * 3200 + row * 64;
      for (int q = 0; q < 64; ++q) acc += ld(g + q);
    }
    p.part[(size_t)blockIdx.y * p.pstride + 25000 + row] = acc;
  }
};

// ------------------------------------------------------------ host side
template <class Op>
static constexpr size_t smem_bytes() {
  return (size_t)STAGES * (BM * BK * 4 + Op::BN * BK * 4);
}

template <class Op>
static cudaError_t opt_in() {
  return cudaFuncSetAttribute((const void*)tc_gemm<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes<Op>());
}

cudaError_t setup() {
  cudaError_t e;
  if ((e = opt_in<Conv2Fwd>()) != cudaSuccess) return e;
  if ((e = opt_in<IpFwd>()) != cudaSuccess) return e;
  if ((e = opt_in<IpWgrad>()) != cudaSuccess) return e;
  if ((e = opt_in<IpDgradUnpool>()) != cudaSuccess) return e;
  if ((e = opt_in<Conv2Dgrad>()) != cudaSuccess) return e;
  if ((e = opt_in<Conv2Wgrad>()) != cudaSuccess) return e;
  return cudaSuccess;
}

static unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

Launch conv2_pool2_launch(const float* w, const float* b, const float* p1, float* p2, uint8_t* m2, int N, int) {
  Launch l;
  Conv2Fwd::Params p{p1, w, b, p2, m2, N};
  l.set((const void*)tc_gemm<Conv2Fwd>, dim3(cdiv(N, 2)), dim3(THREADS), smem_bytes<Conv2Fwd>(), p);
  return l;
}

Launch ip_fwd_launch(const float* x, const float* w, const float* b, float* y, int M, int K, int Nout, bool relu,
                     int) {
  Launch l;
  IpFwd::Params p{x, w, b, y, M, K, Nout, relu ? 1 : 0};
  l.set((const void*)tc_gemm<IpFwd>, dim3(cdiv(Nout, IpFwd::BN), cdiv(M, BM)), dim3(THREADS), smem_bytes<IpFwd>(), p);
  return l;
}

Launch ip_wgrad_launch(const float* dy, const float* x, float* dw, float* db, int M, int K, int Nout, int) {
  Launch l;
  IpWgrad::Params p{dy, x, dw, db, M, K, Nout};
  l.set((const void*)tc_gemm<IpWgrad>, dim3(cdiv(K, IpWgrad::BN), cdiv(Nout, BM)), dim3(THREADS),
        smem_bytes<IpWgrad>(), p);
  return l;
}

Launch ip_dgrad_unpool_launch(const float* dy, const float* w, const uint8_t* m2, float* g2, int N, int) {
  Launch l;
  IpDgradUnpool::Params p{dy, w, m2, g2, N};
  l.set((const void*)tc_gemm<IpDgradUnpool>, dim3(800 / IpDgradUnpool::BN, cdiv(N, BM)), dim3(THREADS),
        smem_bytes<IpDgradUnpool>(), p);
  return l;
}

Launch conv2_dgrad_launch(const float* g2, const float* w, float* dp1, int N, int) {
  Launch l;
  Conv2Dgrad::Params p{g2, w, dp1, N};
  l.set((const void*)tc_gemm<Conv2Dgrad>, dim3(cdiv((long long)N * 144, BM)), dim3(THREADS),
        smem_bytes<Conv2Dgrad>(), p);
  return l;
}

Launch conv2_wgrad_launch(const float* g2, const float* p1, float* part, int splits, int N, int) {
  Launch l;
  Conv2Wgrad::Params p{g2, p1, part, N, splits, 25050};
  l.set((const void*)tc_gemm<Conv2Wgrad>, dim3(4, splits), dim3(THREADS), smem_bytes<Conv2Wgrad>(), p);
  return l;
}

}  // namespace tc
}  // namespace pn
