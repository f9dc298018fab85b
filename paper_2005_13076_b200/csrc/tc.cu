// tc.cu -- tcgen05 TF32 implicit-GEMM kernels for the GEMM-shaped LeNet
// layers.
//
// Engine (one CTA = one 128-row output tile, 8 warps, all producers):
//   * operands are assembled per 32-wide K chunk in a shared-memory ring in
//     the UMMA canonical K-major no-swizzle layout (core matrix = 8 rows x
//     4 K (16 B); LBO = 128 B between the K halves of one MMA, SBO = 1024 B
//     between 8-row groups).  MN-major TF32 descriptors were measured to
//     produce zeros on this part (tools/umma_probe.cu), so transposed global
//     operands are gathered into K-major rows as well;
//   * copy-type operand units move global -> shared with cp.async (16-byte
//     rows, or 4 x 4-byte scalars for transposed operands), issued
//     LOOKAHEAD chunks ahead of the chunk being consumed; the issuing thread
//     later rounds its own units to TF32 in place (cvt.rna: round to
//     nearest) -- pre-rounded packed weights skip that;
//     gather-type units (implicit im2col) are built from activations the CTA
//     staged in shared memory;
//   * one thread issues tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=BN,
//     K=8) x 4 per chunk into a TMEM accumulator and tcgen05.commit's the
//     stage back to the producers through an mbarrier;
//   * the epilogue reads TMEM with tcgen05.ld 32x32b (thread = tile row;
//     warps 4-7 take the upper half of the columns) and applies the layer's
//     fused tail.
#include <cstdint>

#include "tc.h"

namespace pn {
namespace tc {

constexpr int BM = 128;  // tile rows = UMMA M
constexpr int BK = 32;   // K elements per chunk (4 MMAs of K = 8)
constexpr int THREADS = 256;

enum Mode { COPY16 = 0, COPY16_PRE = 1, COPY4 = 2, GATHER = 3 };

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
__device__ __forceinline__ float tf32f(float x) { return __uint_as_float(to_tf32(x)); }
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(to_tf32(v.x)), "r"(to_tf32(v.y)),
               "r"(to_tf32(v.z)), "r"(to_tf32(v.w))
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// UMMA shared-memory descriptor, no swizzle, sm_100 version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// Instruction descriptor: kind::tf32, D = F32, A = B = TF32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// K-major: byte offset of (row r, 16-B K chunk kc) inside a [rows x 32] chunk
__device__ __forceinline__ uint32_t kmaj_off(int r, int kc) {
  return (uint32_t)((r >> 3) * 1024 + kc * 128 + (r & 7) * 16);
}
__device__ __forceinline__ float4 f4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }
__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// ------------------------------------------------------------------ engine
// Op interface:
//   BN, TMEM_COLS, STAGES, A_MODE, B_MODE, STAGE_BYTES, SYNC_AFTER_WAIT
//   Op(params, staging_smem, ring_smem)        decodes the tile
//   int num_k_chunks()
//   void stage(tid)                            one-time staging (engine syncs after)
//   void issue_extra(chunk, tid)               extra cp.async work for a chunk (may be empty)
//   COPY16/_PRE: const float* a_src(r, k, &valid)    16-byte source of A(r, k..k+3)
//   COPY4:       const float* a_src4(r, k, t, &valid) source of A(r, k+t)
//   GATHER:      float4 a(r, k)                    built from staged smem
//   (B likewise with b_src / b_src4 / b)
//   void a_raw(r, k, float4) / b_raw(c, k, float4)   raw copied values (bias sums)
//   void epilogue(row, c0, v[16])              columns c0..c0+15
//   void finish(tid)                           after epilogue + __syncthreads
template <class Op>
__device__ __forceinline__ void issue_chunk(Op& op, uint32_t As, uint32_t Bs, int k0, int tid) {
  constexpr int BN = Op::BN;
  if (Op::A_MODE != GATHER) {
#pragma unroll
    for (int q = 0; q < BM * (BK / 4) / THREADS; ++q) {
      const int u = tid + q * THREADS, r = u & (BM - 1), kc = u >> 7;
      const uint32_t dst = As + kmaj_off(r, kc);
      if (Op::A_MODE == COPY4) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          bool v;
          const float* s = op.a_src4(r, k0 + kc * 4, t, v);
          cp4(dst + 4 * t, s, v);
        }
      } else {
        bool v;
        const float* s = op.a_src(r, k0 + kc * 4, v);
        cp16(dst, s, v);
      }
    }
  }
  if (Op::B_MODE != GATHER) {
    for (int u = tid; u < BN * (BK / 4); u += THREADS) {
      const int c = u % BN, kc = u / BN;
      const uint32_t dst = Bs + kmaj_off(c, kc);
      if (Op::B_MODE == COPY4) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          bool v;
          const float* s = op.b_src4(c, k0 + kc * 4, t, v);
          cp4(dst + 4 * t, s, v);
        }
      } else {
        bool v;
        const float* s = op.b_src(c, k0 + kc * 4, v);
        cp16(dst, s, v);
      }
    }
  }
}

template <class Op>
__device__ __forceinline__ void produce_chunk(Op& op, uint32_t As, uint32_t Bs, int k0, int tid) {
  constexpr int BN = Op::BN;
#pragma unroll
  for (int q = 0; q < BM * (BK / 4) / THREADS; ++q) {
    const int u = tid + q * THREADS, r = u & (BM - 1), kc = u >> 7;
    const uint32_t dst = As + kmaj_off(r, kc);
    if (Op::A_MODE == GATHER) {
      sts128(dst, op.a(r, k0 + kc * 4));
    } else if (Op::A_MODE != COPY16_PRE) {
      const float4 v = lds128(dst);
      op.a_raw(r, k0 + kc * 4, v);
      sts128(dst, v);
    }
  }
  for (int u = tid; u < BN * (BK / 4); u += THREADS) {
    const int c = u % BN, kc = u / BN;
    const uint32_t dst = Bs + kmaj_off(c, kc);
    if (Op::B_MODE == GATHER) {
      sts128(dst, op.b(c, k0 + kc * 4));
    } else if (Op::B_MODE != COPY16_PRE) {
      const float4 v = lds128(dst);
      op.b_raw(c, k0 + kc * 4, v);
      sts128(dst, v);
    }
  }
}

template <class Op>
__global__ void __launch_bounds__(THREADS) tc_gemm(const __grid_constant__ typename Op::Params prm) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int S = Op::STAGES;
  constexpr int L = S - 2 > 0 ? S - 2 : 1;  // cp.async lookahead (chunks)
  __shared__ uint64_t bars[S + 1];
  __shared__ uint32_t tmem_base;
  constexpr int BN = Op::BN;
  constexpr int A_BYTES = BM * BK * 4;
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = A_BYTES + B_BYTES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Op op(prm, smem + S * STAGE, smem);
  if (tid == 0) {
    for (int s = 0; s <= S; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, Op::TMEM_COLS);
  op.stage(tid);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t sbase = smem_u32(smem);
  constexpr uint32_t idesc = make_idesc(BM, BN);
  const int nk = op.num_k_chunks();
  // prologue: chunks 0 .. L-1 in flight
#pragma unroll 1
  for (int c = 0; c < L; ++c) {
    if (c < nk) {
      op.issue_extra(c, tid);
      issue_chunk(op, sbase + (c % S) * STAGE, sbase + (c % S) * STAGE + A_BYTES, c * BK, tid);
    }
    cp_commit();
  }
#pragma unroll 1
  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % S;
    const int c = kb + L;
    if (c < nk) {
      const int s2 = c % S;
      if (c >= S) mbar_wait(&bars[s2], ((c / S) - 1) & 1);
      op.issue_extra(c, tid);
      issue_chunk(op, sbase + s2 * STAGE, sbase + s2 * STAGE + A_BYTES, c * BK, tid);
    }
    cp_commit();
    cp_wait<L>();
    if (Op::SYNC_AFTER_WAIT) __syncthreads();
    const uint32_t As = sbase + s * STAGE, Bs = As + A_BYTES;
    produce_chunk(op, As, Bs, kb * BK, tid);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < BK / 8; ++k)
        mma_tf32(tbase, make_desc(As + k * 256, 128, 1024), make_desc(Bs + k * 256, 128, 1024), idesc,
                 (kb | k) != 0);
      mma_commit(&bars[s]);
      if (kb == nk - 1) mma_commit(&bars[S]);
    }
  }
  cp_wait<0>();
  // epilogue: warps 0-3 columns [0, BN/2), warps 4-7 [BN/2, BN) (BN >= 32),
  // or warps 0-3 only for BN = 16
  const int row = (warp & 3) * 32 + lane;
  constexpr int HALF = BN >= 32 ? BN / 2 : BN;
  const bool active = BN >= 32 || warp < 4;
  const int cbeg = (BN >= 32 && warp >= 4) ? HALF : 0;
  if (nk > 0) {
    mbar_wait(&bars[S], 0);
    tc_fence_after();
    if (active) {
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + HALF; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + ((uint32_t)((warp & 3) * 32) << 16) + c0, v);
        op.epilogue(row, c0, v);
      }
    }
  } else if (active) {  // empty K range (a weight-gradient split with no images)
#pragma unroll 1
    for (int c0 = cbeg; c0 < cbeg + HALF; c0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
      op.epilogue(row, c0, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  op.finish(tid);
  if (warp == 0) tmem_dealloc(tbase, Op::TMEM_COLS);
}

// common no-op hooks
struct OpBase {
  static constexpr bool SYNC_AFTER_WAIT = false;
  __device__ void stage(int) {}
  __device__ void issue_extra(int, int) {}
  __device__ void a_raw(int, int, float4) {}
  __device__ void b_raw(int, int, float4) {}
  __device__ void finish(int) {}
  __device__ float4 a(int, int) const { return zero4(); }
  __device__ float4 b(int, int) const { return zero4(); }
  __device__ const float* a_src(int, int, bool& v) const { v = false; return nullptr; }
  __device__ const float* b_src(int, int, bool& v) const { v = false; return nullptr; }
  __device__ const float* a_src4(int, int, int, bool& v) const { v = false; return nullptr; }
  __device__ const float* b_src4(int, int, int, bool& v) const { v = false; return nullptr; }
};

// ------------------------------------------- conv2 + bias + pool2 (+mask)
// rows r = (image n = 2*tile + r/64, position p = ho*8+wo), cols f (50 of 64),
// K = (c,i,j) 500 (+12 zero pad).  A(r,k) = p1[n,c,ho+i,wo+j] gathered from
// the two staged images through a k -> c*144+i*12+j table; B(f,k) = W2[f,k]
// copied with cp.async.
struct Conv2Fwd : OpBase {
  struct Params {
    const float* p1;
    const float* w;
    const float* b;
    float* p2;
    uint8_t* m2;
    int N;
  };
  static constexpr int BN = 64, TMEM_COLS = 64, STAGES = 4;
  static constexpr int A_MODE = GATHER, B_MODE = COPY16;
  static constexpr int STAGE_BYTES = 2 * 2880 * 4 + 512 * 4;
  const Params& p;
  float* img;
  int* koff;
  int n0, rowoff;
  __device__ Conv2Fwd(const Params& q, uint8_t* st, uint8_t*)
      : p(q), img((float*)st), koff((int*)(st + 2 * 2880 * 4)) {
    n0 = blockIdx.x * 2;
    const int r = threadIdx.x & 127, pos = r & 63;
    rowoff = (r >> 6) * 2880 + (pos >> 3) * 12 + (pos & 7);
  }
  __device__ int num_k_chunks() const { return 16; }
  __device__ void stage(int tid) {
    const int cnt = min(2, p.N - n0) * 2880;
    const float4* src = reinterpret_cast<const float4*>(p.p1 + (size_t)n0 * 2880);
    for (int i = tid; i < 2 * 720; i += THREADS)
      reinterpret_cast<float4*>(img)[i] = (i * 4 < cnt) ? __ldg(src + i) : zero4();
    for (int k = tid; k < 512; k += THREADS) {
      const int c = k / 25, rem = k - c * 25, i = rem / 5, j = rem - i * 5;
      koff[k] = k < 500 ? c * 144 + i * 12 + j : -1;
    }
  }
  __device__ float g(int k) const {
    const int o = koff[k];
    return o >= 0 ? img[rowoff + o] : 0.f;
  }
  __device__ float4 a(int, int k) const { return f4(g(k), g(k + 1), g(k + 2), g(k + 3)); }
  __device__ const float* b_src(int f, int k, bool& v) const {
    v = f < 50 && k < 500;
    return v ? p.w + f * 500 + k : p.w;
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
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
};

// ------------------------------------------------------ ip fwd + bias + relu
// y[n,o] = relu(sum_k x[n,k] W[o,k] + b[o]); rows n, cols o (BN 16), K = 800.
struct IpFwd : OpBase {
  struct Params {
    const float* x;
    const float* w;
    const float* b;
    float* y;
    int M, K, Nout, relu;
  };
  static constexpr int BN = 16, TMEM_COLS = 32, STAGES = 4;
  static constexpr int A_MODE = COPY16, B_MODE = COPY16;
  static constexpr int STAGE_BYTES = 0;
  const Params& p;
  int m0, o0;
  __device__ IpFwd(const Params& q, uint8_t*, uint8_t*) : p(q), m0(blockIdx.y * BM), o0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return (p.K + BK - 1) / BK; }
  __device__ const float* a_src(int r, int k, bool& v) const {
    const int m = m0 + r;
    v = m < p.M && k < p.K;
    return v ? p.x + (size_t)m * p.K + k : p.x;
  }
  __device__ const float* b_src(int c, int k, bool& v) const {
    const int o = o0 + c;
    v = o < p.Nout && k < p.K;
    return v ? p.w + (size_t)o * p.K + k : p.w;
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
    const int m = m0 + row;
    if (m >= p.M) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int o = o0 + c0 + j;
      if (o >= p.Nout) break;
      float4 r = f4(v[j] + __ldg(p.b + o), v[j + 1] + __ldg(p.b + o + 1), v[j + 2] + __ldg(p.b + o + 2),
                    v[j + 3] + __ldg(p.b + o + 3));
      if (p.relu) {
        r.x = fmaxf(r.x, 0.f); r.y = fmaxf(r.y, 0.f); r.z = fmaxf(r.z, 0.f); r.w = fmaxf(r.w, 0.f);
      }
      *reinterpret_cast<float4*>(p.y + (size_t)m * p.Nout + o) = r;
    }
  }
};

// --------------------------------------------- ip weight gradient (+ bias)
// dW[o,k] = sum_n dy[n,o] x[n,k]: rows o, cols k (BN 32), K = n (batch).
// Both operands are transposed in global memory: 4-byte cp.async per element
// (a warp covers 32 consecutive rows: coalesced).  db[o] = sum_n dy[n,o]
// (fp32, unrounded) from the raw A values in column tile 0; thread tid always
// owns row o0 + (tid & 127), K sub-chunks tid >> 7 and 2 + (tid >> 7).
struct IpWgrad : OpBase {
  struct Params {
    const float* dy;
    const float* x;
    float* dw;
    float* db;
    int M, K, Nout;
  };
  static constexpr int BN = 32, TMEM_COLS = 32, STAGES = 4;
  static constexpr int A_MODE = COPY4, B_MODE = COPY4;
  static constexpr int STAGE_BYTES = THREADS * 4;
  const Params& p;
  float* red;
  int o0, k0;
  float bacc;
  __device__ IpWgrad(const Params& q, uint8_t* st, uint8_t*)
      : p(q), red((float*)st), o0(blockIdx.y * BM), k0(blockIdx.x * BN), bacc(0.f) {}
  __device__ int num_k_chunks() const { return (p.M + BK - 1) / BK; }
  __device__ const float* a_src4(int r, int n, int t, bool& v) const {
    const int o = o0 + r;
    v = o < p.Nout && n + t < p.M;
    return v ? p.dy + (size_t)(n + t) * p.Nout + o : p.dy;
  }
  __device__ const float* b_src4(int c, int n, int t, bool& v) const {
    const int k = k0 + c;
    v = k < p.K && n + t < p.M;
    return v ? p.x + (size_t)(n + t) * p.K + k : p.x;
  }
  __device__ void a_raw(int, int, float4 v) { bacc += (v.x + v.y) + (v.z + v.w); }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
    const int o = o0 + row;
    if (o >= p.Nout) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int k = k0 + c0 + j;
      if (k >= p.K) break;
      *reinterpret_cast<float4*>(p.dw + (size_t)o * p.K + k) = f4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  __device__ void finish(int tid) {
    red[tid] = bacc;
    __syncthreads();
    if (blockIdx.x == 0 && p.db && tid < 128 && o0 + tid < p.Nout) p.db[o0 + tid] = red[tid] + red[tid + 128];
  }
};

// ------------------------------- ip1 data gradient + pool2 backward (LeNet)
// dp2[n,k] = sum_o dy[n,o] W1[o,k]; rows n, cols k (BN 32 = 2 filters x 16),
// K = o (500).  B(k, o) = W1[o][k] is read transposed (4-byte cp.async).
// Epilogue scatters each dp2 value to its pool2 origin in the dense conv2
// gradient G2[n,f,8,8] (zeros elsewhere).
struct IpDgradUnpool : OpBase {
  struct Params {
    const float* dy;    // [N,500]
    const float* w;     // [500,800]
    const uint8_t* m2;  // [N,800]
    float* g2;          // [N,50,8,8]
    int N;
  };
  static constexpr int BN = 32, TMEM_COLS = 32, STAGES = 4;
  static constexpr int A_MODE = COPY16, B_MODE = COPY4;
  static constexpr int STAGE_BYTES = 0;
  const Params& p;
  int m0, k0;
  __device__ IpDgradUnpool(const Params& q, uint8_t*, uint8_t*) : p(q), m0(blockIdx.y * BM), k0(blockIdx.x * BN) {}
  __device__ int num_k_chunks() const { return 16; }  // 500 -> 512
  __device__ const float* a_src(int r, int o, bool& v) const {
    const int n = m0 + r;
    v = n < p.N && o < 500;
    return v ? p.dy + (size_t)n * 500 + o : p.dy;
  }
  __device__ const float* b_src4(int c, int o, int t, bool& v) const {
    v = o + t < 500;
    return v ? p.w + (size_t)(o + t) * 800 + k0 + c : p.w;
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
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
};

// ------------------------------------------------- conv2 data gradient
// dp1 = col2im(W2^T G2), computed as the GEMM
//   C[(c,i,j), (n,p)] = sum_f W2[f,c,i,j] G2[n,f,p]
// with rows = 5 input channels x 25 taps (+3 zero rows) per M tile (4 tiles),
// cols = 2 images x 64 positions (N = 128), K = f (50 of 64), followed by the
// col2im gather dp1[n,c,h,w] = sum_{i,j} C[(c,i,j), (n, h-i, w-j)] done from
// shared memory (C staged over the drained operand ring).  A = W2^T packed
// TF32 once per backward (pack_w2t); B(p, f) = G2[n,f,p] (4-byte cp.async).
struct Conv2Dgrad : OpBase {
  struct Params {
    const float* g2;
    const float* w2t;  // [4][128][64] TF32, zero padded
    float* dp1;
    int N;
  };
  static constexpr int BN = 128, TMEM_COLS = 128, STAGES = 2;
  static constexpr int A_MODE = COPY16_PRE, B_MODE = COPY4;
  static constexpr int STAGE_BYTES = 0;
  const Params& p;
  float* cs;  // [128 rows][128 cols], over the ring after the MMAs
  int m, n0;
  __device__ Conv2Dgrad(const Params& q, uint8_t*, uint8_t* ring)
      : p(q), cs((float*)ring), m(blockIdx.x), n0(blockIdx.y * 2) {}
  __device__ int num_k_chunks() const { return 2; }
  __device__ const float* a_src(int r, int f, bool& v) const {
    v = true;
    return p.w2t + ((size_t)m * 128 + r) * 64 + f;
  }
  __device__ const float* b_src4(int c, int f, int t, bool& v) const {
    const int n = n0 + (c >> 6);
    v = n < p.N && f + t < 50;
    return v ? p.g2 + (size_t)n * 3200 + (f + t) * 64 + (c & 63) : p.g2;
  }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
    float4* dst = reinterpret_cast<float4*>(cs + row * 128 + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = f4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
  __device__ void finish(int tid) {
    // 2 images x 5 channels x 144 outputs
    for (int o = tid; o < 2 * 5 * 144; o += THREADS) {
      const int img = o / 720, rem = o - img * 720, cl = rem / 144, hw = rem - cl * 144;
      const int n = n0 + img;
      if (n >= p.N) continue;
      const int h = hw / 12, w = hw - h * 12;
      const float* base = cs + (cl * 25) * 128 + img * 64;
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int ho = h - i;
        if ((unsigned)ho >= 8u) continue;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const int wo = w - j;
          if ((unsigned)wo >= 8u) continue;
          acc += base[(i * 5 + j) * 128 + ho * 8 + wo];
        }
      }
      p.dp1[(size_t)n * 2880 + (5 * m + cl) * 144 + hw] = acc;
    }
  }
};

// ------------------------------------------------ conv2 weight gradient
// dW2[f,(c,i,j)] = sum_{n,p} G2[n,f,p] p1[n,c,ho+i,wo+j]; rows (c,i,j) 500 of
// 512 (4 tiles), cols f (50 of 64), K = (n in this split, p): 2 chunks per
// image.  Images are cp.async'ed into a 2-slot smem ring one image ahead;
// A gathered from the staged image, B = G2 rows (16-byte cp.async).  Writes
// split partials [split][f*500 + k] and the bias partial db2[f] = sum G2
// (fp32, from the raw B values; thread tid always owns B row f = tid % 64).
struct Conv2Wgrad : OpBase {
  struct Params {
    const float* g2;
    const float* p1;
    float* part;
    int N, splits, pstride;
  };
  static constexpr int BN = 64, TMEM_COLS = 64, STAGES = 4;
  static constexpr int A_MODE = GATHER, B_MODE = COPY16;
  static constexpr bool SYNC_AFTER_WAIT = true;
  static constexpr int STAGE_BYTES = 2 * 2880 * 4 + THREADS * 4;
  const Params& p;
  float* img;
  float* red;
  int kw0, n0, n1, rowoff;
  bool rvalid;
  float bacc;
  __device__ Conv2Wgrad(const Params& q, uint8_t* st, uint8_t*)
      : p(q), img((float*)st), red((float*)(st + 2 * 2880 * 4)) {
    kw0 = blockIdx.x * BM;
    n0 = (int)((long long)q.N * blockIdx.y / q.splits);
    n1 = (int)((long long)q.N * (blockIdx.y + 1) / q.splits);
    const int kw = kw0 + (threadIdx.x & 127);
    rvalid = kw < 500;
    const int c = kw / 25, rem = kw - c * 25, i = rem / 5, j = rem - i * 5;
    rowoff = c * 144 + i * 12 + j;
    bacc = 0.f;
  }
  __device__ int num_k_chunks() const { return (n1 - n0) * 2; }
  __device__ void issue_extra(int c, int tid) {
    if (c & 1) return;
    const int im = c >> 1;
    const float* src = p.p1 + (size_t)(n0 + im) * 2880;
    const uint32_t dst = smem_u32(img + (im & 1) * 2880);
    for (int i = tid; i < 720; i += THREADS) cp16(dst + i * 16, src + i * 4, true);
  }
  __device__ float4 a(int, int k) const {
    if (!rvalid) return zero4();
    const int im = k >> 6, pos = k & 63, ho = pos >> 3, wo = pos & 7;
    const float* s = img + (im & 1) * 2880 + rowoff + ho * 12 + wo;
    return f4(s[0], s[1], s[2], s[3]);
  }
  __device__ const float* b_src(int f, int k, bool& v) const {
    v = f < 50;
    return v ? p.g2 + (size_t)(n0 + (k >> 6)) * 3200 + f * 64 + (k & 63) : p.g2;
  }
  __device__ void b_raw(int, int, float4 v) { bacc += (v.x + v.y) + (v.z + v.w); }
  __device__ void epilogue(int row, int c0, const float (&v)[16]) const {
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
  __device__ void finish(int tid) {
    red[tid] = bacc;
    __syncthreads();
    if (blockIdx.x == 0 && tid < 50)
      p.part[(size_t)blockIdx.y * p.pstride + 25000 + tid] =
          (red[tid] + red[tid + 64]) + (red[tid + 128] + red[tid + 192]);
  }
};

// --------------------------------------------------------- weight repack
// W2 [f][c][i][j] -> W2t [m (4)][r (128)][f (64)], r = (c - 5m)*25 + i*5 + j,
// TF32-rounded, zero padded (conv2 data-gradient A operand; once per backward).
struct PackW2tP {
  const float* w2;
  float* w2t;
};
__global__ void pack_w2t(const __grid_constant__ PackW2tP p) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 4 * 128 * 64) return;
  const int f = idx & 63, r = (idx >> 6) & 127, m = idx >> 13;
  float v = 0.f;
  if (f < 50 && r < 125) {
    const int c = 5 * m + r / 25, tap = r % 25;
    v = p.w2[f * 500 + c * 25 + tap];
  }
  p.w2t[idx] = tf32f(v);
}

// ------------------------------------------------------------ host side
template <class Op>
static constexpr size_t smem_bytes() {
  return (size_t)Op::STAGES * (BM * BK * 4 + Op::BN * BK * 4) + Op::STAGE_BYTES;
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

Launch pack_w2d_launch(const float* w2, float* w2t) {
  Launch l;
  PackW2tP p{w2, w2t};
  l.set((const void*)pack_w2t, dim3(cdiv(4 * 128 * 64, 256)), dim3(256), 0, p);
  return l;
}

Launch conv2_dgrad_launch(const float* g2, const float* w2t, float* dp1, int N, int) {
  Launch l;
  Conv2Dgrad::Params p{g2, w2t, dp1, N};
  l.set((const void*)tc_gemm<Conv2Dgrad>, dim3(4, cdiv(N, 2)), dim3(THREADS), smem_bytes<Conv2Dgrad>(), p);
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
