// mma_rate.cu -- dev microbenchmark: back-to-back tcgen05.mma issue rate for
// the operand layouts / shapes the kernels use (one CTA, one issuing thread).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
// kind: 0 = tf32 (K=8), 1 = f16 (K=16)
__global__ void bench(int kind, int N, int sw, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 190 * 1024 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t A = smem_u32(smem), B = A + 32768;
    uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    idesc |= kind != 1 ? (2u << 7) | (2u << 10) : 0u;  // tf32 : f16 (A/B type 0 = f16)
    uint64_t ad, bd;
    if (sw) {  // K-major SWIZZLE_128B, SBO 1024
      ad = desc(A, 16, 1024, 2);
      bd = desc(B, 16, 1024, 2);
    } else {  // K-major no swizzle: LBO 128 (K), SBO 256 (rows)
      ad = desc(A, 128, 256, 0);
      bd = desc(B, 128, 256, 0);
    }
    const uint32_t tb = tbase;
    unsigned long long t0 = clock64();
    if (kind == 3) {  // the conv2 tap sequence: 25 taps x 3 k steps, A no-swizzle (LBO 4608, SBO 192), B (LBO 800, SBO 128)
      const uint64_t a0 = desc(A, 4608, 192, 0), b0 = desc(A + 6 * 4608 + 1024, 800, 128, 0);
      for (int r = 0; r < reps; r += 75) {
#pragma unroll
        for (int i = 0; i < 5; ++i)
#pragma unroll
          for (int j = 0; j < 5; ++j)
#pragma unroll
            for (int ks = 0; ks < 3; ++ks)
              asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tb),
                           "l"(a0 + (uint64_t)(((i * 24 + j) * 16 + ks * 2 * 4608) >> 4)),
                           "l"(b0 + (uint64_t)(((i * 5 + j) * 4000 + ks * 1600) >> 4)), "r"(idesc));
      }
    } else if (kind == 5) {  // unrolled x16 with a runtime predicate (setp per MMA)
      for (int r = 0; r < reps; r += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tb),
                       "l"(ad + 2 * u), "l"(bd + 2 * u), "r"(idesc), "r"(r | u));
      }
    } else if (kind == 6) {  // not unrolled, constant accumulate
      for (int r = 0; r < reps; ++r)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tb), "l"(ad + 2 * (r & 3)), "l"(bd + 2 * (r & 3)),
                     "r"(idesc));
    } else if (kind == 4) {  // A in tensor memory (columns 128.. of the allocation), unrolled x16, tf32
      for (int r = 0; r < reps; r += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tb), "r"(tb + 128 + 8 * (u & 7)),
                       "l"(bd + 2 * u), "r"(idesc));
      }
    } else if (kind >= 2) {  // unrolled x16, accumulate, tf32
      for (int r = 0; r < reps; r += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tb), "l"(ad + 2 * u), "l"(bd + 2 * u),
                       "r"(idesc));
      }
    } else
    for (int r = 0; r < reps; ++r) {
      if (kind == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(r));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(r));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    *out = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int reps = 1500;
  for (int kind = 0; kind < 7; ++kind)
    for (int sw = 1; sw < 2; ++sw)
      for (int N : {32, 64, 128, 192}) {
        bench<<<1, 128, 200 * 1024>>>(kind, N, sw, reps, d);
        unsigned long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%s %-6s M=128 N=%3d K=%2d: %6.1f cycles/MMA  (%s)\n", kind == 1 ? "f16 " : kind == 2 ? "tf32u" : kind == 3 ? "conv2" : kind == 4 ? "tf32ts" : kind == 5 ? "tf32p" : kind == 6 ? "tf32l" : "tf32", sw ? "sw128" : "noswz", N,
               kind == 1 ? 16 : 8, (double)c / reps, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
