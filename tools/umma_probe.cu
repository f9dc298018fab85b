// umma_probe.cu -- dev tool: check tcgen05 kind::tf32 smem-descriptor
// conventions (K-major / MN-major, no swizzle) on one 128 x N x 32 tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const float* A_img, const float* B_img, float* D, int N, uint32_t idesc, uint32_t alo,
                      uint32_t aso, uint32_t akstep, uint32_t blo, uint32_t bso, uint32_t bkstep, int a_bytes,
                      int b_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* As = (float*)smem;
  float* Bs = (float*)(smem + a_bytes);
  for (int i = threadIdx.x; i < a_bytes / 4; i += blockDim.x) As[i] = A_img[i];
  for (int i = threadIdx.x; i < b_bytes / 4; i += blockDim.x) Bs[i] = B_img[i];
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
    for (int k = 0; k < 4; ++k) {
      uint32_t a = smem_u32(As) + k * akstep, b = smem_u32(Bs) + k * bkstep;
      uint64_t ad = ((uint64_t)((a & 0x3FFFF) >> 4)) | ((uint64_t)(alo >> 4) << 16) | ((uint64_t)(aso >> 4) << 32) |
                    (1ull << 46);
      uint64_t bd = ((uint64_t)((b & 0x3FFFF) >> 4)) | ((uint64_t)(blo >> 4) << 16) | ((uint64_t)(bso >> 4) << 32) |
                    (1ull << 46);
      uint32_t acc = k > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(
              tbase),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < 4) {
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tbase + ((warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      D[(warp * 32 + lane) * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

static float tf32r(float x) {  // round to nearest (ties away) to 10-bit mantissa
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  const int M = 128, K = 32;
  int Ns[] = {32};
  srand(1);
  for (int N : Ns) {
    std::vector<float> A(M * K), B(N * K), ref(M * N);
    for (auto& v : A) v = tf32r((rand() % 2001 - 1000) / 1000.f);
    for (auto& v : B) v = tf32r((rand() % 2001 - 1000) / 1000.f);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double acc = 0;
        for (int k = 0; k < K; ++k) acc += (double)A[m * K + k] * B[n * K + k];
        ref[m * N + n] = (float)acc;
      }
    // images: K-major (core 8 rows x 4 k): off = (r/8)*1024 + (k/4)*128 + (r%8)*16 + (k%4)*4
    // MN-major (core 8 k x 4 rows): off = (r/4)*128 + (k/8)*(rows*32) + (k%8)*16 + (r%4)*4
    for (int amn = 0; amn < 2; ++amn)
      for (int bmn = 0; bmn < 2; ++bmn)
        for (int swap = 0; swap < 2; ++swap) {
          std::vector<float> Ai(M * K), Bi(N * K);
          for (int r = 0; r < M; ++r)
            for (int k = 0; k < K; ++k) {
              int off = amn ? (r / 4) * 128 + (k / 8) * (M * 32) + (k % 8) * 16 + (r % 4) * 4
                            : (r / 8) * 1024 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
              Ai[off / 4] = A[r * K + k];
            }
          for (int r = 0; r < N; ++r)
            for (int k = 0; k < K; ++k) {
              int off = bmn ? (r / 4) * 128 + (k / 8) * (N * 32) + (k % 8) * 16 + (r % 4) * 4
                            : (r / 8) * 1024 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
              Bi[off / 4] = B[r * K + k];
            }
          uint32_t alo = amn ? M * 32 : 128, aso = amn ? 128 : 1024, ak = amn ? M * 32 : 256;
          uint32_t blo = bmn ? N * 32 : 128, bso = bmn ? 128 : 1024, bk = bmn ? N * 32 : 256;
          if (swap) {
            if (amn) std::swap(alo, aso);
            if (bmn) std::swap(blo, bso);
            if (!amn && !bmn) continue;
          }
          uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amn << 15) | (bmn << 16) | ((N >> 3) << 17) |
                           ((M >> 4) << 24);
          float *dA, *dB, *dD;
          cudaMalloc(&dA, M * K * 4);
          cudaMalloc(&dB, N * K * 4);
          cudaMalloc(&dD, M * N * 4);
          cudaMemcpy(dA, Ai.data(), M * K * 4, cudaMemcpyHostToDevice);
          cudaMemcpy(dB, Bi.data(), N * K * 4, cudaMemcpyHostToDevice);
          cudaMemset(dD, 0, M * N * 4);
          int smem = M * K * 4 + N * K * 4;
          cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          probe<<<1, 128, smem>>>(dA, dB, dD, N, idesc, alo, aso, ak, blo, bso, bk, M * K * 4, N * K * 4);
          cudaError_t e = cudaDeviceSynchronize();
          std::vector<float> D(M * N);
          cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
          double err = 0, mx = 0;
          for (int i = 0; i < M * N; ++i) {
            err = fmax(err, fabs(D[i] - ref[i]));
            mx = fmax(mx, fabs(ref[i]));
          }
          printf("  D[0..2]=%g %g %g ref=%g %g %g | D[last]=%g ref=%g\n", D[0], D[1], D[2], ref[0], ref[1], ref[2], D[M*N-1], ref[M*N-1]);
          printf("N=%3d A_mn=%d B_mn=%d swapLBO/SBO=%d  err=%.3g (max |ref| %.3g) %s\n", N, amn, bmn, swap, err, mx,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
          cudaFree(dA);
          cudaFree(dB);
          cudaFree(dD);
          if (e != cudaSuccess) return 1;
        }
  }
  return 0;
}
