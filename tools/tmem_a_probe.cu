// tmem_a_probe.cu -- dev probe: tcgen05.mma kind::tf32 with the A operand in
// TMEM (written by tcgen05.st.32x32b), B in shared memory (SW128 K-major):
// checks the A layout (lane = row m, column = k) and times batches.
#include <cstdint>
#include <cstdio>
#include <cmath>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__global__ void probe(float* out, int reps, unsigned long long* cyc) {
  __shared__ __align__(1024) float Bs[32 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B[n][k] (n < 32 rows, k < 32), SW128: row n at n*128 B, 16-B chunk c at ((c ^ (n & 7)) * 16)
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32, c = k / 4, e = k % 4;
    Bs[n * 32 + ((c ^ (n & 7)) * 4) + e] = (n == k) ? 1.f : (n == k + 8 ? 2.f : 0.f);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  // A[m][k] = m + 1000*k at lane m, columns 0..31 (k)
  {
    const int m = warp * 32 + lane;
    uint32_t r[32];
    for (int k = 0; k < 32; ++k) r[k] = __float_as_uint((float)m + 1000.f * k);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            tb + ((uint32_t)(warp * 32) << 16)),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bd = desc(smem_u32(Bs));
    unsigned long long t0 = clock64();
    for (int rp = 0; rp < reps; ++rp) {
      for (int k = 0; k < 4; ++k) {  // K steps of 8: A columns 8k.., B +32 B
        const uint32_t acc = k ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + 64),
            "r"(tb + 8 * k), "l"(bd + 2 * k), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)), "r"(rp & 1));
    }
    *cyc = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tb + 64 + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 32; ++n) out[(warp * 32 + lane) * 32 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}
int main() {
  float* d;
  unsigned long long* c;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaMalloc(&c, 8);
  probe<<<1, 128>>>(d, 1, c);
  float h[128 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  // expected D[m][n] = sum_k A[m][k] B[n][k] = A[m][n] (n < 32: B[n][n]=1) + 2*A[m][n-8] (n >= 8)
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      // A values rounded to TF32 by the tensor core (truncation): compare loosely
      const double a = m + 1000.0 * n, a2 = n >= 8 ? m + 1000.0 * (n - 8) : 0.0;
      const double e = a + 2 * a2;
      if (fabs(h[m * 32 + n] - e) > 1e-3 * fabs(e) + 0.5) {
        if (bad < 8) printf("m %d n %d got %f want %f\n", m, n, h[m * 32 + n], e);
        ++bad;
      }
    }
  printf("bad %d\n", bad);
  for (int reps : {100, 1000}) {
    probe<<<1, 128>>>(d, reps, c);
    unsigned long long cc;
    cudaMemcpy(&cc, c, 8, cudaMemcpyDeviceToHost);
    printf("round trip of 4 MMAs (A in TMEM) + commit: %.1f cycles\n", (double)cc / reps);
  }
  return 0;
}
