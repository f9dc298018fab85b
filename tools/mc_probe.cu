// mc_probe.cu -- dev probe: a CUDA multicast object over this one GPU (NVLS
// team of one), bound to device memory, and multimem.ld_reduce / multimem.st
// through its multicast address.  Prints whether each step works.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x)                                                          \
  do {                                                                 \
    CUresult r_ = (x);                                                 \
    if (r_ != CUDA_SUCCESS) {                                          \
      const char* s_ = nullptr;                                        \
      cuGetErrorString(r_, &s_);                                       \
      printf("FAIL %s: %s\n", #x, s_ ? s_ : "?");                      \
      return 1;                                                        \
    }                                                                  \
  } while (0)

__global__ void mc_kernel(float* mc, float* uc, float* out, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 >= n) return;
  float a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "l"(mc + i)
               : "memory");
  out[i] = a, out[i + 1] = b, out[i + 2] = c, out[i + 3] = d;
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(a * 2.f), "f"(b * 2.f),
               "f"(c * 2.f), "f"(d * 2.f)
               : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int mcs = 0;
  CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("multicast supported: %d\n", mcs);
  const size_t n = 1 << 20, bytes = n * 4;
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.size = bytes;
  size_t gran = 0;
  CUmemGenericAllocationHandle mc;
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                            CU_MEM_HANDLE_TYPE_NONE};
  for (int t = 0; t < 3 && cr != CUDA_SUCCESS; ++t) {
    mp.handleTypes = hts[t];
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    mp.size = ((bytes + gran - 1) / gran) * gran;
    cr = cuMulticastCreate(&mc, &mp);
    const char* es = nullptr;
    cuGetErrorString(cr, &es);
    printf("handle type %d: min granularity %zu size %zu -> cuMulticastCreate %s\n", (int)hts[t], gran, mp.size, es);
  }
  if (cr != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t ug = 0;
  CK(cuMemGetAllocationGranularity(&ug, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = ((mp.size + ug - 1) / ug) * ug;
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, sz, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, sz, 0));
  CUdeviceptr uc_va, mc_va;
  CK(cuMemAddressReserve(&uc_va, sz, 0, 0, 0));
  CK(cuMemMap(uc_va, sz, 0, phys, 0));
  CK(cuMemAddressReserve(&mc_va, sz, 0, 0, 0));
  CK(cuMemMap(mc_va, sz, 0, mc, 0));
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc_va, sz, &ad, 1));
  CK(cuMemSetAccess(mc_va, sz, &ad, 1));
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
  cudaMemcpy((void*)uc_va, h.data(), bytes, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, bytes);
  mc_kernel<<<n / 4 / 256, 256>>>((float*)mc_va, (float*)uc_va, out, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> o(n), w(n);
  cudaMemcpy(o.data(), out, bytes, cudaMemcpyDeviceToHost);
  cudaMemcpy(w.data(), (void*)uc_va, bytes, cudaMemcpyDeviceToHost);
  size_t bad_r = 0, bad_w = 0;
  for (size_t i = 0; i < n; ++i) {
    bad_r += o[i] != h[i];
    bad_w += w[i] != 2.f * h[i];
  }
  printf("ld_reduce mismatches %zu, multimem.st mismatches %zu\n", bad_r, bad_w);
  return 0;
}
