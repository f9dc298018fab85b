// pdl.cuh -- programmatic dependent launch.
// Every kernel of the library is launched with programmatic stream
// serialization and starts with pdl_enter(): wait for the predecessor grid
// (griddepcontrol.wait = its full completion and memory flush), then allow
// the successor to launch.  Invariant: when a kernel starts, every kernel
// except its immediate predecessor has completed, so data produced two or
// more launches back (e.g. the packed weights) may be read before the wait.
// Without the launch attribute both instructions are no-ops.
#pragma once
#include <cstdint>

// ---- dev-only in-graph step timeline (built with -DPN_STEPTRACE; tools/
// step_trace.py).  Per traced kernel: the first CTA's entry, the first
// return from griddepcontrol.wait (= the predecessor's completion) and the
// last CTA's exit, as %globaltimer ns, so the step's critical path can be
// read without a profiler (CUPTI changes how PDL launches overlap).
enum StKernel {
  ST_PACK, ST_CONV1, ST_CONV2F, ST_IPF, ST_IP2, ST_LOSSRED, ST_IP2B, ST_IPG, ST_IPD, ST_RED_IP, ST_CONV2D,
  ST_CONV2W, ST_CONV1W, ST_RED_CONV, ST_SGD, ST_OTHER, ST_N
};
#ifdef PN_STEPTRACE
static __device__ unsigned long long* g_st;  // [ST_N][3] (one copy per translation unit, set by its setter)
__device__ __forceinline__ unsigned long long st_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_mark(int k, int what) {
  if (!g_st) return;
  if (what == 2) atomicMax(g_st + 3 * k + 2, st_now());
  else atomicMin(g_st + 3 * k + what, st_now());
}
#define PN_STEPTRACE_TU(name) \
  void name(unsigned long long* p) { cudaMemcpyToSymbol(g_st, &p, sizeof(p)); }
#else
__device__ __forceinline__ void st_mark(int, int) {}
#define PN_STEPTRACE_TU(name) \
  void name(unsigned long long*) {}
#endif
// entry / exit of kernel k, by thread 0 of each CTA
#define ST_BEGIN(k) do { if (threadIdx.x == 0) st_mark((k), 0); } while (0)
#define ST_END(k) do { if (threadIdx.x == 0) st_mark((k), 2); } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
// pdl_enter() that also records the wait's return for kernel k (step trace)
__device__ __forceinline__ void pdl_enter_k(int k) {
  pdl_wait();
  if ((threadIdx.x & 31) == 0) st_mark(k, 1);
  pdl_trigger();
}
