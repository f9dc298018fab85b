// runtime.h -- host-side executor types of the C ABI implementation.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/pn.h"

namespace pn {

// Everything that changes from one training step to the next.
// The backward fork (an event record + side-stream wait) adds no dependency to
// the main stream, so the kernel after it launches programmatically after ip2's
// backward; ip1's data gradient then reads its da1 operand after the wait.
// (Shared by net.cu and tc.cu; compile-time knob for A/B builds.)
#ifndef FORK_PDL
#define FORK_PDL 1
#endif

struct StepArgs {
  const float* x = nullptr;
  const uint8_t* x8 = nullptr;  // byte input (fused LeNet plan: normalised inside conv1's loads)
  const int32_t* labels = nullptr;
  float* loss = nullptr;
  float lr = 0.f, mom = 0.f, decay = 0.f, gscale = 1.f;
  const float* lr_dev = nullptr;  // learning rate in device memory (then lr is unused)
};

// One kernel launch with its single __grid_constant__ parameter block.
struct Launch {
  const void* func = nullptr;
  dim3 grid, block;
  dim3 cluster{1, 1, 1};  // thread-block cluster dims (1 = none)
  int prio = 0;           // launch priority attribute (0 = the stream's)
  size_t smem = 0;
  std::vector<unsigned char> arg;
  template <class P>
  void set(const void* f, dim3 g, dim3 b, size_t s, const P& p) {
    func = f;
    grid = g;
    block = b;
    smem = s;
    arg.resize(sizeof(P));
    std::memcpy(arg.data(), &p, sizeof(P));
  }
  template <class P>
  P& params() {
    return *reinterpret_cast<P*>(arg.data());
  }
  // planned launches allow programmatic dependent launch (pdl.cuh) unless PN_PDL=0
  static bool pdl() {
    static const bool on = [] {
      const char* e = getenv("PN_PDL");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  // pdl_ok: the previous operation on `st` is the planned predecessor kernel
  // (inside a phase / a captured step); stand-alone launches stay fully
  // stream-ordered (the kernels' griddepcontrol instructions are then no-ops)
  cudaError_t launch(cudaStream_t st, bool pdl_ok = false) {
    void* a[1] = {arg.data()};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    unsigned n = 0;
    if (pdl_ok && pdl()) {
      at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cluster.x * cluster.y * cluster.z > 1) {
      at[n].id = cudaLaunchAttributeClusterDimension;
      at[n].val.clusterDim.x = cluster.x;
      at[n].val.clusterDim.y = cluster.y;
      at[n++].val.clusterDim.z = cluster.z;
    }
    if (prio != 0) {
      at[n].id = cudaLaunchAttributePriority;
      at[n++].val.priority = prio;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelExC(&cfg, func, a);
  }
};

// A stage = one kernel launch (or one non-kernel action such as an NCCL
// collective or a cross-stream event) of the plan.
struct Stage {
  std::string name;
  Launch L;
  std::function<void(Launch&, const StepArgs&)> patch;  // refresh step-dependent args
  std::function<cudaError_t(cudaStream_t)> custom;     // non-kernel action
  bool side = false;  // in a step (graph or eager phase run): launched on the side stream, between fork and join
  // 0: always; 1: only when phases run on their own (net_forward / net_backward /
  // sgd_update / net_infer), skipped in a captured whole step; 2: only in a
  // captured whole step (its replacement there, e.g. the loss sum off the
  // critical path, the conv bucket reduced inside the solver)
  int mode = 0;
  bool transparent = false;  // non-kernel stage that adds no dependency to its own stream (a fork's event
                             // record): the next kernel may still launch programmatically after the previous one
};

}  // namespace pn
