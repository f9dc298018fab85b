// pdl.cuh -- programmatic dependent launch.
// Every kernel of the library is launched with programmatic stream
// serialization and starts with pdl_enter(): wait for the predecessor grid
// (griddepcontrol.wait = its full completion and memory flush), then allow
// the successor to launch.  Invariant: when a kernel starts, every kernel
// except its immediate predecessor has completed, so data produced two or
// more launches back (e.g. the packed weights) may be read before the wait.
// Without the launch attribute both instructions are no-ops.
#pragma once
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
