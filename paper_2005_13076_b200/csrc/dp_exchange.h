// dp_exchange.h -- the fused data-parallel exchange + solver (dp_exchange.cu;
// SURVEY §8(f) NEXT #1): NCCL symmetric windows over the flat gradient,
// parameter and momentum buffers and one kernel that reduces each rank's
// shard over NVLink (multimem / peer loads), applies SGD and writes the
// updated shard to every rank.
#pragma once
#include <nccl.h>

#include <string>

#include "pn.h"
#include "runtime.h"

namespace pn {
struct DpxState;  // opaque (windows, device communicator)
// collective over the communicator's ranks: every rank calls it with buffers
// of the same size n (floats, a multiple of 4) allocated by ncclMemAlloc
pn_status dpx_setup(ncclComm_t comm, float* grads, float* params, float* hist, long long n, int sms, DpxState** out,
                    std::string* err);
void dpx_destroy(DpxState* s);
bool dpx_multimem(const DpxState* s);
Launch dpx_launch(const DpxState* s, float* params, float* hist, long long n);
void dpx_patch(Launch& l, float lr, float mom, float decay, float gscale, const float* lr_dev);
}  // namespace pn
