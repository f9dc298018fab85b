// tc.cu -- placeholder until the tcgen05 kernels land: setup() reports
// "not supported", so net_create(PN_TF32) fails loudly (no fallback).
#include "tc.h"
namespace pn {
namespace tc {
cudaError_t setup() { return cudaErrorNotSupported; }
Launch conv2_pool2_launch(const float*, const float*, const float*, float*, uint8_t*, int, int) { return Launch(); }
Launch ip_fwd_launch(const float*, const float*, const float*, float*, int, int, int, bool, int) { return Launch(); }
Launch ip_wgrad_launch(const float*, const float*, float*, float*, int, int, int, int) { return Launch(); }
Launch ip_dgrad_unpool_launch(const float*, const float*, const uint8_t*, float*, int, int) { return Launch(); }
Launch conv2_dgrad_launch(const float*, const float*, float*, int, int) { return Launch(); }
Launch conv2_wgrad_launch(const float*, const float*, float*, int, int, int) { return Launch(); }
}  // namespace tc
}  // namespace pn
