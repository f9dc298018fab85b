// kernels.h -- declarations of every __global__ kernel of the library.
#pragma once
#include "params.h"
#include "pdl.cuh"

namespace pn {
// generic per-layer kernels (kernels_generic.cu)
__global__ void conv_fwd_generic(const __grid_constant__ ConvFwdP p);
__global__ void conv_bwd_data_generic(const __grid_constant__ ConvBwdDataP p);
__global__ void conv_bwd_weight_generic(const __grid_constant__ ConvBwdWeightP p);
__global__ void reduce_partials(const __grid_constant__ ReduceP p);
__global__ void reduce_partials_multi(const __grid_constant__ ReduceMultiP p);
__global__ void pool_fwd_generic(const __grid_constant__ PoolFwdP p);
__global__ void pool_bwd_generic(const __grid_constant__ PoolBwdP p);
// planes per block of pool_bwd_plane (inputs per plane HW)
__host__ __device__ inline int pool_bwd_planes(int HW) { return HW >= 1024 ? 1 : 1024 / HW; }
template <int KH, int KW, int SH, int SW>
__global__ void pool_bwd_plane(const __grid_constant__ PoolBwdP p);
__global__ void gemm_generic(const __grid_constant__ GemmP p);
__global__ void gemm_splitk_reduce(const __grid_constant__ GemmP p);
__global__ void stem_fwd(const __grid_constant__ StemP p);
__global__ void stem_wgrad(const __grid_constant__ StemP p);
size_t stem_wgrad_smem(int C, int H, int W, int ph, int pw, int HWp);
constexpr int kStemKmax = 75;  // stem_wgrad: C x kh x kw (the cifar10_quick stem: 3 x 5 x 5)
constexpr int STEM_FG_HOST = 8;  // stem kernels: filters per block (kernels_generic.cu STEM_FG)
template <int AT, int BT>
__global__ void gemm_tiled(const __grid_constant__ GemmP p);
__global__ void ip_fwd_rows(const __grid_constant__ IpRowsP p);
__global__ void colsum_generic(const __grid_constant__ ColSumP p);
__global__ void relu_fwd_generic(const __grid_constant__ ReluP p);
__global__ void relu_bwd_generic(const __grid_constant__ ReluP p);
__global__ void softmax_loss_generic(const __grid_constant__ SoftmaxLossP p);
__global__ void softmax_fwd_generic(const __grid_constant__ SoftmaxP p);
__global__ void softmax_bwd_generic(const __grid_constant__ SoftmaxP p);
__global__ void accuracy_generic(const __grid_constant__ AccuracyP p);
__global__ void accuracy_reduce(const __grid_constant__ AccReduceP p);
__global__ void loss_reduce(const __grid_constant__ LossReduceP p);
__global__ void sgd_update_kernel(const __grid_constant__ SgdP p);
__global__ void ingest_u8(const __grid_constant__ IngestP p);
__global__ void mask_convert(const __grid_constant__ MaskExpandP p);
__global__ void tf32_copy(const __grid_constant__ Tf32CopyP p);

// fused LeNet kernels (kernels_lenet.cu)
__global__ void lenet_conv1_pool1(const __grid_constant__ Conv1Pool1P p);
__global__ void lenet_conv2_pool2_simt(const __grid_constant__ Conv2Pool2P p);
__global__ void lenet_ip2_loss(const __grid_constant__ Ip2LossP p);
__global__ void lenet_ip2_bwd(const __grid_constant__ Ip2BwdP p);
__global__ void lenet_unpool2(const __grid_constant__ Unpool2P p);
__global__ void lenet_conv1_wgrad(const __grid_constant__ Conv1WgradP p);
__global__ void lenet_conv2_dgrad_simt(const __grid_constant__ ConvBwdDataP p);
__global__ void lenet_conv2_wgrad_simt(const __grid_constant__ ConvBwdWeightP p);
#ifndef C2_IMGS_DEF
#define C2_IMGS_DEF 2
#endif
constexpr int kC2Imgs = C2_IMGS_DEF;  // fp32 conv2 forward: images per CTA round (160 threads each)
constexpr int kConv2DgradSimtSmem = (50 * 20 * 5 * 8 + 2 * 50 * 16 * 8) * 4;

constexpr int kGemmTile = 64;
#ifndef KWG
#define KWG 32
#endif
constexpr int kWgradSplits = KWG;
// conv1 weight gradient (fused LeNet plan): images per block
#ifndef CW_IMGS_DEF
#define CW_IMGS_DEF 4
#endif
constexpr int CW_IMGS = CW_IMGS_DEF;
// ip2 + softmax-loss: samples (warps) per block
#ifndef IP2_SPB
#define IP2_SPB 4
#endif
// SGD blocks per SM (grid-stride over float4 groups)
#ifndef SGD_BPS
#define SGD_BPS 8
#endif
// conv1 + pool1 (SIMT): filters per thread (2 or 4; compile-time knob for A/B
// builds) and the block size that covers conv1's 20 filters with one warp per group
#ifndef C1_FPT
#define C1_FPT 4
#endif
constexpr int C1_THREADS = 32 * (20 / C1_FPT);
#ifndef C1_MINB
#define C1_MINB 2  // conv1 + pool1: resident blocks per SM the register budget is sized for
#endif
}  // namespace pn
