/*
 * pn.h -- C ABI of the B200-native LeNet-style training path
 * (arxiv 2005.13076, "Using PHAST to port Caffe library").
 *
 * The paper's system is Caffe's Net/Solver/Layer stack: a net of
 * layers exchanging Blobs (data + diff), run feed-forward in order and
 * back-propagated in reverse order after the loss, then updated by the
 * solver.  This header exposes exactly that: build a net from a layer spec,
 * forward, backward, solver update, plus blob access.  SPEC.md S:509-544 gives
 * the operation list (net_build / net_forward / net_backward / sgd_step) and
 * S:580 the spec text format.
 *
 * Conventions (all functions):
 *  - Plain C types only; no C++ types or exceptions cross this boundary.
 *  - Every function returns a pn_status; on non-OK, pn_last_error() returns a
 *    thread-local human-readable message.
 *  - "stream" is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is stream-ordered; nothing synchronises the
 *    host except net_sync_errors(), net_get_blob(..., host) and the *_host
 *    entry points, which say so.
 *  - Ownership: the library owns every blob (activations, masks, parameters,
 *    parameter diffs, momentum history), allocated in net_create on the net's
 *    device and freed in net_destroy.  Caller-owned input buffers (images,
 *    labels, loss output) must stay alive until the stream work that uses them
 *    completes, as with any CUDA async API.
 *  - Layout: every blob is NCHW fp32 row-major.  Labels are int32 class
 *    ids.  Inner-product weights are [num_output, K] (Listing 1).
 *  - Errors: PN_ERR_INVALID_ARG (NULL / bad enum / size mismatch),
 *    PN_ERR_PARSE (spec syntax, unknown key), PN_ERR_UNKNOWN_LAYER,
 *    PN_ERR_DANGLING_BLOB (bottom not produced earlier), PN_ERR_SHAPE (shape
 *    inference failure, non-positive output size), PN_ERR_LABEL_RANGE
 *    (a label outside [0, classes): detected on the device, reported by
 *    net_sync_errors), PN_ERR_CUDA, PN_ERR_NCCL, PN_ERR_STATE (call
 *    order misuse, e.g. backward before forward, or a blob that the fused plan
 *    does not materialise).
 */
#ifndef PN_H
#define PN_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pn_net pn_net; /* opaque; one per device */

typedef enum {
  PN_OK = 0,
  PN_ERR_INVALID_ARG = 1,
  PN_ERR_PARSE = 2,
  PN_ERR_UNKNOWN_LAYER = 3,
  PN_ERR_DANGLING_BLOB = 4,
  PN_ERR_SHAPE = 5,
  PN_ERR_LABEL_RANGE = 6,
  PN_ERR_CUDA = 7,
  PN_ERR_NCCL = 8,
  PN_ERR_STATE = 9
} pn_status;

/* net_create flags */
enum {
  PN_FP32 = 0,      /* fp32 SIMT FFMA contractions (1e-5 parity class)        */
  PN_TF32 = 1,      /* TF32 tcgen05 tensor-core contractions, fp32 accumulate,
                       operands rounded to nearest (2e-3 parity class)         */
  PN_LAYERWISE = 2, /* one generic kernel per layer, every blob materialised
                       (debug / teacher-forcing plan); default is the fused
                       plan when the net matches a fused pattern              */
  PN_3XTF32 = 4     /* with PN_FP32 on the fused LeNet plan: ip1's three
                       contractions as 3xTF32 tcgen05 MMAs over hi / lo
                       operand copies (x = hi + lo; A_lo B_hi + A_hi B_lo +
                       A_hi B_hi, fp32 accumulate): 1e-5 parity class; ignored
                       with PN_TF32 or on the layerwise plan                  */
};

/* which buffer of a blob */
enum { PN_DATA = 0, PN_DIFF = 1, PN_MASK = 2, PN_HISTORY = 3 };

/* Solver settings (Caffe SGD, R11). lr_policy: 0 fixed,
 * 1 inv: lr = base_lr * (1 + gamma*iter)^(-power), evaluated on the host in
 * double and rounded to fp32 once per step. */
typedef struct {
  float base_lr, momentum, weight_decay, gamma, power;
  int lr_policy;
} pn_sgd;

/* Build a net.  spec_text: NUL-terminated "[input]" + "[layer]"
 * sections of key = value lines (unknown keys are PN_ERR_PARSE).
 * batch: images per forward on this device (fixed for the net's lifetime).
 * device: CUDA ordinal.  flags: PN_FP32 | PN_TF32, optionally | PN_LAYERWISE
 * (and PN_FP32 | PN_3XTF32: the fp32 class with ip1 on 3xTF32 tensor cores).
 * Parameters start at zero; set them with net_set_param. */
pn_status net_create(const char* spec_text, int batch, int device, int flags,
                     pn_net** out);
void net_destroy(pn_net* net);
const char* pn_last_error(void);

/* Describe the net.  Blob i in [0, count): name (library-owned string),
 * dims (N,C,H,W), is_param (1 for "<layer>.w" / "<layer>.b" parameters),
 * materialised (0 if the fused plan never writes it to memory). */
pn_status net_blob_count(const pn_net* net, int* count);
pn_status net_blob_info(const pn_net* net, int i, const char** name,
                        int dims[4], int* is_param, int* materialised);
/* Total learnable floats (sum of all weights and biases). */
pn_status net_param_count(const pn_net* net, int64_t* count);
/* Library-owned device pointer of a blob's DATA / DIFF / HISTORY buffer
 * (HISTORY: momentum, parameters only).  Valid until net_destroy. */
pn_status net_blob_ptr(pn_net* net, const char* name, int which,
                       void** dev_ptr);

/* Copy count floats into parameter blob `name` ("conv1.w", "ip2.b", ...)
 * from src (device pointer, or host pointer if src_on_host; a host copy is
 * synchronous).  count must equal the blob's element count. */
pn_status net_set_param(pn_net* net, const char* name, const float* src,
                        int64_t count, int src_on_host, void* stream);
/* Copy a blob buffer out.  which = PN_DATA / PN_DIFF / PN_HISTORY copy fp32
 * values; PN_MASK copies the max-pool origin mask of a Pooling layer's top
 * as int32 plane-local indices h*W+w (R5).  bytes must equal the
 * blob's element count times 4.  dst_on_host: synchronous host copy. */
pn_status net_get_blob(pn_net* net, const char* name, int which, void* dst,
                       int64_t bytes, int dst_on_host, void* stream);
/* Overwrite a blob buffer (teacher forcing: feed a stage the oracle's
 * inputs).  PN_MASK takes int32 plane-local indices. */
pn_status net_put_blob(pn_net* net, const char* name, int which,
                       const void* src, int64_t bytes, int src_on_host,
                       void* stream);

/* Forward (P:94 feed-forward).  x: device N*C*H*W fp32, labels:
 * device N int32, loss: device float (may be NULL).  Also leaves the class
 * probabilities in blob "prob" and the predictions (lowest-index argmax) in
 * blob "pred" (int32 values stored in the blob's 4-byte slots). */
pn_status net_forward(pn_net* net, const float* x, const int32_t* labels,
                      float* loss, void* stream);
/* Backward in reverse layer order.  Overwrites every parameter
 * diff (equivalent to S:573's zero-then-accumulate).  With data parallelism
 * enabled the diffs are summed over ranks (NCCL) before returning. */
pn_status net_backward(pn_net* net, void* stream);
/* Solver update: for every parameter, in fp32 without FMA:
 * g = diff*(1/nranks) + weight_decay*w; v = momentum*v + lr*g; w -= v,
 * with lr the policy value at `iter`. */
pn_status sgd_update(pn_net* net, const pn_sgd* sgd, int64_t iter,
                     void* stream);
/* forward + backward + sgd_update as one CUDA-graph replay on `stream`. */
pn_status net_train_step(pn_net* net, const float* x, const int32_t* labels,
                         const pn_sgd* sgd, int64_t iter, float* loss,
                         void* stream);
/* Same step from HOST buffers (e2e path): copies x (N*C*H*W floats) and
 * labels (N int32) host->device, runs the step, copies the loss back to
 * *loss_host and synchronises `stream`.  Host buffers should be pinned. */
pn_status net_train_step_host(pn_net* net, const float* x_host,
                              const int32_t* labels_host, const pn_sgd* sgd,
                              int64_t iter, float* loss_host, void* stream);
/* Forward-only (inference) from the same graph machinery. */
pn_status net_infer(pn_net* net, const float* x, const int32_t* labels,
                    float* loss, void* stream);

/* Byte input (data ingestion).  Images arrive as the
 * datasets store them, one unsigned byte per pixel, N*C*H*W; the input blob is
 * x = fl(fl(byte * scale) - mean[c,h,w]) (S:604 MNIST: scale 1/256, no mean;
 * S:613 CIFAR: scale 1/256 minus the per-pixel mean), two IEEE fp32
 * roundings, no FMA.  The fused LeNet plan applies it inside conv1's own
 * loads (no fp32 input is ever stored); other plans run one ingest kernel
 * into a library-owned fp32 input buffer first.
 * net_set_input_transform: scale > 0; mean_host = NULL or count = C*H*W host
 *   floats (copied).  Default: scale 1/256, no mean.  Invalidates the captured
 *   graphs (they are re-captured on the next step). */
pn_status net_set_input_transform(pn_net* net, float scale,
                                  const float* mean_host, int64_t count);
/* net_train_step from a device byte batch x8 (N*C*H*W bytes, caller-owned,
 * stream-ordered like net_train_step's x). */
pn_status net_train_step_u8(pn_net* net, const uint8_t* x8,
                            const int32_t* labels, const pn_sgd* sgd,
                            int64_t iter, float* loss, void* stream);
/* nsteps consecutive training steps from HOST byte batches (the end-to-end
 * data path): batch s is x8_host[s*N*C*H*W ...], labels_host[s*N ...]
 * (pinned memory for overlap).  Three device input slots: the host->device
 * copies (bytes, labels, the step's learning rate) of the next batches run on
 * a library copy stream while the current step computes; in the fused LeNet
 * plan each three consecutive steps replay as one captured graph whose loss
 * read-backs run on a side branch; step s's loss lands in losses_host[s].
 * Iterations iter0 .. iter0+nsteps-1.  Synchronises `stream` before
 * returning. */
pn_status net_train_steps_u8_host(pn_net* net, const uint8_t* x8_host,
                                  const int32_t* labels_host, int64_t nsteps,
                                  const pn_sgd* sgd, int64_t iter0,
                                  float* losses_host, void* stream);
/* Dataset files (host only, no GPU needed).
 * pn_idx_read: an unsigned-byte IDX file (MNIST images: 3 dims N,28,28;
 *   labels: 1 dim N).  Fills ndims/dims (up to 4, big-endian sizes decoded);
 *   copies the payload to dst when dst != NULL (cap bytes available).
 *   PN_ERR_PARSE: wrong magic / data type / truncated or oversized file.
 * pn_cifar_read: a CIFAR-10 binary batch (records: 1 label byte, 3072 pixel
 *   bytes in CHW order).  *count = records; pixels (count*3072 bytes) and
 *   labels (count int32) filled when non-NULL (cap records available).
 *   PN_ERR_PARSE: size not a multiple of 3073 or a label byte > 9. */
pn_status pn_idx_read(const char* path, uint8_t* dst, int64_t cap, int* ndims,
                      int64_t dims[4]);
pn_status pn_cifar_read(const char* path, uint8_t* pixels, int32_t* labels,
                        int64_t cap, int64_t* count);

/* Teacher forcing / profiling: the plan is a list of stages (one kernel
 * launch each).  Stage i of the forward (phase 0), backward (phase 1) or
 * update (phase 2) list can be run alone against the current blob contents. */
pn_status net_stage_count(const pn_net* net, int phase, int* count);
pn_status net_stage_name(const pn_net* net, int phase, int i,
                         const char** name);
/* Whether stage i runs in a whole captured step: 0 always, 1 only when the
 * phases run on their own (net_forward / net_backward / sgd_update /
 * net_infer), 2 only inside a whole step (net_train_step*: e.g. the loss sum
 * moved to the backward's side branch, the conv bucket reduced inside the
 * solver). */
pn_status net_stage_mode(const pn_net* net, int phase, int i, int* mode);
pn_status net_run_stage(pn_net* net, int phase, int i, const float* x,
                        const int32_t* labels, void* stream);
/* Per-stage kernel durations on `stream`: one pass through the plan in order
 * (x, labels, sgd, iter as for net_train_step); every kernel stage is
 * launched once, then captured `steps` times back to back into a CUDA graph
 * that is replayed between two CUDA events, so ms_out[phase-major stage
 * order] = mean device milliseconds per launch (kernel + in-graph launch
 * gap, no host launch rate).  Forward / backward stages overwrite their
 * outputs from inputs they do not write; the solver stage applies `steps`
 * updates (profiling changes the parameters).  Non-kernel stages report 0.
 * Synchronises.  n_out: number of entries written (cap >= total stages). */
pn_status net_profile_stages(pn_net* net, const float* x,
                             const int32_t* labels, const pn_sgd* sgd,
                             int64_t iter, int steps, float* ms_out, int cap,
                             int* n_out, void* stream);
/* Number of kernels one net_train_step launches on the device. */
pn_status net_launches_per_step(const pn_net* net, int* n);

/* SURVEY §8(f) NEXT #1 (P:76 multi-GPU roadmap; P:94 / S:536-544 solver):
 * fuse the gradient exchange with the solver.  Collective over the ranks of
 * net_dp_init (every rank calls it, after net_dp_init).  The flat gradient,
 * parameter and momentum buffers become NCCL symmetric windows (parameters
 * and momentum are moved into ncclMemAlloc memory, values kept; pointers from
 * net_blob_ptr taken before are stale) and the backward's bucket allreduces
 * plus the solver are replaced by one kernel: an NVLink barrier, each rank
 * reduces its shard of the gradients over the ranks (NVLS multimem
 * ld_reduce, or peer loads in rank order when the team has no multicast
 * object), applies SGD and stores the updated shard of w and the momentum to
 * every rank, a second barrier.  PN_ERR_STATE without a communicator,
 * PN_ERR_NCCL when NCCL refuses the windows or the device communicator. */
pn_status net_dp_fused_exchange(pn_net* net);

/* Dev-only: in-graph step timeline.  Only in a library built with
 * -DPN_STEPTRACE (else PN_ERR_STATE).  Synchronises the device; when
 * host_out is non-NULL copies the per-kernel record gathered since the last
 * call into it (16 x 3 uint64 %globaltimer ns: first CTA entry, first return
 * from the PDL wait, last CTA exit; kernel order as enum StKernel in
 * csrc/pdl.cuh), then re-arms the record. */
pn_status net_steptrace(pn_net* net, unsigned long long* host_out);

/* Synchronise `stream` and surface device-side errors (label range). */
pn_status net_sync_errors(pn_net* net, void* stream);

/* Data parallelism (R13).  Rank 0 calls pn_nccl_unique_id and
 * broadcasts the 128 bytes; every rank then calls net_dp_init.  Afterwards
 * net_backward allreduces the parameter diffs (sum) over NCCL, overlapped
 * with the rest of the backward pass, and sgd_update scales by 1/nranks. */
pn_status pn_nccl_unique_id(void* out128);
pn_status net_dp_init(pn_net* net, int nranks, int rank, const void* id128);

/* TEST HOOK: data parallelism without NCCL for n <= 8 nets on ONE device
 * (NCCL cannot place two ranks on one GPU), to check the exchange semantics
 * of R13 (sum over ranks, 1/G in the solver) on a single-GPU box.  Create a
 * group, then give each net its rank (net_dp_init_loopback); drive each net
 * from its own host thread with the EAGER phases (net_forward, net_backward,
 * sgd_update: net_train_step returns PN_ERR_STATE).  Each bucket's exchange
 * synchronises the calling rank's stream, meets the other ranks at a host
 * barrier, and rank 0 sums the bucket over the ranks' gradient buffers in
 * rank order on the device.  The group must outlive its nets' exchanges;
 * pn_loopback_destroy after every net using it is destroyed. */
pn_status pn_loopback_create(int n, void** group);
void pn_loopback_destroy(void* group);
pn_status net_dp_init_loopback(pn_net* net, void* group, int rank);

#ifdef __cplusplus
}
#endif
#endif /* PN_H */
