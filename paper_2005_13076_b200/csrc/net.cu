// net.cu -- the C ABI (include/pn.h): spec parsing, shape inference, device
// memory, the stage plan (fused LeNet or layerwise), eager execution, CUDA
// graph capture/replay with per-step kernel-node patching, profiling, and the
// NCCL data-parallel gradient exchange.
//
// The paper's Net runs every layer forward in order and back-propagates in
// reverse order after the loss; the solver then updates.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <mutex>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pn.h"
#include "dp_exchange.h"
#include "kernels.h"
#include "runtime.h"
#include "tc.h"
#include "tc_conv.h"

#ifndef PIPE_SLOTS
#define PIPE_SLOTS 6  // pipelined host loop: input slots = steps per captured graph (A/B knob; 3 -> 6: e2e 5.49 -> 5.56 M img/s)
#endif
#ifndef WG2_SPLITS
#define WG2_SPLITS 0  // conv2 weight-gradient image splits (0: SMs / 4; compile-time knob for A/B builds)
#endif

using namespace pn;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static pn_status fail(pn_status s, const std::string& m) {
  g_err = m;
  return s;
}
#define CU(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      return fail(PN_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)
#define NC(x)                                                                        \
  do {                                                                               \
    ncclResult_t r_ = (x);                                                           \
    if (r_ != ncclSuccess)                                                           \
      return fail(PN_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));     \
  } while (0)
#define TRY(x)                  \
  do {                          \
    pn_status s_ = (x);         \
    if (s_ != PN_OK) return s_; \
  } while (0)

extern "C" const char* pn_last_error(void) { return g_err.c_str(); }

// -------------------------------------------------------------- spec model
namespace {

enum LType { L_CONV, L_POOL, L_IP, L_RELU, L_LOSS, L_SOFTMAX, L_ACC };

struct Layer {
  LType type;
  std::string name, bottom, top;
  int in[4] = {0, 0, 0, 0}, out[4] = {0, 0, 0, 0};
  int F = 0, kh = 0, kw = 0, sh = 1, sw = 1, ph = 0, pw = 0;  // conv / pool
  int G = 1;                                                  // conv groups (Caffe `group`)
  int method = 0;                                             // pool
  int K = 0, Nout = 0;                                        // ip
  bool bias = true;
  float slope = 0.f;
  int top_k = 1;  // accuracy
  // parameters (conv / ip)
  int64_t wcount = 0, bcount = 0, off = -1;  // offset of w in the flat buffers, b follows w
  int64_t part_off = -1;                     // partial-sum region (split wgrads)
  int splits = 0;
  // layerwise TF32 plan (tc_conv.cu): forward and weight gradient over
  // materialised TF32 operands (plan tp, weight copy Wf [F][kp]); data
  // gradient as an implicit GEMM over gathered G (swizzled W' image bdg)
  bool tc_conv = false, tc_dgrad = false, tma_fwd = false;
  bool stem = false;  // layerwise TF32 plan: conv -> MAX pool -> in-place ReLU fused (stem_fwd / stem_wgrad)
  // the stem's forward as the plane tap GEMM (TF32) + pooling with the ReLU
  // fused (conv output in stem_conv), its backward still stem_wgrad
  bool stem_plane = false;
  float* stem_conv = nullptr;
  bool tap_fwd = false, tap_dgrad = false;  // stride-1 tap GEMM over NHWC (tc_conv.cu)
  bool wtap = false;  // weight gradient as a tap GEMM over shifted X boxes (tc_conv.cu conv_wgrad_taps)
  // forward / data gradient over halo-staged channel planes (tc_plane.cu)
  bool plane_f = false, plane_d = false;
  tcc::PlanePlan pf{}, pd{};
  float* wpl_f = nullptr;  // [T][Kq][F][4]
  float* wpl_d = nullptr;  // [T][Kq][C][4]
  int cp_in = 0, cp_out = 0;                // NHWC channel pitches of x and of G
  float* wtap_f = nullptr;                  // [T][F][cp_in]
  float* wtap_d = nullptr;                  // [T][C][cp_out]
  tcc::ConvTmaPlan tp{};
  float* wf = nullptr;   // Wf [F][kp] (materialised forward)
  float* bfwd = nullptr; // swizzled W image (gathered forward)
  float* bdg = nullptr;  // swizzled W' image (gathered data gradient)
  int fwd_rows = 0, fwd_nk = 0, dg_rows = 0, dg_nk = 0;
};

struct Blob {
  std::string name;
  int dims[4] = {0, 0, 0, 0};
  bool is_param = false, materialised = true, is_input = false;
  float* data = nullptr;
  float* diff = nullptr;
  float* hist = nullptr;
  int32_t* m32 = nullptr;  // layerwise max-pool mask (plane-local)
  uint8_t* m8 = nullptr;   // fused max-pool mask (window offset)
  int pool_layer = -1;     // index of the pooling layer producing it
  int64_t count() const { return (int64_t)dims[0] * dims[1] * dims[2] * dims[3]; }
};

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
  return a == std::string::npos ? "" : s.substr(a, b - a + 1);
}

typedef std::vector<std::pair<std::string, std::string>> KV;

bool allowed_key(const std::string& type, const std::string& k) {
  static const char* common[] = {"name", "type", "bottom", "top"};
  for (auto c : common)
    if (k == c) return true;
  static const char* geo[] = {"kernel_size", "kernel_h", "kernel_w", "stride", "stride_h",
                              "stride_w",    "pad",      "pad_h",    "pad_w"};
  if (type == "Convolution") {
    if (k == "num_output" || k == "bias_term" || k == "group") return true;
    for (auto g : geo)
      if (k == g) return true;
  } else if (type == "Pooling") {
    if (k == "pool") return true;
    for (auto g : geo)
      if (k == g) return true;
  } else if (type == "InnerProduct") {
    return k == "num_output" || k == "bias_term";
  } else if (type == "ReLU") {
    return k == "negative_slope";
  } else if (type == "Accuracy") {
    return k == "top_k";
  }
  return false;
}

const std::string* get(const KV& kv, const std::string& k) {
  for (auto& p : kv)
    if (p.first == k) return &p.second;
  return nullptr;
}

bool parse_int(const std::string& s, int* v) {
  char* e = nullptr;
  long x = strtol(s.c_str(), &e, 10);
  if (!e || *e) return false;
  *v = (int)x;
  return true;
}

int conv_out(int in, int k, int s, int p) {
  int num = in + 2 * p - k;
  if (in <= 0 || k <= 0 || s <= 0 || p < 0 || num < 0) return -1;
  return num / s + 1;
}
// DESIGN.md R4 (Caffe ceil sizing)
int pool_out(int in, int k, int s, int p) {
  int num = in + 2 * p - k;
  if (in <= 0 || k <= 0 || s <= 0 || p < 0 || p >= k || num < 0) return -1;
  int o = (num + s - 1) / s + 1;
  if (p > 0 && (o - 1) * s >= in + p) o--;
  return o;
}

}  // namespace

// -------------------------------------------------------------------- net
// one instantiated graph of phases [0, nph): the node of every stage (flat
// phase-major order; null for non-kernel stages) and the parameter block it
// was last given, so a re-patch touches only the nodes whose arguments changed
struct GraphExec {
  cudaGraphExec_t ex = nullptr;
  cudaGraph_t g = nullptr;
  std::vector<cudaGraphNode_t> nodes;
  std::vector<std::vector<unsigned char>> args;
  StepArgs a;
  void drop() {
    if (ex) cudaGraphExecDestroy(ex);
    if (g) cudaGraphDestroy(g);
    ex = nullptr;
    g = nullptr;
    nodes.clear();
    args.clear();
  }
};

// Test hook: an in-process "communicator" for n nets on ONE
// device, each driven eagerly from its own host thread.  The exchange stage
// of rank r synchronises its stream, meets the others at a host barrier, and
// rank 0 sums the bucket over the ranks' gradient buffers in rank order on
// the device (the same semantics as the NCCL sum; not capturable in a graph).
struct pn_loop {
  int n = 0;
  std::vector<pn_net*> nets;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct pn_net {
  int device = 0, batch = 0, flags = 0;
  bool tf32 = false, fused = false;
  // PN_3XTF32 (fused fp32 LeNet plan): ip1's contractions as 3xTF32 on the tensor
  // cores over per-step hi / lo operand copies (tc.cu Ip3Fwd / Ip3Grad)
  bool x3 = false;
  float *w1h = nullptr, *w1l = nullptr, *w1th = nullptr, *w1tl = nullptr;     // [500][800], [800][512]
  float *p2h = nullptr, *p2l = nullptr, *p2Th = nullptr, *p2Tl = nullptr;     // [N][800], [800][npad]
  float *da1h = nullptr, *da1l = nullptr, *da1Th = nullptr, *da1Tl = nullptr; // [N][500], [500][npad]
  std::vector<Layer> layers;
  std::vector<Layer> acc_layers;  // Accuracy (forward only; read the chain's blobs)
  std::vector<Blob> blobs;
  std::string input_name;
  int classes = 0;

  float* params = nullptr;
  float* grads = nullptr;
  float* hist = nullptr;
  int64_t nparams = 0;      // padded total
  int64_t nlearn = 0;       // unpadded learnable count
  float* partials = nullptr;
  int64_t npartials = 0;
  float* row_loss = nullptr;
  tc::PackP pack{};      // TF32 weight copies for the tensor-core plan
  // TF32 plan operand copies (see tc.cu): transposes padded to npad columns
  int npad = 0;
  float* p2T = nullptr;       // [800][npad]
  float* p1c = nullptr;       // pool1 in the conv2 tap-GEMM layout (tc.h)
  // byte input (NEXT #4): x = byte * x_scale - x_mean[pixel]
  float x_scale = 1.f / 256.f;
  float* x_mean = nullptr;    // [C*H*W] device, or null
  float* xin = nullptr;       // fp32 input written by the ingest kernel (layerwise plans)
  static constexpr int kSlots = PIPE_SLOTS;  // pipelined host input: device slots (copies run up to kSlots-1 steps ahead)
  uint8_t* h2d_x8[kSlots] = {};
  int32_t* h2d_y[kSlots] = {};
  float* h2d_loss = nullptr;  // [kSlots]
  float* h2d_lr = nullptr;    // [kSlots]: each slot's learning rate (its graph reads it: no per-step patch)
  float* lr_pinned = nullptr; // host (pinned) learning rates of the steps of one call
  int64_t lr_pinned_cap = 0;
  float* loss_pinned = nullptr;  // host (pinned) per-step losses of the pipelined loop
  float* hs_x = nullptr;         // net_train_step_host: device staging of one batch (on this net's device)
  int32_t* hs_y = nullptr;
  float* hs_loss = nullptr;
  int64_t loss_pinned_cap = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copied[kSlots] = {}, ev_used[kSlots] = {};
  float* da1r = nullptr;      // [N][500]
  float* da1rT = nullptr;     // [500][npad]
  float* part_b1 = nullptr;   // [splits][500]  ip1 bias-gradient partials
  float* part_db2 = nullptr;  // [rowtiles][50] conv2 bias-gradient partials
  unsigned* err = nullptr;
  int32_t* acc_flags = nullptr;  // per-row top-k hits of the Accuracy layers
  std::vector<void*> allocs;

  std::vector<Stage> phase[3];  // 0 fwd, 1 bwd, 2 update
  bool forward_done = false;
  StepArgs last;  // for eager stage patching

  cudaStream_t cap = nullptr;  // capture stream
  // captured graphs: the train step, forward-only inference, and one train
  // step per input slot of the pipelined host loop (their arguments then
  // differ only in the learning rate)
  GraphExec step, infer, slot[kSlots];
  // the pipelined loop's kSlots consecutive steps as ONE graph (one host launch
  // per kSlots steps): waits on the slots' copy events, the steps, the per-step
  // loss read-backs (destination patched per launch) and the slot-free events
  cudaGraphExec_t multi = nullptr;
  cudaGraph_t multi_g = nullptr;
  cudaGraphNode_t multi_d2h[kSlots] = {};
  float multi_mom = 0.f, multi_decay = 0.f, multi_gscale = 0.f;  // solver settings baked into `multi`
  cudaStream_t aux = nullptr;  // capture-side branch of the loss read-backs
  cudaEvent_t ev_loss[kSlots] = {}, ev_aux = nullptr;
  int launches_per_step = 0;
  // TF32 fused plan: the packed weight copies (pack.w1f ...) no longer match
  // the parameters (set through the ABI): packed before the next run
  bool pack_dirty = true;
  unsigned long long* bar = nullptr;
  bool conv_tail = false;  // the conv bucket's solver as conv1's weight-gradient tail (build_fused_lenet)
  std::vector<ReduceP> conv_segs;  // the conv bucket's partial sums (the step's solver reduces them)

  // data parallel
  int nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  pn_loop* loop = nullptr;          // test-hook exchange (instead of comm)
  void* nccl_grads = nullptr;       // gradient buffer from ncclMemAlloc (registered with the communicator)
  void* nccl_reg = nullptr;         // ncclCommRegister handle
  // the fused exchange + solver (net_dp_fused_exchange, dp_exchange.cu): parameters and
  // momentum moved to ncclMemAlloc buffers, the three symmetric windows, the device communicator
  DpxState* dpx = nullptr;
  void* nccl_params = nullptr;
  void* nccl_hist = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ip = nullptr, ev_conv = nullptr, ev_done = nullptr;
  // single-GPU step: a side stream for independent backward branches
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_ipd = nullptr;
  int64_t bucket_split = 0;  // params [0, split) = ip bucket, [split, n) = conv bucket
  int tc_sms = 148;
  bool tmap_failed = false;
  // layerwise TF32 plan: shared workspaces of the weight-gradient operands
  float* col_ws = nullptr;  // colT [kpad][pitch]
  float* gemm_ws = nullptr;  // split-K partials of the register-tiled fp32 GEMM (add_gemm)
  size_t gemm_ws_floats = 0;
  float* gm_ws = nullptr;   // Gm   [fpad][pitch]

  int blob(const std::string& n) const {
    for (size_t i = 0; i < blobs.size(); ++i)
      if (blobs[i].name == n) return (int)i;
    return -1;
  }
  template <class T>
  pn_status alloc(T** p, size_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, count * sizeof(T) + 16);
    if (e != cudaSuccess) return fail(PN_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    cudaMemset(v, 0, count * sizeof(T) + 16);
    allocs.push_back(v);
    *p = (T*)v;
    return PN_OK;
  }
};

// ------------------------------------------------------------ spec parsing
static pn_status parse_and_infer(pn_net* net, const char* text) {
  std::vector<std::pair<std::string, KV>> sections;
  std::istringstream in(text);
  std::string raw;
  int lineno = 0;
  while (std::getline(in, raw)) {
    ++lineno;
    std::string line = raw.substr(0, raw.find('#'));
    line = trim(line);
    if (line.empty()) continue;
    if (line.front() == '[' && line.back() == ']') {
      sections.push_back({trim(line.substr(1, line.size() - 2)), KV()});
      continue;
    }
    size_t eq = line.find('=');
    if (sections.empty() || eq == std::string::npos)
      return fail(PN_ERR_PARSE, "spec line " + std::to_string(lineno) + ": expected key = value");
    sections.back().second.push_back({trim(line.substr(0, eq)), trim(line.substr(eq + 1))});
  }
  if (sections.empty() || sections[0].first != "input")
    return fail(PN_ERR_PARSE, "spec must start with an [input] section");
  int C = 0, H = 0, W = 0;
  for (auto& kv : sections[0].second) {
    int v = 0;
    if (kv.first == "name") net->input_name = kv.second;
    else if (kv.first == "channels" && parse_int(kv.second, &v)) C = v;
    else if (kv.first == "height" && parse_int(kv.second, &v)) H = v;
    else if (kv.first == "width" && parse_int(kv.second, &v)) W = v;
    else return fail(PN_ERR_PARSE, "[input]: bad key or value '" + kv.first + "'");
  }
  if (net->input_name.empty() || C <= 0 || H <= 0 || W <= 0)
    return fail(PN_ERR_SHAPE, "[input] needs name, channels, height, width > 0");
  Blob in_blob;
  in_blob.name = net->input_name;
  in_blob.dims[0] = net->batch; in_blob.dims[1] = C; in_blob.dims[2] = H; in_blob.dims[3] = W;
  in_blob.is_input = true;
  in_blob.materialised = false;
  net->blobs.push_back(in_blob);

  for (size_t si = 1; si < sections.size(); ++si) {
    if (sections[si].first != "layer") return fail(PN_ERR_PARSE, "unknown section [" + sections[si].first + "]");
    const KV& kv = sections[si].second;
    const std::string* type = get(kv, "type");
    const std::string *name = get(kv, "name"), *bottom = get(kv, "bottom"), *top = get(kv, "top");
    if (!type) return fail(PN_ERR_PARSE, "layer without type");
    Layer L;
    if (*type == "Convolution") L.type = L_CONV;
    else if (*type == "Pooling") L.type = L_POOL;
    else if (*type == "InnerProduct") L.type = L_IP;
    else if (*type == "ReLU") L.type = L_RELU;
    else if (*type == "SoftmaxWithLoss") L.type = L_LOSS;
    else if (*type == "Softmax") L.type = L_SOFTMAX;
    else if (*type == "Accuracy") L.type = L_ACC;
    else return fail(PN_ERR_UNKNOWN_LAYER, "unknown layer type " + *type);
    for (auto& p : kv)
      if (!allowed_key(*type, p.first)) return fail(PN_ERR_PARSE, "unknown key '" + p.first + "' for " + *type);
    if (!name || !bottom || !top) return fail(PN_ERR_PARSE, "layer needs name, bottom, top");
    L.name = *name; L.bottom = *bottom; L.top = *top;
    int bi = net->blob(L.bottom);
    if (bi < 0) return fail(PN_ERR_DANGLING_BLOB, "layer " + L.name + ": bottom '" + L.bottom + "' not produced earlier");
    memcpy(L.in, net->blobs[bi].dims, sizeof(L.in));
    auto geo = [&](const char* base, int def, int* h, int* w) -> bool {
      std::string b = base;
      const std::string* both = get(kv, b == "kernel" ? "kernel_size" : b);
      const std::string* hs = get(kv, b + "_h");
      const std::string* ws = get(kv, b + "_w");
      *h = *w = def;
      if (both && !(parse_int(*both, h) && parse_int(*both, w))) return false;
      if (hs && !parse_int(*hs, h)) return false;
      if (ws && !parse_int(*ws, w)) return false;
      return *h >= 0 && *w >= 0;
    };
    if (L.type == L_CONV || L.type == L_POOL) {
      if (!geo("kernel", -1, &L.kh, &L.kw) || L.kh <= 0 || L.kw <= 0 || !geo("stride", 1, &L.sh, &L.sw) ||
          !geo("pad", 0, &L.ph, &L.pw))
        return fail(PN_ERR_PARSE, "layer " + L.name + ": bad kernel/stride/pad");
    }
    L.out[0] = L.in[0];
    if (L.type == L_CONV) {
      const std::string* no = get(kv, "num_output");
      if (!no || !parse_int(*no, &L.F) || L.F <= 0) return fail(PN_ERR_PARSE, L.name + ": num_output");
      const std::string* bt = get(kv, "bias_term");
      L.bias = !(bt && *bt == "false");
      int Ho = conv_out(L.in[2], L.kh, L.sh, L.ph), Wo = conv_out(L.in[3], L.kw, L.sw, L.pw);
      if (Ho < 1 || Wo < 1) return fail(PN_ERR_SHAPE, L.name + ": non-positive output size");
      const std::string* gs = get(kv, "group");
      if (gs && (!parse_int(*gs, &L.G) || L.G < 1)) return fail(PN_ERR_PARSE, L.name + ": group");
      if (L.in[1] % L.G || L.F % L.G) return fail(PN_ERR_SHAPE, L.name + ": group must divide channels and num_output");
      L.out[1] = L.F; L.out[2] = Ho; L.out[3] = Wo;
      L.wcount = (int64_t)L.F * (L.in[1] / L.G) * L.kh * L.kw;
      L.bcount = L.bias ? L.F : 0;
    } else if (L.type == L_POOL) {
      const std::string* pm = get(kv, "pool");
      if (!pm || *pm == "MAX") L.method = 0;
      else if (*pm == "AVE") L.method = 1;
      else return fail(PN_ERR_PARSE, L.name + ": pool must be MAX or AVE");
      int Hp = pool_out(L.in[2], L.kh, L.sh, L.ph), Wp = pool_out(L.in[3], L.kw, L.sw, L.pw);
      if (Hp < 1 || Wp < 1) return fail(PN_ERR_SHAPE, L.name + ": non-positive output size");
      if (L.method == 0 && L.kh * L.kw > 255) return fail(PN_ERR_SHAPE, L.name + ": window too large");
      L.out[1] = L.in[1]; L.out[2] = Hp; L.out[3] = Wp;
    } else if (L.type == L_IP) {
      const std::string* no = get(kv, "num_output");
      if (!no || !parse_int(*no, &L.Nout) || L.Nout <= 0) return fail(PN_ERR_PARSE, L.name + ": num_output");
      const std::string* bt = get(kv, "bias_term");
      L.bias = !(bt && *bt == "false");
      L.K = L.in[1] * L.in[2] * L.in[3];
      L.out[1] = L.Nout; L.out[2] = 1; L.out[3] = 1;
      L.wcount = (int64_t)L.Nout * L.K;
      L.bcount = L.bias ? L.Nout : 0;
    } else if (L.type == L_RELU) {
      const std::string* s = get(kv, "negative_slope");
      L.slope = s ? (float)atof(s->c_str()) : 0.f;
      if (!(L.slope >= 0.f)) return fail(PN_ERR_PARSE, L.name + ": negative_slope must be >= 0");
      memcpy(L.out, L.in, sizeof(L.out));
    } else if (L.type == L_SOFTMAX) {
      if (L.top == L.bottom) return fail(PN_ERR_PARSE, L.name + ": Softmax cannot run in place");
      memcpy(L.out, L.in, sizeof(L.out));
    } else if (L.type == L_ACC) {
      const std::string* k = get(kv, "top_k");
      const int D = L.in[1] * L.in[2] * L.in[3];
      if (k && !parse_int(*k, &L.top_k)) return fail(PN_ERR_PARSE, L.name + ": top_k");
      if (L.top_k < 1 || L.top_k > D) return fail(PN_ERR_SHAPE, L.name + ": top_k must be in [1, classes]");
      L.out[0] = L.out[1] = L.out[2] = L.out[3] = 1;
    } else {
      net->classes = L.in[1] * L.in[2] * L.in[3];
      L.out[1] = L.out[2] = L.out[3] = 1;
      L.out[0] = 1;
    }
    if (L.type == L_RELU && L.top == L.bottom) {
      // in place: blob already exists
    } else {
      if (net->blob(L.top) >= 0) return fail(PN_ERR_PARSE, "blob '" + L.top + "' produced twice");
      Blob b;
      b.name = L.top;
      memcpy(b.dims, L.out, sizeof(b.dims));
      if (L.type == L_POOL) b.pool_layer = (int)net->layers.size();
      net->blobs.push_back(b);
    }
    if (L.type == L_ACC) net->acc_layers.push_back(L);  // test-phase side output, off the chain
    else net->layers.push_back(L);
  }
  if (net->layers.empty() || net->layers.back().type != L_LOSS)
    return fail(PN_ERR_SHAPE, "the net must end with a SoftmaxWithLoss layer");
  for (size_t i = 0; i + 1 < net->layers.size(); ++i)
    if (net->layers[i].type == L_LOSS) return fail(PN_ERR_SHAPE, "SoftmaxWithLoss must be last");
  return PN_OK;
}

// fused LeNet pattern: conv(1->20,5x5) pool(MAX2/2) conv(20->50,5x5) pool(MAX2/2)
// ip(800->500) relu(in place, 0) ip(500->10) loss on a 1x28x28 input.
static bool is_lenet(const pn_net* n) {
  const auto& L = n->layers;
  if (L.size() != 8) return false;
  auto conv = [](const Layer& l, int C, int F) {
    return l.type == L_CONV && l.in[1] == C && l.F == F && l.kh == 5 && l.kw == 5 && l.sh == 1 && l.sw == 1 &&
           l.ph == 0 && l.pw == 0 && l.bias && l.G == 1;
  };
  auto pool = [](const Layer& l) {
    return l.type == L_POOL && l.method == 0 && l.kh == 2 && l.kw == 2 && l.sh == 2 && l.sw == 2 && l.ph == 0 &&
           l.pw == 0;
  };
  return conv(L[0], 1, 20) && L[0].in[2] == 28 && L[0].in[3] == 28 && L[0].bottom == n->input_name && pool(L[1]) &&
         L[1].bottom == L[0].top && conv(L[2], 20, 50) && L[2].bottom == L[1].top && pool(L[3]) &&
         L[3].bottom == L[2].top && L[4].type == L_IP && L[4].Nout == 500 && L[4].bias && L[4].bottom == L[3].top &&
         L[5].type == L_RELU && L[5].slope == 0.f && L[5].top == L[5].bottom && L[5].bottom == L[4].top &&
         L[6].type == L_IP && L[6].Nout == 10 && L[6].bias && L[6].bottom == L[4].top && L[7].type == L_LOSS &&
         L[7].bottom == L[6].top;
}

// ---------------------------------------------------------- memory layout
static pn_status allocate(pn_net* net) {
  // Parameters in reverse layer order so the data-parallel buckets are
  // contiguous (ip bucket first); each blob 16-byte aligned.
  int64_t off = 0;
  bool seen_conv = false;
  for (int i = (int)net->layers.size() - 1; i >= 0; --i) {
    Layer& L = net->layers[i];
    if (L.type != L_CONV && L.type != L_IP) continue;
    if (L.type == L_CONV && !seen_conv) {
      seen_conv = true;
      net->bucket_split = off;
    }
    L.off = off;
    off += L.wcount + L.bcount;
    off = (off + 3) & ~3LL;
    net->nlearn += L.wcount + L.bcount;
  }
  if (!seen_conv) net->bucket_split = off;
  net->nparams = off;
  TRY(net->alloc(&net->params, off));
  TRY(net->alloc(&net->grads, off));
  TRY(net->alloc(&net->hist, off));
  // parameter blobs
  for (auto& L : net->layers) {
    if (L.off < 0) continue;
    Blob w;
    w.name = L.name + ".w";
    w.is_param = true;
    if (L.type == L_CONV) { w.dims[0] = L.F; w.dims[1] = L.in[1] / L.G; w.dims[2] = L.kh; w.dims[3] = L.kw; }
    else { w.dims[0] = L.Nout; w.dims[1] = L.K; w.dims[2] = 1; w.dims[3] = 1; }
    w.data = net->params + L.off; w.diff = net->grads + L.off; w.hist = net->hist + L.off;
    net->blobs.push_back(w);
    if (L.bcount) {
      Blob b;
      b.name = L.name + ".b";
      b.is_param = true;
      b.dims[0] = (int)L.bcount; b.dims[1] = b.dims[2] = b.dims[3] = 1;
      b.data = net->params + L.off + L.wcount; b.diff = net->grads + L.off + L.wcount;
      b.hist = net->hist + L.off + L.wcount;
      net->blobs.push_back(b);
    }
  }
  // partial-sum regions for split weight gradients
  int64_t poff = 0;
  for (auto& L : net->layers) {
    if (L.off < 0) continue;
    // conv1's fused weight gradient is a light SIMT kernel: CW_IMGS images per
    // CTA (4 at batch 512: 128 CTAs, each beside a conv2 weight-gradient CTA;
    // spreading them over all 148 SMs measured 12 us slower -- the grid barrier
    // of the conv tail then waits for SMs other kernels hold)
    L.splits = (net->fused && &L == &net->layers[0]) ? (net->batch + CW_IMGS - 1) / CW_IMGS : kWgradSplits;
    // the tensor-core conv2 weight gradient runs 4 row tiles x splits CTAs: one per SM
    if (net->fused && net->tf32 && &L == &net->layers[2])  // conv2 weight gradient: one CTA per SM (4 row tiles)
      L.splits = std::max(1, std::min(net->batch, WG2_SPLITS > 0 ? WG2_SPLITS : net->tc_sms / 4));
    if (net->fused && !net->tf32 && &L == &net->layers[2])  // fp32 SIMT conv2 weight gradient: one block per SM
      L.splits = std::max(1, std::min(net->batch, net->tc_sms));
    if (L.stem)  // stem_wgrad: two blocks per SM over image splits
      L.splits = std::max(1, std::min(net->batch, 2 * net->tc_sms));
    if (L.tc_conv) {
      L.tp = tcc::conv_tma_plan(net->batch, L.in[1], L.kh, L.kw, L.F, L.out[2], L.out[3], L.bias ? 1 : 0,
                                net->tc_sms, L.G);
      L.splits = L.tp.wg_splits;
      L.wtap = tcc::wgrad_taps_ok(L.in[1], L.in[3], L.out[3], L.F, L.kh, L.kw, L.sh, L.sw, L.G);
      if (L.wtap) L.splits = tcc::wgrad_taps_splits(net->batch, L.out[2], L.out[3], L.in[1], L.F, L.kh, L.kw, net->tc_sms);
    }
    L.part_off = poff;
    poff += (int64_t)L.splits * (L.wcount + L.bcount);
  }
  net->npartials = poff;
  TRY(net->alloc(&net->partials, poff > 0 ? poff : 1));
  TRY(net->alloc(&net->row_loss, net->batch));
  if (net->tf32) {
    TRY(net->alloc(&net->pack.w1f, tc::kW1fFloats));
    TRY(net->alloc(&net->pack.w1t, tc::kW1tFloats));
    TRY(net->alloc(&net->pack.w2c, tc::kW2cFloats));
    TRY(net->alloc(&net->pack.w2t, tc::kW2tFloats));
    TRY(net->alloc(&net->bar, 1));  // grid-barrier counter of the conv solver tail (conv1 weight gradient)
    net->npad = (net->batch + 3) & ~3;  // TMA row pitch must be a multiple of 16 B
    TRY(net->alloc(&net->p2T, (size_t)800 * net->npad));
    TRY(net->alloc(&net->p1c, (size_t)((net->batch + 1) / 2) * tc::kP1cPairFloats));
    TRY(net->alloc(&net->da1r, (size_t)net->batch * 500));
    TRY(net->alloc(&net->da1rT, (size_t)500 * net->npad));
    TRY(net->alloc(&net->part_b1, (size_t)kWgradSplits * 500));
    TRY(net->alloc(&net->part_db2, (size_t)tc::db2_partials(net->batch) * 50));
  }
  if (net->x3) {
    const size_t N = net->batch;
    net->npad = (net->batch + 3) & ~3;
    for (float** b : {&net->w1h, &net->w1l}) TRY(net->alloc(b, (size_t)500 * 800));
    for (float** b : {&net->w1th, &net->w1tl}) TRY(net->alloc(b, (size_t)800 * 512));
    for (float** b : {&net->p2h, &net->p2l}) TRY(net->alloc(b, N * 800));
    for (float** b : {&net->p2Th, &net->p2Tl}) TRY(net->alloc(b, (size_t)800 * net->npad));
    for (float** b : {&net->da1h, &net->da1l}) TRY(net->alloc(b, N * 500));
    for (float** b : {&net->da1Th, &net->da1Tl}) TRY(net->alloc(b, (size_t)500 * net->npad));
  }
  size_t col_n = 0, gm_n = 0;
  if (net->layers[0].stem_plane) {
    Layer& S0 = net->layers[0];
    TRY(net->alloc(&S0.wpl_f, (size_t)S0.kh * S0.kw * S0.pf.Kq * S0.F * 4));
    TRY(net->alloc(&S0.stem_conv, (size_t)net->batch * S0.F * S0.out[2] * S0.out[3]));
    col_n = std::max(col_n, (size_t)S0.pf.tiles * S0.pf.a_bytes / 4);
  }
  for (auto& L : net->layers) {  // layerwise TF32 plan: packed conv weight images, wgrad workspaces
    if (L.tc_conv) {
      const size_t T = (size_t)L.kh * L.kw;
      if (L.tap_fwd) TRY(net->alloc(&L.wtap_f, T * L.F * L.cp_in));  // inner = per-group slots
      else if (L.tma_fwd) TRY(net->alloc(&L.wf, (size_t)L.F * L.tp.kp));
      else TRY(net->alloc(&L.bfwd, (size_t)L.fwd_rows * L.fwd_nk * 32));
      if (L.tap_dgrad) TRY(net->alloc(&L.wtap_d, T * L.in[1] * L.cp_out));
      if (L.plane_f) TRY(net->alloc(&L.wpl_f, T * L.pf.Kq * L.F * 4));
      if (L.plane_d) TRY(net->alloc(&L.wpl_d, T * L.pd.Kq * L.in[1] * 4));
      if (L.plane_f) col_n = std::max(col_n, (size_t)L.pf.tiles * L.pf.a_bytes / 4);
      if (L.plane_d) col_n = std::max(col_n, (size_t)L.pd.tiles * L.pd.a_bytes / 4);
      if (L.tap_fwd) col_n = std::max(col_n, (size_t)net->batch * L.in[2] * L.in[3] * L.cp_in * L.G);
      if (L.tap_dgrad) col_n = std::max(col_n, (size_t)net->batch * L.out[2] * L.out[3] * L.cp_out * L.G);
      if (L.tc_dgrad && !L.tap_dgrad) TRY(net->alloc(&L.bdg, (size_t)L.dg_rows * L.dg_nk * 32));
      col_n = std::max(col_n, L.tp.col_floats);
      if (L.wtap) col_n = std::max(col_n, (size_t)net->batch * L.in[1] * L.in[2] * L.in[3] * L.kw);  // X's shifted copies
      gm_n = std::max(gm_n, L.tp.g_floats);
    }
  }
  if (col_n) {
    TRY(net->alloc(&net->col_ws, col_n));
    TRY(net->alloc(&net->gm_ws, gm_n));
  }
  TRY(net->alloc(&net->err, 1));
  {  // split-K workspace of the fp32 inner products (up to 8 slices of the largest of their GEMMs)
    size_t mx = 0;
    const bool fp32_ip = !(net->fused && net->tf32);
    for (auto& L : net->layers)
      if (L.type == L_IP && fp32_ip)
        mx = std::max({mx, (size_t)net->batch * L.Nout, (size_t)L.Nout * L.K, (size_t)net->batch * L.K});
    if (mx) {
      net->gemm_ws_floats = 8 * mx;
      TRY(net->alloc(&net->gemm_ws, net->gemm_ws_floats));
    }
  }
  if (!net->acc_layers.empty()) TRY(net->alloc(&net->acc_flags, net->batch));
  // activation blobs (the fused plan never stores conv1's output or its
  // gradient, nor conv2's output; conv2's gradient is the dense unpooled G2)
  std::string skip_data1, skip_data2;
  if (net->fused) {
    skip_data1 = net->layers[0].top;
    skip_data2 = net->layers[2].top;
  }
  if (net->layers[0].stem) skip_data1 = net->layers[0].top;  // the stem's conv output stays on chip
  for (auto& b : net->blobs) {
    if (b.is_param || b.is_input) continue;
    int64_t n = b.count();
    if (b.name == skip_data1) { b.materialised = false; continue; }  // (no data, no gradient)
    if (b.name == skip_data2) b.materialised = false;
    else TRY(net->alloc(&b.data, n));
    TRY(net->alloc(&b.diff, n));
    if (b.pool_layer >= 0 && net->layers[b.pool_layer].method == 0) {
      if (net->fused) TRY(net->alloc(&b.m8, n));
      else TRY(net->alloc(&b.m32, n));
    }
  }
  // classifier outputs
  Blob prob, pred, loss;
  prob.name = "prob"; prob.dims[0] = net->batch; prob.dims[1] = net->classes; prob.dims[2] = prob.dims[3] = 1;
  pred.name = "pred"; pred.dims[0] = net->batch; pred.dims[1] = pred.dims[2] = pred.dims[3] = 1;
  loss.name = "loss"; loss.dims[0] = loss.dims[1] = loss.dims[2] = loss.dims[3] = 1;
  int li = net->blob(net->layers.back().top);
  net->blobs.erase(net->blobs.begin() + li);  // the loss layer's top is "loss"
  for (Blob* b : {&prob, &pred, &loss}) {
    TRY(net->alloc(&b->data, b->count()));
    net->blobs.push_back(*b);
  }
  return PN_OK;
}

static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// ------------------------------------------------------------- plan build
static const float* in_data(pn_net* net, const Layer& L, bool* is_x) {
  *is_x = (L.bottom == net->input_name);
  return *is_x ? nullptr : net->blobs[net->blob(L.bottom)].data;
}

// whether stage s runs in a captured whole step (full) or a phase run on its own
static bool in_run(const Stage& s, bool full) { return s.mode == 0 || (s.mode == 2) == full; }

static void add(std::vector<Stage>& v, const std::string& name, const Launch& L,
                std::function<void(Launch&, const StepArgs&)> patch = nullptr) {
  Stage s;
  s.name = name;
  s.L = L;
  s.patch = patch;
  v.push_back(s);
}

// grads[w (and b)] = sum over the layer's split partials (fixed order)
static void add_reduce_multi(std::vector<Stage>& v, const std::string& name, const std::vector<ReduceP>& segs,
                             bool late = false);
// a layer's split weight-gradient partials: 8 warps per 32 outputs, every
// load of a pass in flight (reduce.cuh) -- hundreds of splits (stem_wgrad)
// in two L2 round trips instead of one per 8 splits
static void add_reduce(pn_net* net, std::vector<Stage>& v, const Layer& L, bool with_bias = true) {
  const int stride = (int)(L.wcount + L.bcount);
  ReduceP r{net->partials + L.part_off, net->grads + L.off, with_bias ? stride : (int)L.wcount, L.splits, stride};
  if (L.wtap) r.pw = (int)L.wcount, r.pk = L.in[1] * L.kh * L.kw, r.pc = L.in[1], r.pt = L.kh * L.kw;
  add_reduce_multi(v, L.name + ".wgrad_reduce", {r});
}


static void add_reduce_multi(std::vector<Stage>& v, const std::string& name, const std::vector<ReduceP>& segs,
                             bool late) {
  ReduceMultiP m{};
  m.late = late ? 1 : 0;
  m.nseg = (int)segs.size();
  m.total = 0;
  for (size_t i = 0; i < segs.size() && i < 6; ++i) {
    m.seg[i] = segs[i];
    m.total += (segs[i].n + 31) / 32;  // 32-output blocks
  }
  Launch l;
  l.set((const void*)reduce_partials_multi, dim3(m.total), dim3(256), 0, m);
  add(v, name, l);
}

static void add_loss(pn_net* net, std::vector<Stage>& fwd) {
  LossReduceP lr{net->row_loss, nullptr, net->blobs[net->blob("loss")].data, net->batch, 1.f / net->batch};
  Launch l;
  l.set((const void*)loss_reduce, dim3(1), dim3(256), 0, lr);
  add(fwd, "loss_reduce", l, [](Launch& l, const StepArgs& a) { l.params<LossReduceP>().loss_out = a.loss; });
}

// The layerwise TF32 plan's stem: a first convolution on the data input
// (stride 1, 3 x 5 x 5 filters), read only by a MAX pooling layer whose output
// an in-place ReLU (slope 0) follows -- cifar10_quick's conv1 -> pool1 ->
// relu1.  Fused by stem_fwd (the conv plane stays in shared memory)
// and stem_wgrad (the weight gradient straight from the pooled gradient and
// origins).
static bool is_stem(const pn_net* net) {
  if (!net->tf32 || net->layers.size() < 3) return false;
  const Layer &C = net->layers[0], &P = net->layers[1], &R = net->layers[2];
  if (C.type != L_CONV || C.bottom != net->input_name || C.G != 1 || C.in[1] != 3 || C.kh != 5 || C.kw != 5 ||
      C.sh != 1 || C.sw != 1 || C.top == C.bottom)
    return false;
  if (P.type != L_POOL || P.method != 0 || P.bottom != C.top || P.top == C.top || P.kh != P.kw || P.sh != P.sw ||
      P.ph != P.pw)
    return false;
  if (R.type != L_RELU || R.bottom != P.top || R.top != P.top || R.slope != 0.f) return false;
  if (C.F > 32) return false;  // stem_wgrad: lane = filter
  for (size_t i = 2; i < net->layers.size(); ++i)
    if (net->layers[i].bottom == C.top) return false;
  for (const Layer& A : net->acc_layers)
    if (A.bottom == C.top) return false;
  return true;
}
static size_t stem_fwd_smem(const Layer& C) {
  const int Hpad = C.in[2] + 2 * C.ph, Wpad = C.in[3] + 2 * C.pw, Wq = (C.out[3] + 3) & ~3;
  return (size_t)(C.in[1] * Hpad * (Wpad + 8) + C.in[1] * C.kh * C.kw * STEM_FG_HOST + STEM_FG_HOST * C.out[2] * Wq) * 4;
}
static StemP stem_params(pn_net* net) {
  const Layer &C = net->layers[0], &P = net->layers[1];
  Blob& y = net->blobs[net->blob(P.top)];
  StemP s{};
  s.w = net->params + C.off;
  s.b = C.bias ? net->params + C.off + C.wcount : nullptr;
  s.y = y.data, s.mask = y.m32, s.dy = y.diff;
  s.part_w = net->partials + C.part_off;
  s.N = net->batch, s.C = C.in[1], s.H = C.in[2], s.W = C.in[3], s.F = C.F, s.kh = C.kh, s.kw = C.kw;
  s.ph = C.ph, s.pw = C.pw, s.Ho = C.out[2], s.Wo = C.out[3];
  s.pk = P.kh, s.ps = P.sh, s.pp = P.ph, s.Hp = P.out[2], s.Wp = P.out[3];
  s.splits = C.splits, s.pstride = (int)(C.wcount + C.bcount), s.relu = 1;
  return s;
}

// C = A B on the register-tiled fp32 GEMM when the operand layouts allow
// float4 loads (a unit stride on K or on M / N, the other a multiple of 4,
// 16-B aligned bases), else the generic strided kernel
static Launch gemm_launch(const GemmP& g) {
  Launch l;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const int at = g.sak == 1 && g.sam % 4 == 0 ? 0 : (g.sam == 1 && g.sak % 4 == 0 ? 1 : -1);
  const int bt = g.sbk == 1 && g.sbn % 4 == 0 ? 0 : (g.sbn == 1 && g.sbk % 4 == 0 ? 1 : -1);
  if (at < 0 || bt < 0 || !al(g.A) || !al(g.B)) {
    l.set((const void*)gemm_generic, dim3(cdiv(g.N, 64), cdiv(g.M, 64), std::max(1, g.splits)), dim3(256), 0, g);
    return l;
  }
  const void* f = at == 0 ? (bt == 0 ? (const void*)gemm_tiled<0, 0> : (const void*)gemm_tiled<0, 1>)
                          : (bt == 0 ? (const void*)gemm_tiled<1, 0> : (const void*)gemm_tiled<1, 1>);
  l.set(f, dim3(cdiv(g.N, 32), cdiv(g.M, 64), std::max(1, g.splits)), dim3(128), 0, g);
  return l;
}

// K split for the register-tiled GEMM: about four 128-thread blocks per SM,
// >= 4 K steps of 16 per slice, <= 8 slices (the fp32 plans' 64 x 32 tiles
// alone leave most SMs with one block)
static int gemm_splits(const pn_net* net, const GemmP& g, bool generic) {
  const long long blocks = generic ? (long long)cdiv(g.N, 64) * cdiv(g.M, 64) : (long long)cdiv(g.N, 32) * cdiv(g.M, 64);
  const int nkt = (g.K + 15) / 16;
  // the generic 64 x 64 kernel (odd strides: e.g. a 10-output layer's weight
  // gradient, one tile over K = batch) splits down to 2 K steps per slice
  int s = (int)std::min<long long>(generic ? 16 : 8, std::max<long long>(1, 4LL * net->tc_sms / blocks));
  s = std::max(1, std::min(s, nkt / (generic ? 2 : 4)));
  return getenv("PN_NO_SPLITK") ? 1 : s;
}

// C = A B as stages: the GEMM (K split into raw partials in gemm_ws when it
// pays) + the fixed-order sum of the slices with bias / ReLU
static void add_gemm(pn_net* net, std::vector<Stage>& v, const std::string& name, GemmP g,
                     std::function<void(Launch&, const StepArgs&)> patch = nullptr) {
  g.splits = 1;
  Launch l = gemm_launch(g);
  {
    const int s = gemm_splits(net, g, l.func == (const void*)gemm_generic);
    if (s > 1 && (size_t)s * g.M * g.N <= net->gemm_ws_floats) {
      g.splits = s;
      g.part = net->gemm_ws;
      l = gemm_launch(g);
      add(v, name, l, patch);
      Launch r;
      r.set((const void*)gemm_splitk_reduce,
            dim3((unsigned)std::min<long long>(8LL * net->tc_sms, cdiv((long long)g.M * g.N, 256))), dim3(256), 0, g);
      add(v, name + ".splitk_reduce", r);
      return;
    }
  }
  add(v, name, l, patch);
}

static void build_layerwise(pn_net* net) {
  auto& fwd = net->phase[0];
  auto& bwd = net->phase[1];
  const int N = net->batch;
  // TF32 plan: an in-place ReLU (slope 0) right after a convolution runs in
  // the convolution's epilogue (its forward stage disappears; its backward,
  // which reads the output sign, stays)
  std::vector<bool> relu_in_conv(net->layers.size(), false);
  for (size_t li = 0; li + 1 < net->layers.size(); ++li) {
    const Layer &L = net->layers[li], &R = net->layers[li + 1];
    if (L.type == L_CONV && L.tc_conv && R.type == L_RELU && R.bottom == L.top && R.top == L.top && R.slope == 0.f)
      relu_in_conv[li + 1] = true;
  }
  const bool stem = net->layers[0].stem;
  for (size_t li = 0; li < net->layers.size(); ++li) {
    Layer& L = net->layers[li];
    bool isx = false;
    const float* x = in_data(net, L, &isx);
    Blob* top = L.type == L_LOSS ? nullptr : &net->blobs[net->blob(L.top)];
    Launch l;
    if (relu_in_conv[li]) continue;
    if (stem && li <= 2) {  // conv -> MAX pool -> ReLU in one kernel (is_stem)
      if (li == 0 && L.stem_plane) {
        // conv1 on the tensor cores (plane tap GEMM, + bias), then pool1 with
        // relu1 fused (the mask is the pooling's, as stem_wgrad reads it)
        const Layer& Pl = net->layers[1];
        Blob& py = net->blobs[net->blob(Pl.top)];
        add(fwd, L.name + ".wpack[tc]", tcc::plane_wpack_launch(L.pf, net->params + L.off, L.wpl_f, L.in[1], L.F, L.kh,
                                                                L.kw, 0));
        add(fwd, L.name + ".planes[tc]",
            tcc::plane_pack_launch(L.pf, x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.ph, L.pw),
            [](Launch& l, const StepArgs& a) { l.params<tcc::PlanePackP>().src = a.x; });
        add(fwd, L.name + ".fwd[tc]",
            tcc::plane_conv_launch(L.pf, net->col_ws, L.wpl_f, L.bias ? net->params + L.off + L.wcount : nullptr,
                                   nullptr, L.stem_conv, N, L.out[2], L.out[3], L.F, L.kh, L.kw, 0, net->tc_sms));
        PoolFwdP pp{L.stem_conv, py.data, py.m32, N, L.F, L.out[2], L.out[3], Pl.kh, Pl.kw, Pl.sh, Pl.sw, Pl.ph, Pl.pw,
                    Pl.out[2], Pl.out[3], 0, 1};
        Launch lp;
        lp.set((const void*)pool_fwd_generic,
               dim3((unsigned)std::min<long long>(cdiv(py.count(), 256), 16LL * net->tc_sms)), dim3(256), 0, pp);
        add(fwd, Pl.name + "+" + net->layers[2].name + ".fwd", lp);
      } else if (li == 0) {
        l.set((const void*)stem_fwd, dim3(cdiv(L.F, STEM_FG_HOST), N), dim3(256), stem_fwd_smem(L), stem_params(net));
        add(fwd, L.name + "+" + net->layers[1].name + "+" + net->layers[2].name + ".fwd", l,
            [](Launch& l, const StepArgs& a) { l.params<StemP>().x = a.x; });
      }
      continue;
    }
    if (L.type == L_CONV && L.tc_conv) {
      // im2col + GEMM, engine chosen at net_create:
      // stride-1 tap GEMM over NHWC, materialised TF32 column matrix col
      // [m][k] streamed by TMA, or the column matrix gathered straight into
      // shared memory
      const bool relu = li + 1 < net->layers.size() && relu_in_conv[li + 1];
      const float* bias = L.bias ? net->params + L.off + L.wcount : nullptr;
      auto xpatch = [](Launch& l, const StepArgs& a) { l.params<Im2colTP>().x = a.x; };
      if (L.plane_f) {
        add(fwd, L.name + ".wpack[tc]", tcc::plane_wpack_launch(L.pf, net->params + L.off, L.wpl_f, L.in[1], L.F, L.kh,
                                                                L.kw, 0));
      } else if (L.tap_fwd) {
        PackTapsP pk{net->params + L.off, L.wtap_f, L.F, L.in[1], L.kh, L.kw, L.cp_in, 0, L.G};
        add(fwd, L.name + ".wpack[tc]", tcc::pack_taps_launch(pk));
      } else if (L.tma_fwd) {
        PackPlainP pk{net->params + L.off, L.wf, L.F, L.tp.K, L.tp.kp};
        add(fwd, L.name + ".wpack[tc]", tcc::pack_plain_launch(pk));
      } else {
        ConvPackP pk{net->params + L.off, L.bfwd, L.F, L.in[1], L.kh, L.kw, L.fwd_rows, L.fwd_nk, 0};
        add(fwd, L.name + ".wpack[tc]", tcc::pack_launch(pk));
      }
      if (L.plane_d) {
        add(fwd, L.name + ".wpack_dgrad[tc]", tcc::plane_wpack_launch(L.pd, net->params + L.off, L.wpl_d, L.F,
                                                                      L.in[1], L.kh, L.kw, 1));
      } else if (L.tap_dgrad) {
        PackTapsP pd{net->params + L.off, L.wtap_d, L.F, L.in[1], L.kh, L.kw, L.cp_out, 1, L.G};
        add(fwd, L.name + ".wpack_dgrad[tc]", tcc::pack_taps_launch(pd));
      } else if (L.tc_dgrad) {
        ConvPackP pd{net->params + L.off, L.bdg, L.F, L.in[1], L.kh, L.kw, L.dg_rows, L.dg_nk, 1};
        add(fwd, L.name + ".wpack_dgrad[tc]", tcc::pack_launch(pd));
      }
      if (L.plane_f) {
        // stride 1: halo-staged channel planes (TF32), then the plane tap GEMM
        add(fwd, L.name + ".planes[tc]",
            tcc::plane_pack_launch(L.pf, x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.ph, L.pw),
            isx ? [](Launch& l, const StepArgs& a) { l.params<tcc::PlanePackP>().src = a.x; }
                : std::function<void(Launch&, const StepArgs&)>());
        add(fwd, L.name + (relu ? ".fwd+relu[tc]" : ".fwd[tc]"),
            tcc::plane_conv_launch(L.pf, net->col_ws, L.wpl_f, bias, nullptr, top->data, N, L.out[2], L.out[3], L.F,
                                   L.kh, L.kw, relu ? 1 : 0, net->tc_sms));
      } else if (L.tap_fwd) {
        // stride 1: x to NHWC (TF32), then the tap GEMM (no column matrix)
        NhwcP nh{x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.cp_in * L.G, L.G, L.cp_in};
        add(fwd, L.name + ".nhwc[tc]", tcc::nhwc_launch(nh),
            isx ? [](Launch& l, const StepArgs& a) { l.params<NhwcP>().x = a.x; }
                : std::function<void(Launch&, const StepArgs&)>());
        Launch lt;
        if (!tcc::tap_launch(net->col_ws, N, L.in[2], L.in[3], L.cp_in * L.G, L.wtap_f, L.F, L.cp_in, L.kh, L.kw,
                             L.ph, L.pw, 1, L.out[2], L.out[3], L.F, bias, relu ? 1 : 0, nullptr, top->data, &lt, L.G,
                             L.cp_in))
          net->tmap_failed = true;
        add(fwd, L.name + (relu ? ".fwd+relu[tc]" : ".fwd[tc]"), lt);
      } else if (L.tma_fwd) {
        Im2colTP ic{x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.out[2],
                    L.out[3], L.tp.K, L.tp.K, L.tp.kp};
        add(fwd, L.name + ".im2col[tc]", tcc::im2col_rows_launch(ic),
            isx ? xpatch : std::function<void(Launch&, const StepArgs&)>());
        Launch lg;
        if (!tcc::gemm_fwd_launch(L.tp, net->col_ws, L.wf, bias, top->data, relu ? 1 : 0, &lg)) net->tmap_failed = true;
        add(fwd, L.name + (relu ? ".fwd+relu[tc]" : ".fwd[tc]"), lg);
      } else {
        ConvTcP p{x, L.bfwd, bias, top->data, N, L.in[1], L.in[2], L.in[3], L.F, L.kh, L.kw, L.sh, L.sw, L.ph, L.pw,
                  L.out[2], L.out[3], L.tp.K, L.fwd_nk, L.fwd_rows, relu ? 1 : 0, nullptr};
        add(fwd, L.name + (relu ? ".fwd+relu[tc]" : ".fwd[tc]"), tcc::conv_fwd_launch(p),
            isx ? [](Launch& l, const StepArgs& a) { l.params<ConvTcP>().x = a.x; }
                : std::function<void(Launch&, const StepArgs&)>());
      }
    } else if (L.type == L_CONV) {
      ConvFwdP p{x, net->params + L.off, L.bias ? net->params + L.off + L.wcount : nullptr, top->data,
                 N, L.in[1], L.in[2], L.in[3], L.F, L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.out[2], L.out[3], L.G};
      l.set((const void*)conv_fwd_generic, dim3(cdiv((long long)N * L.F * L.out[2] * L.out[3], 256)), dim3(256), 0, p);
      add(fwd, L.name + ".fwd", l, isx ? [](Launch& l, const StepArgs& a) { l.params<ConvFwdP>().x = a.x; }
                                       : std::function<void(Launch&, const StepArgs&)>());
    } else if (L.type == L_POOL) {
      PoolFwdP p{x, top->data, top->m32, N, L.in[1], L.in[2], L.in[3], L.kh, L.kw, L.sh, L.sw, L.ph, L.pw,
                 L.out[2], L.out[3], L.method, 0};
      l.set((const void*)pool_fwd_generic,
            dim3((unsigned)std::min<long long>(cdiv(top->count(), 256), 16LL * net->tc_sms)), dim3(256), 0, p);
      add(fwd, L.name + ".fwd", l);
    } else if (L.type == L_IP && (long long)cdiv(L.Nout, 64) * cdiv(N, 64) < net->tc_sms) {
      // few output tiles: split-K rows kernel instead of the 64x64-tile GEMM
      IpRowsP p{x, net->params + L.off, L.bias ? net->params + L.off + L.wcount : nullptr, top->data,
                N, L.K, L.Nout, 0};
      l.set((const void*)ip_fwd_rows, dim3(cdiv(N, 4), cdiv(L.Nout, 8)), dim3(256), 0, p);
      add(fwd, L.name + ".fwd", l, isx ? [](Launch& l, const StepArgs& a) { l.params<IpRowsP>().x = a.x; }
                                       : std::function<void(Launch&, const StepArgs&)>());
    } else if (L.type == L_IP) {
      GemmP p{x, net->params + L.off, top->data, L.bias ? net->params + L.off + L.wcount : nullptr,
              N, L.Nout, L.K, L.K, 1, 1, L.K, 0};
      add_gemm(net, fwd, L.name + ".fwd", p, isx ? [](Launch& l, const StepArgs& a) { l.params<GemmP>().A = a.x; }
                                                 : std::function<void(Launch&, const StepArgs&)>());
    } else if (L.type == L_SOFTMAX) {
      SoftmaxP p{x, nullptr, top->data, N, L.in[1] * L.in[2] * L.in[3]};
      l.set((const void*)softmax_fwd_generic, dim3(cdiv(N, 8)), dim3(256), 0, p);
      add(fwd, L.name + ".fwd", l, isx ? [](Launch& l, const StepArgs& a) { l.params<SoftmaxP>().x = a.x; }
                                       : std::function<void(Launch&, const StepArgs&)>());
    } else if (L.type == L_RELU) {
      ReluP p{x, nullptr, top->data, top->count(), L.slope};
      l.set((const void*)relu_fwd_generic, dim3(std::max(1u, std::min(cdiv(top->count() / 4, 256), 8u * net->tc_sms))),
            dim3(256), 0, p);
      add(fwd, L.name + ".fwd", l);
    } else {
      Blob& bb = net->blobs[net->blob(L.bottom)];
      SoftmaxLossP p{x, nullptr, net->blobs[net->blob("prob")].data,
                     (int32_t*)net->blobs[net->blob("pred")].data, bb.diff, net->row_loss, net->err,
                     N, net->classes, 1.f / N};
      l.set((const void*)softmax_loss_generic, dim3(cdiv(N, 8)), dim3(256), 0, p);
      add(fwd, L.name + ".fwd+bwd", l, [](Launch& l, const StepArgs& a) { l.params<SoftmaxLossP>().labels = a.labels; });
      add_loss(net, fwd);
    }
  }
  // An in-place ReLU (slope 0) whose output feeds a pooling layer or a TF32
  // convolution's data gradient is back-propagated inside that consumer's
  // backward kernel (dx *= (y > 0)): its backward stage disappears.
  std::vector<bool> relu_bwd_fused(net->layers.size(), false);
  for (size_t li = 0; li + 1 < net->layers.size(); ++li) {
    const Layer &R = net->layers[li], &C = net->layers[li + 1];
    if (R.type == L_RELU && R.top == R.bottom && R.slope == 0.f && R.bottom != net->input_name &&
        C.bottom == R.top && (C.type == L_POOL || (C.type == L_CONV && C.tc_dgrad)))
      relu_bwd_fused[li] = true;
  }
  // backward, reverse order
  for (int li = (int)net->layers.size() - 1; li >= 0; --li) {
    Layer& L = net->layers[li];
    bool isx = false;
    const float* x = in_data(net, L, &isx);
    if (L.type == L_LOSS) continue;  // gradient produced with the forward
    if (relu_bwd_fused[li]) continue;
    if (stem && li <= 2) {  // the stem's backward: its weight gradient from the pooled gradient (is_stem)
      if (li == 0) {
        Launch l;
        const Layer& Pl = net->layers[1];
        l.set((const void*)stem_wgrad, dim3(L.splits), dim3(256),
              stem_wgrad_smem(L.in[1], L.in[2], L.in[3], L.ph, L.pw, Pl.out[2] * Pl.out[3]), stem_params(net));
        add(bwd, L.name + ".wgrad", l, [](Launch& l, const StepArgs& a) { l.params<StemP>().x = a.x; });
        add_reduce(net, bwd, L);
      }
      continue;
    }
    const float* relu_y = (li > 0 && relu_bwd_fused[li - 1]) ? net->blobs[net->blob(L.bottom)].data : nullptr;
    Blob& top = net->blobs[net->blob(L.top)];
    Blob* bot = isx ? nullptr : &net->blobs[net->blob(L.bottom)];
    Launch l;
    if (L.type == L_CONV && L.tc_conv) {
      // weight gradient: colT = im2col(x)^T and Gm = G as [F][m] (TF32), then the
      // TMA-fed GEMM into split partials, then their fixed-order sum
      const int K = L.tp.K;
      Launch lw;
      bool ok;
      if (L.wtap) {
        // the tap GEMM over TMA-staged segments (no column matrix): X as kw
        // column-shifted TF32 copies in the column workspace, G as Gw
        tcc::ShiftCopyP xc{x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.kw, L.pw};
        add(bwd, L.name + ".wgrad.xshift[tc]", tcc::shift_copies_launch(xc),
            isx ? [](Launch& l, const StepArgs& a) { l.params<tcc::ShiftCopyP>().x = a.x; }
                : std::function<void(Launch&, const StepArgs&)>());
        tcc::GwP gp{top.diff, net->gm_ws, N, L.F, L.out[2], L.out[3]};
        add(bwd, L.name + ".wgrad.gw[tc]", tcc::gw_launch(gp));
        ok = tcc::wgrad_taps_launch(net->col_ws, net->gm_ws, N, L.in[1], L.in[2], L.in[3], L.out[2], L.out[3], L.F,
                                    L.kh, L.kw, L.ph, L.pw, L.bias ? 1 : 0, net->partials + L.part_off,
                                    (int)(L.wcount + L.bcount), L.splits, &lw);
      } else {
        Im2colTP ic{x, net->col_ws, N, L.in[1], L.in[2], L.in[3], L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.out[2],
                    L.out[3], K, L.G * (K + (L.bias ? 1 : 0)), L.tp.pitch_m, L.G, K + (L.bias ? 1 : 0)};
        add(bwd, L.name + ".wgrad.im2col[tc]", tcc::im2col_t_launch(ic),
            isx ? [](Launch& l, const StepArgs& a) { l.params<Im2colTP>().x = a.x; }
                : std::function<void(Launch&, const StepArgs&)>());
        GmP gp{top.diff, net->gm_ws, N, L.F, L.out[2] * L.out[3], L.tp.pitch_m};
        add(bwd, L.name + ".wgrad.gm[tc]", tcc::gm_launch(gp));
        ok = tcc::gemm_wgrad_launch(L.tp, net->col_ws, net->gm_ws, net->partials + L.part_off,
                                    (int)(L.wcount + L.bcount), &lw);
      }
      if (!ok) net->tmap_failed = true;
      add(bwd, L.name + ".wgrad[tc]", lw);
      add_reduce(net, bwd, L);
      if (bot && L.plane_d) {
        // data gradient as the convolution of G with the flipped,
        // channel-transposed filter (pad k - 1 - p) over halo-staged planes of G
        add(bwd, L.name + ".dgrad.planes[tc]",
            tcc::plane_pack_launch(L.pd, top.diff, net->col_ws, N, L.F, L.out[2], L.out[3], L.kh - 1 - L.ph,
                                   L.kw - 1 - L.pw));
        add(bwd, L.name + (relu_y ? ".dgrad+relu_bwd[tc]" : ".dgrad[tc]"),
            tcc::plane_conv_launch(L.pd, net->col_ws, L.wpl_d, nullptr, relu_y, bot->diff, N, L.in[2], L.in[3],
                                   L.in[1], L.kh, L.kw, 0, net->tc_sms));
      } else if (bot && L.tap_dgrad) {
        // data gradient: col2im(W^T G) = sum over taps of G shifted
        // by (p - i, p - j) times W_t^T -- G to NHWC, then the tap GEMM
        NhwcP nh{top.diff, net->col_ws, N, L.F, L.out[2], L.out[3], L.cp_out * L.G, L.G, L.cp_out};
        add(bwd, L.name + ".dgrad.nhwc[tc]", tcc::nhwc_launch(nh));
        Launch lt;
        if (!tcc::tap_launch(net->col_ws, N, L.out[2], L.out[3], L.cp_out * L.G, L.wtap_d, L.in[1], L.cp_out, L.kh,
                             L.kw, L.ph, L.pw, -1, L.in[2], L.in[3], L.in[1], nullptr, 0, relu_y, bot->diff, &lt, L.G,
                             L.cp_out))
          net->tmap_failed = true;
        add(bwd, L.name + (relu_y ? ".dgrad+relu_bwd[tc]" : ".dgrad[tc]"), lt);
      } else if (bot && L.tc_dgrad) {
        // data gradient: col2im(W^T G) = W' (*) G, stride 1, pad
        // kh-1-p, as an implicit GEMM gathering G (+ the in-place ReLU below)
        ConvTcP q{top.diff, L.bdg, nullptr, bot->diff, N, L.F, L.out[2], L.out[3], L.in[1], L.kh, L.kw, 1, 1,
                  L.kh - 1 - L.ph, L.kw - 1 - L.pw, L.in[2], L.in[3], L.F * L.kh * L.kw, L.dg_nk, L.dg_rows, 0,
                  relu_y};
        add(bwd, L.name + (relu_y ? ".dgrad+relu_bwd[tc]" : ".dgrad[tc]"), tcc::conv_fwd_launch(q));
      } else if (bot) {
        ConvBwdDataP q{top.diff, net->params + L.off, bot->diff, N, L.in[1], L.in[2], L.in[3], L.F, L.kh, L.kw,
                       L.sh, L.sw, L.ph, L.pw, L.out[2], L.out[3], L.G};
        Launch l2;
        l2.set((const void*)conv_bwd_data_generic, dim3(cdiv(bot->count(), 256)), dim3(256), 0, q);
        add(bwd, L.name + ".dgrad", l2);
      }
    } else if (L.type == L_CONV) {
      ConvBwdWeightP p{top.diff, x, net->partials + L.part_off, L.bcount ? net->partials + L.part_off + L.wcount : nullptr,
                       N, L.in[1], L.in[2], L.in[3], L.F, L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.out[2], L.out[3],
                       L.splits, (int)(L.wcount + L.bcount), L.G};
      l.set((const void*)conv_bwd_weight_generic, dim3(L.F * (L.in[1] / L.G), L.splits), dim3(256), 0, p);
      add(bwd, L.name + ".wgrad", l, isx ? [](Launch& l, const StepArgs& a) { l.params<ConvBwdWeightP>().x = a.x; }
                                         : std::function<void(Launch&, const StepArgs&)>());
      add_reduce(net, bwd, L);
      if (bot) {
        ConvBwdDataP q{top.diff, net->params + L.off, bot->diff, N, L.in[1], L.in[2], L.in[3], L.F, L.kh, L.kw,
                       L.sh, L.sw, L.ph, L.pw, L.out[2], L.out[3], L.G};
        Launch l2;
        l2.set((const void*)conv_bwd_data_generic, dim3(cdiv(bot->count(), 256)), dim3(256), 0, q);
        add(bwd, L.name + ".dgrad", l2);
      }
    } else if (L.type == L_POOL) {
      PoolBwdP p{top.diff, top.m32, bot->diff, N, L.in[1], L.in[2], L.in[3], L.kh, L.kw, L.sh, L.sw, L.ph, L.pw,
                 L.out[2], L.out[3], L.method, relu_y};
      // plane-staged kernel when a plane's gradients + origins fit shared memory
      const int P = pool_bwd_planes(L.in[2] * L.in[3]);
      const size_t psmem = (size_t)P * L.out[2] * L.out[3] * 8 + (size_t)(L.in[2] + L.in[3]) * 4 + 16;
      if (psmem <= 48 * 1024) {  // (3x3 / 2x2 stride-2 windows: compile-time geometry)
        const void* fn = (L.kh == 3 && L.kw == 3 && L.sh == 2 && L.sw == 2) ? (const void*)pool_bwd_plane<3, 3, 2, 2>
                         : (L.kh == 2 && L.kw == 2 && L.sh == 2 && L.sw == 2) ? (const void*)pool_bwd_plane<2, 2, 2, 2>
                                                                               : (const void*)pool_bwd_plane<0, 0, 0, 0>;
        l.set(fn, dim3((unsigned)std::min<long long>(cdiv((long long)N * L.in[1], P), 16LL * net->tc_sms)), dim3(256),
              psmem, p);
      } else {
        l.set((const void*)pool_bwd_generic,
              dim3((unsigned)std::min<long long>(cdiv(bot->count(), 256), 16LL * net->tc_sms)), dim3(256), 0, p);
      }
      add(bwd, L.name + (relu_y ? ".bwd+relu_bwd" : ".bwd"), l);
    } else if (L.type == L_IP) {
      // dW = dy^T x : A(m=o,k=n) = dy[n*Nout+o], B(k=n, n=k') = x[n*K+k']
      GemmP w{top.diff, x, net->grads + L.off, nullptr, L.Nout, L.K, N, 1, L.Nout, L.K, 1, 0};
      add_gemm(net, bwd, L.name + ".wgrad", w, isx ? [](Launch& l, const StepArgs& a) { l.params<GemmP>().B = a.x; }
                                                   : std::function<void(Launch&, const StepArgs&)>());
      if (L.bcount) {
        ColSumP c{top.diff, net->grads + L.off + L.wcount, N, L.Nout};
        Launch l2;
        l2.set((const void*)colsum_generic, dim3(L.Nout), dim3(256), 0, c);
        add(bwd, L.name + ".bgrad", l2);
      }
      if (bot) {
        GemmP d{top.diff, net->params + L.off, bot->diff, nullptr, N, L.K, L.Nout, L.Nout, 1, L.K, 1, 0};
        add_gemm(net, bwd, L.name + ".dgrad", d);
      }
    } else if (L.type == L_SOFTMAX) {
      if (bot) {
        SoftmaxP p{top.diff, top.data, bot->diff, N, L.in[1] * L.in[2] * L.in[3]};
        l.set((const void*)softmax_bwd_generic, dim3(cdiv(N, 8)), dim3(256), 0, p);
        add(bwd, L.name + ".bwd", l);
      }
    } else if (L.type == L_RELU) {
      ReluP p{top.diff, top.data, bot->diff, top.count(), L.slope};
      l.set((const void*)relu_bwd_generic, dim3(std::max(1u, std::min(cdiv(top.count() / 4, 256), 8u * net->tc_sms))),
            dim3(256), 0, p);
      add(bwd, L.name + ".bwd", l);
    }
  }
}

// fork: the side stream continues after everything enqueued so far on the main one
static void add_fork(pn_net* net, std::vector<Stage>& v, const char* name, cudaEvent_t ev) {
  Stage f;
  f.name = name;
  f.custom = [net, ev](cudaStream_t st) -> cudaError_t {
    cudaError_t e = cudaEventRecord(ev, st);
    return e != cudaSuccess ? e : cudaStreamWaitEvent(net->side, ev, 0);
  };
  f.transparent = FORK_PDL != 0;
  v.push_back(f);
}

static Stage solver_stage(pn_net* net, const std::string& name, bool ip, bool conv, const std::vector<ReduceP>* segs);

static void build_fused_lenet(pn_net* net) {
  auto& fwd = net->phase[0];
  auto& bwd = net->phase[1];
  const int N = net->batch;
  Layer &c1 = net->layers[0], &c2 = net->layers[2], &i1 = net->layers[4], &i2 = net->layers[6];
  Blob& p1 = net->blobs[net->blob(net->layers[1].top)];
  Blob& cv2 = net->blobs[net->blob(c2.top)];
  Blob& p2 = net->blobs[net->blob(net->layers[3].top)];
  Blob& a1 = net->blobs[net->blob(i1.top)];
  Blob& lg = net->blobs[net->blob(i2.top)];
  float* P = net->params;
  float* G = net->grads;
  // ---- forward
  // TF32 weight copies for the contractions: written by the solver of the
  // previous step (lenet_solver), or packed once after the parameters were
  // set through the ABI (ensure_packed)
  const bool dp = net->comm || net->loop;
  net->conv_tail = false;
  if (net->x3)  // W1 as hi / lo copies (+ transposes) first: off ip1's critical path (read after conv1, conv2)
    add(fwd, "ip1.wsplit[3x]", tc::split3_launch({P + i1.off, net->w1h, net->w1l, net->w1th, net->w1tl, 500, 800, 512}));
  if (net->tf32 && !dp && !getenv("PN_NO_TAIL")) {  // every conv1 weight-gradient block resident at the barrier
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)lenet_conv1_wgrad, 320, 0);
    net->conv_tail = c1.splits <= occ * net->tc_sms;
  }
  if (net->tf32) {
    net->pack.w1 = P + i1.off;
    net->pack.w2 = P + c2.off;
  }
  {
    // TF32 plan: pool1 is consumed only by conv2's contractions, so it is
    // stored TF32-rounded; the mask is taken before rounding
    // items (image, pooled position) split evenly over 2 blocks per SM
    // (at least one block per image pair: a block's range then touches <= 3 images)
    const int blocks = std::max(std::max(1, std::min(C1_MINB * net->tc_sms, N * 144 / 32)), (N + 1) / 2);
    const int per = (int)cdiv((long long)N * 144, blocks);
    Conv1Pool1P p{nullptr, P + c1.off, P + c1.off + 500, p1.data, p1.m8, N, net->tf32 ? 1 : 0, net->p1c, per};
    Launch l;
    if (net->tf32 && !getenv("PN_C1_SIMT"))  // TF32 plan: implicit GEMM on the tensor cores (tc_conv1.cu)
      l = tc::conv1_pool1_tc_launch(p, net->tc_sms);
    else
      l.set((const void*)lenet_conv1_pool1, dim3(cdiv((long long)N * 144, per)), dim3(C1_THREADS), 0, p);
    add(fwd, net->tf32 && !getenv("PN_C1_SIMT") ? "conv1+pool1[tc]" : "conv1+pool1", l, [net](Launch& l, const StepArgs& a) {
      Conv1Pool1P& q = l.params<Conv1Pool1P>();
      q.x = a.x, q.x8 = a.x8, q.x_scale = net->x_scale, q.x_mean = net->x_mean;
    });
  }
  if (net->tf32) {
    add(fwd, "conv2+pool2[tc]", tc::conv2_pool2_launch(net->pack.w2c, P + c2.off + 25000, net->p1c, p2.data,
                                                        net->p2T, p2.m8, N, net->npad, net->tc_sms));
  } else {
    Conv2Pool2P p{p1.data, P + c2.off, P + c2.off + 25000, p2.data, p2.m8, N};
    Launch l;
    l.set((const void*)lenet_conv2_pool2_simt, dim3(std::min(net->tc_sms, (int)cdiv(N, kC2Imgs))), dim3(160 * kC2Imgs),
          (50 * 20 * 28 + kC2Imgs * 2880) * 4, p);
    add(fwd, "conv2+pool2", l);
  }
  if (net->tf32) {
    add(fwd, "ip1+relu[tc]", tc::ip1_fwd_launch(p2.data, net->pack.w1f, P + i1.off + i1.wcount, a1.data, N));
  } else if (net->x3) {
    // W1 and p2 as hi / lo copies (+ the transposes the gradients read), then 3xTF32
    add(fwd, "p2.split[3x]", tc::split3_launch({p2.data, net->p2h, net->p2l, net->p2Th, net->p2Tl, N, 800, net->npad}));
    add(fwd, "ip1+relu[3x]",
        tc::ip1_fwd3_launch(net->p2h, net->p2l, net->w1h, net->w1l, P + i1.off + i1.wcount, a1.data, N));
  } else {
    GemmP g{p2.data, P + i1.off, a1.data, P + i1.off + i1.wcount, N, 500, 800, 800, 1, 1, 800, 1};
    add_gemm(net, fwd, "ip1+relu", g);
  }
  {
    Ip2LossP p{a1.data, P + i2.off, P + i2.off + 5000, nullptr, lg.data,
               net->blobs[net->blob("prob")].data, (int32_t*)net->blobs[net->blob("pred")].data, lg.diff,
               net->row_loss, net->err, N, 1.f / N};
    Launch l;
    l.set((const void*)lenet_ip2_loss, dim3(cdiv(N, IP2_SPB)), dim3(IP2_SPB * 32), 0, p);
    add(fwd, "ip2+softmax_loss", l, [](Launch& l, const StepArgs& a) { l.params<Ip2LossP>().labels = a.labels; });
    add_loss(net, fwd);
    // in a whole TF32 step the loss sum runs on the backward's side branch
    // (below), off the critical path: ip2's backward follows ip2+loss directly
    if (net->tf32 && net->side) fwd.back().mode = 1;
  }
  // ---- backward (reverse order).  Split-partial reductions are merged per
  // gradient bucket: one launch for the ip bucket (ready before the NCCL ip
  // allreduce), one for the conv bucket at the end.
  auto seg = [](const float* part, float* out, int n, int splits, int stride) {
    return ReduceP{part, out, n, splits, stride};
  };
  std::vector<ReduceP> ip_segs, conv_segs;
  ip_segs.push_back(seg(net->partials + i2.part_off, G + i2.off, 5010, i2.splits, 5010));
  {
    Ip2BwdP p{lg.diff, a1.data, P + i2.off, a1.diff, net->partials + i2.part_off,
              net->partials + i2.part_off + 5000, N, i2.splits, 5010,
              net->da1r, net->da1rT, net->part_b1, net->npad};
    Launch l;
    l.set((const void*)lenet_ip2_bwd, dim3(4, i2.splits), dim3(128), 0, p);
    add(bwd, "ip2.bwd+relu1.bwd", l);
  }
  // the ip weight gradients (+ the ip bucket reduction) run on a side
  // stream, concurrently with ip1's data gradient and the conv backward
  // (their CTAs co-reside: 97 KB of shared memory each); joined before the
  // solver.  With data parallelism the ip bucket's allreduce is issued from
  // the same side branch, right after its reduction.
  const bool fork = net->tf32 && net->side;
  if (net->tf32) {
    ip_segs.push_back(seg(net->part_b1, G + i1.off + i1.wcount, 500, i2.splits, 500));
    if (fork) add_fork(net, bwd, "fork[side]", net->ev_fork);
    add(bwd, "ip1.wgrad[tc]", tc::ip1_wgrad_launch(net->da1rT, net->p2T, G + i1.off, N, net->npad));
    if (fork) bwd.back().side = true;
    // the ip partials come from ip2's backward, two launches back (pdl.cuh)
    add_reduce_multi(bwd, "ip.bucket_reduce", ip_segs, true);
    if (fork) {
      bwd.back().side = true;
      add_loss(net, bwd);
      bwd.back().name = "loss_reduce[side]";
      bwd.back().side = true;
      bwd.back().mode = 2;
    }
    add(bwd, "ip1.dgrad+unpool2[tc]",
        tc::ip1_dgrad_unpool_launch(net->da1r, net->pack.w1t, p2.m8, cv2.diff, net->part_db2, N));
    if (fork && net->conv_tail) {
      // a whole single-GPU step updates the ip layers on the side branch once
      // ip1's data gradient (the last reader of W1t) is done: overlaps the conv backward
      add_fork(net, bwd, "fork2[side]", net->ev_ipd);
      bwd.back().mode = 2;
      bwd.push_back(solver_stage(net, "ip.solver[tc]", true, false, nullptr));
      bwd.back().side = true;
      bwd.back().mode = 2;
    }
    conv_segs.push_back(seg(net->part_db2, G + c2.off + 25000, 50, tc::db2_partials(N), 50));
  } else if (net->x3) {
    add(bwd, "da1.split[3x]", tc::split3_launch({a1.diff, net->da1h, net->da1l, net->da1Th, net->da1Tl, N, 500, net->npad}));
    // dW1[o][k] = sum_n da1[n][o] p2[n][k]: A = da1^T [500][N], B = p2^T [800][N]
    add(bwd, "ip1.wgrad[3x]", tc::ip1_grad3_launch(net->da1Th, net->da1Tl, 500, N, net->npad, net->p2Th, net->p2Tl, 800,
                                                    net->npad, G + i1.off, 800));
    ColSumP c{a1.diff, G + i1.off + i1.wcount, N, 500};
    Launch l2;
    l2.set((const void*)colsum_generic, dim3(500), dim3(256), 0, c);
    add(bwd, "ip1.bgrad", l2);
    add_reduce_multi(bwd, "ip.bucket_reduce", ip_segs, true);
    // dp2[n][k] = sum_o da1[n][o] W1[o][k]: A = da1 [N][500], B = W1^T [800][512]
    add(bwd, "ip1.dgrad[3x]", tc::ip1_grad3_launch(net->da1h, net->da1l, N, 500, 500, net->w1th, net->w1tl, 800, 512,
                                                    p2.diff, 800));
    Unpool2P u{p2.diff, p2.m8, cv2.diff, N};
    Launch l4;
    l4.set((const void*)lenet_unpool2, dim3(cdiv((long long)N * 3200, 256)), dim3(256), 0, u);
    add(bwd, "pool2.bwd", l4);
  } else {
    GemmP w{a1.diff, p2.data, G + i1.off, nullptr, 500, 800, N, 1, 500, 800, 1, 0};
    add_gemm(net, bwd, "ip1.wgrad", w);
    ColSumP c{a1.diff, G + i1.off + i1.wcount, N, 500};
    Launch l2;
    l2.set((const void*)colsum_generic, dim3(500), dim3(256), 0, c);
    add(bwd, "ip1.bgrad", l2);
    add_reduce_multi(bwd, "ip.bucket_reduce", ip_segs, true);
    GemmP d{a1.diff, P + i1.off, p2.diff, nullptr, N, 800, 500, 500, 1, 800, 1, 0};
    add_gemm(net, bwd, "ip1.dgrad", d);
    Unpool2P u{p2.diff, p2.m8, cv2.diff, N};
    Launch l4;
    l4.set((const void*)lenet_unpool2, dim3(cdiv((long long)N * 3200, 256)), dim3(256), 0, u);
    add(bwd, "pool2.bwd", l4);
  }
  if (net->tf32) {
    // (a side branch for conv2's weight gradient measured slower: both conv2
    // backward kernels are persistent over every SM and cannot co-reside)
    add(bwd, "conv2.dgrad[tc]", tc::conv2_dgrad_launch(cv2.diff, net->pack.w2t, p1.diff, N, net->tc_sms));
    add(bwd, "conv2.wgrad[tc]", tc::conv2_wgrad_launch(cv2.diff, p1.data, net->partials + c2.part_off, c2.splits, N));
    // conv2.b comes from the ip1 dgrad epilogue's partials
    conv_segs.push_back(seg(net->partials + c2.part_off, G + c2.off, 25000, c2.splits, 25050));
  } else {
    ConvBwdDataP q{cv2.diff, P + c2.off, p1.diff, N, 20, 12, 12, 50, 5, 5, 1, 1, 0, 0, 8, 8};
    Launch l;
    l.set((const void*)lenet_conv2_dgrad_simt, dim3(std::min(net->tc_sms, (int)cdiv(N, 2))), dim3(480),
          kConv2DgradSimtSmem, q);
    add(bwd, "conv2.dgrad", l);
    ConvBwdWeightP w{cv2.diff, p1.data, net->partials + c2.part_off, net->partials + c2.part_off + 25000,
                     N, 20, 12, 12, 50, 5, 5, 1, 1, 0, 0, 8, 8, c2.splits, 25050};
    Launch l2;
    l2.set((const void*)lenet_conv2_wgrad_simt, dim3(c2.splits), dim3(512), 0, w);
    add(bwd, "conv2.wgrad", l2);
    conv_segs.push_back(seg(net->partials + c2.part_off, G + c2.off, 25050, c2.splits, 25050));
  }
  {
    Conv1WgradP p{p1.diff, p1.m8, nullptr, net->partials + c1.part_off, net->partials + c1.part_off + 500, N,
                  c1.splits, 520};
    Launch l;
    l.set((const void*)lenet_conv1_wgrad, dim3(c1.splits), dim3(320), 0, p);
    add(bwd, "conv1.wgrad", l, [net](Launch& l, const StepArgs& a) {
      Conv1WgradP& q = l.params<Conv1WgradP>();
      q.x = a.x, q.x8 = a.x8, q.x_scale = net->x_scale, q.x_mean = net->x_mean;
    });
    conv_segs.push_back(seg(net->partials + c1.part_off, G + c1.off, 520, c1.splits, 520));
  }
  net->conv_segs = conv_segs;
  if (net->conv_tail) {
    // a whole single-GPU TF32 step ends in conv1's weight gradient: after a
    // grid barrier its threads reduce the conv bucket's partials, apply SGD
    // and write the W2 copies (no bucket-reduction or solver launch); with
    // data parallelism the bucket is reduced and all-reduced first, then the
    // solver (phase 2)
    bwd.back().mode = 1;
    Stage t = bwd.back();
    t.name = "conv1.wgrad+solver";
    t.mode = 2;
    Conv1WgradP& q = t.L.params<Conv1WgradP>();
    q.tail = 1;
    q.bar = net->bar;
    q.sp = solver_stage(net, "", false, true, &net->conv_segs).L.params<SolverP>();
    auto base = t.patch;
    t.patch = [base](Launch& l, const StepArgs& a) {
      base(l, a);
      SolverP& s = l.params<Conv1WgradP>().sp;
      s.lr = a.lr; s.mom = a.mom; s.decay = a.decay; s.gscale = a.gscale; s.lr_dev = a.lr_dev;
    };
    bwd.push_back(t);
  }
  add_reduce_multi(bwd, "conv.bucket_reduce", conv_segs);
  if (net->conv_tail) bwd.back().mode = 1;
  if (fork) {  // the ip branch joins before the solver (its gradients are ready)
    Stage j;
    j.name = "join[side]";
    j.custom = [net](cudaStream_t st) -> cudaError_t {
      cudaError_t e = cudaEventRecord(net->ev_join, net->side);
      return e != cudaSuccess ? e : cudaStreamWaitEvent(st, net->ev_join, 0);
    };
    bwd.push_back(j);
  }
}

// the fused TF32 solver over a part of the parameters: ip (the ip layers:
// ip1 weight tiles + the plain ip2 / ip1-bias ranges), conv (the conv bucket
// as reduce segments: `segs`, or its already-reduced gradients)
static Stage solver_stage(pn_net* net, const std::string& name, bool ip, bool conv, const std::vector<ReduceP>* segs) {
  const Layer &c1 = net->layers[0], &c2 = net->layers[2], &i1 = net->layers[4], &i2 = net->layers[6];
  float* G = net->grads;
  SolverP p{};
  p.w = net->params, p.g = G, p.v = net->hist;
  p.w1_off = i1.off, p.w2_off = c2.off;
  p.w1f = net->pack.w1f, p.w1t = net->pack.w1t, p.w2c = net->pack.w2c, p.w2t = net->pack.w2t;
  if (ip) {
    p.w1_tiles = 400;
    p.plain_lo[0] = i2.off, p.plain_hi[0] = i2.off + i2.wcount + i2.bcount;
    p.plain_lo[1] = i1.off + i1.wcount, p.plain_hi[1] = i1.off + i1.wcount + i1.bcount;
    p.nplain = 2;
  }
  if (conv && segs) {
    p.nseg = (int)segs->size();
    for (int k = 0; k < p.nseg && k < 4; ++k) p.seg[k] = (*segs)[k];
  } else if (conv) {  // gradients already reduced: one-split segments over the gradient blob
    const int n2 = (int)(c2.wcount + c2.bcount), n1 = (int)(c1.wcount + c1.bcount);
    p.seg[0] = ReduceP{G + c2.off, G + c2.off, n2, 1, n2};
    p.seg[1] = ReduceP{G + c1.off, G + c1.off, n1, 1, n1};
    p.nseg = 2;
  }
  Stage s;
  s.name = name;
  s.L = tc::lenet_solver_launch(p);
  s.patch = [](Launch& l, const StepArgs& a) {
    SolverP& q = l.params<SolverP>();
    q.lr = a.lr; q.mom = a.mom; q.decay = a.decay; q.gscale = a.gscale; q.lr_dev = a.lr_dev;
  };
  return s;
}

static void build_update(pn_net* net) {
  if (net->dpx) {  // data parallel, fused: the exchange and the solver in one kernel (dp_exchange.cu)
    add(net->phase[2], "exchange+solver[nvlink]", dpx_launch(net->dpx, net->params, net->hist, net->nparams),
        [](Launch& l, const StepArgs& a) { dpx_patch(l, a.lr, a.mom, a.decay, a.gscale, a.lr_dev); });
    if (net->fused && net->tf32) {  // the TF32 weight copies of the exchanged parameters
      net->pack.w1 = net->params + net->layers[4].off;
      net->pack.w2 = net->params + net->layers[2].off;
      add(net->phase[2], "wpack[tc]", tc::pack_weights_launch(net->pack));
    }
    return;
  }
  if (net->fused && net->tf32) {  // reduce (conv bucket) + SGD + the TF32 weight copies
    net->phase[2].push_back(solver_stage(net, "solver[tc]", true, true, nullptr));
    // the whole single-GPU step: the ip part ran on the side branch and the
    // conv bucket's at the end of conv1's weight gradient (build_fused_lenet)
    if (net->conv_tail) net->phase[2].back().mode = 1;
    return;
  }
  SgdP p{net->params, net->grads, net->hist, net->nparams, 0.f, 0.f, 0.f, 1.f, nullptr};
  Launch l;
  long long n4 = net->nparams / 4;
  l.set((const void*)sgd_update_kernel, dim3(std::max(1u, std::min(cdiv(n4, 256), 148u * SGD_BPS))), dim3(256), 0, p);
  add(net->phase[2], "sgd", l, [](Launch& l, const StepArgs& a) {
    SgdP& q = l.params<SgdP>();
    q.lr = a.lr; q.mom = a.mom; q.decay = a.decay; q.gscale = a.gscale; q.lr_dev = a.lr_dev;
  });
}

// data-parallel exchange stages (inserted into the backward list)
__global__ void loopback_sum(const __grid_constant__ LoopSumP p) {
  // rank-order sum of one bucket over the ranks' buffers, written back to all
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.count; i += stride) {
    float s = p.buf[0][i];
    for (int r = 1; r < p.n; ++r) s += p.buf[r][i];
    for (int r = 0; r < p.n; ++r) p.buf[r][i] = s;
  }
}

static void add_dp_stages(pn_net* net) {
  if (!net->comm && !net->loop) return;  // (a 1-rank communicator still runs the full exchange path)
  if (net->dpx) return;                  // the fused exchange runs in the solver's place (build_update)
  auto& bwd = net->phase[1];
  // position: after the last stage producing a gradient of the ip bucket
  // (the inner-product layers' parameters, which lead the flat buffer):
  // stages are named "<layer>.<op>"; the fused plan reduces the bucket in
  // "ip.bucket_reduce" (on the side branch when the plan forks)
  size_t pos = 0;
  bool fused_reduce = false, on_side = false;
  for (size_t i = 0; i < bwd.size(); ++i)
    if (bwd[i].name == "ip.bucket_reduce") {
      pos = i + 1;
      fused_reduce = true;
      on_side = bwd[i].side;
    }
  for (size_t i = 0; i < bwd.size() && !fused_reduce; ++i)
    for (const Layer& L : net->layers)
      if (L.type == L_IP && bwd[i].name.compare(0, L.name.size() + 1, L.name + ".") == 0) pos = i + 1;
  auto allreduce = [net](int64_t off, int64_t cnt, cudaEvent_t ready) -> std::function<cudaError_t(cudaStream_t)> {
    if (net->loop)
      return [net, off, cnt](cudaStream_t st) -> cudaError_t {
        cudaError_t e = cudaStreamSynchronize(st);  // this rank's bucket is complete
        if (e != cudaSuccess) return e;
        net->loop->barrier();
        if (net->rank == 0 && cnt > 0) {
          LoopSumP q{};
          q.n = net->loop->n;
          q.count = cnt;
          for (int r = 0; r < q.n; ++r) q.buf[r] = net->loop->nets[r]->grads + off;
          Launch l;
          l.set((const void*)loopback_sum, dim3(std::min<long long>(1184, (cnt + 255) / 256)), dim3(256), 0, q);
          if ((e = l.launch(st)) != cudaSuccess) return e;
          if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        }
        net->loop->barrier();
        return cudaSuccess;
      };
    return [net, off, cnt, ready](cudaStream_t st) -> cudaError_t {
      cudaError_t e = cudaEventRecord(ready, st);
      if (e != cudaSuccess) return e;
      e = cudaStreamWaitEvent(net->comm_stream, ready, 0);
      if (e != cudaSuccess) return e;
      if (cnt > 0 && ncclAllReduce(net->grads + off, net->grads + off, cnt, ncclFloat, ncclSum, net->comm,
                                   net->comm_stream) != ncclSuccess)
        return cudaErrorUnknown;
      return cudaSuccess;
    };
  };
  Stage s1;
  s1.name = "allreduce[ip bucket]";
  s1.custom = allreduce(0, net->bucket_split, net->ev_ip);
  s1.side = on_side;
  s1.transparent = on_side;  // (on the side branch it adds nothing to the main stream)
  bwd.insert(bwd.begin() + pos, s1);
  Stage s2;
  s2.name = "allreduce[conv bucket]";
  s2.custom = allreduce(net->bucket_split, net->nparams - net->bucket_split, net->ev_conv);
  bwd.push_back(s2);
  if (net->comm) {
    Stage s3;
    s3.name = "join[comm]";
    s3.custom = [net](cudaStream_t st) -> cudaError_t {
      cudaError_t e = cudaEventRecord(net->ev_done, net->comm_stream);
      if (e != cudaSuccess) return e;
      return cudaStreamWaitEvent(st, net->ev_done, 0);
    };
    bwd.push_back(s3);
  }
}

// Accuracy layers (test-phase side outputs): after the forward
// chain, in both plans, on the blobs it materialised
static pn_status add_accuracy(pn_net* net) {
  for (auto& L : net->acc_layers) {
    const Blob& b = net->blobs[net->blob(L.bottom)];
    if (!b.materialised || !b.data)
      return fail(PN_ERR_STATE, L.name + ": bottom '" + L.bottom + "' is not materialised by this plan");
    const int D = L.in[1] * L.in[2] * L.in[3];
    AccuracyP a{b.data, nullptr, net->acc_flags, net->err, net->batch, D, L.top_k};
    Launch l;
    l.set((const void*)accuracy_generic, dim3(cdiv(net->batch, 8)), dim3(256), 0, a);
    add(net->phase[0], L.name + ".fwd", l, [](Launch& l, const StepArgs& s) { l.params<AccuracyP>().labels = s.labels; });
    AccReduceP r{net->acc_flags, net->blobs[net->blob(L.top)].data, net->batch};
    Launch l2;
    l2.set((const void*)accuracy_reduce, dim3(1), dim3(256), 0, r);
    add(net->phase[0], L.name + ".reduce", l2);
  }
  return PN_OK;
}

static pn_status build_plan(pn_net* net) {
  for (auto& ph : net->phase) ph.clear();
  if (net->fused) build_fused_lenet(net);
  else build_layerwise(net);
  TRY(add_accuracy(net));
  build_update(net);
  add_dp_stages(net);
  {  // side-branch kernels at the highest launch priority: scheduled ahead of the
     // pending CTAs of the persistent conv backward kernels (PN_SIDE_PRIO=0: off)
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* e = getenv("PN_SIDE_PRIO");
    if (!(e && e[0] == '0'))
      for (auto& ph : net->phase)
        for (auto& s : ph)
          if (s.side && !s.custom) s.L.prio = hi;
  }
  int n = 0;
  for (auto& ph : net->phase)
    for (auto& s : ph)
      if (!s.custom && in_run(s, true)) ++n;
  net->launches_per_step = n;
  return PN_OK;
}

// --------------------------------------------------------------- execution
// pdl_ok: this stage directly follows its planned predecessor kernel
static pn_status run_stage(pn_net* net, Stage& s, const StepArgs& a, cudaStream_t st, bool pdl_ok = false) {
  if (s.custom) {
    cudaError_t e = s.custom(st);
    if (e != cudaSuccess) return fail(net->comm ? PN_ERR_NCCL : PN_ERR_CUDA, "stage " + s.name + " failed");
    return PN_OK;
  }
  if (s.patch) s.patch(s.L, a);
  cudaError_t e = s.L.launch(st, pdl_ok);
  if (e != cudaSuccess) return fail(PN_ERR_CUDA, "launch " + s.name + ": " + cudaGetErrorString(e));
  return PN_OK;
}

static pn_status ensure_packed(pn_net* net, cudaStream_t st);

// a phase run eagerly: its first kernel follows whatever the caller enqueued
static pn_status run_phase(pn_net* net, int ph, const StepArgs& a, cudaStream_t st) {
  TRY(ensure_packed(net, st));
  bool prev_kernel = false;  // (main stream; side-stream kernels run without PDL)
  for (auto& s : net->phase[ph]) {
    if (!in_run(s, false)) continue;
    if (s.side) {
      TRY(run_stage(net, s, a, net->side, false));
      continue;
    }
    TRY(run_stage(net, s, a, st, prev_kernel));
    if (!s.transparent) prev_kernel = !s.custom;
  }
  return PN_OK;
}

// the TF32 weight copies after the parameters changed through the ABI (the
// solver keeps them current from then on); stand-alone, stream-ordered
static pn_status ensure_packed(pn_net* net, cudaStream_t st) {
  if (!(net->fused && net->tf32) || !net->pack_dirty) return PN_OK;
  CU(cudaSetDevice(net->device));
  CU(tc::pack_weights_launch(net->pack).launch(st));
  net->pack_dirty = false;
  return PN_OK;
}

static StepArgs make_args(pn_net* net, const float* x, const int32_t* labels, float* loss, const pn_sgd* sgd,
                          int64_t iter) {
  StepArgs a;
  a.x = x;
  a.labels = labels;
  a.loss = loss;
  if (sgd) {
    double lr = sgd->base_lr;
    if (sgd->lr_policy == 1) lr = (double)sgd->base_lr * pow(1.0 + (double)sgd->gamma * (double)iter, -(double)sgd->power);
    a.lr = (float)lr;
    a.mom = sgd->momentum;
    a.decay = sgd->weight_decay;
  }
  a.gscale = 1.f / (float)net->nranks;
  return a;
}

static bool same_args(const StepArgs& a, const StepArgs& b) {
  return a.x == b.x && a.x8 == b.x8 && a.lr_dev == b.lr_dev && a.labels == b.labels && a.loss == b.loss && a.lr == b.lr && a.mom == b.mom &&
         a.decay == b.decay && a.gscale == b.gscale;
}

// capture phases [0, nph) into an executable graph; record kernel nodes
static pn_status capture(pn_net* net, int nph, const StepArgs& a, GraphExec& E) {
  if (!net->cap) CU(cudaStreamCreateWithFlags(&net->cap, cudaStreamNonBlocking));
  E.drop();
  CU(cudaStreamBeginCapture(net->cap, cudaStreamCaptureModeThreadLocal));
  bool prev_kernel = false;  // the captured step is one fixed sequence across phases
  for (int ph = 0; ph < nph; ++ph)
    for (auto& s : net->phase[ph]) {
      if (!in_run(s, nph == 3)) continue;
      cudaStream_t on = s.side ? net->side : net->cap;
      pn_status st = run_stage(net, s, a, on, s.side ? false : prev_kernel);
      if (!s.side && !s.transparent) prev_kernel = !s.custom;
      if (st != PN_OK) {
        cudaGraph_t g;
        cudaStreamEndCapture(net->cap, &g);
        E.drop();
        return st;
      }
      cudaGraphNode_t node = nullptr;
      if (!s.custom) {
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CU(cudaStreamGetCaptureInfo(on, &cs, nullptr, nullptr, &deps, &nd));
        node = nd ? deps[0] : nullptr;
      }
      E.nodes.push_back(node);
      E.args.push_back(s.L.arg);
    }
  CU(cudaStreamEndCapture(net->cap, &E.g));
  CU(cudaGraphInstantiate(&E.ex, E.g, 0));  // (the graph is kept: its node handles address the exec's nodes)
  E.a = a;
  return PN_OK;
}

static pn_status patch_graph(pn_net* net, int nph, const StepArgs& a, GraphExec& E) {
  size_t i = 0;
  for (int ph = 0; ph < nph; ++ph)
    for (auto& s : net->phase[ph]) {
      if (!in_run(s, nph == 3)) continue;
      const size_t k = i++;
      if (s.custom || !s.patch) continue;
      s.patch(s.L, a);
      if (s.L.arg == E.args[k]) continue;  // unchanged in this exec
      cudaKernelNodeParams kp{};
      void* args[1] = {s.L.arg.data()};
      kp.func = (void*)s.L.func;
      kp.gridDim = s.L.grid;
      kp.blockDim = s.L.block;
      kp.sharedMemBytes = (unsigned)s.L.smem;
      kp.kernelParams = args;
      CU(cudaGraphExecKernelNodeSetParams(E.ex, E.nodes[k], &kp));
      E.args[k] = s.L.arg;
    }
  E.a = a;
  return PN_OK;
}

// launch graph E of phases [0, nph) with arguments a (capture on first use)
static pn_status replay(pn_net* net, int nph, const StepArgs& a, GraphExec& E, cudaStream_t st) {
  if (net->loop && nph >= 2)
    return fail(PN_ERR_STATE, "a loopback data-parallel net runs its phases eagerly (net_forward / net_backward / "
                              "sgd_update): its exchange synchronises on the host");
  TRY(ensure_packed(net, st));
  if (!E.ex) TRY(capture(net, nph, a, E));
  else if (!same_args(a, E.a)) TRY(patch_graph(net, nph, a, E));
  CU(cudaGraphLaunch(E.ex, st));
  net->last = a;
  net->forward_done = true;
  return PN_OK;
}

static void drop_graphs(pn_net* net) {
  net->step.drop();
  net->infer.drop();
  for (auto& g : net->slot) g.drop();
  if (net->multi) cudaGraphExecDestroy(net->multi);
  if (net->multi_g) cudaGraphDestroy(net->multi_g);
  net->multi = nullptr;
  net->multi_g = nullptr;
}


// ------------------------------------------------------------------ C ABI
#define CHECK_NET(n) \
  if (!(n)) return fail(PN_ERR_INVALID_ARG, "net is NULL")

extern "C" pn_status net_create(const char* spec, int batch, int device, int flags, pn_net** out) {
  if (!spec || !out || batch <= 0 || device < 0 || (flags & ~7)) return fail(PN_ERR_INVALID_ARG, "net_create: bad argument");
  *out = nullptr;
  std::unique_ptr<pn_net> net(new pn_net());
  net->device = device;
  net->batch = batch;
  net->flags = flags;
  net->tf32 = flags & PN_TF32;
  TRY(parse_and_infer(net.get(), spec));  // host-only: spec errors need no GPU
  CU(cudaSetDevice(device));
  net->fused = !(flags & PN_LAYERWISE) && is_lenet(net.get());
  net->x3 = (flags & PN_3XTF32) && !net->tf32 && net->fused;
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  net->tc_sms = sms;
  int max_nk = 1;
  if (net->tf32 && !net->fused) {
    // layerwise TF32 plan: every convolution on the general tcgen05 kernels
    // (tc_conv.cu); the data gradient needs stride 1 and pad < kernel (else
    // the generic fp32 kernel computes it)
    net->layers[0].stem = is_stem(net.get()) && !getenv("PN_NO_STEM");
    {
      Layer& S0 = net->layers[0];
      S0.stem_plane = S0.stem && !getenv("PN_NO_STEM_PLANE") && S0.sh == 1 && S0.sw == 1 && S0.G == 1 &&
                      tcc::plane_plan(batch, S0.in[1], S0.out[2], S0.out[3], S0.F, S0.kh, S0.kw, &S0.pf);
    }
    for (auto& L : net->layers) {
      if (L.type != L_CONV || L.stem) continue;
      const int Cg = L.in[1] / L.G, Fg = L.F / L.G;
      // grouped layers run on the tap GEMM only: stride 1,
      // >= 16 channels per group (else the generic fp32 kernels)
      if (L.G > 1 && !(L.sh == 1 && L.sw == 1 && Cg >= 16 && Fg >= 16)) continue;
      L.tc_conv = true;
      // forward: tap GEMM for stride-1 layers with >= 16 input channels,
      // materialised im2col for strided layers with K >= 256 (AlexNet conv1),
      // else the gather kernel (C = 3, K = 75: cifar conv1)
      L.tap_fwd = L.sh == 1 && L.sw == 1 && Cg >= 16;
      // NHWC channel slots: per group a multiple of 32 when grouped (chunks
      // never straddle groups), else a multiple of 4
      L.cp_in = L.G > 1 ? (Cg + 31) / 32 * 32 : (L.in[1] + 3) / 4 * 4;
      L.cp_out = L.G > 1 ? (Fg + 31) / 32 * 32 : (L.F + 3) / 4 * 4;
      L.tma_fwd = !L.tap_fwd && L.in[1] * L.kh * L.kw >= 256;
      if (!L.tma_fwd && !L.tap_fwd) {
        L.fwd_rows = tcc::fwd_rows_pad(L.F);
        L.fwd_nk = (L.in[1] * L.kh * L.kw + 31) / 32;
        max_nk = std::max(max_nk, L.fwd_nk);
      }
      L.tc_dgrad = L.bottom != net->input_name && L.sh == 1 && L.sw == 1 && L.ph < L.kh && L.pw < L.kw;
      L.tap_dgrad = L.tc_dgrad && Fg >= 16;
      L.plane_f = L.tap_fwd && L.G == 1 &&
                  tcc::plane_plan(batch, L.in[1], L.out[2], L.out[3], L.F, L.kh, L.kw, &L.pf);
      L.plane_d = L.tap_dgrad && L.G == 1 &&
                  tcc::plane_plan(batch, L.F, L.in[2], L.in[3], L.in[1], L.kh, L.kw, &L.pd);
      if (L.tc_dgrad && !L.tap_dgrad) {
        L.dg_rows = tcc::fwd_rows_pad(L.in[1]);
        L.dg_nk = (L.F * L.kh * L.kw + 31) / 32;
        max_nk = std::max(max_nk, L.dg_nk);
      }
    }
  }
  TRY(allocate(net.get()));
  if (net->layers[0].stem) {
    const Layer &C = net->layers[0], &P = net->layers[1];
    CU(cudaFuncSetAttribute((const void*)stem_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, stem_fwd_smem(C)));
    CU(cudaFuncSetAttribute((const void*)stem_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)stem_wgrad_smem(C.in[1], C.in[2], C.in[3], C.ph, C.pw, P.out[2] * P.out[3])));
  }
  CU(cudaFuncSetAttribute((const void*)lenet_conv2_pool2_simt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (50 * 20 * 28 + kC2Imgs * 2880) * 4));
  CU(cudaFuncSetAttribute((const void*)lenet_conv2_dgrad_simt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kConv2DgradSimtSmem));
  if (net->tf32 || net->x3) {
    cudaError_t e = net->fused ? tc::setup() : tcc::setup(max_nk);
    if (e != cudaSuccess) return fail(PN_ERR_CUDA, std::string("tc setup: ") + cudaGetErrorString(e));
  }
  if (net->fused && net->tf32) {  // side stream of the single-GPU backward (build_fused_lenet)
    {  // the side branch at the highest priority: its small kernels are scheduled ahead of the
       // pending CTAs of the persistent conv backward kernels (PN_SIDE_PRIO=0: default priority)
      int lo = 0, hi = 0;
      CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const char* e = getenv("PN_SIDE_PRIO");
      CU(cudaStreamCreateWithPriority(&net->side, cudaStreamNonBlocking, (e && e[0] == '0') ? 0 : hi));
    }
    CU(cudaEventCreateWithFlags(&net->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&net->ev_join, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&net->ev_ipd, cudaEventDisableTiming));
  }
  TRY(build_plan(net.get()));
  if (net->tf32 && (!tc::tensor_maps_ok() || net->tmap_failed)) return fail(PN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  CU(cudaDeviceSynchronize());
  *out = net.release();
  return PN_OK;
}

extern "C" void net_destroy(pn_net* net) {
  if (!net) return;
  cudaSetDevice(net->device);
  cudaDeviceSynchronize();
  drop_graphs(net);
  if (net->cap) cudaStreamDestroy(net->cap);
  if (net->dpx) dpx_destroy(net->dpx);
  if (net->comm && net->nccl_reg) ncclCommDeregister(net->comm, net->nccl_reg);
  if (net->nccl_grads) ncclMemFree(net->nccl_grads);
  if (net->nccl_params) ncclMemFree(net->nccl_params);
  if (net->nccl_hist) ncclMemFree(net->nccl_hist);
  if (net->comm) ncclCommDestroy(net->comm);
  if (net->comm_stream) cudaStreamDestroy(net->comm_stream);
  for (cudaEvent_t e : {net->ev_ip, net->ev_conv, net->ev_done, net->ev_fork, net->ev_join, net->ev_ipd})
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < pn_net::kSlots; ++b) {
    if (net->ev_copied[b]) cudaEventDestroy(net->ev_copied[b]);
    if (net->ev_used[b]) cudaEventDestroy(net->ev_used[b]);
  }
  if (net->side) cudaStreamDestroy(net->side);
  if (net->copy) cudaStreamDestroy(net->copy);
  if (net->aux) cudaStreamDestroy(net->aux);
  for (cudaEvent_t e : net->ev_loss)
    if (e) cudaEventDestroy(e);
  if (net->ev_aux) cudaEventDestroy(net->ev_aux);
  if (net->loss_pinned) cudaFreeHost(net->loss_pinned);
  if (net->lr_pinned) cudaFreeHost(net->lr_pinned);
  for (void* p : net->allocs) cudaFree(p);
  delete net;
}

extern "C" pn_status net_blob_count(const pn_net* net, int* count) {
  CHECK_NET(net);
  if (!count) return fail(PN_ERR_INVALID_ARG, "count is NULL");
  *count = (int)net->blobs.size();
  return PN_OK;
}

extern "C" pn_status net_blob_info(const pn_net* net, int i, const char** name, int dims[4], int* is_param,
                                   int* materialised) {
  CHECK_NET(net);
  if (i < 0 || i >= (int)net->blobs.size()) return fail(PN_ERR_INVALID_ARG, "blob index out of range");
  const Blob& b = net->blobs[i];
  if (name) *name = b.name.c_str();
  if (dims) memcpy(dims, b.dims, sizeof(b.dims));
  if (is_param) *is_param = b.is_param;
  if (materialised) *materialised = b.materialised;
  return PN_OK;
}

extern "C" pn_status net_param_count(const pn_net* net, int64_t* count) {
  CHECK_NET(net);
  if (!count) return fail(PN_ERR_INVALID_ARG, "count is NULL");
  *count = net->nlearn;
  return PN_OK;
}

static pn_status find_blob(pn_net* net, const char* name, Blob** b) {
  if (!name) return fail(PN_ERR_INVALID_ARG, "blob name is NULL");
  int i = net->blob(name);
  if (i < 0) return fail(PN_ERR_INVALID_ARG, std::string("no blob named ") + name);
  *b = &net->blobs[i];
  return PN_OK;
}

extern "C" pn_status net_blob_ptr(pn_net* net, const char* name, int which, void** p) {
  CHECK_NET(net);
  Blob* b;
  TRY(find_blob(net, name, &b));
  if (!p) return fail(PN_ERR_INVALID_ARG, "out pointer is NULL");
  void* r = which == PN_DATA ? (void*)b->data : which == PN_DIFF ? (void*)b->diff
          : which == PN_HISTORY ? (void*)b->hist : nullptr;
  if (!r) return fail(PN_ERR_STATE, std::string(name) + ": buffer not materialised by this plan");
  if (b->is_param && which == PN_DATA) net->pack_dirty = true;  // the caller may write the parameters
  *p = r;
  return PN_OK;
}

extern "C" pn_status net_set_param(pn_net* net, const char* name, const float* src, int64_t count, int on_host,
                                   void* stream) {
  CHECK_NET(net);
  Blob* b;
  TRY(find_blob(net, name, &b));
  if (!b->is_param) return fail(PN_ERR_INVALID_ARG, std::string(name) + " is not a parameter");
  if (!src || count != b->count()) return fail(PN_ERR_INVALID_ARG, "net_set_param: count mismatch");
  CU(cudaSetDevice(net->device));
  net->pack_dirty = true;
  cudaStream_t st = (cudaStream_t)stream;
  if (on_host) {
    CU(cudaMemcpyAsync(b->data, src, count * 4, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
  } else {
    CU(cudaMemcpyAsync(b->data, src, count * 4, cudaMemcpyDeviceToDevice, st));
  }
  return PN_OK;
}

static pn_status mask_io(pn_net* net, Blob* b, int32_t* m32, bool to32, cudaStream_t st) {
  const Layer& L = net->layers[b->pool_layer];
  MaskExpandP p{b->m8, m32, b->dims[0], b->dims[1], L.in[2], L.in[3], L.kh, L.kw, L.sh, L.sw, L.ph, L.pw,
                b->dims[2], b->dims[3], to32 ? 1 : 0};
  Launch l;
  l.set((const void*)mask_convert, dim3(cdiv(b->count(), 256)), dim3(256), 0, p);
  CU(l.launch(st));
  return PN_OK;
}

static pn_status blob_io(pn_net* net, const char* name, int which, void* buf, int64_t bytes, int on_host,
                         void* stream, bool put) {
  CHECK_NET(net);
  Blob* b;
  TRY(find_blob(net, name, &b));
  if (!buf) return fail(PN_ERR_INVALID_ARG, "buffer is NULL");
  if (bytes != b->count() * 4) return fail(PN_ERR_INVALID_ARG, "byte count mismatch");
  CU(cudaSetDevice(net->device));
  cudaStream_t st = (cudaStream_t)stream;
  void* dev = nullptr;
  int32_t* tmp = nullptr;
  if (which == PN_MASK) {
    if (b->pool_layer < 0 || net->layers[b->pool_layer].method != 0)
      return fail(PN_ERR_INVALID_ARG, std::string(name) + " has no max-pool mask");
    if (b->m32) dev = b->m32;
    else {
      CU(cudaMallocAsync((void**)&tmp, bytes, st));
      dev = tmp;
    }
  } else {
    if (which != PN_DATA && which != PN_DIFF && which != PN_HISTORY) return fail(PN_ERR_INVALID_ARG, "bad which");
    dev = which == PN_DATA ? (void*)b->data : which == PN_DIFF ? (void*)b->diff : (void*)b->hist;
    if (!dev) return fail(b->is_input || b->is_param ? PN_ERR_INVALID_ARG : PN_ERR_STATE,
                          std::string(name) + ": buffer not materialised by this plan");
  }
  cudaMemcpyKind kind = on_host ? (put ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost) : cudaMemcpyDeviceToDevice;
  if (put && b->is_param && which == PN_DATA) net->pack_dirty = true;
  if (put) {
    CU(cudaMemcpyAsync(dev, buf, bytes, kind, st));
    if (tmp) TRY(mask_io(net, b, tmp, false, st));
    if (net->tf32 && net->fused) {
      // keep the tensor-core operand copies of an overwritten blob in sync
      Tf32CopyP c{nullptr, nullptr, nullptr, 0, 0, 0};
      if (b->name == net->layers[3].top && which == PN_DATA)
        c = Tf32CopyP{b->data, nullptr, net->p2T, net->batch, 800, net->npad};
      else if (b->name == net->layers[4].top && which == PN_DIFF)
        c = Tf32CopyP{b->diff, net->da1r, net->da1rT, net->batch, 500, net->npad};
      if (c.src) {
        Launch l;
        l.set((const void*)tf32_copy, dim3(cdiv((long long)c.R * c.C, 256)), dim3(256), 0, c);
        CU(l.launch(st));
      }
      if (b->name == net->layers[1].top && which == PN_DATA) CU(tc::pack_p1c_launch(b->data, net->p1c, net->batch).launch(st));
    }
  } else {
    if (tmp) TRY(mask_io(net, b, tmp, true, st));
    CU(cudaMemcpyAsync(buf, dev, bytes, kind, st));
  }
  if (tmp) CU(cudaFreeAsync(tmp, st));
  if (on_host) CU(cudaStreamSynchronize(st));
  return PN_OK;
}

extern "C" pn_status net_get_blob(pn_net* net, const char* name, int which, void* dst, int64_t bytes, int on_host,
                                  void* stream) {
  return blob_io(net, name, which, dst, bytes, on_host, stream, false);
}
extern "C" pn_status net_put_blob(pn_net* net, const char* name, int which, const void* src, int64_t bytes,
                                  int on_host, void* stream) {
  return blob_io(net, name, which, const_cast<void*>(src), bytes, on_host, stream, true);
}

extern "C" pn_status net_forward(pn_net* net, const float* x, const int32_t* labels, float* loss, void* stream) {
  CHECK_NET(net);
  if (!x || !labels) return fail(PN_ERR_INVALID_ARG, "x and labels are required");
  CU(cudaSetDevice(net->device));
  StepArgs a = make_args(net, x, labels, loss, nullptr, 0);
  net->last = a;
  TRY(run_phase(net, 0, a, (cudaStream_t)stream));
  net->forward_done = true;
  return PN_OK;
}

extern "C" pn_status net_backward(pn_net* net, void* stream) {
  CHECK_NET(net);
  if (!net->forward_done) return fail(PN_ERR_STATE, "net_backward before net_forward");
  CU(cudaSetDevice(net->device));
  TRY(run_phase(net, 1, net->last, (cudaStream_t)stream));
  return PN_OK;
}

extern "C" pn_status sgd_update(pn_net* net, const pn_sgd* sgd, int64_t iter, void* stream) {
  CHECK_NET(net);
  if (!sgd || iter < 0 || (sgd->lr_policy != 0 && sgd->lr_policy != 1))
    return fail(PN_ERR_INVALID_ARG, "sgd_update: bad solver settings");
  CU(cudaSetDevice(net->device));
  StepArgs a = make_args(net, net->last.x, net->last.labels, net->last.loss, sgd, iter);
  TRY(run_phase(net, 2, a, (cudaStream_t)stream));
  return PN_OK;
}

extern "C" pn_status net_train_step(pn_net* net, const float* x, const int32_t* labels, const pn_sgd* sgd,
                                    int64_t iter, float* loss, void* stream) {
  CHECK_NET(net);
  if (!x || !labels || !sgd || iter < 0 || (sgd->lr_policy != 0 && sgd->lr_policy != 1))
    return fail(PN_ERR_INVALID_ARG, "net_train_step: bad argument");
  CU(cudaSetDevice(net->device));
  StepArgs a = make_args(net, x, labels, loss, sgd, iter);
  return replay(net, 3, a, net->step, (cudaStream_t)stream);
}

extern "C" pn_status net_infer(pn_net* net, const float* x, const int32_t* labels, float* loss, void* stream) {
  CHECK_NET(net);
  if (!x || !labels) return fail(PN_ERR_INVALID_ARG, "x and labels are required");
  CU(cudaSetDevice(net->device));
  StepArgs a = make_args(net, x, labels, loss, nullptr, 0);
  return replay(net, 1, a, net->infer, (cudaStream_t)stream);
}

extern "C" pn_status net_train_step_host(pn_net* net, const float* xh, const int32_t* lh, const pn_sgd* sgd,
                                         int64_t iter, float* loss_host, void* stream) {
  CHECK_NET(net);
  if (!xh || !lh || !loss_host) return fail(PN_ERR_INVALID_ARG, "host buffers are required");
  CU(cudaSetDevice(net->device));
  cudaStream_t st = (cudaStream_t)stream;
  const Blob& in = net->blobs[net->blob(net->input_name)];
  if (!net->hs_x) {  // owned by the net, on its device, freed by net_destroy
    TRY(net->alloc(&net->hs_x, (size_t)in.count()));
    TRY(net->alloc(&net->hs_y, (size_t)net->batch));
    TRY(net->alloc(&net->hs_loss, 1));
  }
  CU(cudaMemcpyAsync(net->hs_x, xh, in.count() * 4, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(net->hs_y, lh, net->batch * 4, cudaMemcpyHostToDevice, st));
  TRY(net_train_step(net, net->hs_x, net->hs_y, sgd, iter, net->hs_loss, stream));
  CU(cudaMemcpyAsync(loss_host, net->hs_loss, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return PN_OK;
}

// ------------------------------------------------ byte input (NEXT #4)
static int64_t input_count(pn_net* net) { return net->blobs[net->blob(net->input_name)].count(); }

extern "C" pn_status net_set_input_transform(pn_net* net, float scale, const float* mean_host, int64_t count) {
  CHECK_NET(net);
  const Blob& in = net->blobs[net->blob(net->input_name)];
  const int64_t per = in.count() / net->batch;
  if (!(scale > 0.f) || (mean_host && count != per))
    return fail(PN_ERR_INVALID_ARG, "input transform: scale > 0 and a mean of C*H*W floats (or none)");
  CU(cudaSetDevice(net->device));
  net->x_scale = scale;
  if (mean_host) {
    if (!net->x_mean) TRY(net->alloc(&net->x_mean, (size_t)per));
    CU(cudaMemcpy(net->x_mean, mean_host, per * 4, cudaMemcpyHostToDevice));
  } else {
    net->x_mean = nullptr;
  }
  // the transform is a kernel parameter of the captured graphs: re-capture
  drop_graphs(net);
  return PN_OK;
}

// the step's arguments for a byte batch: the fused LeNet plan normalises the
// bytes inside conv1's own loads; any other plan gets them through the ingest
// kernel into an fp32 input buffer first
static pn_status byte_args(pn_net* net, const uint8_t* x8, StepArgs& a, cudaStream_t st) {
  if (net->fused) {
    a.x = nullptr;
    a.x8 = x8;
    return PN_OK;
  }
  const int64_t n = input_count(net);
  if (!net->xin) TRY(net->alloc(&net->xin, (size_t)n));
  IngestP q{x8, net->xin, n, (int)(n / net->batch), net->x_scale, net->x_mean};
  Launch l;
  l.set((const void*)ingest_u8, dim3(cdiv((n + 3) / 4, 256)), dim3(256), 0, q);
  CU(l.launch(st));
  a.x = net->xin;
  a.x8 = nullptr;
  return PN_OK;
}


extern "C" pn_status net_train_step_u8(pn_net* net, const uint8_t* x8, const int32_t* labels, const pn_sgd* sgd,
                                       int64_t iter, float* loss, void* stream) {
  CHECK_NET(net);
  if (!x8 || !labels || !sgd || iter < 0 || (sgd->lr_policy != 0 && sgd->lr_policy != 1))
    return fail(PN_ERR_INVALID_ARG, "net_train_step_u8: bad argument");
  CU(cudaSetDevice(net->device));
  StepArgs a = make_args(net, nullptr, labels, loss, sgd, iter);
  TRY(byte_args(net, x8, a, (cudaStream_t)stream));
  return replay(net, 3, a, net->step, (cudaStream_t)stream);
}

extern "C" pn_status net_train_steps_u8_host(pn_net* net, const uint8_t* x8_host, const int32_t* labels_host,
                                             int64_t nsteps, const pn_sgd* sgd, int64_t iter0, float* losses_host,
                                             void* stream) {
  CHECK_NET(net);
  if (!x8_host || !labels_host || !losses_host || !sgd || nsteps < 0 || iter0 < 0)
    return fail(PN_ERR_INVALID_ARG, "net_train_steps_u8_host: bad argument");
  CU(cudaSetDevice(net->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nx = input_count(net);
  if (!net->copy) {
    CU(cudaStreamCreateWithFlags(&net->copy, cudaStreamNonBlocking));
    for (int b = 0; b < pn_net::kSlots; ++b) {
      CU(cudaEventCreateWithFlags(&net->ev_copied[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&net->ev_used[b], cudaEventDisableTiming));
      TRY(net->alloc(&net->h2d_x8[b], (size_t)nx));
      TRY(net->alloc(&net->h2d_y[b], (size_t)net->batch));
    }
    TRY(net->alloc(&net->h2d_loss, pn_net::kSlots));
    TRY(net->alloc(&net->h2d_lr, pn_net::kSlots));
    // the slots start free
    for (int b = 0; b < pn_net::kSlots; ++b) CU(cudaEventRecord(net->ev_used[b], st));
  }
  if (net->lr_pinned_cap < nsteps) {  // the steps' learning rates, staged in pinned memory
    if (net->lr_pinned) cudaFreeHost(net->lr_pinned);
    net->lr_pinned = nullptr;
    net->lr_pinned_cap = 0;
    CU(cudaMallocHost(&net->lr_pinned, nsteps * sizeof(float)));
    net->lr_pinned_cap = nsteps;
  }
  for (int64_t s = 0; s < nsteps; ++s) net->lr_pinned[s] = make_args(net, nullptr, nullptr, nullptr, sgd, iter0 + s).lr;
  if (net->loss_pinned_cap < nsteps) {  // the D2H loss reads land in pinned memory (asynchronous)
    if (net->loss_pinned) cudaFreeHost(net->loss_pinned);
    net->loss_pinned = nullptr;
    net->loss_pinned_cap = 0;
    CU(cudaMallocHost(&net->loss_pinned, nsteps * sizeof(float)));
    net->loss_pinned_cap = nsteps;
  }
  // slot b's step arguments (fixed device pointers; the learning rate rides in h2d_lr[b])
  auto slot_args = [&](int b, int64_t s, StepArgs& a) -> pn_status {
    a = make_args(net, nullptr, net->h2d_y[b], net->h2d_loss + b, sgd, iter0 + s);
    a.lr = 0.f;
    a.lr_dev = net->h2d_lr + b;
    return byte_args(net, net->h2d_x8[b], a, st);
  };
  auto issue_copies = [&](int64_t s) -> pn_status {
    const int b = (int)(s % pn_net::kSlots);
    CU(cudaStreamWaitEvent(net->copy, net->ev_used[b], 0));  // step s - kSlots is done with slot b
    CU(cudaMemcpyAsync(net->h2d_x8[b], x8_host + s * nx, nx, cudaMemcpyHostToDevice, net->copy));
    CU(cudaMemcpyAsync(net->h2d_y[b], labels_host + s * net->batch, net->batch * 4, cudaMemcpyHostToDevice,
                       net->copy));
    CU(cudaMemcpyAsync(net->h2d_lr + b, net->lr_pinned + s, 4, cudaMemcpyHostToDevice, net->copy));
    CU(cudaEventRecord(net->ev_copied[b], net->copy));
    return PN_OK;
  };
  int64_t s0 = 0;
  TRY(ensure_packed(net, st));
  if (net->fused && nsteps >= pn_net::kSlots && !getenv("PN_NO_MULTI")) {
    {  // momentum / decay / 1/G are kernel arguments of the captured steps: re-capture when they change
      const StepArgs h = make_args(net, nullptr, nullptr, nullptr, sgd, iter0);
      if (net->multi && (h.mom != net->multi_mom || h.decay != net->multi_decay || h.gscale != net->multi_gscale)) {
        CU(cudaStreamSynchronize(st));
        cudaGraphExecDestroy(net->multi);
        cudaGraphDestroy(net->multi_g);
        net->multi = nullptr;
        net->multi_g = nullptr;
      }
    }
    if (!net->multi) {  // capture the kSlots-step graph once (slot arguments never change)
      if (!net->cap) CU(cudaStreamCreateWithFlags(&net->cap, cudaStreamNonBlocking));
      if (!net->aux) {
        CU(cudaStreamCreateWithFlags(&net->aux, cudaStreamNonBlocking));
        for (auto& e : net->ev_loss) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&net->ev_aux, cudaEventDisableTiming));
      }
      CU(cudaStreamBeginCapture(net->cap, cudaStreamCaptureModeThreadLocal));
      pn_status err = PN_OK;
      bool prev_kernel = false;
      for (int b = 0; b < pn_net::kSlots && err == PN_OK; ++b) {
        StepArgs a;
        if ((err = slot_args(b, b, a)) != PN_OK) break;
        if (cudaStreamWaitEvent(net->cap, net->ev_copied[b], cudaEventWaitExternal) != cudaSuccess) { err = PN_ERR_CUDA; break; }
        prev_kernel = false;
        for (int ph = 0; ph < 3 && err == PN_OK; ++ph)
          for (auto& stg : net->phase[ph]) {
            if (!in_run(stg, true)) continue;
            cudaStream_t on = stg.side ? net->side : net->cap;
            if ((err = run_stage(net, stg, a, on, stg.side ? false : prev_kernel)) != PN_OK) break;
            if (!stg.side && !stg.transparent) prev_kernel = !stg.custom;
          }
        if (err != PN_OK) break;
        // the loss read-back on a side branch (the next step does not wait for it)
        if (cudaEventRecord(net->ev_loss[b], net->cap) != cudaSuccess ||
            cudaStreamWaitEvent(net->aux, net->ev_loss[b], 0) != cudaSuccess ||
            cudaMemcpyAsync(net->loss_pinned + b, net->h2d_loss + b, 4, cudaMemcpyDeviceToHost, net->aux) != cudaSuccess) {
          err = PN_ERR_CUDA;
          break;
        }
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        if (cudaStreamGetCaptureInfo(net->aux, &cs, nullptr, nullptr, &deps, &nd) != cudaSuccess || nd == 0) { err = PN_ERR_CUDA; break; }
        net->multi_d2h[b] = deps[0];
        if (cudaEventRecordWithFlags(net->ev_used[b], net->cap, cudaEventRecordExternal) != cudaSuccess) { err = PN_ERR_CUDA; break; }
      }
      if (err == PN_OK && (cudaEventRecord(net->ev_aux, net->aux) != cudaSuccess ||
                           cudaStreamWaitEvent(net->cap, net->ev_aux, 0) != cudaSuccess))
        err = PN_ERR_CUDA;  // the read-backs join before the graph ends
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(net->cap, &g);
      if (err != PN_OK || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return err != PN_OK ? err : fail(PN_ERR_CUDA, "capture of the pipelined steps failed");
      }
      CU(cudaGraphInstantiate(&net->multi, g, 0));
      net->multi_g = g;
      const StepArgs h = make_args(net, nullptr, nullptr, nullptr, sgd, iter0);
      net->multi_mom = h.mom;
      net->multi_decay = h.decay;
      net->multi_gscale = h.gscale;
    }
    for (; s0 + pn_net::kSlots <= nsteps; s0 += pn_net::kSlots) {
      for (int b = 0; b < pn_net::kSlots; ++b) TRY(issue_copies(s0 + b));
      for (int b = 0; b < pn_net::kSlots; ++b)
        CU(cudaGraphExecMemcpyNodeSetParams1D(net->multi, net->multi_d2h[b], net->loss_pinned + s0 + b,
                                              net->h2d_loss + b, 4, cudaMemcpyDeviceToHost));
      CU(cudaGraphLaunch(net->multi, st));
    }
    net->forward_done = true;
  }
  // the remaining steps one graph launch each (kSlots input slots: the copies
  // of the next batches on the copy stream run under step s)
  for (int64_t s = s0; s < nsteps; ++s) {
    const int b = (int)(s % pn_net::kSlots);
    CU(cudaStreamWaitEvent(net->copy, net->ev_used[b], 0));  // step s-2 is done with slot b
    CU(cudaMemcpyAsync(net->h2d_x8[b], x8_host + s * nx, nx, cudaMemcpyHostToDevice, net->copy));
    CU(cudaMemcpyAsync(net->h2d_y[b], labels_host + s * net->batch, net->batch * 4, cudaMemcpyHostToDevice,
                       net->copy));
    CU(cudaMemcpyAsync(net->h2d_lr + b, net->lr_pinned + s, 4, cudaMemcpyHostToDevice, net->copy));
    CU(cudaEventRecord(net->ev_copied[b], net->copy));
    CU(cudaStreamWaitEvent(st, net->ev_copied[b], 0));
    StepArgs a = make_args(net, nullptr, net->h2d_y[b], net->h2d_loss + b, sgd, iter0 + s);
    a.lr = 0.f;  // read from the slot on the device instead: slot b's graph needs no patching
    a.lr_dev = net->h2d_lr + b;
    TRY(byte_args(net, net->h2d_x8[b], a, st));
    TRY(replay(net, 3, a, net->slot[b], st));  // slot b's own graph: only the lr changes
    CU(cudaMemcpyAsync(net->loss_pinned + s, net->h2d_loss + b, 4, cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(net->ev_used[b], st));
  }
  CU(cudaStreamSynchronize(st));
  std::memcpy(losses_host, net->loss_pinned, nsteps * sizeof(float));
  return PN_OK;
}

// ------------------------------------------------ dataset files (NEXT #4)
// MNIST IDX (big-endian magic 0x00000800 | type << 8 | ndims, then ndims
// big-endian uint32 sizes, then the data; type 0x08 = unsigned byte) and the
// CIFAR-10 binary batches (records of 1 label byte + 3072 pixel bytes, CHW).
static bool read_all(const char* path, std::vector<uint8_t>& buf) {
  FILE* f = fopen(path, "rb");
  if (!f) return false;
  uint8_t tmp[1 << 16];
  size_t n;
  while ((n = fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
  fclose(f);
  return true;
}

extern "C" pn_status pn_idx_read(const char* path, uint8_t* dst, int64_t cap, int* ndims, int64_t dims[4]) {
  if (!path || !ndims || !dims) return fail(PN_ERR_INVALID_ARG, "pn_idx_read: NULL argument");
  std::vector<uint8_t> b;
  if (!read_all(path, b)) return fail(PN_ERR_INVALID_ARG, std::string("cannot read ") + path);
  if (b.size() < 4 || b[0] != 0 || b[1] != 0 || b[2] != 0x08 || b[3] < 1 || b[3] > 4)
    return fail(PN_ERR_PARSE, "not an unsigned-byte IDX file (magic)");
  const int nd = b[3];
  if (b.size() < 4 + 4 * (size_t)nd) return fail(PN_ERR_PARSE, "truncated IDX header");
  int64_t total = 1;
  for (int i = 0; i < nd; ++i) {
    const uint8_t* q = &b[4 + 4 * i];
    dims[i] = ((int64_t)q[0] << 24) | ((int64_t)q[1] << 16) | ((int64_t)q[2] << 8) | q[3];
    total *= dims[i];
  }
  *ndims = nd;
  const size_t off = 4 + 4 * (size_t)nd;
  if (b.size() != off + (size_t)total) return fail(PN_ERR_PARSE, "IDX size does not match its header");
  if (dst) {
    if (cap < total) return fail(PN_ERR_INVALID_ARG, "pn_idx_read: destination too small");
    std::memcpy(dst, b.data() + off, (size_t)total);
  }
  return PN_OK;
}

extern "C" pn_status pn_cifar_read(const char* path, uint8_t* pixels, int32_t* labels, int64_t cap, int64_t* count) {
  if (!path || !count) return fail(PN_ERR_INVALID_ARG, "pn_cifar_read: NULL argument");
  std::vector<uint8_t> b;
  if (!read_all(path, b)) return fail(PN_ERR_INVALID_ARG, std::string("cannot read ") + path);
  if (b.empty() || b.size() % 3073) return fail(PN_ERR_PARSE, "CIFAR-10 binary: size is not a multiple of 3073");
  const int64_t n = (int64_t)(b.size() / 3073);
  *count = n;
  if (pixels || labels) {
    if (cap < n) return fail(PN_ERR_INVALID_ARG, "pn_cifar_read: destination too small");
    for (int64_t i = 0; i < n; ++i) {
      const uint8_t* r = b.data() + i * 3073;
      if (r[0] > 9) return fail(PN_ERR_PARSE, "CIFAR-10 binary: label byte > 9");
      if (labels) labels[i] = r[0];
      if (pixels) std::memcpy(pixels + i * 3072, r + 1, 3072);
    }
  }
  return PN_OK;
}

extern "C" pn_status net_stage_count(const pn_net* net, int phase, int* count) {
  CHECK_NET(net);
  if (phase < 0 || phase > 2 || !count) return fail(PN_ERR_INVALID_ARG, "bad phase");
  *count = (int)net->phase[phase].size();
  return PN_OK;
}

extern "C" pn_status net_stage_name(const pn_net* net, int phase, int i, const char** name) {
  CHECK_NET(net);
  if (phase < 0 || phase > 2 || i < 0 || i >= (int)net->phase[phase].size() || !name)
    return fail(PN_ERR_INVALID_ARG, "bad stage");
  *name = net->phase[phase][i].name.c_str();
  return PN_OK;
}

extern "C" pn_status net_stage_mode(const pn_net* net, int phase, int i, int* mode) {
  CHECK_NET(net);
  if (phase < 0 || phase > 2 || i < 0 || i >= (int)net->phase[phase].size() || !mode)
    return fail(PN_ERR_INVALID_ARG, "bad stage");
  *mode = net->phase[phase][i].mode;
  return PN_OK;
}

extern "C" pn_status net_run_stage(pn_net* net, int phase, int i, const float* x, const int32_t* labels,
                                   void* stream) {
  CHECK_NET(net);
  if (phase < 0 || phase > 2 || i < 0 || i >= (int)net->phase[phase].size())
    return fail(PN_ERR_INVALID_ARG, "bad stage");
  CU(cudaSetDevice(net->device));
  StepArgs a = net->last;
  if (x) a.x = x;
  if (labels) a.labels = labels;
  TRY(ensure_packed(net, (cudaStream_t)stream));
  return run_stage(net, net->phase[phase][i], a, (cudaStream_t)stream);
}

extern "C" pn_status net_profile_stages(pn_net* net, const float* x, const int32_t* labels, const pn_sgd* sgd,
                                        int64_t iter, int steps, float* ms_out, int cap, int* n_out, void* stream) {
  CHECK_NET(net);
  int total = 0;
  for (auto& ph : net->phase) total += (int)ph.size();
  if (!x || !labels || !sgd || steps <= 0 || !ms_out || cap < total) return fail(PN_ERR_INVALID_ARG, "bad argument");
  CU(cudaSetDevice(net->device));
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  // one pass through the plan in order.  Every kernel stage (each overwrites
  // its outputs from inputs it does not write, so repeats are idempotent --
  // except the solver, which then applies `steps` updates: the net's
  // parameters are changed by profiling) is captured `steps` times back to
  // back into one CUDA graph and replayed between two events: the mean is the
  // kernel's device duration plus the graph's launch-to-launch gap, without
  // the host launch rate (which bounds eager back-to-back launches on a slow
  // host).  Non-kernel stages (events, collectives) report 0.
  StepArgs a = make_args(net, x, labels, nullptr, sgd, iter);
  if (!net->cap) CU(cudaStreamCreateWithFlags(&net->cap, cudaStreamNonBlocking));
  int k = 0;
  for (int ph = 0; ph < 3; ++ph)
    for (auto& stg : net->phase[ph]) {
      if (stg.custom) {
        ms_out[k++] = 0.f;
        continue;
      }
      TRY(run_stage(net, stg, a, st));
      CU(cudaStreamSynchronize(st));
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      CU(cudaStreamBeginCapture(net->cap, cudaStreamCaptureModeThreadLocal));
      pn_status cs = PN_OK;
      for (int i = 0; i < steps && cs == PN_OK; ++i) cs = run_stage(net, stg, a, net->cap);
      cudaError_t ce = cudaStreamEndCapture(net->cap, &g);
      if (cs != PN_OK) {
        if (g) cudaGraphDestroy(g);
        return cs;
      }
      CU(ce);
      CU(cudaGraphInstantiate(&ge, g, 0));
      CU(cudaGraphLaunch(ge, st));  // warm
      CU(cudaEventRecord(e0, st));
      CU(cudaGraphLaunch(ge, st));
      CU(cudaEventRecord(e1, st));
      CU(cudaEventSynchronize(e1));
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, e0, e1));
      ms_out[k++] = ms / steps;
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  if (n_out) *n_out = total;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  net->forward_done = true;
  return PN_OK;
}

extern "C" pn_status net_launches_per_step(const pn_net* net, int* n) {
  CHECK_NET(net);
  if (!n) return fail(PN_ERR_INVALID_ARG, "n is NULL");
  *n = net->launches_per_step;
  return PN_OK;
}

// dev-only in-graph step timeline (pdl.cuh; libpn built with -DPN_STEPTRACE)
namespace pn {
void st_set_lenet(unsigned long long*);
void st_set_generic(unsigned long long*);
namespace tc {
void st_set_tc(unsigned long long*);
void st_set_c1(unsigned long long*);
}  // namespace tc
}  // namespace pn

extern "C" pn_status net_steptrace(pn_net* net, unsigned long long* host_out) {
  CHECK_NET(net);
#ifndef PN_STEPTRACE
  (void)host_out;
  return fail(PN_ERR_STATE, "libpn was built without -DPN_STEPTRACE");
#else
  CU(cudaSetDevice(net->device));
  static unsigned long long* buf = nullptr;
  const size_t bytes = ST_N * 3 * sizeof(unsigned long long);
  if (!buf) {
    CU(cudaMalloc(&buf, bytes));
    pn::st_set_lenet(buf);
    pn::st_set_generic(buf);
    pn::tc::st_set_tc(buf);
    pn::tc::st_set_c1(buf);
  }
  CU(cudaDeviceSynchronize());
  if (host_out) CU(cudaMemcpy(host_out, buf, bytes, cudaMemcpyDeviceToHost));
  std::vector<unsigned long long> init(ST_N * 3);
  for (int k = 0; k < ST_N; ++k) init[3 * k] = init[3 * k + 1] = ~0ull, init[3 * k + 2] = 0;
  CU(cudaMemcpy(buf, init.data(), bytes, cudaMemcpyHostToDevice));
  return PN_OK;
#endif
}

extern "C" pn_status net_sync_errors(pn_net* net, void* stream) {
  CHECK_NET(net);
  CU(cudaSetDevice(net->device));
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  unsigned e = 0;
  CU(cudaMemcpy(&e, net->err, 4, cudaMemcpyDeviceToHost));
  if (e) {
    CU(cudaMemset(net->err, 0, 4));
    return fail(PN_ERR_LABEL_RANGE, "a label was outside [0, classes)");
  }
  return PN_OK;
}

extern "C" pn_status pn_nccl_unique_id(void* out128) {
  if (!out128) return fail(PN_ERR_INVALID_ARG, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  memcpy(out128, &id, 128);
  return PN_OK;
}

// point the parameter blobs' diffs at the current gradient buffer
static void repoint_diffs(pn_net* net) {
  for (auto& L : net->layers) {
    if (L.off < 0) continue;
    int wi = net->blob(L.name + ".w"), bi = net->blob(L.name + ".b");
    if (wi >= 0) net->blobs[wi].diff = net->grads + L.off;
    if (bi >= 0) net->blobs[bi].diff = net->grads + L.off + L.wcount;
  }
}

// NEXT #1: the exchange and the solver fused into one kernel
// over NCCL symmetric windows (dp_exchange.cu).  Collective: every rank calls
// it after net_dp_init.  Parameters and momentum move into ncclMemAlloc
// buffers (their contents kept), the plan is rebuilt.
extern "C" pn_status net_dp_fused_exchange(pn_net* net) {
  CHECK_NET(net);
  if (!net->comm) return fail(PN_ERR_STATE, "net_dp_fused_exchange needs net_dp_init (an NCCL communicator)");
  if (net->dpx) return PN_OK;
  CU(cudaSetDevice(net->device));
  CU(cudaDeviceSynchronize());
  const size_t bytes = (size_t)net->nparams * 4;
  void *P = nullptr, *V = nullptr;
  NC(ncclMemAlloc(&P, bytes));
  NC(ncclMemAlloc(&V, bytes));
  CU(cudaMemcpy(P, net->params, bytes, cudaMemcpyDeviceToDevice));
  CU(cudaMemcpy(V, net->hist, bytes, cudaMemcpyDeviceToDevice));
  net->nccl_params = P, net->nccl_hist = V;
  net->params = (float*)P, net->hist = (float*)V;
  for (auto& L : net->layers) {
    if (L.off < 0) continue;
    int wi = net->blob(L.name + ".w"), bi = net->blob(L.name + ".b");
    if (wi >= 0) net->blobs[wi].data = net->params + L.off, net->blobs[wi].hist = net->hist + L.off;
    if (bi >= 0) net->blobs[bi].data = net->params + L.off + L.wcount, net->blobs[bi].hist = net->hist + L.off + L.wcount;
  }
  std::string err;
  if (dpx_setup(net->comm, net->grads, net->params, net->hist, net->nparams, net->tc_sms, &net->dpx, &err) != PN_OK)
    return fail(PN_ERR_NCCL, err);
  net->pack_dirty = true;
  drop_graphs(net);
  TRY(build_plan(net));
  return PN_OK;
}

extern "C" pn_status net_dp_init(pn_net* net, int nranks, int rank, const void* id128) {
  CHECK_NET(net);
  if (nranks < 1 || rank < 0 || rank >= nranks || !id128) return fail(PN_ERR_INVALID_ARG, "net_dp_init: bad rank");
  if (net->comm || net->loop) return fail(PN_ERR_STATE, "data parallelism already initialised");
  CU(cudaSetDevice(net->device));
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  NC(ncclCommInitRank(&net->comm, nranks, id, rank));
  net->nranks = nranks;
  net->rank = rank;
  // the flat gradient buffer (both buckets) from NCCL's allocator and
  // registered with the communicator, so NCCL can use NVLink SHARP (NVLS,
  // in-switch reduction) / zero-copy paths for the bucket allreduces
  const size_t bytes = (size_t)net->nparams * 4;
  void* buf = nullptr;
  NC(ncclMemAlloc(&buf, bytes));
  CU(cudaMemset(buf, 0, bytes));
  net->nccl_grads = buf;
  net->grads = (float*)buf;
  repoint_diffs(net);
  NC(ncclCommRegister(net->comm, buf, bytes, &net->nccl_reg));
  CU(cudaStreamCreateWithFlags(&net->comm_stream, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&net->ev_ip, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&net->ev_conv, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&net->ev_done, cudaEventDisableTiming));
  drop_graphs(net);
  TRY(build_plan(net));
  return PN_OK;
}

extern "C" pn_status pn_loopback_create(int n, void** group) {
  if (n < 1 || n > 8 || !group) return fail(PN_ERR_INVALID_ARG, "pn_loopback_create: 1 <= n <= 8");
  pn_loop* g = new pn_loop();
  g->n = n;
  g->nets.assign(n, nullptr);
  *group = g;
  return PN_OK;
}

extern "C" void pn_loopback_destroy(void* group) { delete static_cast<pn_loop*>(group); }

extern "C" pn_status net_dp_init_loopback(pn_net* net, void* group, int rank) {
  CHECK_NET(net);
  pn_loop* g = static_cast<pn_loop*>(group);
  if (!g || rank < 0 || rank >= g->n) return fail(PN_ERR_INVALID_ARG, "net_dp_init_loopback: bad group or rank");
  if (net->comm || net->loop) return fail(PN_ERR_STATE, "data parallelism already initialised");
  for (pn_net* o : g->nets)
    if (o && o->device != net->device) return fail(PN_ERR_INVALID_ARG, "loopback ranks must share one device");
  if (g->nets[rank]) return fail(PN_ERR_INVALID_ARG, "loopback rank already taken");
  CU(cudaSetDevice(net->device));
  g->nets[rank] = net;
  net->loop = g;
  net->nranks = g->n;
  net->rank = rank;
  drop_graphs(net);
  TRY(build_plan(net));
  return PN_OK;
}
