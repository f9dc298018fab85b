// dp_exchange.cu -- SURVEY §8(f) NEXT #1: the data-parallel gradient
// exchange fused with the solver (a18 + a17; the paper's multi-GPU roadmap,
// P:76, and its "recalculates some values" update, P:94 / S:536-544).
//
// One kernel over NVLink peer memory replaces the bucket allreduces and the
// solver launch: the gradient, parameter and momentum buffers are NCCL
// symmetric windows (ncclMemAlloc + ncclCommWindowRegister), and through
// NCCL's device API (ncclDevComm, LSA = load/store-accessible team) each
// rank r of G
//   1. meets the others at an LSA barrier (every rank's gradients final),
//   2. for its shard r of the flat parameters: sums the G ranks' gradients
//      -- multimem.ld_reduce on the NVLS multicast address (the switch adds
//      them) when the team has one, else loads from every peer's window in
//      rank order (deterministic) --, applies SGD (sgd_one; the 1/G of
//      R13 in gscale) to its local copy of w and the momentum, and writes the
//      updated w and v to every rank: multimem.st (one multicast store) or
//      one store per peer,
//   3. meets the others again (every rank's shard landed everywhere).
// Same bytes on the wire as reduce-scatter + all-gather, no NCCL launches,
// no separate solver pass.  (A single B200 gives a one-rank team: the peer
// path with G = 1 runs in the GPU tests; the multicast path needs an NVLS
// team of >= 2 GPUs -- a multicast object of one device is refused by the
// driver here, tools/mc_probe.cu.)
#include <cuda/atomic>

#include <nccl.h>
#include <nccl_device.h>

#include "dp_exchange.h"
#include "pdl.cuh"
#include "sgd.cuh"

namespace pn {
namespace dpx {

struct Params {
  ncclDevComm dc;
  ncclWindow_t wg, ww, wv;  // gradients, parameters, momentum (same layout on every rank)
  float* w;                 // this rank's parameters / momentum (its window's local memory)
  float* v;
  long long n4;             // float4 elements of the flat buffers
  int multimem;
  float lr, mom, decay, gscale;
  const float* lr_dev;
};

__device__ __forceinline__ float4 ld_reduce4(const float* mc) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}
__device__ __forceinline__ void st_mc4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(256) exchange_sgd(const __grid_constant__ Params p) {
  pdl_enter();
  ncclCoopCta cta;
  ncclLsaBarrierSession<ncclCoopCta> bar(cta, p.dc, ncclTeamTagLsa(), blockIdx.x, p.multimem != 0);
  bar.sync(cta, cuda::memory_order_acq_rel);  // every rank's gradients are final
  const float lr = p.lr_dev ? __ldg(p.lr_dev) : p.lr;
  const int G = p.dc.lsaSize, me = p.dc.lsaRank;
  const long long lo = p.n4 * me / G, hi = p.n4 * (me + 1) / G;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
    float4 g;
    if (p.multimem) {
      g = ld_reduce4((const float*)ncclGetLsaMultimemPointer(p.wg, 16 * i, p.dc));
    } else {  // rank order: the same sum on every rank that owns the shard
      g = *(const float4*)ncclGetLsaPointer(p.wg, 16 * i, 0);
      for (int r = 1; r < G; ++r) {
        const float4 t = *(const float4*)ncclGetLsaPointer(p.wg, 16 * i, r);
        g.x += t.x, g.y += t.y, g.z += t.z, g.w += t.w;
      }
    }
    float4 w = reinterpret_cast<float4*>(p.w)[i], v = reinterpret_cast<float4*>(p.v)[i];
    sgd_one(w.x, g.x, v.x, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.y, g.y, v.y, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.z, g.z, v.z, lr, p.mom, p.decay, p.gscale);
    sgd_one(w.w, g.w, v.w, lr, p.mom, p.decay, p.gscale);
    if (p.multimem) {
      st_mc4((float*)ncclGetLsaMultimemPointer(p.ww, 16 * i, p.dc), w);
      st_mc4((float*)ncclGetLsaMultimemPointer(p.wv, 16 * i, p.dc), v);
    } else {
      for (int r = 0; r < G; ++r) {
        *(float4*)ncclGetLsaPointer(p.ww, 16 * i, r) = w;
        *(float4*)ncclGetLsaPointer(p.wv, 16 * i, r) = v;
      }
    }
  }
  bar.sync(cta, cuda::memory_order_acq_rel);  // every rank's shard has landed everywhere
}

struct State {
  ncclComm_t comm = nullptr;
  ncclDevComm dc{};
  bool dc_ok = false;
  ncclWindow_t wg = nullptr, ww = nullptr, wv = nullptr;
  bool multimem = false;
  int blocks = 0;
};

}  // namespace dpx

pn_status dpx_setup(ncclComm_t comm, float* grads, float* params, float* hist, long long n, int sms, DpxState** out,
                    std::string* err) {
  auto* s = new dpx::State();
  s->comm = comm;
  auto bad = [&](const char* what, ncclResult_t r) {
    *err = std::string(what) + ": " + ncclGetErrorString(r);
    dpx_destroy(reinterpret_cast<DpxState*>(s));
    return PN_ERR_NCCL;
  };
  const size_t bytes = (size_t)n * 4;
  ncclResult_t r;
  if ((r = ncclCommWindowRegister(comm, grads, bytes, &s->wg, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)
    return bad("ncclCommWindowRegister(grads)", r);
  if ((r = ncclCommWindowRegister(comm, params, bytes, &s->ww, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)
    return bad("ncclCommWindowRegister(params)", r);
  if ((r = ncclCommWindowRegister(comm, hist, bytes, &s->wv, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess)
    return bad("ncclCommWindowRegister(hist)", r);
  int nranks = 1;
  ncclCommCount(comm, &nranks);
  s->blocks = sms;  // one LSA barrier per CTA
  ncclDevCommRequirements req{};
  req.lsaBarrierCount = s->blocks;
  req.lsaMultimem = nranks > 1;  // an NVLS team needs >= 2 GPUs
  r = ncclDevCommCreate(comm, &req, &s->dc);
  if (r != ncclSuccess && req.lsaMultimem) {  // no NVLS on this system: peer loads / stores
    req.lsaMultimem = false;
    r = ncclDevCommCreate(comm, &req, &s->dc);
  }
  if (r != ncclSuccess) return bad("ncclDevCommCreate", r);
  s->dc_ok = true;
  s->multimem = req.lsaMultimem;
  *out = reinterpret_cast<DpxState*>(s);
  return PN_OK;
}

void dpx_destroy(DpxState* st) {
  auto* s = reinterpret_cast<dpx::State*>(st);
  if (!s) return;
  if (s->dc_ok) ncclDevCommDestroy(s->comm, &s->dc);
  if (s->wg) ncclCommWindowDeregister(s->comm, s->wg);
  if (s->ww) ncclCommWindowDeregister(s->comm, s->ww);
  if (s->wv) ncclCommWindowDeregister(s->comm, s->wv);
  delete s;
}

bool dpx_multimem(const DpxState* st) { return reinterpret_cast<const dpx::State*>(st)->multimem; }

Launch dpx_launch(const DpxState* st, float* params, float* hist, long long n) {
  const auto* s = reinterpret_cast<const dpx::State*>(st);
  dpx::Params p{};
  p.dc = s->dc;
  p.wg = s->wg, p.ww = s->ww, p.wv = s->wv;
  p.w = params, p.v = hist;
  p.n4 = n / 4;
  p.multimem = s->multimem ? 1 : 0;
  Launch l;
  l.set((const void*)dpx::exchange_sgd, dim3(s->blocks), dim3(256), 0, p);
  return l;
}

void dpx_patch(Launch& l, float lr, float mom, float decay, float gscale, const float* lr_dev) {
  dpx::Params& q = l.params<dpx::Params>();
  q.lr = lr, q.mom = mom, q.decay = decay, q.gscale = gscale, q.lr_dev = lr_dev;
}

}  // namespace pn
