// Solver-level C ABI (SURVEY.md §8(b) "What the C-ABI layer must export"): a per-rank
// context owning a stream and an NCCL communicator, a Cox state that owns its
// workspaces, and bs_cox_run, the whole cox_fit loop (solvers.py:422-450) in native code
// (same kernels and order as paper_2010_16114_b200/solvers.py:cox_fit, collectives over
// NCCL).  A host without Python can drive a fit with these five calls; the Python package
// keeps its own loop over the same kernels.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"), so the library still loads where
// NCCL is absent; a context with size 1 needs no NCCL at all.
#include "bsb200.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

using namespace bs;

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.Reduce = reinterpret_cast<decltype(api.Reduce)>(dlsym(h, "ncclReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString &&
             api.Reduce && api.Broadcast && api.GroupStart && api.GroupEnd;
  });
  return api;
}

}  // namespace

struct bs_ctx {
  int rank, size, device;
  cudaStream_t stream;
  ncclComm_t comm;
};

struct bs_cox {
  bs_ctx* ctx;
  const void* X;
  int xdtype, dtype;
  int64_t m, n_loc;
  const void* delta;
  const int64_t* cuts;
  double lam, sigma, clamp;
  void* beta;
  void* grad;
  // owned device buffers
  double* xb;  // m + 1: X beta (reduced), ||beta||_1
  void *Xbeta, *w, *W, *pd;
  double* dmpd;
  double* loglik;
  int* flags;
  void *ws_xb, *ws_risk, *ws_pd, *ws_grad, *ws_fused, *ws_red;
  int64_t n_xb, n_risk, n_pd, n_grad, n_fused, n_red;
  bool fused;
  bool xb_fresh;  // xb holds the last fused pass's local partial for the current beta
};

namespace {

int nccl_err(const char* what, ncclResult_t r) {
  set_error("%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return BS_ENCCL;
}

int dalloc(void** p, int64_t bytes) {
  *p = nullptr;
  if (bytes <= 0) bytes = 256;
  if (cudaMalloc(p, size_t(bytes)) != cudaSuccess) return BS_ECUDA;
  return cudaMemset(*p, 0, size_t(bytes)) == cudaSuccess ? BS_OK : BS_ECUDA;
}

int allreduce_sum_f64(bs_ctx* c, double* buf, int64_t count) {
  if (c->size <= 1 || count == 0) return BS_OK;
  const ncclResult_t r = nccl().AllReduce(buf, buf, size_t(count), ncclFloat64, ncclSum, c->comm, c->stream);
  return r == ncclSuccess ? BS_OK : nccl_err("allreduce", r);
}

// scn m + ||beta||_1, reduced over ranks (solvers.py:436; _xbeta in solvers.py)
int cox_xbeta(bs_cox* s) {
  bs_ctx* c = s->ctx;
  int rc = bs_reduce(s->beta, s->dtype, s->n_loc, BS_SUM, BS_T_ABS, s->xb + s->m, s->ws_red, s->n_red, c->stream);
  if (rc) return rc;
  rc = bs_cox_xbeta(s->X, s->xdtype, s->beta, s->dtype, s->m, s->n_loc, s->xb, s->ws_xb, s->n_xb, c->stream);
  if (rc) return rc;
  s->xb_fresh = false;
  return allreduce_sum_f64(c, s->xb, s->m + 1);
}

bool converged(std::vector<double>& h, int window, double tol, double f) {  // solvers.py:54-70
  h.push_back(f);
  if (int(h.size()) <= window) return false;
  const double a = h.back(), b = h[h.size() - 1 - size_t(window)];
  return std::fabs(a - b) / (std::fabs(a) + 1.0) < tol;
}

}  // namespace

extern "C" int bs_nccl_unique_id(void* out128) {
  clear_error();
  if (!out128) { set_error("bs_nccl_unique_id: null output"); return BS_EINVAL; }
  if (!nccl().ok) { set_error("bs_nccl_unique_id: libnccl.so.2 not loadable"); return BS_ENCCL; }
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err("bs_nccl_unique_id", r);
  std::memcpy(out128, &id, sizeof(id));
  return BS_OK;
}

extern "C" int bs_ctx_create(int rank, int size, int device, const void* nccl_unique_id, void* stream,
                             bs_ctx_t* out) {
  clear_error();
  if (!out || size < 1 || rank < 0 || rank >= size || device < 0) {
    set_error("bs_ctx_create: bad arguments");
    return BS_EINVAL;
  }
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) { set_error("bs_ctx_create: cudaSetDevice(%d) failed", device); return BS_ECUDA; }
  bs_ctx* c = new bs_ctx{rank, size, device, as_stream(stream), nullptr};
  if (size > 1) {
    if (!nccl_unique_id) { delete c; set_error("bs_ctx_create: size > 1 needs an NCCL unique id"); return BS_EINVAL; }
    if (!nccl().ok) { delete c; set_error("bs_ctx_create: libnccl.so.2 not loadable"); return BS_ENCCL; }
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    const ncclResult_t r = nccl().CommInitRank(&c->comm, size, id, rank);
    if (r != ncclSuccess) { delete c; return nccl_err("bs_ctx_create", r); }
  }
  *out = c;
  return BS_OK;
}

extern "C" int bs_ctx_destroy(bs_ctx_t c) {
  clear_error();
  if (!c) return BS_OK;
  int rc = BS_OK;
  if (c->comm && nccl().ok) {
    const ncclResult_t r = nccl().CommDestroy(c->comm);
    if (r != ncclSuccess) rc = nccl_err("bs_ctx_destroy", r);
  }
  delete c;
  return rc;
}

extern "C" int bs_cox_state_create(bs_ctx_t ctx, const void* X, int xdtype, int dtype, int64_t m, int64_t n_loc,
                                   const void* delta, const int64_t* cuts, double lam, double sigma, void* beta,
                                   void* grad, bs_cox_t* out) {
  clear_error();
  if (!ctx || !out || m < 1 || n_loc < 0 || !delta || (dtype != BS_F32 && dtype != BS_F64) || sigma <= 0 ||
      (n_loc > 0 && (!X || !beta || !grad))) {
    set_error("bs_cox_state_create: bad arguments");
    return BS_EINVAL;
  }
  *out = nullptr;
  cudaSetDevice(ctx->device);
  bs_cox* s = new bs_cox();
  s->ctx = ctx;
  s->X = X;
  s->xdtype = xdtype;
  s->dtype = dtype;
  s->m = m;
  s->n_loc = n_loc;
  s->delta = delta;
  s->cuts = cuts;
  s->lam = lam;
  s->sigma = sigma;
  s->clamp = dtype == BS_F64 ? 700.0 : 85.0;  // solvers.py _EXP_CLAMP
  s->beta = beta;
  s->grad = grad;
  // the fused one-stream pass for float32 X with float32 arithmetic, as cox_fit's default
  s->fused = xdtype == BS_F32 && dtype == BS_F32 && ctx->size >= 1;
  const int64_t es = dtype == BS_F64 ? 8 : 4;
  s->n_xb = bs_cox_xbeta_workspace(xdtype, m, n_loc);
  s->n_risk = bs_cox_risk_workspace(m);
  s->n_pd = bs_cox_pi_delta_workspace(m);
  s->n_grad = bs_cox_grad_workspace(xdtype, m, n_loc);
  s->n_fused = s->fused ? bs_cox_grad_xbeta_workspace(xdtype, m, n_loc) : 0;
  s->n_red = bs_reduce_workspace(std::max<int64_t>(n_loc, 1));
  int rc = BS_OK;
  void* p = nullptr;
  rc |= dalloc(&p, 8 * (m + 1)); s->xb = static_cast<double*>(p);
  rc |= dalloc(&s->Xbeta, es * m);
  rc |= dalloc(&s->w, es * m);
  rc |= dalloc(&s->W, es * m);
  rc |= dalloc(&s->pd, es * m);
  rc |= dalloc(&p, 8 * m); s->dmpd = static_cast<double*>(p);
  rc |= dalloc(&p, 8); s->loglik = static_cast<double*>(p);
  rc |= dalloc(&p, 4); s->flags = static_cast<int*>(p);
  rc |= dalloc(&s->ws_xb, s->n_xb);
  rc |= dalloc(&s->ws_risk, s->n_risk);
  rc |= dalloc(&s->ws_pd, s->n_pd);
  rc |= dalloc(&s->ws_grad, s->n_grad);
  rc |= dalloc(&s->ws_fused, s->n_fused);
  rc |= dalloc(&s->ws_red, s->n_red);
  if (rc != BS_OK) {
    bs_cox_state_destroy(s);
    set_error("bs_cox_state_create: device allocation failed");
    return BS_ECUDA;
  }
  s->n_xb = std::max<int64_t>(s->n_xb, 256);
  s->n_risk = std::max<int64_t>(s->n_risk, 256);
  s->n_pd = std::max<int64_t>(s->n_pd, 256);
  s->n_grad = std::max<int64_t>(s->n_grad, 256);
  s->n_fused = std::max<int64_t>(s->n_fused, 256);
  s->n_red = std::max<int64_t>(s->n_red, 256);
  *out = s;
  return BS_OK;
}

extern "C" int bs_cox_state_destroy(bs_cox_t s) {
  clear_error();
  if (!s) return BS_OK;
  cudaSetDevice(s->ctx->device);
  void* bufs[] = {s->xb, s->Xbeta, s->w, s->W, s->pd, s->dmpd, s->loglik, s->flags,
                  s->ws_xb, s->ws_risk, s->ws_pd, s->ws_grad, s->ws_fused, s->ws_red};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete s;
  return BS_OK;
}

extern "C" int bs_cox_run(bs_cox_t s, int iters, int trace_every, int monitor_window, double monitor_tol,
                          double* trace_out, int* ntrace_out, int* iters_run, int* flags_out) {
  clear_error();
  if (!s || iters < 0 || trace_every < 0 || monitor_window < 0) { set_error("bs_cox_run: bad arguments"); return BS_EINVAL; }
  bs_ctx* c = s->ctx;
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  if (ntrace_out) *ntrace_out = 0;
  if (iters_run) *iters_run = 0;
  if (flags_out) *flags_out = 0;
  if (iters == 0) return BS_OK;
  const int64_t m = s->m;
  int rc = BS_OK;
  if (cudaMemsetAsync(s->flags, 0, sizeof(int), st) != cudaSuccess) return BS_ECUDA;
  double* trace_dev = nullptr;
  int* fhist = nullptr;
  if (cudaMalloc(&trace_dev, sizeof(double) * size_t(iters)) != cudaSuccess ||
      cudaMalloc(&fhist, sizeof(int) * size_t(iters)) != cudaSuccess) {
    cudaFree(trace_dev);
    set_error("bs_cox_run: device allocation failed");
    return BS_ECUDA;
  }
  std::vector<double> history, host_trace;
  const bool monitor = monitor_window > 0;
  const bool reuse = s->fused && s->xb_fresh;
  int ran = iters;
  auto fail = [&](int code) {
    cudaFree(trace_dev);
    cudaFree(fhist);
    return code;
  };
  if (s->fused && !reuse && (rc = cox_xbeta(s))) return fail(rc);
  for (int it = 0; it < iters; ++it) {
    if (!s->fused) {
      if ((rc = cox_xbeta(s))) return fail(rc);  // scn m + ||beta||_1 (solvers.py:436)
    } else if ((it > 0 || reuse) && (rc = allreduce_sum_f64(c, s->xb, m + 1))) {
      return fail(rc);  // the fused pass's X beta partials
    }
    if ((rc = bs_cox_risk(s->xb, s->delta, s->cuts, s->dtype, m, s->clamp, s->Xbeta, s->w, s->W, s->loglik, s->flags,
                          s->ws_risk, s->n_risk, st)))
      return fail(rc);
    cudaMemcpyAsync(fhist + it, s->flags, sizeof(int), cudaMemcpyDeviceToDevice, st);
    if (trace_every && it % trace_every == 0) {
      if ((rc = bs_cox_objective(s->loglik, s->xb + m, s->lam, trace_dev + it, st))) return fail(rc);
      if (monitor) {  // solvers.py:438-441: the monitor may stop before stepping
        double obj;
        int fl;
        cudaMemcpyAsync(&obj, trace_dev + it, sizeof(double), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&fl, s->flags, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return fail(BS_ECUDA);
        if (fl & BS_FLAG_NONFINITE) { ran = it; break; }
        host_trace.push_back(obj);
        if (converged(history, monitor_window, monitor_tol, obj)) { ran = it + 1; break; }
      }
    }
    if ((rc = bs_cox_pi_delta(s->w, s->W, s->delta, s->cuts, s->dtype, m, 0, m, s->pd, s->dmpd, s->flags, s->ws_pd,
                              s->n_pd, st)))
      return fail(rc);
    if (s->fused)
      rc = bs_cox_grad_xbeta(s->X, s->xdtype, s->dmpd, s->dtype, m, s->n_loc, s->grad, s->beta, s->sigma, s->lam, s->xb,
                             s->flags, 1, s->ws_fused, s->n_fused, st);
    else
      rc = bs_cox_grad_step(s->X, s->xdtype, s->dmpd, s->dtype, m, s->n_loc, s->grad, s->beta, s->sigma, s->lam, 1,
                            s->xb + m, s->flags, s->ws_grad, s->n_grad, st);
    if (rc) return fail(rc);
  }
  // first iteration whose risk weights went nonfinite, as cox_fit reports it
  std::vector<int> fl(size_t(std::max(ran, 1)), 0);
  std::vector<double> tr(size_t(iters), 0.0);
  int final_flags = 0;
  if (ran > 0) cudaMemcpyAsync(fl.data(), fhist, sizeof(int) * size_t(ran), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(tr.data(), trace_dev, sizeof(double) * size_t(iters), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&final_flags, s->flags, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(BS_ECUDA);
  int stop = ran;
  for (int it = 0; it < ran; ++it)
    if (fl[size_t(it)] & BS_FLAG_NONFINITE) { stop = it; break; }
  for (int it = 0; it < ran; ++it) final_flags |= fl[size_t(it)] & BS_FLAG_CLAMPED;
  if (stop < ran) final_flags |= BS_FLAG_NONFINITE;
  int nt = 0;
  if (monitor) {
    for (int it = 0, k = 0; it < stop; ++it)
      if (trace_every && it % trace_every == 0) {
        if (trace_out) trace_out[nt] = host_trace[size_t(k)];
        ++nt;
        ++k;
      }
  } else {
    for (int it = 0; it < stop; ++it)
      if (trace_every && it % trace_every == 0) {
        if (trace_out) trace_out[nt] = tr[size_t(it)];
        ++nt;
      }
  }
  s->xb_fresh = s->fused && ran == iters && !(final_flags & BS_FLAG_NONFINITE);
  if (ntrace_out) *ntrace_out = nt;
  if (iters_run) *iters_run = stop;
  if (flags_out) *flags_out = final_flags;
  fail(BS_OK);
  if (final_flags & BS_FLAG_NONFINITE) {
    set_error("bs_cox_run: nonfinite risk weights at iteration %d; rescale X or lower sigma", stop);
    return BS_ENUMERIC;
  }
  return BS_OK;
}

// ---------------------------------------------------------------------------
// NMF (solvers.py:73-185): nmf_multiplicative / nmf_apg as one native loop.  The
// reduce-scatter of scn b (distlinalg.py:251-252) and the all-gather of Vt are NCCL
// reduces / broadcasts per rank block inside one group, so uneven partition_of blocks
// need no padding.
// ---------------------------------------------------------------------------
struct bs_nmf {
  bs_ctx* ctx;
  const void* X;
  int dtype, r;
  int64_t m, n_loc, m_loc, m_lo;
  double eps;
  void* Vt;  // r x m_loc (caller)
  void* W;   // r x n_loc (caller)
  void *WXt, *P, *tmp;  // owned: r x m_loc; r x m (size > 1); r x m (size > 1)
  double *red, *scan, *VtV, *direct;  // scan: {min, sum X^2, nonfinite, scales ready, min Vt, min W}
  int* guard;                          // objective cancellation flag (bs_nmf_objective)
  void* xscale;                        // integer GEMM block scales (float32 X)
  void *ws_gram, *ws_wxt, *ws_prep, *ws_vt, *ws_w, *ws_res, *ws_red;
  int64_t n_gram, n_wxt, n_prep, n_vt, n_w, n_res, n_red;
};

namespace {

void part_of(int64_t ext, int p, int q, int64_t* lo, int64_t* hi) {  // partition_of (distarray.py:55-65)
  const int64_t base = ext / p, extra = ext % p;
  *lo = q * base + std::min<int64_t>(q, extra);
  *hi = *lo + base + (q < extra ? 1 : 0);
}

ncclDataType_t nccl_type(int dtype) { return dtype == BS_F64 ? ncclFloat64 : ncclFloat32; }

int nmf_reduce_scatter(bs_nmf* s) {  // P (r x m) summed over ranks, block q -> rank q's WXt
  bs_ctx* c = s->ctx;
  const int64_t es = s->dtype == BS_F64 ? 8 : 4;
  const NcclApi& api = nccl();
  api.GroupStart();
  for (int q = 0; q < c->size; ++q) {
    int64_t lo, hi;
    part_of(s->m, c->size, q, &lo, &hi);
    if (hi == lo) continue;
    const ncclResult_t r = api.Reduce(static_cast<char*>(s->P) + lo * s->r * es, s->WXt, size_t((hi - lo) * s->r),
                                      nccl_type(s->dtype), ncclSum, q, c->comm, c->stream);
    if (r != ncclSuccess) { api.GroupEnd(); return nccl_err("reduce-scatter", r); }
  }
  const ncclResult_t r = api.GroupEnd();
  return r == ncclSuccess ? BS_OK : nccl_err("reduce-scatter", r);
}

int nmf_allgather(bs_nmf* s) {  // Vt blocks -> tmp (r x m)
  bs_ctx* c = s->ctx;
  const int64_t es = s->dtype == BS_F64 ? 8 : 4;
  const NcclApi& api = nccl();
  api.GroupStart();
  for (int q = 0; q < c->size; ++q) {
    int64_t lo, hi;
    part_of(s->m, c->size, q, &lo, &hi);
    if (hi == lo) continue;
    const ncclResult_t r = api.Broadcast(s->Vt, static_cast<char*>(s->tmp) + lo * s->r * es, size_t((hi - lo) * s->r),
                                         nccl_type(s->dtype), q, c->comm, c->stream);
    if (r != ncclSuccess) { api.GroupEnd(); return nccl_err("all-gather", r); }
  }
  const ncclResult_t r = api.GroupEnd();
  return r == ncclSuccess ? BS_OK : nccl_err("all-gather", r);
}

int allreduce_f64(bs_ctx* c, double* buf, int64_t count, ncclRedOp_t op) {
  if (c->size <= 1 || count == 0) return BS_OK;
  const ncclResult_t r = nccl().AllReduce(buf, buf, size_t(count), ncclFloat64, op, c->comm, c->stream);
  return r == ncclSuccess ? BS_OK : nccl_err("allreduce", r);
}

}  // namespace

extern "C" int bs_nmf_state_create(bs_ctx_t ctx, const void* X, int dtype, int64_t m, int64_t n_loc, int r,
                                   double eps, void* Vt, void* W, bs_nmf_t* out) {
  clear_error();
  if (!ctx || !out || m < 1 || n_loc < 0 || r < 1 || (dtype != BS_F32 && dtype != BS_F64) ||
      (ctx->size == 1 && !Vt) || (n_loc > 0 && (!X || !W))) {
    set_error("bs_nmf_state_create: bad arguments");
    return BS_EINVAL;
  }
  *out = nullptr;
  cudaSetDevice(ctx->device);
  bs_nmf* s = new bs_nmf();
  s->ctx = ctx;
  s->X = X;
  s->dtype = dtype;
  s->r = r;
  s->m = m;
  s->n_loc = n_loc;
  s->eps = eps;
  s->Vt = Vt;
  s->W = W;
  int64_t hi;
  part_of(m, ctx->size, ctx->rank, &s->m_lo, &hi);
  s->m_loc = hi - s->m_lo;
  const int64_t es = dtype == BS_F64 ? 8 : 4;
  s->n_gram = std::max<int64_t>(bs_gram_workspace(r, n_loc), 256);
  s->n_wxt = std::max<int64_t>(bs_nmf_wxt_workspace(dtype, m, n_loc, r), 256);
  s->n_prep = std::max<int64_t>(bs_nmf_prepare_workspace(m, n_loc), 256);
  s->n_res = std::max<int64_t>(bs_nmf_residual_workspace(m, n_loc), 256);
  s->n_red = std::max<int64_t>(bs_reduce_workspace(std::max<int64_t>(r * std::max(s->m_loc, n_loc), 1)), 256);
  s->n_vt = std::max<int64_t>(bs_nmf_vt_step_workspace(r, s->m_loc), 256);
  s->n_w = std::max<int64_t>(bs_nmf_w_step_workspace(dtype, m, n_loc, r), 256);
  int rc = BS_OK;
  void* p = nullptr;
  rc |= dalloc(&s->WXt, es * r * std::max<int64_t>(s->m_loc, 1));
  if (ctx->size > 1) {
    rc |= dalloc(&s->P, es * r * m);
    rc |= dalloc(&s->tmp, es * r * m);
  } else {
    s->P = s->WXt;  // one rank: scn b lands in WXt, Vt is the full factor
    s->tmp = Vt;
  }
  rc |= dalloc(&p, 8 * (int64_t(r) * r + 1)); s->red = static_cast<double*>(p);
  rc |= dalloc(&p, 64); s->scan = static_cast<double*>(p);
  rc |= dalloc(&p, 16); s->direct = static_cast<double*>(p);
  rc |= dalloc(&p, 16); s->guard = static_cast<int*>(p);
  s->xscale = nullptr;
  if (dtype == BS_F32) rc |= dalloc(&s->xscale, std::max<int64_t>(bs_nmf_xscale_bytes(m, n_loc), 16));
  rc |= dalloc(&p, 8 * int64_t(r) * r); s->VtV = static_cast<double*>(p);
  rc |= dalloc(&s->ws_gram, s->n_gram);
  rc |= dalloc(&s->ws_wxt, s->n_wxt);
  rc |= dalloc(&s->ws_prep, s->n_prep);
  rc |= dalloc(&s->ws_res, s->n_res);
  rc |= dalloc(&s->ws_red, s->n_red);
  rc |= dalloc(&s->ws_vt, s->n_vt);
  rc |= dalloc(&s->ws_w, s->n_w);
  if (rc != BS_OK) {
    bs_nmf_state_destroy(s);
    set_error("bs_nmf_state_create: device allocation failed");
    return BS_ECUDA;
  }
  *out = s;
  return BS_OK;
}

extern "C" int bs_nmf_state_destroy(bs_nmf_t s) {
  clear_error();
  if (!s) return BS_OK;
  cudaSetDevice(s->ctx->device);
  void* bufs[] = {s->WXt,     s->red,     s->scan,    s->VtV,  s->direct, s->guard,  s->xscale,
                  s->ws_gram, s->ws_wxt, s->ws_prep, s->ws_vt, s->ws_w,   s->ws_res, s->ws_red};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (s->ctx->size > 1) {
    if (s->P) cudaFree(s->P);
    if (s->tmp) cudaFree(s->tmp);
  }
  delete s;
  return BS_OK;
}

extern "C" int bs_nmf_run(bs_nmf_t s, int algo, int iters, int trace_every, double* trace_out, int* ntrace_out) {
  clear_error();
  if (!s || iters < 0 || trace_every < 0 || (algo != BS_NMF_MU && algo != BS_NMF_APG)) {
    set_error("bs_nmf_run: bad arguments");
    return BS_EINVAL;
  }
  bs_ctx* c = s->ctx;
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  if (ntrace_out) *ntrace_out = 0;
  if (iters == 0) return BS_OK;
  const int r = s->r;
  const int64_t rr = int64_t(r) * r;
  double* trace_dev = nullptr;
  if (cudaMalloc(&trace_dev, sizeof(double) * size_t(iters)) != cudaSuccess) {
    set_error("bs_nmf_run: device allocation failed");
    return BS_ECUDA;
  }
  auto done = [&](int code) {
    cudaFree(trace_dev);
    return code;
  };
  int rc;
  // WWt of the entering W (scn d, solvers.py:151)
  if ((rc = bs_gram(s->W, s->dtype, r, s->n_loc, s->red, s->ws_gram, s->n_gram, st))) return done(rc);
  if ((rc = allreduce_f64(c, s->red, rr, ncclSum))) return done(rc);
  // the X pass of this call (_nmf_check, solvers.py:139-141): min, sum X^2, integer-GEMM scales;
  // the integer path also needs finite X and nonnegative factors (the solver keeps them so)
  if ((rc = bs_nmf_prepare(s->X, s->dtype, s->m, s->n_loc, s->scan, s->xscale, s->ws_prep, s->n_prep, st)))
    return done(rc);
  if ((rc = bs_reduce(s->Vt, s->dtype, int64_t(r) * s->m_loc, BS_MIN, BS_T_NONE, s->scan + 4, s->ws_red, s->n_red,
                      st)) ||
      (rc = bs_reduce(s->W, s->dtype, int64_t(r) * s->n_loc, BS_MIN, BS_T_NONE, s->scan + 5, s->ws_red, s->n_red,
                      st)))
    return done(rc);
  if ((rc = allreduce_f64(c, s->scan, 1, ncclMin)) || (rc = allreduce_f64(c, s->scan + 1, 1, ncclSum)) ||
      (rc = allreduce_f64(c, s->scan + 2, 1, ncclMax)) || (rc = allreduce_f64(c, s->scan + 4, 2, ncclMin)))
    return done(rc);
  double h[6];
  cudaMemcpyAsync(h, s->scan, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return done(BS_ECUDA);
  if (!(s->n_loc == 0 && c->size == 1) && h[0] < 0) {
    set_error("NMF requires nonnegative data");
    return done(BS_EINVAL);
  }
  const bool use_i8 = h[3] == 1.0 && h[2] == 0.0 && h[4] >= 0.0 && h[5] >= 0.0;
  const void* xs = use_i8 ? s->xscale : nullptr;
  // Gram-identity guard (solvers.py _KAPPA_*): float64 1e6, integer path 16, 3xTF32 always direct
  const double kappa = s->dtype == BS_F64 ? 1e6 : (use_i8 && r <= 64) ? 16.0 : -1.0;
  for (int it = 0; it < iters; ++it) {
    if ((rc = bs_nmf_wxt(s->X, s->W, s->dtype, s->m, s->n_loc, r, s->P, xs, s->ws_wxt, s->n_wxt, st)))
      return done(rc);
    if (c->size > 1 && (rc = nmf_reduce_scatter(s))) return done(rc);
    // Vt half-step (solvers.py:152-156 / 173-176)
    if ((rc = bs_nmf_vt_step(algo, s->Vt, s->WXt, s->red, s->dtype, r, s->m_loc, s->eps, s->VtV, nullptr, s->ws_vt,
                             s->n_vt, st)))
      return done(rc);
    if (c->size > 1 && ((rc = allreduce_f64(c, s->VtV, rr, ncclSum)) || (rc = nmf_allgather(s)))) return done(rc);
    // W half-step + next WWt + objective cross term (solvers.py:155-159 / 177-182)
    if ((rc = bs_nmf_w_step(algo, s->X, s->tmp, s->W, s->VtV, s->dtype, s->m, s->n_loc, r, s->eps, s->red, xs,
                            s->ws_w, s->n_w, st)))
      return done(rc);
    if ((rc = allreduce_f64(c, s->red, rr + 1, ncclSum))) return done(rc);
    if (trace_every && it % trace_every == 0) {
      if ((rc = bs_nmf_objective(s->scan + 1, s->red, s->VtV, r, trace_dev + it, s->guard, kappa, st)) ||
          (rc = bs_nmf_residual(s->X, s->tmp, s->W, s->dtype, s->m, s->n_loc, r, s->direct, s->guard, s->ws_res,
                                s->n_res, st)) ||
          (rc = allreduce_f64(c, s->direct, 1, ncclSum)) ||
          (rc = bs_nmf_objective_select(s->guard, s->direct, trace_dev + it, st)))
        return done(rc);
    }
  }
  std::vector<double> tr(size_t(iters), 0.0);
  cudaMemcpyAsync(tr.data(), trace_dev, sizeof(double) * size_t(iters), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return done(BS_ECUDA);
  int nt = 0;
  for (int it = 0; it < iters; ++it)
    if (trace_every && it % trace_every == 0) {
      if (trace_out) trace_out[nt] = tr[size_t(it)];
      ++nt;
    }
  if (ntrace_out) *ntrace_out = nt;
  return done(BS_OK);
}

// ---------------------------------------------------------------------------
// MDS (solvers.py:188-305): mds_fit as one native loop; theta is all-gathered with
// grouped NCCL broadcasts per rank block.
// ---------------------------------------------------------------------------
struct bs_mds {
  bs_ctx* ctx;
  const void* Y;
  int dtype, q, perturb;
  int64_t n, lo, n_loc;
  double wsum;
  void* theta;                 // q x n_loc (caller)
  void *full, *zsum, *T;       // owned: q x n (size > 1), n_loc, q x n_loc
  double* red;
  int* flags;
  void* ws;
  int64_t n_ws;
};

extern "C" int bs_mds_state_create(bs_ctx_t ctx, const void* Y, int dtype, int64_t n, int64_t n_loc, int q,
                                   int perturb, void* theta, bs_mds_t* out) {
  clear_error();
  if (!ctx || !out || n < 2 || n_loc < 0 || q < 1 || (dtype != BS_F32 && dtype != BS_F64) ||
      (n_loc > 0 && (!Y || !theta))) {
    set_error("bs_mds_state_create: bad arguments");
    return BS_EINVAL;
  }
  *out = nullptr;
  cudaSetDevice(ctx->device);
  bs_mds* s = new bs_mds();
  s->ctx = ctx;
  s->Y = Y;
  s->dtype = dtype;
  s->q = q;
  s->perturb = perturb ? 1 : 0;
  s->n = n;
  s->n_loc = n_loc;
  s->wsum = double(n - 1);  // W_sums (solvers.py:231)
  s->theta = theta;
  int64_t hi;
  part_of(n, ctx->size, ctx->rank, &s->lo, &hi);
  if (hi - s->lo != n_loc) {
    delete s;
    set_error("bs_mds_state_create: n_loc %lld is not this rank's partition_of(n) block", (long long)n_loc);
    return BS_EINVAL;
  }
  const int64_t es = dtype == BS_F64 ? 8 : 4;
  s->n_ws = std::max<int64_t>(bs_mds_pass_workspace(dtype, n, n_loc, q), 256);
  int rc = BS_OK;
  void* p = nullptr;
  if (ctx->size > 1) rc |= dalloc(&s->full, es * q * n);
  else s->full = theta;
  rc |= dalloc(&s->zsum, es * std::max<int64_t>(n_loc, 1));
  rc |= dalloc(&s->T, es * q * std::max<int64_t>(n_loc, 1));
  rc |= dalloc(&p, 16); s->red = static_cast<double*>(p);
  rc |= dalloc(&p, 4); s->flags = static_cast<int*>(p);
  rc |= dalloc(&s->ws, s->n_ws);
  if (rc != BS_OK) {
    bs_mds_state_destroy(s);
    set_error("bs_mds_state_create: device allocation failed");
    return BS_ECUDA;
  }
  *out = s;
  return BS_OK;
}

extern "C" int bs_mds_state_destroy(bs_mds_t s) {
  clear_error();
  if (!s) return BS_OK;
  cudaSetDevice(s->ctx->device);
  if (s->ctx->size > 1 && s->full) cudaFree(s->full);
  void* bufs[] = {s->zsum, s->T, s->red, s->flags, s->ws};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete s;
  return BS_OK;
}

extern "C" int bs_mds_run(bs_mds_t s, int iters, int trace_every, double* trace_out, int* ntrace_out) {
  clear_error();
  if (!s || iters < 0 || trace_every < 0) { set_error("bs_mds_run: bad arguments"); return BS_EINVAL; }
  bs_ctx* c = s->ctx;
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  if (ntrace_out) *ntrace_out = 0;
  if (iters == 0) return BS_OK;
  const int64_t es = s->dtype == BS_F64 ? 8 : 4;
  double* hist = nullptr;
  if (cudaMalloc(&hist, sizeof(double) * 2 * size_t(iters)) != cudaSuccess) {
    set_error("bs_mds_run: device allocation failed");
    return BS_ECUDA;
  }
  auto done = [&](int code) {
    cudaFree(hist);
    return code;
  };
  if (cudaMemsetAsync(s->flags, 0, sizeof(int), st) != cudaSuccess) return done(BS_ECUDA);
  int rc;
  for (int it = 0; it < iters; ++it) {
    if (c->size > 1) {  // all-gather theta (solvers.py:272, _theta_full)
      const NcclApi& api = nccl();
      api.GroupStart();
      for (int qr = 0; qr < c->size; ++qr) {
        int64_t lo, hi;
        part_of(s->n, c->size, qr, &lo, &hi);
        if (hi == lo) continue;
        const ncclResult_t r = api.Broadcast(s->theta, static_cast<char*>(s->full) + lo * s->q * es,
                                             size_t((hi - lo) * s->q), nccl_type(s->dtype), qr, c->comm, st);
        if (r != ncclSuccess) { api.GroupEnd(); return done(nccl_err("all-gather", r)); }
      }
      const ncclResult_t r = api.GroupEnd();
      if (r != ncclSuccess) return done(nccl_err("all-gather", r));
    }
    if ((rc = bs_mds_pass(s->Y, s->full, s->dtype, s->n, s->lo, s->n_loc, s->q, s->perturb, 0, s->red, s->zsum, s->T,
                          s->ws, s->n_ws, st)))
      return done(rc);
    if ((rc = allreduce_f64(c, s->red, 2, ncclSum))) return done(rc);
    cudaMemcpyAsync(hist + 2 * it, s->red, 2 * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if ((rc = bs_mds_update(s->theta, s->zsum, s->T, s->dtype, s->q, s->n_loc, s->wsum, s->red, s->perturb, s->flags,
                            st)))
      return done(rc);
  }
  std::vector<double> h(2 * size_t(iters));
  int fl = 0;
  cudaMemcpyAsync(h.data(), hist, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&fl, s->flags, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return done(BS_ECUDA);
  int last = iters;
  const bool failed = fl & BS_FLAG_DEGENERATE;
  if (failed)
    for (int it = 0; it < iters; ++it)
      if (h[2 * size_t(it) + 1] > 0) { last = it + 1; break; }
  int nt = 0;
  for (int it = 0; it < last; ++it)
    if (trace_every && it % trace_every == 0) {
      if (trace_out) trace_out[nt] = h[2 * size_t(it)];
      ++nt;
    }
  if (ntrace_out) *ntrace_out = nt;
  if (failed) {
    set_error("coincident embedding points; rerun with perturb=True");
    return done(BS_EDEGEN);
  }
  return done(BS_OK);
}
