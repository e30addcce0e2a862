// Conjugate gradient on the device (replaces proj/src/solver.cpp:24-108).
//
// Same recurrence, stopping rule and exit check as the reference cg_solve:
// x0 = 0, stop when |r|/|b| < tol (recurrence residual), recompute the true
// residual |A x - b|/|b| at exit, NonConvergence past max_iterations. All
// scalars live on the device (CgState); one iteration is
//
//   p_update : x += alpha p ; p = r + beta p      (x update deferred by one step)
//   operator : q = M p with |q|^2 = <p, A p> from the Dslash epilogue   [fused]
//              or Ap = op(p) followed by dot(p, Ap)                     [callback]
//   alpha    : rr / pAp                              (1-thread kernel)
//   update   : r -= alpha A p, |r|^2 — fused into the last Dslash epilogue, so
//              A p is never written [fused], or a streaming kernel [callback]
//   end      : rel = sqrt(rr')/|b|, history, convergence, beta, rr <- rr'
//
// With one rank the whole loop is captured once into a CUDA graph with a
// device-side while node (cudaGraphSetConditional from the `end` kernel), so a
// solve is a single graph launch with no host round trips. With several ranks
// the scalars are summed by the transport (NCCL allreduce) before `alpha` and
// `end`, and the host polls the converged flag once per iteration.
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <cmath>
#include <cstring>
#include <functional>
#include <list>
#include <map>
#include <string>

#include "objects.hpp"

using namespace lbcu;

namespace {

constexpr int kSlotPap = 8, kSlotRR = 10, kSlotB2 = 12, kSlotTrue = 14;
constexpr int kSlotR = 0, kSlotP = 1, kSlotQ = 2, kSlotT = 3, kSlotAp = 4, kSlotTmp2 = 5, kSlotS = 6, kSlotW = 7;
constexpr int kSlotGD = 16;  // single-reduction CG: (gamma, delta) side by side

struct Fused {
  enum Kind { H, EO } kind;
  const lbcu_gauge_s* g;
  double mass;
};

void ensure_hist(lbcu_ctx_s* ctx, long long n) {
  if (ctx->hist_cap >= n) return;
  if (ctx->dhist) LBCU_CUDA(cudaFree(ctx->dhist));
  ctx->dhist = nullptr;
  LBCU_CUDA(cudaMalloc(&ctx->dhist, sizeof(double) * n));
  ctx->hist_cap = n;
}

double* slot(lbcu_ctx_s* ctx, int k) { return ctx->dscal + k; }

// One fused iteration body (everything stream-ordered on ctx->stream).
void fused_body(lbcu_ctx_s* ctx, const Fused& F, lbcu_spinor_s* x, lbcu_spinor_s* r,
                lbcu_spinor_s* p, lbcu_spinor_s* q, lbcu_spinor_s* t, unsigned long long handle,
                int use_graph) {
  Transport* T = ctx->world->t.get();
  const double A = 4.0 + F.mass;
  // one rank: alpha and the end-of-iteration step run in the last block of
  // the reductions that produce pAp and rr' (two launches fewer per iteration)
  const bool fuse = T->nranks() == 1 && std::getenv("LBCU_CG_FUSE_SCALARS") == nullptr;
  auto scalar_alpha = [&](HopCall& h) {
    if (fuse) {
      h.post = POST_ALPHA;
      return;
    }
  };
  auto scalar_end = [&](HopCall& h) {
    if (fuse) {
      h.post = POST_END;
      h.handle = handle;
      h.use_graph = use_graph;
    }
  };
  auto after_pap = [&] {
    if (fuse) return;
    T->allreduce(ctx->rank, slot(ctx, kSlotPap), 1, ctx->stream);
    cg_scalar_alpha(ctx, slot(ctx, kSlotPap));
  };
  cg_p_update(ctx, p, r, x);
  if (F.kind == Fused::EO) {
    HopCall a;  // t_o = H_oe p_e
    a.in = p;
    a.out = t;
    a.g = F.g;
    a.out_parity = 1;
    hop_apply(ctx, a);
    HopCall b;  // q_e = Mhat p_e = A p - H_eo t / 4A ; |q|^2
    b.in = t;
    b.out = q;
    b.x = p;
    b.g = F.g;
    b.out_parity = 0;
    b.a = A;
    b.b = -1.0 / (4.0 * A);
    b.epi = EPI_STORE_NORM;
    b.result = slot(ctx, kSlotPap);
    scalar_alpha(b);
    hop_apply(ctx, b);
    after_pap();
    HopCall c;  // t_o = H_oe g5 q
    c.in = q;
    c.out = t;
    c.g = F.g;
    c.out_parity = 1;
    c.s5in = -1.0;
    hop_apply(ctx, c);
    HopCall d;  // Ap = g5 Mhat g5 q ; r -= alpha Ap ; |r|^2
    d.in = t;
    d.out = q;  // unused by EPI_CG
    d.x = q;
    d.r = r;
    d.g = F.g;
    d.out_parity = 0;
    d.a = A;
    d.b = -1.0 / (4.0 * A);
    d.s5acc = -1.0;
    d.epi = EPI_CG;
    d.alpha = &ctx->dcg->alpha;
    d.result = slot(ctx, kSlotRR);
    scalar_end(d);
    hop_apply(ctx, d);
  } else {
    HopCall a;  // q = D p ; |q|^2 = <p, D^dag D p>
    a.in = p;
    a.out = q;
    a.x = p;
    a.g = F.g;
    a.out_parity = 2;
    a.a = A;
    a.b = -0.5;
    a.epi = EPI_STORE_NORM;
    a.result = slot(ctx, kSlotPap);
    scalar_alpha(a);
    hop_apply(ctx, a);
    after_pap();
    HopCall b;  // Ap = g5 D g5 q ; r -= alpha Ap ; |r|^2
    b.in = q;
    b.out = q;  // unused by EPI_CG (in == out is never written)
    b.x = q;
    b.r = r;
    b.g = F.g;
    b.out_parity = 2;
    b.a = A;
    b.b = -0.5;
    b.s5in = -1.0;
    b.s5acc = -1.0;
    b.epi = EPI_CG;
    b.alpha = &ctx->dcg->alpha;
    b.result = slot(ctx, kSlotRR);
    scalar_end(b);
    hop_apply(ctx, b);
  }
  if (fuse) return;
  T->allreduce(ctx->rank, slot(ctx, kSlotRR), 1, ctx->stream);
  cg_scalar_end(ctx, slot(ctx, kSlotRR), handle, use_graph);
}

// w = A v with delta = (v, A v) = |M v|^2 from the first operator's epilogue
// (A = Mhat^dag Mhat or D^dag D, the dagger as g5 M g5), written to *delta.
void apply_a_delta(lbcu_ctx_s* ctx, const Fused& F, lbcu_spinor_s* v, lbcu_spinor_s* q, lbcu_spinor_s* t,
                   lbcu_spinor_s* w, double* delta) {
  const double A = 4.0 + F.mass;
  if (F.kind == Fused::EO) {
    HopCall a;  // t_o = H_oe v_e
    a.in = v;
    a.out = t;
    a.g = F.g;
    a.out_parity = 1;
    hop_apply(ctx, a);
    HopCall b;  // q_e = Mhat v ; |q|^2
    b.in = t;
    b.out = q;
    b.x = v;
    b.g = F.g;
    b.out_parity = 0;
    b.a = A;
    b.b = -1.0 / (4.0 * A);
    b.epi = EPI_STORE_NORM;
    b.result = delta;
    hop_apply(ctx, b);
    HopCall c;  // t_o = H_oe g5 q
    c.in = q;
    c.out = t;
    c.g = F.g;
    c.out_parity = 1;
    c.s5in = -1.0;
    hop_apply(ctx, c);
    HopCall d;  // w = g5 Mhat g5 q
    d.in = t;
    d.out = w;
    d.x = q;
    d.g = F.g;
    d.out_parity = 0;
    d.a = A;
    d.b = -1.0 / (4.0 * A);
    d.s5acc = -1.0;
    hop_apply(ctx, d);
  } else {
    HopCall a;  // q = D v ; |q|^2
    a.in = v;
    a.out = q;
    a.x = v;
    a.g = F.g;
    a.out_parity = 2;
    a.a = A;
    a.b = -0.5;
    a.epi = EPI_STORE_NORM;
    a.result = delta;
    hop_apply(ctx, a);
    HopCall b;  // w = g5 D g5 q
    b.in = q;
    b.out = w;
    b.x = q;
    b.g = F.g;
    b.out_parity = 2;
    b.a = A;
    b.b = -0.5;
    b.s5in = -1.0;
    b.s5acc = -1.0;
    hop_apply(ctx, b);
  }
}

// One single-reduction iteration (Chronopoulos & Gear 1989): the same
// iterates and stopping rule as the reference recurrence in exact
// arithmetic, but |r|^2 and (r, A r) are summed across ranks in ONE
// allreduce per iteration instead of two (pAp, then rr), at the price of two
// more streamed vectors (s = A p, w = A r). For multi-rank runs whose local
// volume is small enough that the allreduce latency outweighs that traffic.
void cg1_body(lbcu_ctx_s* ctx, const Fused& F, lbcu_spinor_s* x, lbcu_spinor_s* r, lbcu_spinor_s* p,
              lbcu_spinor_s* q, lbcu_spinor_s* t, lbcu_spinor_s* sv, lbcu_spinor_s* w) {
  double* gd = slot(ctx, kSlotGD);
  cg1_update(ctx, p, sv, x, r, w, gd);             // gamma' = |r'|^2
  apply_a_delta(ctx, F, r, q, t, w, gd + 1);       // w' = A r', delta' = (r', A r')
  ctx->world->t->allreduce(ctx->rank, gd, 2, ctx->stream);
  cg1_scalar_end(ctx, gd);
}

bool single_reduce(const lbcu_ctx_s* ctx, int dr) {
  const char* e = std::getenv("LBCU_CG_SINGLE_REDUCE");
  if (e && e[0] == '1') return true;
  if (e && e[0] == '0') return false;
  // auto: two streamed vectors more per iteration (4 passes of a parity
  // field, 256 dr B per even site) against one ~15-20 us allreduce fewer at
  // ~6.5 TB/s: worth it below ~5e5 dr-weighted sites per rank
  return ctx->geo.nranks > 1 && static_cast<double>(ctx->geo.vh) * dr < 5e5;
}

void callback_body(lbcu_ctx_s* ctx, lbcu_linop op, void* user, lbcu_spinor_s* x, lbcu_spinor_s* r,
                   lbcu_spinor_s* p, lbcu_spinor_s* ap) {
  Transport* T = ctx->world->t.get();
  cg_p_update(ctx, p, r, x);
  const int rc = op(user, ap, p);
  if (rc != 0) throw Error(rc, std::string("linear operator callback failed: ") + lbcu_last_error());
  blas_dot(ctx, p, ap, slot(ctx, kSlotPap));
  T->allreduce(ctx->rank, slot(ctx, kSlotPap), 2, ctx->stream);
  cg_scalar_alpha(ctx, slot(ctx, kSlotPap));
  cg_r_update(ctx, r, ap, slot(ctx, kSlotRR));
  T->allreduce(ctx->rank, slot(ctx, kSlotRR), 1, ctx->stream);
  cg_scalar_end(ctx, slot(ctx, kSlotRR), 0, 0);
}

// Graph cache: one instantiated while-loop per context, fused problem and
// field set. The key holds the handles AND the device state the captured
// kernels bake in (base pointers, link storage format), and every entry that
// names a handle is dropped (cudaGraphExecDestroy) when that handle is
// destroyed or its links are re-uploaded (graph_cache_forget, called from
// api.cpp) and when the context is destroyed (graph_cache_clear): a replay
// can never see freed memory or a stale kernel specialisation, even when a
// new handle is allocated at a recycled address.
struct GraphKey {
  int kind, fmt;
  const void *g, *x, *r, *p, *q, *t;              // handles
  const void *gb, *xb, *rb, *pb, *qb, *tb;        // device bases
  double mass;
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
  bool names(const void* h) const { return g == h || x == h || r == h || p == h || q == h || t == h; }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec;
  long long body_kernels;
};
std::mutex g_graph_mu;
std::map<const lbcu_ctx_s*, std::list<GraphEntry>> g_graphs;  // node-stable per context
constexpr size_t kMaxGraphsPerCtx = 16;

bool graphs_enabled() {
  const char* e = std::getenv("LBCU_CG_GRAPH");
  return !(e && e[0] == '0');
}

// Returned by value: the cache may be pruned by another thread afterwards.
GraphEntry graph_for(lbcu_ctx_s* ctx, const Fused& F, lbcu_spinor_s* x, lbcu_spinor_s* r,
                     lbcu_spinor_s* p, lbcu_spinor_s* q, lbcu_spinor_s* t) {
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.kind = F.kind;
  key.fmt = F.g->fmt;
  key.g = F.g;
  key.x = x;
  key.r = r;
  key.p = p;
  key.q = q;
  key.t = t;
  key.gb = F.g->base;
  key.xb = x->base;
  key.rb = r->base;
  key.pb = p->base;
  key.qb = q->base;
  key.tb = t->base;
  key.mass = F.mass;
  std::lock_guard<std::mutex> lk(g_graph_mu);
  auto& list = g_graphs[ctx];
  for (auto it = list.begin(); it != list.end(); ++it)
    if (it->key == key) {
      list.splice(list.begin(), list, it);  // most recently used first
      return list.front();
    }
  cudaGraph_t graph;
  LBCU_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  LBCU_CUDA(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  LBCU_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const long long before = ctx->launches;
  LBCU_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
  try {
    fused_body(ctx, F, x, r, p, q, t, static_cast<unsigned long long>(handle), 1);
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(ctx->stream, &dummy);
    cudaGraphDestroy(graph);
    throw;
  }
  LBCU_CUDA(cudaStreamEndCapture(ctx->stream, &body));
  GraphEntry e;
  e.key = key;
  e.body_kernels = ctx->launches - before;
  ctx->launches = before;  // captured, not launched
  LBCU_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
  LBCU_CUDA(cudaGraphDestroy(graph));
  list.push_front(e);
  while (list.size() > kMaxGraphsPerCtx) {  // least recently used
    LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaGraphExecDestroy(list.back().exec);
    list.pop_back();
  }
  return e;
}

void check_settings(const lbcu_cg_settings* s) {  // solver.cpp:26-28
  if (!s) throw Error(LBCU_CONTRACT_VIOLATION, "cg: null settings");
  if (!(s->tolerance > 0.0 && s->tolerance < 1.0))
    throw Error(LBCU_CONFIG_ERROR, "cg tolerance must lie in (0, 1)");
  if (s->max_iterations < 1) throw Error(LBCU_CONFIG_ERROR, "cg max iterations must be >= 1");
}

double read_b2(lbcu_ctx_s* ctx, const lbcu_spinor_s* rhs) {
  blas_sqnorm(ctx, rhs, slot(ctx, kSlotB2));
  ctx->world->t->allreduce(ctx->rank, slot(ctx, kSlotB2), 1, ctx->stream);
  LBCU_CUDA(cudaMemcpyAsync(ctx->hscal + kSlotB2, slot(ctx, kSlotB2), sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  return ctx->hscal[kSlotB2];
}

// Shared driver. apply(out, in) computes A for the true residual.
int run_cg(lbcu_ctx_s* ctx, const lbcu_cg_settings* st, lbcu_spinor_s* rhs, lbcu_spinor_s* x,
           lbcu_cg_outcome* outc, double* history, const Fused* fused, lbcu_linop op,
           void* user, const std::function<void(lbcu_spinor_s*, lbcu_spinor_s*)>& apply) {
  check_settings(st);
  if (!x || !rhs || x->ctx != ctx || rhs->ctx != ctx || x->dr != rhs->dr || x->subset != rhs->subset)
    throw Error(LBCU_CONTRACT_VIOLATION, "cg: rhs and x disagree on context, dr or subset");
  if (x == rhs) throw Error(LBCU_CONTRACT_VIOLATION, "cg: solution must not alias rhs");
  lbcu_cg_outcome out{};
  const int dr = rhs->dr, sub = rhs->subset;
  lbcu_spinor_s* r = scratch_spinor(ctx, dr, sub, 200 + kSlotR);
  lbcu_spinor_s* p = scratch_spinor(ctx, dr, sub, 200 + kSlotP);
  lbcu_spinor_s* q = scratch_spinor(ctx, dr, sub, 200 + kSlotQ);
  lbcu_spinor_s* t = scratch_spinor(ctx, dr, LBCU_ODD, 200 + kSlotT);
  ensure_hist(ctx, st->max_iterations + 1);

  const bool use_graph = fused && ctx->world->t->capturable() && ctx->geo.nranks == 1 && graphs_enabled() &&
                         !(std::getenv("LBCU_CG_SINGLE_REDUCE") && std::getenv("LBCU_CG_SINGLE_REDUCE")[0] == '1');
  GraphEntry ge{};
  if (use_graph) {  // capture + instantiate (first solve on these fields) outside the timed region
    if (fused->kind == Fused::EO) {  // make sure lazily allocated buffers exist before capture
      (void)scratch_spinor(ctx, dr, LBCU_ODD, 200 + kSlotT);
    }
    ge = graph_for(ctx, *fused, x, r, p, q, t);
  }
  const bool cg1 = fused && !use_graph && single_reduce(ctx, dr);
  lbcu_spinor_s* sv = cg1 ? scratch_spinor(ctx, dr, sub, 200 + kSlotS) : nullptr;  // allocated untimed
  lbcu_spinor_s* w = cg1 ? scratch_spinor(ctx, dr, sub, 200 + kSlotW) : nullptr;

  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->world->t->barrier(ctx->rank);  // solver.cpp:36
  LBCU_CUDA(cudaEventRecord(ctx->ev[14], ctx->stream));
  blas_zero(ctx, x);
  const double b2 = read_b2(ctx, rhs);
  if (b2 == 0.0) {  // solver.cpp:40: x = 0, zero iterations
    if (outc) *outc = out;
    return LBCU_OK;
  }
  blas_copy(ctx, r, rhs);
  blas_zero(ctx, p);
  cg_scalar_init(ctx, slot(ctx, kSlotB2), st->tolerance, st->max_iterations);
  if (cg1) {  // s = 0 ; w = A b, delta_0 = (b, A b) ; gamma_0 = |b|^2 (already summed)
    blas_zero(ctx, sv);
    double* gd = slot(ctx, kSlotGD);
    apply_a_delta(ctx, *fused, r, q, t, w, gd + 1);
    ctx->world->t->allreduce(ctx->rank, gd + 1, 1, ctx->stream);
    LBCU_CUDA(cudaMemcpyAsync(gd, slot(ctx, kSlotB2), sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    cg1_scalar_start(ctx, gd);
  }

  if (use_graph) {
    LBCU_CUDA(cudaGraphLaunch(ge.exec, ctx->stream));
    LBCU_CUDA(cudaMemcpyAsync(ctx->hcg, ctx->dcg, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
    LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->launches += ge.body_kernels * ctx->hcg->k;
  } else if (fused) {
    // host loop one iteration ahead: iteration k + 1 is enqueued before the
    // state of iteration k is read back, so the device never idles on the
    // host round trip; a speculative iteration after convergence is a no-op
    // on x, p and the state (device.cuh: cg_post_*; blas.cu: k_cg_p)
    for (int e = 0; e < 2; ++e)
      if (!ctx->ev_cg[e]) LBCU_CUDA(cudaEventCreateWithFlags(&ctx->ev_cg[e], cudaEventDisableTiming));
    for (int k = 0; k < st->max_iterations; ++k) {
      if (cg1) cg1_body(ctx, *fused, x, r, p, q, t, sv, w);
      else fused_body(ctx, *fused, x, r, p, q, t, 0, 0);
      CgState* h = ctx->hcg + 1 + (k & 1);
      LBCU_CUDA(cudaMemcpyAsync(h, ctx->dcg, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
      LBCU_CUDA(cudaEventRecord(ctx->ev_cg[k & 1], ctx->stream));
      if (k == 0) continue;
      LBCU_CUDA(cudaEventSynchronize(ctx->ev_cg[(k - 1) & 1]));
      if (ctx->hcg[1 + ((k - 1) & 1)].done) break;
    }
    LBCU_CUDA(cudaMemcpyAsync(ctx->hcg, ctx->dcg, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
    LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    for (int k = 0; k < st->max_iterations; ++k) {  // the callback runs exactly once per iteration
      callback_body(ctx, op, user, x, r, p, q);
      LBCU_CUDA(cudaMemcpyAsync(ctx->hcg, ctx->dcg, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
      LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
      if (ctx->hcg->done) break;
    }
  }
  const CgState cs = *ctx->hcg;
  out.iterations = cs.k;
  out.rel_residual = cs.rel;
  out.best_residual = cs.best;
  if (history && cs.k > 0)
    LBCU_CUDA(cudaMemcpy(history, ctx->dhist, sizeof(double) * cs.k, cudaMemcpyDeviceToHost));
  if (!cs.conv) {
    if (outc) *outc = out;
    throw Error(LBCU_NON_CONVERGENCE, "cg failed to converge after " + std::to_string(cs.k) +
                                          " iterations, best relative residual " +
                                          std::to_string(cs.best));
  }
  if (!cg1) cg_x_final(ctx, x, p);  // the single-reduction update keeps x current
  // true residual from scratch (solver.cpp:74-76)
  lbcu_spinor_s* ap = scratch_spinor(ctx, dr, sub, 200 + kSlotAp);
  apply(ap, x);
  blas_axpy(ctx, ap, -1.0, 0.0, rhs);
  blas_sqnorm(ctx, ap, slot(ctx, kSlotTrue));
  ctx->world->t->allreduce(ctx->rank, slot(ctx, kSlotTrue), 1, ctx->stream);
  LBCU_CUDA(cudaEventRecord(ctx->ev[15], ctx->stream));
  LBCU_CUDA(cudaMemcpyAsync(ctx->hscal + kSlotTrue, slot(ctx, kSlotTrue), sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  out.true_rel_residual = std::sqrt(ctx->hscal[kSlotTrue]) / std::sqrt(b2);
  float ms = 0.f;
  LBCU_CUDA(cudaEventElapsedTime(&ms, ctx->ev[14], ctx->ev[15]));
  out.seconds = ms * 1e-3;
  if (outc) *outc = out;
  return LBCU_OK;
}

thread_local std::string tl_err;

int guard(const std::function<int()>& f) {
  try {
    return f();
  } catch (const Error& e) {
    tl_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    tl_err = e.what();
    return LBCU_CONTRACT_VIOLATION;
  }
}

}  // namespace

namespace lbcu {

void graph_cache_forget(const lbcu_ctx_s* ctx, const void* handle) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  auto it = g_graphs.find(ctx);
  if (it == g_graphs.end()) return;
  for (auto e = it->second.begin(); e != it->second.end();) {
    if (e->key.names(handle)) {
      cudaGraphExecDestroy(e->exec);
      e = it->second.erase(e);
    } else {
      ++e;
    }
  }
}

void graph_cache_clear(const lbcu_ctx_s* ctx) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  auto it = g_graphs.find(ctx);
  if (it == g_graphs.end()) return;
  for (auto& e : it->second) cudaGraphExecDestroy(e.exec);
  g_graphs.erase(it);
}

size_t graph_cache_size(const lbcu_ctx_s* ctx) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  auto it = g_graphs.find(ctx);
  return it == g_graphs.end() ? 0 : it->second.size();
}

}  // namespace lbcu

// api.cpp owns lbcu_last_error(); solver errors are forwarded into it.
extern "C" int lbcu_internal_set_error(const char* msg);

extern "C" {

int lbcu_cg_solve(lbcu_ctx c, lbcu_linop op, void* user, lbcu_spinor rhs, lbcu_spinor x,
                  const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome, double* history) {
  const int rc = guard([&] {
    if (!c || !op) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve: null context or operator");
    LBCU_CUDA(cudaSetDevice(c->device));
    return run_cg(c, settings, rhs, x, outcome, history, nullptr, op, user,
                  [&](lbcu_spinor_s* out, lbcu_spinor_s* in) {
                    const int r = op(user, out, in);
                    if (r != 0) throw Error(r, "linear operator callback failed");
                  });
  });
  if (rc != LBCU_OK) lbcu_internal_set_error(tl_err.c_str());
  return rc;
}

int lbcu_cg_solve_h(lbcu_gauge g, double mass, lbcu_spinor rhs, lbcu_spinor x,
                    const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome, double* history) {
  const int rc = guard([&] {
    if (!g || !rhs) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_h: null argument");
    if (rhs->subset != LBCU_FULL) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_h: needs FULL fields");
    if (g->dr != rhs->dr) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_h: representation mismatch");
    lbcu_ctx_s* ctx = rhs->ctx;
    LBCU_CUDA(cudaSetDevice(ctx->device));
    Fused F{Fused::H, g, mass};
    return run_cg(ctx, settings, rhs, x, outcome, history, &F, nullptr, nullptr,
                  [&](lbcu_spinor_s* out, lbcu_spinor_s* in) {
                    if (lbcu_h(out, g, in, mass) != 0) throw Error(LBCU_CUDA_ERROR, lbcu_last_error());
                  });
  });
  if (rc != LBCU_OK) lbcu_internal_set_error(tl_err.c_str());
  return rc;
}

int lbcu_cg_solve_eo(lbcu_gauge g, double mass, lbcu_spinor rhs, lbcu_spinor x,
                     const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome, double* history) {
  const int rc = guard([&] {
    if (!g || !rhs) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_eo: null argument");
    if (rhs->subset != LBCU_EVEN) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_eo: needs EVEN fields");
    if (g->dr != rhs->dr) throw Error(LBCU_CONTRACT_VIOLATION, "cg_solve_eo: representation mismatch");
    lbcu_ctx_s* ctx = rhs->ctx;
    LBCU_CUDA(cudaSetDevice(ctx->device));
    Fused F{Fused::EO, g, mass};
    return run_cg(ctx, settings, rhs, x, outcome, history, &F, nullptr, nullptr,
                  [&](lbcu_spinor_s* out, lbcu_spinor_s* in) {
                    if (lbcu_mhat_dag_mhat(out, g, in, mass) != 0)
                      throw Error(LBCU_CUDA_ERROR, lbcu_last_error());
                  });
  });
  if (rc != LBCU_OK) lbcu_internal_set_error(tl_err.c_str());
  return rc;
}

}  // extern "C"
