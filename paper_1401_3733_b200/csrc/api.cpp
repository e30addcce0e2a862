// C-ABI entry points (include/lbcu.h). Every function converts exceptions to
// status codes + a thread-local message, mirroring the reference's exception
// taxonomy (proj/include/latbench/errors.hpp:9-63).
#include <cstring>
#include <string>
#include <thread>

#include "objects.hpp"

using namespace lbcu;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define API_BEGIN try {
#define API_END                                      \
  }                                                  \
  catch (const lbcu::Error& e) {                     \
    return fail(e.code, e.what());                   \
  }                                                  \
  catch (const std::exception& e) {                  \
    return fail(LBCU_CONTRACT_VIOLATION, e.what());  \
  }                                                  \
  return LBCU_OK;

void need(bool ok, const char* what) {
  if (!ok) throw Error(LBCU_CONTRACT_VIOLATION, what);
}

void bind(lbcu_ctx_s* c) { LBCU_CUDA(cudaSetDevice(c->device)); }

void check_pair(const lbcu_spinor_s* a, const lbcu_spinor_s* b, const char* who) {
  need(a && b, who);
  if (a->ctx != b->ctx || a->dr != b->dr || a->subset != b->subset)
    throw Error(LBCU_CONTRACT_VIOLATION,
                std::string(who) + ": spinor fields disagree on context, dr or subset");
}

void check_dirac(const lbcu_spinor_s* out, const lbcu_gauge_s* g, const lbcu_spinor_s* in,
                 const char* who) {  // kernels.cpp:15-21
  need(out && g && in, who);
  if (out->ctx != in->ctx || g->ctx != in->ctx)
    throw Error(LBCU_CONTRACT_VIOLATION, std::string(who) + ": geometry mismatch");
  if (g->dr != in->dr || out->dr != in->dr)
    throw Error(LBCU_CONTRACT_VIOLATION,
                std::string(who) + ": gauge and spinor representations disagree");
  if (out == in) throw Error(LBCU_CONTRACT_VIOLATION, std::string(who) + ": output must not alias input");
}

lbcu_spinor_s* new_spinor(lbcu_ctx_s* ctx, int dr, int subset) {
  if (dr < 1) throw Error(LBCU_CONFIG_ERROR, "spinor dr must be >= 1");
  if (subset < LBCU_FULL || subset > LBCU_ODD) throw Error(LBCU_CONFIG_ERROR, "bad subset");
  auto* s = new lbcu_spinor_s;
  s->ctx = ctx;
  s->dr = dr;
  s->subset = subset;
  const int npar = subset == LBCU_FULL ? 2 : 1;
  const size_t blk = static_cast<size_t>(4 * dr) * ctx->geo.stride;
  s->elems = blk * npar;
  cudaError_t e = cudaMalloc(&s->base, s->elems * sizeof(double2));
  if (e != cudaSuccess) {
    delete s;
    throw Error(LBCU_CUDA_ERROR, std::string("spinor allocation failed: ") + cudaGetErrorString(e));
  }
  LBCU_CUDA(cudaMemsetAsync(s->base, 0, s->elems * sizeof(double2), ctx->stream));
  if (subset == LBCU_FULL) {
    s->par[0] = s->base;
    s->par[1] = s->base + blk;
  } else {
    s->par[subset == LBCU_EVEN ? 0 : 1] = s->base;
  }
  return s;
}

void free_spinor(lbcu_spinor_s* s) {
  if (!s) return;
  if (s->base) cudaFree(s->base);
  delete s;
}

// Mhat and friends need temporaries of the opposite parity.
constexpr int kSlotTmp = 100;

}  // namespace

namespace lbcu {

lbcu_spinor_s* scratch_spinor(lbcu_ctx_s* ctx, int dr, int subset, int slot) {
  auto key = std::make_tuple(dr, subset, slot);
  auto it = ctx->scratch.find(key);
  if (it != ctx->scratch.end()) return it->second;
  lbcu_spinor_s* s = new_spinor(ctx, dr, subset);
  ctx->scratch[key] = s;
  return s;
}

}  // namespace lbcu

// ===================================================================== ABI
extern "C" {

const char* lbcu_last_error(void) { return g_last_error.c_str(); }
int lbcu_abi_version(void) { return LBCU_ABI_VERSION; }

int lbcu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

long long lbcu_flops_per_site(int kernel, int dr, int real_rep) {  // flops.cpp:14-25
  const long long d = dr;
  switch (kernel) {
    case LBCU_KERNEL_SQNORM: return 16 * d;
    case LBCU_KERNEL_MULADD: return 32 * d;
    case LBCU_KERNEL_DIRAC: return 8 * (4 * d + 2 * d * d * (real_rep ? 4 : 8) + 8 * d) + 24 * d;
  }
  return 0;
}

int lbcu_rep_dim(int rep, int n, int* dr, int* real_links) {
  API_BEGIN
  *dr = rep_dim(rep, n);
  *real_links = rep == LBCU_REP_ADJOINT;
  API_END
}

int lbcu_check_geometry(const int global[4], const int grid[4], int rank, int enforce_floor,
                        int local_out[4]) {
  API_BEGIN
  const Geometry g = build_geometry(global, grid, rank, enforce_floor != 0);
  if (local_out)
    for (int d = 0; d < 4; ++d) local_out[d] = g.local[d];
  API_END
}

int lbcu_host_spinor_random(const int global[4], const int grid[4], int rank, int dr, uint64_t seed,
                            uint64_t field_index, double* out) {
  API_BEGIN
  const Geometry g = build_geometry(global, grid, rank, false);
  need(out != nullptr && dr >= 1, "lbcu_host_spinor_random: bad arguments");
  host_spinor_random(g, dr, seed, field_index, out);
  API_END
}

int lbcu_host_gauge_random(const int global[4], const int grid[4], int rank, int group_rank, int rep,
                           int links, uint64_t seed, double eps, int nthreads, double* out) {
  API_BEGIN
  const Geometry g = build_geometry(global, grid, rank, false);
  need(out != nullptr, "lbcu_host_gauge_random: null output");
  if (links < LBCU_LINKS_UNIT || links > LBCU_LINKS_NEAR_UNIT)
    throw Error(LBCU_CONFIG_ERROR, "unknown link generator");
  host_gauge_random(g, group_rank, rep, links, seed, eps, nthreads, out);
  API_END
}

int lbcu_plan_faces(const int global[4], const int grid[4], int rank, int input_parity,
                    int partner[8], int count[8], int32_t* sites) {
  API_BEGIN
  const Geometry g = build_geometry(global, grid, rank, false);
  const FacePlan p = plan_faces(g);
  int64_t off = 0;
  for (int f = 0; f < 8; ++f) {
    partner[f] = p.partner[f];
    count[f] = static_cast<int>(p.count[f]);
    if (sites)
      for (int64_t j = 0; j < p.count[f]; ++j)
        sites[off + j] = static_cast<int32_t>(face_site(g, f, input_parity & 1, j));
    off += p.count[f];
  }
  API_END
}

// ---- worlds ---------------------------------------------------------------
int lbcu_world_single(lbcu_world* out) {
  API_BEGIN
  auto* w = new lbcu_world_s;
  w->t = make_single_transport();
  *out = w;
  API_END
}

int lbcu_world_threads(int nranks, lbcu_world* out) {
  API_BEGIN
  auto* w = new lbcu_world_s;
  w->t = make_thread_transport(nranks);
  *out = w;
  API_END
}

int lbcu_world_threads_direct(int nranks, lbcu_world* out) {
  API_BEGIN
  auto* w = new lbcu_world_s;
  w->t = make_thread_transport(nranks, true);
  *out = w;
  API_END
}

int lbcu_world_ipc(int nranks, int rank, const char* name, const unsigned char* nccl_id, lbcu_world* out) {
  API_BEGIN
  need(out != nullptr, "lbcu_world_ipc: null output");
  auto* w = new lbcu_world_s;
  try {
    w->t = make_ipc_transport(nranks, rank, name, nccl_id);
  } catch (...) {
    delete w;
    throw;
  }
  *out = w;
  API_END
}

int lbcu_world_set_direct(lbcu_world w, int on) {
  API_BEGIN
  need(w != nullptr, "lbcu_world_set_direct: null world");
  w->t->set_direct(on != 0);
  API_END
}

int lbcu_nccl_unique_id(unsigned char id[128]) {
  API_BEGIN
  nccl_unique_id(id);
  API_END
}

int lbcu_world_nccl(int nranks, int rank, const unsigned char id[128], lbcu_world* out) {
  API_BEGIN
  auto* w = new lbcu_world_s;
  try {
    w->t = make_nccl_transport(nranks, rank, id);
  } catch (...) {
    delete w;
    throw;
  }
  *out = w;
  API_END
}

int lbcu_world_destroy(lbcu_world w) {
  API_BEGIN
  delete w;
  API_END
}

// ---- contexts ---------------------------------------------------------------
int lbcu_ctx_create(lbcu_world w, int rank, int device, const int global[4], const int grid[4],
                    int enforce_floor, lbcu_ctx* out) {
  API_BEGIN
  need(out != nullptr, "lbcu_ctx_create: null output");
  auto ctx = std::make_unique<lbcu_ctx_s>();
  ctx->geo = build_geometry(global, grid, rank, enforce_floor != 0);
  if (!w) {
    w = new lbcu_world_s;
    w->t = make_single_transport();
    ctx->owns_world = true;
  }
  ctx->world = w;
  if (w->t->nranks() != ctx->geo.nranks) {
    if (ctx->owns_world) delete w;
    throw Error(LBCU_CONTRACT_VIOLATION, "world size does not match the configured grid");
  }
  ctx->rank = rank;
  ctx->device = device;
  ctx->plan = plan_faces(ctx->geo);
  const Geometry& g = ctx->geo;
  if (g.vh * 2 > INT32_MAX / 2)
    throw Error(LBCU_CONFIG_ERROR, "local volume too large for 32-bit site indexing");
  DevGeo& dg = ctx->dgeo;
  for (int d = 0; d < 4; ++d) {
    dg.L[d] = g.local[d];
    dg.wrap[d] = g.decomposed[d] ? 0 : 1;
  }
  dg.sx[3] = 1;
  dg.sx[2] = g.local[3];
  dg.sx[1] = g.local[2] * g.local[3];
  dg.sx[0] = g.local[1] * g.local[2] * g.local[3];
  dg.vh = static_cast<int>(g.vh);
  dg.stride = g.stride;

  LBCU_CUDA(cudaSetDevice(device));
  w->t->bind_device(device);
  LBCU_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;  // the halo pack runs ahead of the interior stencil
  LBCU_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  LBCU_CUDA(cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, prio_hi));
  LBCU_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  LBCU_CUDA(cudaEventCreateWithFlags(&ctx->ev_pack, cudaEventDisableTiming));
  LBCU_CUDA(cudaEventCreateWithFlags(&ctx->ev_comm, cudaEventDisableTiming));
  for (auto& e : ctx->ev) LBCU_CUDA(cudaEventCreate(&e));
  w->t->attach(rank, device);
  ctx->max_partials = static_cast<int>(2 * ((g.vh + 31) / 32) + 4096);  // hop blocks >= 32 threads
  LBCU_CUDA(cudaMalloc(&ctx->partials, sizeof(double) * 2 * ctx->max_partials));
  LBCU_CUDA(cudaMalloc(&ctx->dscal, sizeof(double) * 64));
  LBCU_CUDA(cudaMemset(ctx->dscal, 0, sizeof(double) * 64));
  LBCU_CUDA(cudaMallocHost(&ctx->hscal, sizeof(double) * 64));
  LBCU_CUDA(cudaMalloc(&ctx->dcg, sizeof(CgState)));
  LBCU_CUDA(cudaMallocHost(&ctx->hcg, 3 * sizeof(CgState)));  // [0] final, [1..2] per-iteration ring

  if (g.any_decomposed) {  // interior / boundary site lists per parity
    for (int p = 0; p < 2; ++p) {
      std::vector<int> in, bd;
      for (int64_t s = 0; s < g.volume; ++s) {
        int c[4];
        int64_t r = s;
        for (int d = 3; d >= 0; --d) {
          c[d] = static_cast<int>(r % g.local[d]);
          r /= g.local[d];
        }
        if (((c[0] + c[1] + c[2] + c[3]) & 1) != p) continue;
        bool edge = false;
        for (int d = 0; d < 4; ++d)
          if (g.decomposed[d] && (c[d] == 0 || c[d] == g.local[d] - 1)) edge = true;
        (edge ? bd : in).push_back(static_cast<int>(s >> 1));
      }
      ctx->nint[p] = static_cast<int>(in.size());
      ctx->nbnd[p] = static_cast<int>(bd.size());
      // a run of consecutive cb indices (only T decomposed): the interior
      // launch then indexes directly (no list load, warp-shared z hops)
      ctx->int_lo[p] = -1;
      if (!in.empty() && in.back() - in.front() + 1 == static_cast<int>(in.size())) ctx->int_lo[p] = in.front();
      LBCU_CUDA(cudaMalloc(&ctx->ilist[p], sizeof(int) * std::max<size_t>(1, in.size())));
      LBCU_CUDA(cudaMalloc(&ctx->blist[p], sizeof(int) * std::max<size_t>(1, bd.size())));
      if (!in.empty())
        LBCU_CUDA(cudaMemcpy(ctx->ilist[p], in.data(), sizeof(int) * in.size(), cudaMemcpyHostToDevice));
      if (!bd.empty())
        LBCU_CUDA(cudaMemcpy(ctx->blist[p], bd.data(), sizeof(int) * bd.size(), cudaMemcpyHostToDevice));
    }
  }
  *out = ctx.release();
  API_END
}

int lbcu_ctx_destroy(lbcu_ctx c) {
  API_BEGIN
  if (!c) return LBCU_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaStreamSynchronize(c->comm_stream);
  graph_cache_clear(c);
  host_pipe_release(c);
  for (auto& kv : c->scratch) free_spinor(kv.second);
  for (auto& kv : c->halo)
    for (int p = 0; p < 2; ++p)
      for (int f = 0; f < 8; ++f) {
        if (kv.second.send[p][f]) cudaFree(kv.second.send[p][f]);
        if (kv.second.recv[p][f]) cudaFree(kv.second.recv[p][f]);
      }
  for (int p = 0; p < 2; ++p) {
    if (c->ilist[p]) cudaFree(c->ilist[p]);
    if (c->blist[p]) cudaFree(c->blist[p]);
  }
  cudaFree(c->partials);
  cudaFree(c->dscal);
  cudaFreeHost(c->hscal);
  cudaFree(c->dcg);
  cudaFreeHost(c->hcg);
  if (c->dhist) cudaFree(c->dhist);
  if (c->staging) cudaFree(c->staging);
  for (auto& e : c->ev) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_fork);
  cudaEventDestroy(c->ev_pack);
  for (int e = 0; e < 2; ++e)
    if (c->ev_cg[e]) cudaEventDestroy(c->ev_cg[e]);
  cudaEventDestroy(c->ev_comm);
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->comm_stream);
  if (c->owns_world) delete c->world;
  delete c;
  API_END
}

int lbcu_ctx_synchronize(lbcu_ctx c) {
  API_BEGIN
  bind(c);
  LBCU_CUDA(cudaStreamSynchronize(c->stream));
  API_END
}

void* lbcu_ctx_stream(lbcu_ctx c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int lbcu_ctx_local(lbcu_ctx c, int local[4]) {
  API_BEGIN
  for (int d = 0; d < 4; ++d) local[d] = c->geo.local[d];
  API_END
}

int lbcu_barrier(lbcu_ctx c) {
  API_BEGIN
  bind(c);
  LBCU_CUDA(cudaStreamSynchronize(c->stream));
  c->world->t->barrier(c->rank);
  API_END
}

int lbcu_allreduce_sum(lbcu_ctx c, double* values, int n) {
  API_BEGIN
  need(c && values && n >= 1 && n <= 16, "allreduce_sum: 1..16 values");
  bind(c);
  double* d = c->dscal + 40;
  LBCU_CUDA(cudaMemcpyAsync(d, values, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  c->world->t->allreduce(c->rank, d, n, c->stream);
  LBCU_CUDA(cudaMemcpyAsync(values, d, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LBCU_CUDA(cudaStreamSynchronize(c->stream));
  API_END
}

long long lbcu_ctx_kernel_launches(lbcu_ctx c) { return c ? c->launches : -1; }
long long lbcu_ctx_cached_solves(lbcu_ctx c) {
  return c ? static_cast<long long>(graph_cache_size(c)) : -1;
}

int lbcu_event_record(lbcu_ctx c, int slot) {
  API_BEGIN
  need(slot >= 0 && slot < 16, "event slot out of range");
  bind(c);
  LBCU_CUDA(cudaEventRecord(c->ev[slot], c->stream));
  API_END
}

int lbcu_event_elapsed_ms(lbcu_ctx c, int a, int b, float* ms) {
  API_BEGIN
  need(a >= 0 && a < 16 && b >= 0 && b < 16, "event slot out of range");
  bind(c);
  LBCU_CUDA(cudaEventSynchronize(c->ev[b]));
  LBCU_CUDA(cudaEventElapsedTime(ms, c->ev[a], c->ev[b]));
  API_END
}

// ---- gauge -----------------------------------------------------------------
int lbcu_gauge_create(lbcu_ctx c, int group_rank, int rep, int bc_time, lbcu_gauge* out) {
  API_BEGIN
  need(c && out, "lbcu_gauge_create: null argument");
  bind(c);
  auto g = std::make_unique<lbcu_gauge_s>();
  g->ctx = c;
  g->n = group_rank;
  g->rep = rep;
  g->dr = rep_dim(rep, group_rank);
  g->real = rep == LBCU_REP_ADJOINT;
  if (bc_time != LBCU_BC_PERIODIC && bc_time != LBCU_BC_ANTIPERIODIC_T)
    throw Error(LBCU_CONFIG_ERROR, "unknown time boundary condition");
  g->bc = bc_time;
  const size_t esz = g->real ? sizeof(double) : sizeof(double2);
  const size_t bytes = 2 * 4 * static_cast<size_t>(g->dr) * g->dr * c->geo.stride * esz;
  LBCU_CUDA(cudaMalloc(&g->base, bytes));  // make_gauge: zero links until uploaded
  LBCU_CUDA(cudaMemsetAsync(g->base, 0, bytes, c->stream));
  g->fmt = 0;
  *out = g.release();
  API_END
}

int lbcu_gauge_upload(lbcu_gauge g, const double* host) {
  API_BEGIN
  need(g && host, "lbcu_gauge_upload: null argument");
  bind(g->ctx);
  graph_cache_forget(g->ctx, g);  // the link buffer and its storage format may change
  gauge_upload(g->ctx, g, host);
  API_END
}

int lbcu_gauge_download(lbcu_gauge g, double* host) {
  API_BEGIN
  need(g && host, "lbcu_gauge_download: null argument");
  bind(g->ctx);
  gauge_download(g->ctx, g, host);
  API_END
}

int lbcu_gauge_generate(lbcu_gauge g, int links, uint64_t seed, double eps) {
  API_BEGIN
  need(g != nullptr, "lbcu_gauge_generate: null gauge");
  if (links < LBCU_LINKS_UNIT || links > LBCU_LINKS_NEAR_UNIT)
    throw Error(LBCU_CONFIG_ERROR, "unknown link generator");
  lbcu_ctx_s* c = g->ctx;
  bind(c);
  graph_cache_forget(c, g);
  if (g->rep == LBCU_REP_ANTISYMMETRIC && g->n == 4 && g->compact_ok) {
    // SU(4) fundamental elements -> real SO(6) storage (or kept as AS4)
    gauge_adopt_fundamental(c, g, gauge_generate_dense(c, g, links, seed, eps, true));
  } else {
    gauge_adopt_dense(c, g, gauge_generate_dense(c, g, links, seed, eps, false));
  }
  API_END
}

int lbcu_spinor_random(lbcu_spinor s, uint64_t seed, uint64_t field_index) {
  API_BEGIN
  need(s != nullptr, "lbcu_spinor_random: null field");
  bind(s->ctx);
  spinor_generate(s->ctx, s, seed, field_index);
  API_END
}

int lbcu_gauge_upload_fundamental(lbcu_gauge g, const double* host) {
  API_BEGIN
  need(g && host, "lbcu_gauge_upload_fundamental: null argument");
  bind(g->ctx);
  graph_cache_forget(g->ctx, g);
  gauge_upload_fundamental(g->ctx, g, host);
  API_END
}

int lbcu_gauge_set_compact(lbcu_gauge g, int enable) {
  API_BEGIN
  need(g != nullptr, "lbcu_gauge_set_compact: null gauge");
  g->compact_ok = enable != 0;
  API_END
}

int lbcu_gauge_storage(lbcu_gauge g, int* format, double* reconstruction_error) {
  API_BEGIN
  need(g != nullptr, "lbcu_gauge_storage: null gauge");
  if (format) *format = g->fmt;
  if (reconstruction_error) *reconstruction_error = g->compact_err;
  API_END
}

int lbcu_gauge_destroy(lbcu_gauge g) {
  API_BEGIN
  if (!g) return LBCU_OK;
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  graph_cache_forget(g->ctx, g);
  cudaFree(g->base);
  delete g;
  API_END
}

// ---- spinors ---------------------------------------------------------------
int lbcu_spinor_create(lbcu_ctx c, int dr, int subset, lbcu_spinor* out) {
  API_BEGIN
  need(c && out, "lbcu_spinor_create: null argument");
  bind(c);
  *out = new_spinor(c, dr, subset);
  API_END
}

int lbcu_spinor_upload(lbcu_spinor s, const double* host) {
  API_BEGIN
  need(s && host, "lbcu_spinor_upload: null argument");
  bind(s->ctx);
  spinor_upload(s->ctx, s, host);
  API_END
}

int lbcu_spinor_download(lbcu_spinor s, double* host) {
  API_BEGIN
  need(s && host, "lbcu_spinor_download: null argument");
  bind(s->ctx);
  spinor_download(s->ctx, s, host);
  API_END
}

int lbcu_spinor_subset(lbcu_spinor s) { return s ? s->subset : -1; }

int lbcu_spinor_destroy(lbcu_spinor s) {
  API_BEGIN
  if (!s) return LBCU_OK;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  graph_cache_forget(s->ctx, s);
  free_spinor(s);
  API_END
}

// ---- operators -------------------------------------------------------------
int lbcu_dphi(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass) {
  API_BEGIN
  check_dirac(out, g, in, "apply_dirac");
  need(out->subset == LBCU_FULL && in->subset == LBCU_FULL, "apply_dirac: needs FULL fields");
  bind(in->ctx);
  HopCall hc;
  hc.in = in;
  hc.out = out;
  hc.x = in;
  hc.g = g;
  hc.out_parity = 2;
  hc.a = 4.0 + mass;
  hc.b = -0.5;
  hop_apply(in->ctx, hc);
  API_END
}

int lbcu_dphi_host(lbcu_gauge g, double mass, int nfields, const double* const* in,
                   double* const* out) {
  API_BEGIN
  need(g && in && out && nfields >= 0, "dphi_host: null argument");
  for (int k = 0; k < nfields; ++k) need(in[k] && out[k], "dphi_host: null field buffer");
  bind(g->ctx);
  dphi_host_batch(g->ctx, g, mass, nfields, in, out);
  API_END
}

int lbcu_g5dphi(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass) {
  API_BEGIN
  check_dirac(out, g, in, "g5dphi");
  need(out->subset == LBCU_FULL && in->subset == LBCU_FULL, "g5dphi: needs FULL fields");
  bind(in->ctx);
  HopCall hc;
  hc.in = in;
  hc.out = out;
  hc.x = in;
  hc.g = g;
  hc.out_parity = 2;
  hc.a = 4.0 + mass;
  hc.b = -0.5;
  hc.s5x = -1.0;
  hc.s5acc = -1.0;
  hop_apply(in->ctx, hc);
  API_END
}

int lbcu_dphi_eo(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in) {
  API_BEGIN
  check_dirac(out, g, in, "dphi_eo");
  need(out->has(0) && in->has(1), "dphi_eo: needs an even output and an odd input");
  bind(in->ctx);
  HopCall hc;
  hc.in = in;
  hc.out = out;
  hc.g = g;
  hc.out_parity = 0;
  hc.b = -0.5;
  hop_apply(in->ctx, hc);
  API_END
}

int lbcu_dphi_oe(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in) {
  API_BEGIN
  check_dirac(out, g, in, "dphi_oe");
  need(out->has(1) && in->has(0), "dphi_oe: needs an odd output and an even input");
  bind(in->ctx);
  HopCall hc;
  hc.in = in;
  hc.out = out;
  hc.g = g;
  hc.out_parity = 1;
  hc.b = -0.5;
  hop_apply(in->ctx, hc);
  API_END
}

namespace {
// out_e = Mhat in_e (optionally gamma5 Mhat gamma5 in_e) through an odd temporary
void mhat_impl(lbcu_spinor_s* out, const lbcu_gauge_s* g, const lbcu_spinor_s* in, double mass,
               bool g5sandwich) {
  lbcu_ctx_s* ctx = in->ctx;
  lbcu_spinor_s* t = scratch_spinor(ctx, in->dr, LBCU_ODD, kSlotTmp);
  const double A = 4.0 + mass;
  HopCall h1;
  h1.in = in;
  h1.out = t;
  h1.g = g;
  h1.out_parity = 1;
  h1.b = 1.0;
  h1.s5in = g5sandwich ? -1.0 : 1.0;
  hop_apply(ctx, h1);
  HopCall h2;
  h2.in = t;
  h2.out = out;
  h2.x = in;
  h2.g = g;
  h2.out_parity = 0;
  h2.a = A;
  h2.b = -1.0 / (4.0 * A);
  if (g5sandwich) h2.s5acc = -1.0;  // g5 (A g5 x - H t/4A) = A x -/+ ...
  hop_apply(ctx, h2);
}
}  // namespace

int lbcu_mhat(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass) {
  API_BEGIN
  check_dirac(out, g, in, "mhat");
  need(out->has(0) && in->has(0), "mhat: needs even fields");
  bind(in->ctx);
  mhat_impl(out, g, in, mass, false);
  API_END
}

int lbcu_mhat_dag_mhat(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass) {
  API_BEGIN
  check_dirac(out, g, in, "mhat_dag_mhat");
  need(out->has(0) && in->has(0), "mhat_dag_mhat: needs even fields");
  bind(in->ctx);
  lbcu_spinor_s* q = scratch_spinor(in->ctx, in->dr, out->subset, kSlotTmp + 1);
  mhat_impl(q, g, in, mass, false);
  mhat_impl(out, g, q, mass, true);
  API_END
}

int lbcu_h(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass) {
  API_BEGIN  // solver.cpp:9-15 with both gamma5 folded into the second Dslash
  check_dirac(out, g, in, "apply_h");
  need(out->subset == LBCU_FULL && in->subset == LBCU_FULL, "apply_h: needs FULL fields");
  bind(in->ctx);
  lbcu_spinor_s* q = scratch_spinor(in->ctx, in->dr, LBCU_FULL, kSlotTmp + 2);
  HopCall h1;
  h1.in = in;
  h1.out = q;
  h1.x = in;
  h1.g = g;
  h1.a = 4.0 + mass;
  h1.b = -0.5;
  hop_apply(in->ctx, h1);
  HopCall h2;  // g5 D g5 q: input g5, lower x sign cancels, lower hop sign flips
  h2.in = q;
  h2.out = out;
  h2.x = q;
  h2.g = g;
  h2.a = 4.0 + mass;
  h2.b = -0.5;
  h2.s5in = -1.0;
  h2.s5acc = -1.0;
  hop_apply(in->ctx, h2);
  API_END
}

// ---- vector ops ------------------------------------------------------------
namespace {
double fetch_scalar(lbcu_ctx_s* c, int slot, int n) {
  c->world->t->allreduce(c->rank, c->dscal + slot, n, c->stream);
  LBCU_CUDA(cudaMemcpyAsync(c->hscal + slot, c->dscal + slot, sizeof(double) * n,
                            cudaMemcpyDeviceToHost, c->stream));
  LBCU_CUDA(cudaStreamSynchronize(c->stream));
  return c->hscal[slot];
}
constexpr int kSlotSq = 0, kSlotDot = 2;
}  // namespace

int lbcu_sqnorm(lbcu_spinor f, double* out) {
  API_BEGIN
  need(f && out, "sqnorm: null argument");
  bind(f->ctx);
  blas_sqnorm(f->ctx, f, f->ctx->dscal + kSlotSq);
  *out = fetch_scalar(f->ctx, kSlotSq, 1);
  API_END
}

int lbcu_mul_add(lbcu_spinor psi2, double c_re, double c_im, lbcu_spinor psi1) {
  API_BEGIN
  check_pair(psi2, psi1, "mul_add");
  bind(psi1->ctx);
  blas_axpy(psi1->ctx, psi2, c_re, c_im, psi1);
  API_END
}

int lbcu_dot(lbcu_spinor a, lbcu_spinor b, double* re, double* im) {
  API_BEGIN
  check_pair(a, b, "dot");
  bind(a->ctx);
  blas_dot(a->ctx, a, b, a->ctx->dscal + kSlotDot);
  *re = fetch_scalar(a->ctx, kSlotDot, 2);
  *im = a->ctx->hscal[kSlotDot + 1];
  API_END
}

int lbcu_axpy(lbcu_spinor y, double a_re, double a_im, lbcu_spinor x) {
  API_BEGIN
  check_pair(y, x, "axpy");
  bind(x->ctx);
  blas_axpy(x->ctx, y, a_re, a_im, x);
  API_END
}

int lbcu_xpay(lbcu_spinor y, double a_re, double a_im, lbcu_spinor x) {
  API_BEGIN
  check_pair(y, x, "xpay");
  bind(x->ctx);
  blas_xpay(x->ctx, y, a_re, a_im, x);
  API_END
}

int lbcu_copy(lbcu_spinor dst, lbcu_spinor src) {
  API_BEGIN
  check_pair(dst, src, "copy_interior");
  bind(src->ctx);
  blas_copy(src->ctx, dst, src);
  API_END
}

int lbcu_zero(lbcu_spinor f) {
  API_BEGIN
  need(f != nullptr, "zero_interior: null field");
  bind(f->ctx);
  blas_zero(f->ctx, f);
  API_END
}

int lbcu_gamma5(lbcu_spinor f) {
  API_BEGIN
  need(f != nullptr, "apply_gamma5: null field");
  bind(f->ctx);
  blas_gamma5(f->ctx, f);
  API_END
}

}  // extern "C"

extern "C" int lbcu_internal_set_error(const char* msg) {
  g_last_error = msg ? msg : "";
  return 0;
}
