// Library objects behind the opaque C-ABI handles, and the launcher entry
// points the .cu translation units provide.
#pragma once

#include <map>
#include <mutex>
#include <tuple>

#include "device.cuh"
#include "lbcu_internal.hpp"

struct lbcu_ctx_s;

struct lbcu_spinor_s {
  lbcu_ctx_s* ctx = nullptr;
  int dr = 0;
  int subset = LBCU_FULL;
  double2* base = nullptr;
  double2* par[2] = {nullptr, nullptr};  // parity blocks of 4 dr x stride elements, 32-site tiles
  size_t elems = 0;                      // double2 elements over present parities
  bool has(int p) const { return par[p] != nullptr; }
};

struct lbcu_gauge_s {
  lbcu_ctx_s* ctx = nullptr;
  int n = 0, rep = 0, dr = 0, bc = 0;
  bool real = false;
  // [2 parity][4 mu][entries][stride]: GF_FULL dense dr x dr (double2, or
  // double for real links, BC sign baked in); compact formats (links.cuh)
  // store double2 entries and apply the BC sign in the kernels
  void* base = nullptr;
  int fmt = 0;
  bool compact_ok = true;     // lbcu_gauge_set_compact
  double compact_err = -1.0;  // max reconstruction error seen at the last upload
};

namespace lbcu {

enum Epi { EPI_STORE = 0, EPI_STORE_NORM = 1, EPI_CG = 2 };

struct HaloBufs {
  double2* send[2][8] = {};  // by output parity, face
  double2* recv[2][8] = {};
  // direct transports: one receive arena [parity][face][epoch & 1] of `slot`
  // double2 each, mapped by every peer and owned by the world's transport
  // (Transport::map_arena frees it; lbcu_ctx_destroy does not)
  double2* arena = nullptr;
  size_t slot = 0;
  size_t cap = 0;  // double2 per buffer
};

}  // namespace lbcu

struct lbcu_ctx_s {
  lbcu_world_s* world = nullptr;
  bool owns_world = false;
  int rank = 0, device = 0;
  lbcu::Geometry geo;
  lbcu::FacePlan plan;
  lbcu::DevGeo dgeo{};
  cudaStream_t stream = nullptr;
  cudaStream_t comm_stream = nullptr;  // halo pack + exchange (decomposed runs), high priority
  cudaEvent_t ev_fork = nullptr, ev_pack = nullptr, ev_comm = nullptr;
  cudaEvent_t ev[16] = {};
  // reduction workspace
  double* partials = nullptr;
  int max_partials = 0;
  double* dscal = nullptr;  // 64 device scalars (reduction results)
  double* hscal = nullptr;  // pinned mirror
  // interior / boundary site lists per output parity (decomposed runs only)
  int* ilist[2] = {nullptr, nullptr};
  int* blist[2] = {nullptr, nullptr};
  int nint[2] = {0, 0}, nbnd[2] = {0, 0};
  int int_lo[2] = {-1, -1};  // first cb of a contiguous interior, -1: use ilist
  std::map<int, lbcu::HaloBufs> halo;  // keyed by dr
  std::map<std::tuple<int, int, int>, lbcu_spinor_s*> scratch;  // (dr, subset, slot)
  lbcu::CgState* dcg = nullptr;
  lbcu::CgState* hcg = nullptr;  // pinned, 3: final state + 2-slot per-iteration ring
  double* dhist = nullptr;
  long long hist_cap = 0;
  void* staging = nullptr;  // device staging buffer for host<->device layout transposes
  size_t staging_bytes = 0;
  long long launches = 0;
  long long xepoch = 0;  // halo exchanges so far (direct transports: arena / event slot)
  cudaEvent_t ev_cg[2] = {nullptr, nullptr};  // per-iteration CG state copies (host loop)
  // host-field pipeline (lbcu_dphi_host): 2 slots, copy-in / copy-out streams
  struct HostPipe {
    size_t bytes = 0;
    void* stage_in[2] = {};
    void* stage_out[2] = {};
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_in_free[2] = {}, ev_out[2] = {}, ev_d2h[2] = {};
  } pipe;
};

namespace lbcu {

// ---- launchers (stream-ordered on ctx->stream) --------------------------
struct HopCall {
  const lbcu_spinor_s* in = nullptr;
  lbcu_spinor_s* out = nullptr;
  const lbcu_spinor_s* x = nullptr;  // diagonal term (same parity set as out)
  lbcu_spinor_s* r = nullptr;        // EPI_CG residual
  const lbcu_gauge_s* g = nullptr;
  int out_parity = 2;  // 0 even, 1 odd, 2 both
  double a = 0.0, b = 1.0;
  double s5in = 1.0, s5x = 1.0, s5acc = 1.0;
  int epi = EPI_STORE;
  const double* alpha = nullptr;  // EPI_CG scalar (device)
  double* result = nullptr;       // reduction output (device), EPI != STORE
  // CG scalar step fused into the reduction's last block (single rank only)
  int post = POST_NONE;
  unsigned long long handle = 0;
  int use_graph = 0;
};
void hop_apply(lbcu_ctx_s* ctx, const HopCall& c);

// flat BLAS over the present parity blocks (padding included, kept at zero)
void blas_sqnorm(lbcu_ctx_s* ctx, const lbcu_spinor_s* f, double* dres);
void blas_dot(lbcu_ctx_s* ctx, const lbcu_spinor_s* a, const lbcu_spinor_s* b, double* dres2);
void blas_axpy(lbcu_ctx_s* ctx, lbcu_spinor_s* y, double are, double aim, const lbcu_spinor_s* x);
void blas_xpay(lbcu_ctx_s* ctx, lbcu_spinor_s* y, double are, double aim, const lbcu_spinor_s* x);
void blas_copy(lbcu_ctx_s* ctx, lbcu_spinor_s* dst, const lbcu_spinor_s* src);
void blas_zero(lbcu_ctx_s* ctx, lbcu_spinor_s* f);
void blas_gamma5(lbcu_ctx_s* ctx, lbcu_spinor_s* f);
// CG helpers reading scalars from the device CgState
void cg_p_update(lbcu_ctx_s* ctx, lbcu_spinor_s* p, const lbcu_spinor_s* r, lbcu_spinor_s* x);
void cg_r_update(lbcu_ctx_s* ctx, lbcu_spinor_s* r, const lbcu_spinor_s* ap, double* dres);
void cg_x_final(lbcu_ctx_s* ctx, lbcu_spinor_s* x, const lbcu_spinor_s* p);
void cg_scalar_alpha(lbcu_ctx_s* ctx, const double* pap);
void cg_scalar_end(lbcu_ctx_s* ctx, const double* rr_new, unsigned long long graph_handle,
                   int use_graph);
void cg_scalar_init(lbcu_ctx_s* ctx, const double* b2, double tol, long long maxit);
// single-reduction (Chronopoulos-Gear) CG steps, blas.cu
void cg1_update(lbcu_ctx_s* ctx, lbcu_spinor_s* p, lbcu_spinor_s* s, lbcu_spinor_s* x, lbcu_spinor_s* r,
                const lbcu_spinor_s* w, double* dres);
void cg1_scalar_start(lbcu_ctx_s* ctx, const double* gd);
void cg1_scalar_end(lbcu_ctx_s* ctx, const double* gd);

// layout transposes host (reference AoS) <-> device (even-odd SoA)
void spinor_upload(lbcu_ctx_s* ctx, lbcu_spinor_s* s, const double* host);
void spinor_download(lbcu_ctx_s* ctx, const lbcu_spinor_s* s, double* host);
void gauge_upload(lbcu_ctx_s* ctx, lbcu_gauge_s* g, const double* host);
void gauge_download(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, double* host);
void gauge_upload_fundamental(lbcu_ctx_s* ctx, lbcu_gauge_s* g, const double* host);
void gauge_adopt_dense(lbcu_ctx_s* ctx, lbcu_gauge_s* g, void* full);
void gauge_adopt_fundamental(lbcu_ctx_s* ctx, lbcu_gauge_s* g, void* fund);
// on-device keyed generation (generate.cu)
void spinor_generate(lbcu_ctx_s* ctx, lbcu_spinor_s* s, uint64_t seed, uint64_t field);
void* gauge_generate_dense(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, int links, uint64_t seed,
                           double eps, bool fundamental);
// out[k] = D in[k] for host fields, transfers overlapped with the kernels
void dphi_host_batch(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, double mass, int n,
                     const double* const* in, double* const* out);
void host_pipe_release(lbcu_ctx_s* ctx);

// CG graph cache (solver.cpp): drop every instantiated solve that names a
// handle (spinor or gauge) before it is freed or its links are replaced, and
// all of a context's solves when it is destroyed
void graph_cache_forget(const lbcu_ctx_s* ctx, const void* handle);
void graph_cache_clear(const lbcu_ctx_s* ctx);
size_t graph_cache_size(const lbcu_ctx_s* ctx);

// helpers in api.cpp
lbcu_spinor_s* scratch_spinor(lbcu_ctx_s* ctx, int dr, int subset, int slot);
void reduce_slot_reset(lbcu_ctx_s* ctx);
int reduce_blocks_cap(lbcu_ctx_s* ctx);

}  // namespace lbcu
