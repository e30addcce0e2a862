/*
 * lbcu.h — C-ABI of the B200 Wilson-Dirac / CG hot path (latbench-b200).
 *
 * Drop-in boundary for the reference's operator API (latbench, C++20,
 * /root/reference/proj). Every entry point cites the reference interface it
 * replaces. Plain pointers and sizes only; no torch or CUDA types cross it
 * (streams are handed out as opaque void*).
 *
 * Host buffers always use the reference's storage layout for ONE worker's
 * interior (proj/include/latbench/fields.hpp:15-57, geometry.hpp:40-42):
 *   site order   : local lexicographic (t,x,y,z), z fastest
 *   spinor       : [site][spin 4][colour dr] complex<double>   (2 doubles)
 *   gauge        : [site][mu 4][row dr][col dr] complex<double>, or double for
 *                  the adjoint representation (real_links)
 * Device storage is private to the library (even-odd, 32-site tiles).
 *
 * Status codes mirror the reference exception classes
 * (proj/include/latbench/errors.hpp:9-63): a non-zero return carries a
 * thread-local message readable through lbcu_last_error().
 *
 * Calls taking a context are collective over the ranks of its world, one
 * host thread per rank (proj/include/latbench/transport.hpp:15-18).
 */
#ifndef LBCU_H
#define LBCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* the library is built with -fvisibility=hidden: exactly these symbols export */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LBCU_ABI_VERSION 1

/* ---- status codes: errors.hpp:9-63 -------------------------------------- */
enum lbcu_status {
  LBCU_OK = 0,
  LBCU_CONTRACT_VIOLATION = 1, /* ContractViolation      errors.hpp:38-42 */
  LBCU_CONFIG_ERROR = 2,       /* ConfigError / DecompositionError / ParseError */
  LBCU_TRANSPORT_ERROR = 3,    /* TransportError         errors.hpp:44-48 */
  LBCU_NON_CONVERGENCE = 4,    /* NonConvergence         errors.hpp:50-63 */
  LBCU_CUDA_ERROR = 5          /* device-side failure (no reference analogue) */
};

/* group.hpp:12 — same enumerator order */
enum lbcu_rep {
  LBCU_REP_FUNDAMENTAL = 0,
  LBCU_REP_ADJOINT = 1,
  LBCU_REP_SYMMETRIC = 2,
  LBCU_REP_ANTISYMMETRIC = 3
};
/* flops.hpp:7 — same enumerator order */
enum lbcu_kernel { LBCU_KERNEL_SQNORM = 0, LBCU_KERNEL_MULADD = 1, LBCU_KERNEL_DIRAC = 2 };
/* site subsets of a spinor field (even-odd preconditioning; no reference analogue) */
enum lbcu_subset { LBCU_FULL = 0, LBCU_EVEN = 1, LBCU_ODD = 2 };
/* time boundary condition (reference: periodic only, geometry.cpp:117-124) */
enum lbcu_bc { LBCU_BC_PERIODIC = 0, LBCU_BC_ANTIPERIODIC_T = 1 };
/* link generators: unit (fields.cpp:71-84), Haar (fields.cpp:86-107), near-unit exp(i eps H) */
enum lbcu_links { LBCU_LINKS_UNIT = 0, LBCU_LINKS_HAAR = 1, LBCU_LINKS_NEAR_UNIT = 2 };

typedef struct lbcu_world_s* lbcu_world;   /* WorkerGroup, transport.hpp:24-67 */
typedef struct lbcu_ctx_s* lbcu_ctx;       /* Worker + Geometry + ExchangePlan */
typedef struct lbcu_gauge_s* lbcu_gauge;   /* GaugeField, fields.hpp:37-57 */
typedef struct lbcu_spinor_s* lbcu_spinor; /* SpinorField, fields.hpp:15-24 */

/* ---- diagnostics --------------------------------------------------------- */
const char* lbcu_last_error(void);
int lbcu_abi_version(void);
/* 1 when a CUDA device is usable, 0 otherwise (host-only helpers still work) */
int lbcu_device_count(void);

/* ---- host-only helpers (no GPU needed) ----------------------------------- */
/* flops_per_site, flops.hpp:44 / flops.cpp:14-25 */
long long lbcu_flops_per_site(int kernel, int dr, int real_rep);
/* rep_dim / rep_is_real, group.hpp:20-23 */
int lbcu_rep_dim(int rep, int group_rank, int* dr, int* real_links);
/* build_geometry checks, geometry.cpp:70-95 (DecompositionError -> LBCU_CONFIG_ERROR) */
int lbcu_check_geometry(const int global[4], const int grid[4], int rank, int enforce_floor,
                        int local_out[4]);
/* init_spinor_random, fields.cpp:22-40: one worker's interior, reference layout */
int lbcu_host_spinor_random(const int global[4], const int grid[4], int rank, int dr,
                            uint64_t seed, uint64_t field_index, double* out);
/* randomize_gauge_interior, fields.cpp:86-107 (links = HAAR), make_unit_gauge
 * fields.cpp:71-84 (UNIT), or near-unit U = exp(i eps H) (NEAR_UNIT, BASELINE
 * config 3; fundamental only). One worker's interior, reference layout.
 * nthreads <= 0 uses all hardware threads. */
int lbcu_host_gauge_random(const int global[4], const int grid[4], int rank, int group_rank,
                           int rep, int links, uint64_t seed, double eps, int nthreads,
                           double* out);
/* Face schedule of one rank's even-odd halo exchange (host logic of the N>1
 * path, the analogue of build_exchange_plan, transport.cpp:142-171).
 * For face f = 2*mu + dir (dir 0: message to the -mu partner carrying the
 * projected boundary at x_mu = 0; dir 1: to the +mu partner carrying U^dag P
 * psi at x_mu = L_mu - 1): partner[f] (-1 when mu is not decomposed) and
 * count[f] = half-spinor records per message. sites (nullable, length
 * sum(count)) receives, for a given input parity, the LOCAL lexicographic
 * site index packed into each record, in message order. */
int lbcu_plan_faces(const int global[4], const int grid[4], int rank, int input_parity,
                    int partner[8], int count[8], int32_t* sites);

/* ---- worlds (transport) -------------------------------------------------- */
int lbcu_world_single(lbcu_world* out);
/* In-process world: one host thread per rank (the reference's run_workers
 * model, transport.cpp:114-140), device buffers exchanged by peer copies. */
int lbcu_world_threads(int nranks, lbcu_world* out);
/* One process per GPU over NCCL (NVLink / NVSwitch). id: 128 bytes from
 * lbcu_nccl_unique_id on rank 0, broadcast out of band. */
int lbcu_nccl_unique_id(unsigned char id[128]);
int lbcu_world_nccl(int nranks, int rank, const unsigned char id[128], lbcu_world* out);
/* One process per GPU on one node with direct halos (replaces the same
 * halo_exchange, transport.cpp:142-221): the halo pack kernel stores its
 * records straight into the receiving rank's arena over NVLink (CUDA IPC
 * mappings); completion is an interprocess event per exchange, recorded after
 * the pack and waited on by the peer's stream before its boundary kernel, with
 * a host barrier in the POSIX shared-memory segment `name` ("/...", unique per
 * job) between the two. No kernel waits on another rank. nccl_id (nullable):
 * CG sums through NCCL; NULL sums through the segment on the host. */
int lbcu_world_ipc(int nranks, int rank, const char* name, const unsigned char* nccl_id, lbcu_world* out);
/* The thread world with the same direct halo protocol (test and emulation). */
int lbcu_world_threads_direct(int nranks, lbcu_world* out);
/* Collective: direct halos on (1) or message exchange (0; the IPC world then
 * sends the halos through its NCCL communicator). Worlds without a direct
 * mode accept only 0. */
int lbcu_world_set_direct(lbcu_world w, int on);
int lbcu_world_destroy(lbcu_world w);

/* ---- contexts: build_geometry + build_exchange_plan + Worker ------------- */
int lbcu_ctx_create(lbcu_world w, int rank, int device, const int global[4], const int grid[4],
                    int enforce_floor, lbcu_ctx* out);
int lbcu_ctx_destroy(lbcu_ctx c);
int lbcu_ctx_synchronize(lbcu_ctx c);
void* lbcu_ctx_stream(lbcu_ctx c); /* the cudaStream_t all work is issued on */
int lbcu_ctx_local(lbcu_ctx c, int local[4]);
int lbcu_barrier(lbcu_ctx c);      /* Worker::barrier, transport.cpp:79 */
/* Worker::global_sum of host values (transport.cpp:83-100), in place, collective */
int lbcu_allreduce_sum(lbcu_ctx c, double* values, int n);
/* launches of library kernels issued on this context since creation */
long long lbcu_ctx_kernel_launches(lbcu_ctx c);
/* Instantiated CG solve graphs cached by the context (one per fused problem
 * and field set; dropped when a field they name is destroyed or its links are
 * re-uploaded, all of them at lbcu_ctx_destroy). -1 for a null context. */
long long lbcu_ctx_cached_solves(lbcu_ctx c);
/* CUDA-event timing on the context stream (slot 0..15) */
int lbcu_event_record(lbcu_ctx c, int slot);
int lbcu_event_elapsed_ms(lbcu_ctx c, int slot_a, int slot_b, float* ms);

/* ---- gauge field: GaugeField / init_gauge_random ------------------------ */
int lbcu_gauge_create(lbcu_ctx c, int group_rank, int rep, int bc_time, lbcu_gauge* out);
/* upload this rank's interior links (reference layout). bc_time applies the
 * antiperiodic sign to U_0 on the last global time slice on the device. */
int lbcu_gauge_upload(lbcu_gauge g, const double* host);
int lbcu_gauge_download(lbcu_gauge g, double* host); /* as uploaded (no BC sign) */
/* Link storage on the device. Compact exact forms are used when every
 * uploaded link reconstructs to within 1e-12 (checked at upload):
 *   LBCU_GAUGE_SU2 : SU(2) links as 2 complex (fundamental; adjoint rebuilt)
 *   LBCU_GAUGE_R12 : SU(3) fundamental, two rows (third = conj(r0 x r1))
 *   LBCU_GAUGE_AS4R: SU(4) antisymmetric as a real SO(6) matrix in a fixed
 *                    real basis of the 6 (the kernels rotate colour vectors)
 * otherwise LBCU_GAUGE_FULL (dense dr x dr). set_compact(0) before upload
 * forces dense storage. */
enum lbcu_gauge_format {
  LBCU_GAUGE_FULL = 0,
  LBCU_GAUGE_SU2 = 1,
  LBCU_GAUGE_R12 = 2,
  LBCU_GAUGE_AS4 = 3, /* SU(4) antisymmetric formed from fundamental links */
  LBCU_GAUGE_AS4R = 4 /* SU(4) antisymmetric, real basis (36 doubles) */
};
int lbcu_gauge_set_compact(lbcu_gauge g, int enable);
/* Upload the FUNDAMENTAL SU(N) links (host layout [site][mu][N][N] complex,
 * the group elements randomize_gauge_interior draws before represent(),
 * fields.cpp:95-96); the represented link is formed on the fly in the
 * kernels. Supported for the SU(4) antisymmetric representation (BASELINE
 * config 5): stored as LBCU_GAUGE_AS4R when every element is in SU(4) to
 * 1e-12, else as the 16 fundamental entries (LBCU_GAUGE_AS4; also forced by
 * the environment variable LBCU_AS4_STORAGE=fund). */
int lbcu_gauge_upload_fundamental(lbcu_gauge g, const double* host_fundamental);
/* init_gauge_random on the device: the keyed generators of
 * fields.cpp:86-107 / group.cpp:82-114 evaluated per link on the GPU
 * (fundamental SU(2..4), the SU(2) adjoint, SU(4) antisymmetric via
 * AS4R / AS4 storage; links = UNIT / HAAR / NEAR_UNIT). Agrees with the host generator
 * to a few ulp (device transcendentals). */
int lbcu_gauge_generate(lbcu_gauge g, int links, uint64_t seed, double eps);
/* init_spinor_random (fields.cpp:22-40) on the device */
int lbcu_spinor_random(lbcu_spinor s, uint64_t seed, uint64_t field_index);
int lbcu_gauge_storage(lbcu_gauge g, int* format, double* reconstruction_error);
int lbcu_gauge_destroy(lbcu_gauge g);

/* ---- spinor fields: SpinorField ------------------------------------------ */
int lbcu_spinor_create(lbcu_ctx c, int dr, int subset, lbcu_spinor* out);
/* host buffer = the rank's whole interior in reference layout; sites outside
 * the field's subset are ignored on upload and written as zero on download. */
int lbcu_spinor_upload(lbcu_spinor s, const double* host);
int lbcu_spinor_download(lbcu_spinor s, double* host);
int lbcu_spinor_subset(lbcu_spinor s);
int lbcu_spinor_destroy(lbcu_spinor s);

/* ---- operators (collective; each performs its own halo exchange) --------- */
/* apply_dirac, kernels.hpp:19-20: out = (4+m) in - 1/2 sum_mu hops. FULL fields. */
int lbcu_dphi(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass);
/* apply_dirac on HOST fields (reference interior layout): out[k] = D in[k]
 * for k < nfields, with the host->device copy of field k+1 and the
 * device->host copy of field k-1 overlapped with the kernels of field k.
 * Pinned host buffers run at full PCIe duplex. Blocks until all are done. */
int lbcu_dphi_host(lbcu_gauge g, double mass, int nfields, const double* const* in,
                   double* const* out);
/* gamma5 . apply_dirac, as composed in apply_h (solver.cpp:11-12) */
int lbcu_g5dphi(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass);
/* even-odd blocks of D (no reference analogue):
 * D_eo = -1/2 H_eo : odd -> even,  D_oe = -1/2 H_oe : even -> odd */
int lbcu_dphi_eo(lbcu_spinor out_even, lbcu_gauge g, lbcu_spinor in_odd);
int lbcu_dphi_oe(lbcu_spinor out_odd, lbcu_gauge g, lbcu_spinor in_even);
/* Schur complement on even sites: Mhat = (4+m) - D_eo D_oe / (4+m) */
int lbcu_mhat(lbcu_spinor out_even, lbcu_gauge g, lbcu_spinor in_even, double mass);
/* Mhat^dag Mhat = g5 Mhat g5 Mhat */
int lbcu_mhat_dag_mhat(lbcu_spinor out_even, lbcu_gauge g, lbcu_spinor in_even, double mass);
/* apply_h, solver.hpp:32-33: out = g5 D g5 D in = D^dag D in */
int lbcu_h(lbcu_spinor out, lbcu_gauge g, lbcu_spinor in, double mass);

/* ---- vector ops: kernels.hpp:11-44 (interior of the field's subset) ------ */
int lbcu_sqnorm(lbcu_spinor f, double* out);                           /* kernels.cpp:36-39 */
int lbcu_mul_add(lbcu_spinor psi2, double c_re, double c_im, lbcu_spinor psi1); /* :45-49 */
int lbcu_dot(lbcu_spinor a, lbcu_spinor b, double* re, double* im);    /* :67-73 */
int lbcu_axpy(lbcu_spinor y, double a_re, double a_im, lbcu_spinor x); /* :75-79 */
int lbcu_xpay(lbcu_spinor y, double a_re, double a_im, lbcu_spinor x); /* :81-85 */
int lbcu_copy(lbcu_spinor dst, lbcu_spinor src);                       /* :87-91 */
int lbcu_zero(lbcu_spinor f);                                          /* :93-96 */
int lbcu_gamma5(lbcu_spinor f);                                        /* :98-104 */

/* ---- CG: solver.hpp:13-44 ------------------------------------------------ */
typedef struct {
  double tolerance;   /* CgSettings::tolerance, relative residual in (0,1) */
  int max_iterations; /* CgSettings::max_iterations >= 1 */
} lbcu_cg_settings;

typedef struct {
  long iterations;          /* CgOutcome::iterations */
  double rel_residual;      /* recurrence residual at exit */
  double true_rel_residual; /* |A x - b| / |b| recomputed at exit */
  double best_residual;     /* best recurrence residual (NonConvergence payload) */
  double seconds;           /* device time, solve start to true residual */
} lbcu_cg_outcome;

/* LinearOp, solver.hpp:28: out = A(in). Must return 0 on success. */
typedef int (*lbcu_linop)(void* user, lbcu_spinor out, lbcu_spinor in);

/* cg_solve(LinearOp, rhs, settings), solver.cpp:24-82. x is overwritten.
 * history (nullable) receives one relative residual per iteration. */
int lbcu_cg_solve(lbcu_ctx c, lbcu_linop op, void* user, lbcu_spinor rhs, lbcu_spinor x,
                  const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome, double* history);
/* cg_solve(make_h_operator(...)), fused kernels: CG on D^dag D, FULL fields */
int lbcu_cg_solve_h(lbcu_gauge g, double mass, lbcu_spinor rhs, lbcu_spinor x,
                    const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome, double* history);
/* even-odd preconditioned CG on Mhat^dag Mhat, EVEN fields (no reference analogue) */
int lbcu_cg_solve_eo(lbcu_gauge g, double mass, lbcu_spinor rhs_even, lbcu_spinor x_even,
                     const lbcu_cg_settings* settings, lbcu_cg_outcome* outcome,
                     double* history);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* LBCU_H */
