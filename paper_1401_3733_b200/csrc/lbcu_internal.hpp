// Internal host-side types of the latbench-b200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lbcu.h"

namespace lbcu {

// Status-carrying exception; every C-ABI entry point converts it to a code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define LBCU_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::lbcu::Error(LBCU_CUDA_ERROR, std::string(#call " failed: ") +               \
                                               cudaGetErrorString(e_) + " at " __FILE__); \
  } while (0)

int rep_dim(int rep, int n);  // group.cpp:29-38

// One rank's view of the decomposed lattice (proj/src/geometry.cpp:70-130),
// plus the even-odd device indexing.
struct Geometry {
  int global[4]{}, grid[4]{}, local[4]{}, coords[4]{};
  int rank = 0, nranks = 1;
  int64_t volume = 0;  // local interior sites
  int64_t vh = 0;      // sites per parity
  int64_t stride = 0;  // padded component stride (elements) of one parity block
  bool decomposed[4]{};
  bool any_decomposed = false;

  void global_coords(int64_t s, int* gc) const {
    int lc[4];
    int64_t r = s;
    for (int d = 3; d >= 0; --d) {
      lc[d] = static_cast<int>(r % local[d]);
      r /= local[d];
    }
    for (int d = 0; d < 4; ++d) gc[d] = coords[d] * local[d] + lc[d];
  }
};

Geometry build_geometry(const int global[4], const int grid[4], int rank, bool enforce_floor);

void host_spinor_random(const Geometry& geo, int dr, uint64_t seed, uint64_t field, double* out);
void host_gauge_random(const Geometry& geo, int n, int rep, int links, uint64_t seed, double eps,
                       int nthreads, double* out);

// Face schedule for the even-odd halo exchange (see lbcu_plan_faces).
struct FacePlan {
  int partner[8]{};   // f = 2 mu + dir; dir 0 -> -mu partner, dir 1 -> +mu partner
  int64_t count[8]{}; // records per message (half the face)
};
FacePlan plan_faces(const Geometry& geo);
// local lexicographic site of record j on face f for the given input parity
int64_t face_site(const Geometry& geo, int f, int input_parity, int64_t j);

// ---------------------------------------------------------------- transport
struct Transport {
  virtual ~Transport() = default;
  virtual int nranks() const = 0;
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
  // in-place sum of n doubles in device memory across ranks, stream-ordered
  virtual void allreduce(int rank, double* dev, int n, cudaStream_t s) = 0;
  // exchange: for each message i, send send[i] (bytes[i]) to peer_send[i] and
  // receive recv[i] (bytes[i]) from peer_recv[i]; stream-ordered.
  struct Msg {
    const void* send;
    void* recv;
    size_t bytes;
    int peer_send, peer_recv;
  };
  virtual void exchange(int rank, const std::vector<Msg>& msgs, cudaStream_t s) = 0;
  virtual void barrier(int rank) = 0;
  // called by each context after it selected its device
  virtual void bind_device(int /*device*/) {}
  // called by each context once its stream exists (rank known)
  virtual void attach(int /*rank*/, int /*device*/) {}

  // ---- direct halo exchange over peer memory -----------------------------
  // With a direct transport the halo pack kernel stores its records straight
  // into the receiving rank's arena (P2P stores over NVLink for the IPC
  // world), so pack and transfer are one kernel; no send buffers, no copies.
  virtual bool direct() const { return false; }
  // switch a direct transport to message exchange and back (collective;
  // the IPC world then uses its NCCL communicator for the halos)
  virtual void set_direct(bool on) {
    if (on) throw Error(LBCU_TRANSPORT_ERROR, "transport has no direct halo mode");
  }
  // collective, once per key and context: register this rank's receive arena
  // and map every peer's (same size and layout on every rank). The transport
  // takes ownership of `local` and frees it at teardown or when the key is
  // mapped again, once no peer can still store into it.
  virtual void map_arena(int /*rank*/, int /*key*/, void* /*local*/, size_t /*bytes*/) {
    throw Error(LBCU_TRANSPORT_ERROR, "transport has no peer-memory arenas");
  }
  virtual void* peer_arena(int /*rank*/, int /*key*/, int /*peer*/) const { return nullptr; }
  // after the pack kernel of exchange `epoch`: publish its completion
  virtual void post(int /*rank*/, long long /*epoch*/, cudaStream_t /*s*/) {}
  // order stream s after every listed peer's post of exchange `epoch`
  virtual void await(int /*rank*/, long long /*epoch*/, const std::vector<int>& /*peers*/, cudaStream_t /*s*/) {}
};

std::unique_ptr<Transport> make_single_transport();
std::unique_ptr<Transport> make_thread_transport(int nranks, bool direct = false);
// one process per rank on one node: peer-memory halos through CUDA IPC, a
// POSIX shared-memory segment `name` for the bootstrap and the host barrier;
// CG sums through NCCL when `nccl_id` is given, else through the segment
std::unique_ptr<Transport> make_ipc_transport(int nranks, int rank, const char* name,
                                              const unsigned char* nccl_id);
std::unique_ptr<Transport> make_nccl_transport(int nranks, int rank, const unsigned char id[128]);
void nccl_unique_id(unsigned char id[128]);

}  // namespace lbcu

struct lbcu_world_s {
  std::unique_ptr<lbcu::Transport> t;
};
