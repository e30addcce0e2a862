// Transports: the replacement for the reference's in-process message layer
// (proj/src/transport.cpp:12-140).
//
//   single  : one rank, every collective is a no-op.
//   threads : the reference's model (one host thread per worker, generation
//             barrier, fixed-order sums, transport.cpp:28-100) carried over to
//             device buffers: messages are device pointers posted between two
//             barriers and pulled with stream-ordered peer copies. Used for
//             multi-rank runs inside one process (tests, one-GPU emulation of
//             a decomposition).
//   nccl    : one process per GPU; ncclSend/ncclRecv pairs inside a group for
//             halos, ncclAllReduce(double, sum) for CG scalars, all on the
//             context stream (NVLink 5 / NVSwitch). libnccl is dlopen()ed on
//             first use so single-GPU users never load it.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "lbcu_internal.hpp"

namespace lbcu {

namespace {

struct SingleTransport final : Transport {
  int nranks() const override { return 1; }
  bool capturable() const override { return true; }
  void allreduce(int, double*, int, cudaStream_t) override {}
  void exchange(int, const std::vector<Msg>& msgs, cudaStream_t s) override {
    for (const auto& m : msgs)  // self-messages only
      LBCU_CUDA(cudaMemcpyAsync(m.recv, m.send, m.bytes, cudaMemcpyDeviceToDevice, s));
  }
  void barrier(int) override {}
};

struct ThreadTransport final : Transport {
  explicit ThreadTransport(int n) : n_(n), contrib_(n), posted_(n) {}
  int nranks() const override { return n_; }
  bool capturable() const override { return false; }

  // generation barrier (transport.cpp:28-55, without op tagging)
  void sync() {
    std::unique_lock<std::mutex> lk(m_);
    if (++arrived_ == n_) {
      arrived_ = 0;
      ++phase_;
      cv_.notify_all();
      return;
    }
    const uint64_t entered = phase_;
    if (!cv_.wait_for(lk, std::chrono::seconds(600), [&] { return phase_ != entered; }))
      throw Error(LBCU_TRANSPORT_ERROR, "thread transport: barrier timed out");
  }

  void barrier(int) override { sync(); }

  void allreduce(int rank, double* dev, int n, cudaStream_t s) override {
    std::vector<double> loc(n);
    LBCU_CUDA(cudaMemcpyAsync(loc.data(), dev, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    LBCU_CUDA(cudaStreamSynchronize(s));
    contrib_[rank] = loc;
    sync();
    // fixed binary tree over ranks, identical on every rank (transport.cpp:83-100)
    for (int k = 0; k < n; ++k) loc[k] = tree(k, 0, n_);
    sync();
    LBCU_CUDA(cudaMemcpyAsync(dev, loc.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    LBCU_CUDA(cudaStreamSynchronize(s));
  }

  void exchange(int rank, const std::vector<Msg>& msgs, cudaStream_t s) override {
    LBCU_CUDA(cudaStreamSynchronize(s));  // send buffers complete
    posted_[rank] = msgs;
    sync();
    // k-th receive from peer q matches q's k-th send addressed to this rank
    std::vector<int> seen(n_, 0);
    for (const auto& m : msgs) {
      const int q = m.peer_recv;
      int want = seen[q]++, k = 0;
      const Msg* src = nullptr;
      for (const auto& pm : posted_[q])
        if (pm.peer_send == rank && k++ == want) {
          src = &pm;
          break;
        }
      if (!src || src->bytes != m.bytes)
        throw Error(LBCU_TRANSPORT_ERROR, "thread transport: posted message does not match halo");
      LBCU_CUDA(cudaMemcpyAsync(m.recv, src->send, m.bytes, cudaMemcpyDefault, s));
    }
    LBCU_CUDA(cudaStreamSynchronize(s));
    sync();  // nobody reuses a send buffer before every pull finished
  }

 private:
  double tree(int k, int lo, int hi) const {
    if (hi - lo == 1) return contrib_[lo][k];
    const int mid = lo + (hi - lo) / 2;
    return tree(k, lo, mid) + tree(k, mid, hi);
  }
  int n_;
  std::mutex m_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t phase_ = 0;
  std::vector<std::vector<double>> contrib_;
  std::vector<std::vector<Msg>> posted_;
};

// ---- NCCL through dlopen ----------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
      const char* names[] = {"libnccl.so.2", "libnccl.so"};
      for (const char* n : names)
        if ((api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
      if (!api.h) return;
#define LBCU_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
      LBCU_SYM(GetUniqueId);
      LBCU_SYM(CommInitRank);
      LBCU_SYM(CommDestroy);
      LBCU_SYM(GroupStart);
      LBCU_SYM(GroupEnd);
      LBCU_SYM(Send);
      LBCU_SYM(Recv);
      LBCU_SYM(AllReduce);
      LBCU_SYM(GetErrorString);
#undef LBCU_SYM
    });
    if (!api.h || !api.CommInitRank || !api.Send)
      throw Error(LBCU_TRANSPORT_ERROR, "libnccl.so.2 could not be loaded");
    return api;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(LBCU_TRANSPORT_ERROR,
                std::string(what) + ": " + NcclApi::get().GetErrorString(r));
}

struct NcclTransport final : Transport {
  // The communicator is created on first use by a context, after that
  // context has made its device current (ncclCommInitRank binds the device).
  NcclTransport(int n, int rank, const unsigned char id[128]) : n_(n), rank_(rank) {
    NcclApi::get();  // fail early if libnccl is missing
    std::memcpy(&uid_, id, sizeof(uid_));
  }
  void bind_device(int device) override {
    if (comm_) return;
    LBCU_CUDA(cudaSetDevice(device));
    nccl_check(NcclApi::get().CommInitRank(&comm_, n_, uid_, rank_), "ncclCommInitRank");
    LBCU_CUDA(cudaMalloc(&scratch_, sizeof(double)));
  }
  ~NcclTransport() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
    if (scratch_) cudaFree(scratch_);
  }
  int nranks() const override { return n_; }
  bool capturable() const override { return true; }
  ncclComm_t comm() const {
    if (!comm_) throw Error(LBCU_TRANSPORT_ERROR, "NCCL world used before a context bound its device");
    return comm_;
  }
  void allreduce(int, double* dev, int n, cudaStream_t s) override {
    if (n_ == 1) return;  // a sum over one rank is the identity (keeps graphs NCCL-free)
    nccl_check(NcclApi::get().AllReduce(dev, dev, n, ncclDouble, ncclSum, comm(), s),
               "ncclAllReduce");
  }
  void exchange(int, const std::vector<Msg>& msgs, cudaStream_t s) override {
    auto& api = NcclApi::get();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const auto& m : msgs) {
      nccl_check(api.Send(m.send, m.bytes, ncclChar, m.peer_send, comm(), s), "ncclSend");
      nccl_check(api.Recv(m.recv, m.bytes, ncclChar, m.peer_recv, comm(), s), "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
  void barrier(int rank) override {
    cudaStream_t s;
    LBCU_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    allreduce(rank, scratch_, 1, s);
    LBCU_CUDA(cudaStreamSynchronize(s));
    LBCU_CUDA(cudaStreamDestroy(s));
  }

 private:
  int n_, rank_;
  ncclUniqueId uid_;
  ncclComm_t comm_ = nullptr;
  double* scratch_ = nullptr;
};

}  // namespace

std::unique_ptr<Transport> make_single_transport() { return std::make_unique<SingleTransport>(); }
std::unique_ptr<Transport> make_thread_transport(int n) {
  if (n < 1) throw Error(LBCU_CONFIG_ERROR, "thread world needs >= 1 rank");
  return std::make_unique<ThreadTransport>(n);
}
std::unique_ptr<Transport> make_nccl_transport(int n, int rank, const unsigned char id[128]) {
  return std::make_unique<NcclTransport>(n, rank, id);
}
void nccl_unique_id(unsigned char id[128]) {
  ncclUniqueId uid;
  nccl_check(NcclApi::get().GetUniqueId(&uid), "ncclGetUniqueId");
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &uid, sizeof(uid));
}

}  // namespace lbcu
