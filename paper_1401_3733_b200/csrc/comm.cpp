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
//   ipc     : one process per GPU on one node, direct halos: every rank maps
//             the peers' receive arenas (cudaIpcOpenMemHandle) and the halo
//             pack kernel stores its records straight into them over NVLink;
//             completion travels as an interprocess CUDA event per exchange,
//             recorded after the pack and waited on (stream-ordered) before
//             the boundary kernel. A host barrier in a POSIX shared-memory
//             segment separates the record and the wait of each exchange, so
//             no kernel ever spins on another rank. The thread world has the
//             same direct mode (one process, plain pointers) for testing.
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <map>
#include <thread>

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
  ThreadTransport(int n, bool direct) : n_(n), direct_(direct), contrib_(n), posted_(n), events_(n) {}
  ~ThreadTransport() override {
    for (auto& ev : events_)
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    for (auto& kv : arenas_)  // the world owns the receive arenas (map_arena)
      for (void* a : kv.second)
        if (a) cudaFree(a);
  }
  int nranks() const override { return n_; }
  bool capturable() const override { return false; }

  // ---- direct mode (peer arenas are plain device pointers in one process)
  bool direct() const override { return direct_.load(std::memory_order_acquire); }
  // one thread flips the shared mode; callers bracket it with barriers so no
  // rank is inside an exchange (test_direct_halo_toggle_matches)
  void set_direct(bool on) override { direct_.store(on, std::memory_order_release); }
  void attach(int rank, int) override {  // events exist even if direct mode is switched on later
    for (auto& e : events_[rank])
      if (!e) LBCU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // Collective. The world takes ownership of `local` (freed at teardown);
  // re-mapping a key (a new context on the same world) frees the rank's old
  // arena once every rank has switched to the new ones.
  void map_arena(int rank, int key, void* local, size_t) override {
    void* old = nullptr;
    {
      std::lock_guard<std::mutex> lk(m_);
      auto& v = arenas_[key];
      if (v.empty()) v.assign(n_, nullptr);
      old = v[rank];
      v[rank] = local;
    }
    sync();
    if (old && old != local) cudaFree(old);
  }
  void* peer_arena(int, int key, int peer) const override {
    std::lock_guard<std::mutex> lk(m_);
    auto it = arenas_.find(key);
    return it == arenas_.end() ? nullptr : it->second[peer];
  }
  void post(int rank, long long epoch, cudaStream_t s) override {
    LBCU_CUDA(cudaEventRecord(events_[rank][epoch & 1], s));
  }
  void await(int, long long epoch, const std::vector<int>& peers, cudaStream_t s) override {
    sync();  // every rank has recorded this epoch's event
    for (int q : peers) LBCU_CUDA(cudaStreamWaitEvent(s, events_[q][epoch & 1], 0));
  }

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
  std::atomic<bool> direct_;
  mutable std::mutex m_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t phase_ = 0;
  std::vector<std::vector<double>> contrib_;
  std::vector<std::vector<Msg>> posted_;
  std::vector<std::array<cudaEvent_t, 2>> events_;
  std::map<int, std::vector<void*>> arenas_;
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

// ---- one process per GPU, peer-memory halos through CUDA IPC ---------------
constexpr int kIpcMaxRanks = 8;  // one node
constexpr int kIpcMaxKeys = 16;  // arenas (one per representation dimension)
constexpr int kIpcMaxSum = 8;    // doubles per host-path allreduce
constexpr uint64_t kIpcMagic = 0x6c6263752d697063ULL;

struct IpcShared {
  std::atomic<uint64_t> magic;
  std::atomic<uint32_t> arrive;
  std::atomic<uint32_t> gen;
  std::atomic<uint32_t> attached;
  cudaIpcEventHandle_t ev[kIpcMaxRanks][2];
  cudaIpcMemHandle_t mem[kIpcMaxKeys][kIpcMaxRanks];
  double sum[kIpcMaxRanks][kIpcMaxSum];
};

struct IpcTransport final : Transport {
  IpcTransport(int n, int rank, const char* name, const unsigned char* nccl_id) : n_(n), rank_(rank), name_(name) {
    if (n < 1 || n > kIpcMaxRanks) throw Error(LBCU_CONFIG_ERROR, "ipc world: 1..8 ranks on one node");
    if (rank < 0 || rank >= n) throw Error(LBCU_CONTRACT_VIOLATION, "ipc world: rank out of range");
    if (!name || name[0] != '/') throw Error(LBCU_CONFIG_ERROR, "ipc world: segment name must start with '/'");
    if (nccl_id) inner_ = make_nccl_transport(n, rank, nccl_id);
    const size_t bytes = sizeof(IpcShared);
    int fd = -1;
    if (rank == 0) {
      shm_unlink(name);  // a stale segment of an earlier run
      fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, bytes) != 0) throw Error(LBCU_TRANSPORT_ERROR, "ipc world: shm_open/ftruncate failed");
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while ((fd = shm_open(name, O_RDWR, 0600)) < 0) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw Error(LBCU_TRANSPORT_ERROR, "ipc world: rank 0 never created the segment");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(LBCU_TRANSPORT_ERROR, "ipc world: mmap failed");
    sh_ = static_cast<IpcShared*>(p);
    if (rank == 0) {
      sh_->arrive.store(0);
      sh_->gen.store(0);
      sh_->attached.store(0);
      sh_->magic.store(kIpcMagic, std::memory_order_release);
    } else {
      wait_until([&] { return sh_->magic.load(std::memory_order_acquire) == kIpcMagic; });
    }
    sh_->attached.fetch_add(1);
    wait_until([&] { return sh_->attached.load() == static_cast<uint32_t>(n_); });
    host_barrier();
    if (rank == 0) shm_unlink(name);  // every rank holds the mapping now
  }
  ~IpcTransport() override {
    // collective teardown: nobody closes its mappings while a peer may still
    // be inside a collective call (bounded wait, never throws)
    if (sh_) bounded_barrier();
    for (auto& kv : peer_mem_)
      for (int q = 0; q < static_cast<int>(kv.second.size()); ++q)
        if (q != rank_ && kv.second[q]) cudaIpcCloseMemHandle(kv.second[q]);
    for (int q = 0; q < n_; ++q)
      for (int e = 0; e < 2; ++e)
        if (ev_[q][e]) cudaEventDestroy(ev_[q][e]);
    // an exported arena is freed only after every importer closed it
    if (sh_ && !own_arenas_.empty()) bounded_barrier();
    for (auto& kv : own_arenas_) cudaFree(kv.second);
    if (sh_) munmap(sh_, sizeof(IpcShared));
  }
  int nranks() const override { return n_; }
  bool capturable() const override { return false; }
  bool direct() const override { return direct_; }
  void set_direct(bool on) override {
    if (!on && !inner_) throw Error(LBCU_TRANSPORT_ERROR, "ipc world without NCCL: halos must be direct");
    direct_ = on;
  }
  void bind_device(int device) override {
    if (inner_) inner_->bind_device(device);
  }
  void attach(int rank, int) override {
    if (attached_) return;
    for (int e = 0; e < 2; ++e) {
      LBCU_CUDA(cudaEventCreateWithFlags(&ev_[rank][e], cudaEventDisableTiming | cudaEventInterprocess));
      LBCU_CUDA(cudaIpcGetEventHandle(&sh_->ev[rank][e], ev_[rank][e]));
    }
    host_barrier();
    for (int q = 0; q < n_; ++q)
      if (q != rank)
        for (int e = 0; e < 2; ++e) LBCU_CUDA(cudaIpcOpenEventHandle(&ev_[q][e], sh_->ev[q][e]));
    host_barrier();
    attached_ = true;
  }
  // Collective. The world owns `local` from here on: it is freed at world
  // teardown, or when the key is re-mapped (a new context on the same world)
  // after every peer has closed its mapping of the old arena.
  void map_arena(int rank, int key, void* local, size_t) override {
    if (key < 0 || key >= kIpcMaxKeys) throw Error(LBCU_TRANSPORT_ERROR, "ipc world: arena key out of range");
    LBCU_CUDA(cudaIpcGetMemHandle(&sh_->mem[key][rank], local));
    host_barrier();
    auto& v = peer_mem_[key];
    for (int q = 0; q < static_cast<int>(v.size()); ++q)  // a previous context's arenas
      if (q != rank && v[q]) cudaIpcCloseMemHandle(v[q]);
    v.assign(n_, nullptr);
    for (int q = 0; q < n_; ++q)
      if (q != rank)
        LBCU_CUDA(cudaIpcOpenMemHandle(&v[q], sh_->mem[key][q], cudaIpcMemLazyEnablePeerAccess));
    v[rank] = local;
    host_barrier();
    void*& mine = own_arenas_[key];
    if (mine && mine != local) cudaFree(mine);  // every peer closed it before the barrier
    mine = local;
  }
  void* peer_arena(int, int key, int peer) const override {
    auto it = peer_mem_.find(key);
    return it == peer_mem_.end() ? nullptr : it->second[peer];
  }
  void post(int rank, long long epoch, cudaStream_t s) override {
    LBCU_CUDA(cudaEventRecord(ev_[rank][epoch & 1], s));
  }
  void await(int, long long epoch, const std::vector<int>& peers, cudaStream_t s) override {
    host_barrier();  // every rank has recorded this epoch's event
    for (int q : peers) LBCU_CUDA(cudaStreamWaitEvent(s, ev_[q][epoch & 1], 0));
  }
  void allreduce(int rank, double* dev, int n, cudaStream_t s) override {
    if (n_ == 1) return;
    if (inner_) return inner_->allreduce(rank, dev, n, s);
    if (n > kIpcMaxSum) throw Error(LBCU_TRANSPORT_ERROR, "ipc world: host sum of more than 8 values");
    double loc[kIpcMaxSum];
    LBCU_CUDA(cudaMemcpyAsync(loc, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    LBCU_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < n; ++k) sh_->sum[rank][k] = loc[k];
    host_barrier();
    for (int k = 0; k < n; ++k) loc[k] = tree(k, 0, n_);  // fixed order on every rank
    host_barrier();
    LBCU_CUDA(cudaMemcpyAsync(dev, loc, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    LBCU_CUDA(cudaStreamSynchronize(s));
  }
  void exchange(int rank, const std::vector<Msg>& msgs, cudaStream_t s) override {
    if (!inner_) throw Error(LBCU_TRANSPORT_ERROR, "ipc world: message exchange needs NCCL");
    inner_->exchange(rank, msgs, s);
  }
  void barrier(int) override { host_barrier(); }

 private:
  template <class F>
  void wait_until(F&& ready) {
    const auto t0 = std::chrono::steady_clock::now();
    unsigned spins = 0;
    while (!ready()) {
      if (++spins > 4096) {
        sched_yield();
        if ((spins & 0xffff) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
          throw Error(LBCU_TRANSPORT_ERROR, "ipc world: host barrier timed out");
      }
    }
  }
  // teardown barrier: bounded wait, never throws
  void bounded_barrier() {
    const uint32_t g = sh_->gen.load(std::memory_order_acquire);
    if (sh_->arrive.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(n_)) {
      sh_->arrive.store(0, std::memory_order_relaxed);
      sh_->gen.fetch_add(1, std::memory_order_release);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    while (sh_->gen.load(std::memory_order_acquire) == g &&
           std::chrono::steady_clock::now() - t0 < std::chrono::seconds(30))
      sched_yield();
  }
  // generation barrier over the shared segment
  void host_barrier() {
    const uint32_t g = sh_->gen.load(std::memory_order_acquire);
    if (sh_->arrive.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(n_)) {
      sh_->arrive.store(0, std::memory_order_relaxed);
      sh_->gen.fetch_add(1, std::memory_order_release);
      return;
    }
    wait_until([&] { return sh_->gen.load(std::memory_order_acquire) != g; });
  }
  double tree(int k, int lo, int hi) const {
    if (hi - lo == 1) return sh_->sum[lo][k];
    const int mid = lo + (hi - lo) / 2;
    return tree(k, lo, mid) + tree(k, mid, hi);
  }
  int n_, rank_;
  std::string name_;
  IpcShared* sh_ = nullptr;
  std::unique_ptr<Transport> inner_;
  cudaEvent_t ev_[kIpcMaxRanks][2] = {};
  bool attached_ = false;
  bool direct_ = true;
  std::map<int, std::vector<void*>> peer_mem_;
  std::map<int, void*> own_arenas_;  // this rank's receive arenas, by key
};

}  // namespace

std::unique_ptr<Transport> make_single_transport() { return std::make_unique<SingleTransport>(); }
std::unique_ptr<Transport> make_thread_transport(int n, bool direct) {
  if (n < 1) throw Error(LBCU_CONFIG_ERROR, "thread world needs >= 1 rank");
  return std::make_unique<ThreadTransport>(n, direct);
}
std::unique_ptr<Transport> make_ipc_transport(int n, int rank, const char* name, const unsigned char* nccl_id) {
  return std::make_unique<IpcTransport>(n, rank, name, nccl_id);
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
