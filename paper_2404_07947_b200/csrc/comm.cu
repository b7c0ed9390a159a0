// Transports of comm.h: NCCL (one process per GPU) and a thread-rank
// transport for single-device tests.
#include "comm.h"

#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace exg {

// ------------------------------------------------------------------ NCCL ---
namespace {
#define EXG_NCCL(x)                                                                               \
  do {                                                                                            \
    ncclResult_t r_ = (x);                                                                        \
    if (r_ != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + ncclGetErrorString(r_)); \
  } while (0)

class NcclComm final : public Comm {
 public:
  NcclComm(const uint8_t uid[128], int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId id;
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
    std::memcpy(id.internal, uid, 128);
    EXG_NCCL(ncclCommInitRank(&comm_, world, id, rank));
  }
  ~NcclComm() override {
    for (auto& kv : sub_)
      if (kv.second) ncclCommDestroy(kv.second);
    if (comm_) ncclCommDestroy(comm_);
  }
  void prepare_groups(const std::vector<std::vector<int>>& groups) override {
    for (const auto& g : groups) {
      if (g.size() < 2 || sub_.count(g)) continue;
      bool member = false;
      for (int r : g) member |= r == rank_;
      // every rank takes part in the split; non-members get no communicator
      ncclComm_t c = nullptr;
      EXG_NCCL(ncclCommSplit(comm_, member ? split_color(g) : NCCL_SPLIT_NOCOLOR, rank_, &c, nullptr));
      sub_[g] = c;
    }
  }
  bool has_allreduce() const override { return true; }
  void allreduce_sum(float* buf, size_t n, const std::vector<int>& group, cudaStream_t st) override {
    auto it = sub_.find(group);
    if (it == sub_.end() || !it->second) throw std::logic_error("NCCL: TP group was not prepared");
    EXG_NCCL(ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, it->second, st));
  }
  void check_async() override {
    auto one = [](ncclComm_t c) {
      ncclResult_t a = ncclSuccess;
      if (c && ncclCommGetAsyncError(c, &a) == ncclSuccess && a != ncclSuccess && a != ncclInProgress)
        throw std::runtime_error(std::string("NCCL async error: ") + ncclGetErrorString(a));
    };
    one(comm_);
    for (auto& kv : sub_) one(kv.second);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void group_start() override { EXG_NCCL(ncclGroupStart()); }
  void group_end() override { EXG_NCCL(ncclGroupEnd()); }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t st) override {
    EXG_NCCL(ncclSend(buf, bytes, ncclUint8, peer, comm_, st));
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t st) override {
    EXG_NCCL(ncclRecv(buf, bytes, ncclUint8, peer, comm_, st));
  }

 private:
  // the same color on every member: a hash of the member list
  static int split_color(const std::vector<int>& g) {
    uint32_t h = 2166136261u;
    for (int r : g) h = (h ^ (uint32_t)r) * 16777619u;
    return (int)(h & 0x3fffffff);
  }
  ncclComm_t comm_ = nullptr;
  int rank_, world_;
  std::map<std::vector<int>, ncclComm_t> sub_;
};
}  // namespace

void nccl_unique_id(uint8_t uid[128]) {
  ncclUniqueId id;
  EXG_NCCL(ncclGetUniqueId(&id));
  std::memcpy(uid, id.internal, 128);
}

std::unique_ptr<Comm> make_nccl_comm(const uint8_t uid[128], int rank, int world) {
  return std::make_unique<NcclComm>(uid, rank, world);
}

// ---------------------------------------------------------- thread ranks ---
// A send and the matching recv (k-th send src->dst with the k-th recv at dst
// from src) rendezvous in the hub.  Whichever side posts second enqueues, on
// the receiver's stream: wait(event "data ready" of the sender's stream),
// copy, record "copied"; the sender's stream then waits for "copied" before
// it may overwrite the buffer -- the stream-level semantics of a blocking
// NCCL send / recv, with the host threads rendezvousing at each op.
struct LocalHub {
  struct Op {
    const void* src = nullptr;
    void* dst = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;      // poster's stream
    cudaEvent_t ready = nullptr;    // send: data ready on the sender's stream
    cudaEvent_t copied = nullptr;   // set by the pairing: copy done on the receiver's stream
    bool paired = false;
    std::string err;
  };
  explicit LocalHub(int w) : world(w) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<Op*>> sends, recvs;   // key (src, dst)

  void pair(Op* s, Op* r) {
    try {
      if (s->bytes != r->bytes) throw std::runtime_error("LocalComm: send/recv size mismatch");
      EXG_CUDA(cudaStreamWaitEvent(r->st, s->ready, 0));
      if (s->bytes) EXG_CUDA(cudaMemcpyAsync(r->dst, s->src, s->bytes, cudaMemcpyDeviceToDevice, r->st));
      EXG_CUDA(cudaEventCreateWithFlags(&s->copied, cudaEventDisableTiming));
      EXG_CUDA(cudaEventRecord(s->copied, r->st));
    } catch (const std::exception& e) {
      s->err = r->err = e.what();
    }
    s->paired = r->paired = true;
  }
  void post(int me, Op* op, bool is_send, int peer) {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = is_send ? std::make_pair(me, peer) : std::make_pair(peer, me);
    auto& other = is_send ? recvs[key] : sends[key];
    if (!other.empty()) {
      Op* o = other.front();
      other.pop_front();
      if (is_send)
        pair(op, o);
      else
        pair(o, op);
      cv.notify_all();
    } else {
      (is_send ? sends[key] : recvs[key]).push_back(op);
    }
  }
  void wait(Op* op) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return op->paired; });
  }
};

namespace {
class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  ~LocalComm() override { drain(); }
  int rank() const override { return rank_; }
  int world() const override { return hub_->world; }
  void group_start() override { ++depth_; }
  void group_end() override {
    if (--depth_ == 0) complete();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t st) override {
    check_peer(peer);
    auto op = std::make_unique<LocalHub::Op>();
    op->src = buf;
    op->bytes = bytes;
    op->st = st;
    EXG_CUDA(cudaEventCreateWithFlags(&op->ready, cudaEventDisableTiming));
    EXG_CUDA(cudaEventRecord(op->ready, st));
    hub_->post(rank_, op.get(), true, peer);
    pending_.push_back({std::move(op), true});
    if (depth_ == 0) complete();
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t st) override {
    check_peer(peer);
    auto op = std::make_unique<LocalHub::Op>();
    op->dst = buf;
    op->bytes = bytes;
    op->st = st;
    hub_->post(rank_, op.get(), false, peer);
    pending_.push_back({std::move(op), false});
    if (depth_ == 0) complete();
  }

 private:
  struct Pending {
    std::unique_ptr<LocalHub::Op> op;
    bool is_send;
  };
  void check_peer(int peer) const {
    if (peer < 0 || peer >= hub_->world || peer == rank_) throw std::invalid_argument("LocalComm: bad peer");
  }
  void complete() {
    std::string err;
    for (auto& p : pending_) {
      hub_->wait(p.op.get());
      if (!p.op->err.empty()) err = p.op->err;
      if (p.is_send && p.op->copied) EXG_CUDA(cudaStreamWaitEvent(p.op->st, p.op->copied, 0));
      done_.push_back(std::move(p.op));
    }
    pending_.clear();
    // events of completed ops are released once the stream has passed them
    if (done_.size() > 256) drain();
    if (!err.empty()) throw std::runtime_error(err);
  }
  void drain() {
    for (auto& op : done_) {
      if (op->copied) cudaEventSynchronize(op->copied);
      if (op->ready) cudaEventDestroy(op->ready);
      if (op->copied) cudaEventDestroy(op->copied);
    }
    done_.clear();
  }
  std::shared_ptr<LocalHub> hub_;
  int rank_;
  int depth_ = 0;
  std::vector<Pending> pending_;
  std::vector<std::unique_ptr<LocalHub::Op>> done_;
};
}  // namespace

std::shared_ptr<LocalHub> make_local_hub(int world) { return std::make_shared<LocalHub>(world); }

std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalHub> hub, int rank) {
  return std::make_unique<LocalComm>(std::move(hub), rank);
}

}  // namespace exg
