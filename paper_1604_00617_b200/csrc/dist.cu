// Transports for the sharded ACR path (see dist.h).
#include <dlfcn.h>
#include <chrono>
#include <cstring>
#include <nccl.h>
#include <stdexcept>

#include "dist.h"

namespace acr {

// ---------------------------------------------------------------------------
// loopback (virtual ranks = threads of one process)
// ---------------------------------------------------------------------------
struct LoopbackTransport : Transport {
  LoopbackHub* hub;
  int r;
  std::map<int, long long> sseq, rseq;
  LoopbackTransport(LoopbackHub* h, int rank) : hub(h), r(rank) {}
  int rank() const override { return r; }
  int size() const override { return hub->P; }

  void exchange(const std::vector<Msg>& msgs, cudaStream_t st) override {
    std::vector<std::tuple<int, int, long long>> mine;
    // publish sends
    for (const Msg& m : msgs) {
      if (!m.send) continue;
      auto key = std::make_tuple(r, m.peer, sseq[m.peer]++);
      LoopbackHub::Slot s;
      s.ptr = m.ptr;
      s.bytes = m.bytes;
      cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
      cudaEventRecord(s.ready, st);
      {
        std::lock_guard<std::mutex> g(hub->mu);
        hub->slots[key] = s;
      }
      mine.push_back(key);
    }
    hub->cv.notify_all();
    // receives: wait for the matching send, copy on our stream
    for (const Msg& m : msgs) {
      if (m.send) continue;
      auto key = std::make_tuple(m.peer, r, rseq[m.peer]++);
      std::unique_lock<std::mutex> lk(hub->mu);
      if (!hub->cv.wait_for(lk, std::chrono::seconds(120),
                            [&] { return hub->slots.count(key) > 0; }))
        throw std::runtime_error("loopback: receive timed out (schedule mismatch)");
      LoopbackHub::Slot& s = hub->slots[key];
      if (s.bytes != m.bytes) throw std::runtime_error("loopback size mismatch");
      cudaStreamWaitEvent(st, s.ready, 0);
      cudaMemcpyAsync(m.ptr, s.ptr, m.bytes, cudaMemcpyDeviceToDevice, st);
      cudaEventRecord(s.done, st);
      s.finished = true;
      lk.unlock();
      hub->cv.notify_all();
    }
    // our sends: later reuse of the buffers is ordered after the peer's copy
    for (auto& key : mine) {
      std::unique_lock<std::mutex> lk(hub->mu);
      if (!hub->cv.wait_for(lk, std::chrono::seconds(120),
                            [&] { return hub->slots[key].finished; }))
        throw std::runtime_error("loopback: send not consumed (schedule mismatch)");
      LoopbackHub::Slot s = hub->slots[key];
      hub->slots.erase(key);
      lk.unlock();
      cudaStreamWaitEvent(st, s.done, 0);
      cudaEventSynchronize(s.done);
      cudaEventDestroy(s.ready);
      cudaEventDestroy(s.done);
    }
  }

  long long allreduce_max(long long v, cudaStream_t st) override {
    cudaStreamSynchronize(st);
    std::unique_lock<std::mutex> lk(hub->mu);
    const long long my_gen = hub->gen;
    hub->acc = hub->arrived == 0 ? v : (v > hub->acc ? v : hub->acc);
    if (++hub->arrived == hub->P) {
      hub->result = hub->acc;
      hub->arrived = 0;
      hub->gen++;
      hub->cv.notify_all();
    } else {
      if (!hub->cv.wait_for(lk, std::chrono::seconds(120),
                            [&] { return hub->gen != my_gen; }))
        throw std::runtime_error("loopback: all-reduce timed out (schedule mismatch)");
    }
    return hub->result;
  }
};

Transport* make_loopback(LoopbackHub* hub, int rank) {
  return new LoopbackTransport(hub, rank);
}

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed)
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load(std::string* err) {
    if (h) return true;
    // prefer an already-loaded NCCL (torch's), then the usual names
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (h) break;
    }
    for (const char* nm : names) {
      if (h) break;
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      *err = "cannot load libnccl.so.2";
      return false;
    }
#define LOAD(f, s) f = reinterpret_cast<decltype(f)>(dlsym(h, s))
    LOAD(GetUniqueId, "ncclGetUniqueId");
    LOAD(CommInitRank, "ncclCommInitRank");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(AllReduce, "ncclAllReduce");
    LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    if (!GetUniqueId || !CommInitRank || !Send || !Recv || !GroupStart || !GroupEnd ||
        !AllReduce) {
      *err = "libnccl is missing symbols";
      return false;
    }
    return true;
  }
};
static NcclApi g_nccl;

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int r, P;
  long long* dval = nullptr;
  NcclTransport(ncclComm_t c, int rank, int n) : comm(c), r(rank), P(n) {
    cudaMalloc(&dval, sizeof(long long));
  }
  ~NcclTransport() override {
    if (comm && g_nccl.CommDestroy) g_nccl.CommDestroy(comm);
    if (dval) cudaFree(dval);
  }
  int rank() const override { return r; }
  int size() const override { return P; }
  void check(ncclResult_t e) {
    if (e != ncclSuccess)
      throw std::runtime_error(std::string("NCCL: ") +
                               (g_nccl.GetErrorString ? g_nccl.GetErrorString(e) : "error"));
  }
  void exchange(const std::vector<Msg>& msgs, cudaStream_t st) override {
    if (msgs.empty()) return;
    check(g_nccl.GroupStart());
    for (const Msg& m : msgs) {
      if (m.send) check(g_nccl.Send(m.ptr, m.bytes, ncclChar, m.peer, comm, st));
      else check(g_nccl.Recv(m.ptr, m.bytes, ncclChar, m.peer, comm, st));
    }
    check(g_nccl.GroupEnd());
  }
  long long allreduce_max(long long v, cudaStream_t st) override {
    cudaMemcpyAsync(dval, &v, sizeof(v), cudaMemcpyHostToDevice, st);
    check(g_nccl.AllReduce(dval, dval, 1, ncclInt64, ncclMax, comm, st));
    long long out = 0;
    cudaMemcpyAsync(&out, dval, sizeof(out), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return out;
  }
};

int nccl_unique_id(void* out, std::string* err) {
  if (!g_nccl.load(err)) return 1;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) {
    *err = "ncclGetUniqueId failed";
    return 1;
  }
  memcpy(out, &id, sizeof(id));
  return 0;
}

Transport* make_nccl(const void* unique_id, int rank, int nranks, std::string* err) {
  if (!g_nccl.load(err)) return nullptr;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm;
  ncclResult_t e = g_nccl.CommInitRank(&comm, nranks, id, rank);
  if (e != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") +
           (g_nccl.GetErrorString ? g_nccl.GetErrorString(e) : "error");
    return nullptr;
  }
  return new NcclTransport(comm, rank, nranks);
}

}  // namespace acr
