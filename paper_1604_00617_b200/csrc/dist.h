// Transport for the sharded factor/solve.
//
// Ranks own contiguous block-row ranges; per reduction level a rank sends its
// first even block's {Dinv, E, F} to its left neighbour and, in the solve,
// one n x k vector per boundary.  Two implementations:
//   NcclTransport     one process per GPU, ncclSend/ncclRecv on the plan's
//                     stream (NCCL is dlopen'ed: the torch-bundled libnccl when
//                     torch is loaded, else the system one)
//   LoopbackTransport virtual ranks as threads of one process (tests on one
//                     GPU): a send publishes (pointer, ready event); the
//                     receiver's stream waits on it and copies D2D; the
//                     sender's stream then waits on the copy's event.
#pragma once
#include <cuda_runtime.h>
#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

namespace acr {

struct Msg {
  int peer;
  void* ptr;
  size_t bytes;
  bool send;
};

struct Transport {
  virtual ~Transport() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // a group of point-to-point transfers, ordered on `st`
  virtual void exchange(const std::vector<Msg>& msgs, cudaStream_t st) = 0;
  // max of a host integer over all ranks (synchronises `st`)
  virtual long long allreduce_max(long long v, cudaStream_t st) = 0;
};

struct LoopbackHub {
  struct Slot {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;
    cudaEvent_t done = nullptr;
    bool taken = false;
    bool finished = false;
  };
  int P;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::tuple<int, int, long long>, Slot> slots;
  // all-reduce state
  long long gen = 0;
  int arrived = 0;
  long long acc = 0, result = 0;
  explicit LoopbackHub(int p) : P(p) {}
};

Transport* make_loopback(LoopbackHub* hub, int rank);
Transport* make_nccl(const void* unique_id, int rank, int nranks, std::string* err);
int nccl_unique_id(void* out, std::string* err);   // 128 bytes

}  // namespace acr
