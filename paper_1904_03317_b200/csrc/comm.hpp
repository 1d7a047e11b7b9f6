// Inter-rank communication of the level exchanges (ghost import / export-add)
// and CG reductions ("communication ... only involves neighboring
// processors", P:836-845 transfer ghosts).  Two transports with one interface:
//  * NcclComm   one process per GPU, grouped ncclSend/ncclRecv + ncclAllReduce
//               (libnccl loaded at run time: the same libnccl.so.2 torch uses)
//  * ThreadComm all ranks in one process (one host thread + stream per rank,
//               same device): host barriers + event-ordered D2D copies; kernels
//               never wait on each other.  Used to test the multi-rank logic on
//               one GPU.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace gmg {

struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // Exchange one contiguous chunk per peer: to peers[i] send sendbuf[soff[i], soff[i+1]),
  // from peers[i] receive into recvbuf[roff[i], roff[i+1]) -- offsets in elements of
  // esize bytes (8: fp64, 4: fp32 wire format).  Stream-ordered.
  virtual void exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff,
                        void* recvbuf, const std::vector<i64>& roff, size_t esize, cudaStream_t s) = 0;
  // in-place sum over ranks of n doubles (device memory), stream-ordered
  virtual void allreduce(double* buf, int n, cudaStream_t s) = 0;
  virtual bool capturable() const = 0;   // may be captured in a CUDA graph
};

// ---------------------------------------------------------------- threads
struct LocalWorld {
  explicit LocalWorld(int n);
  ~LocalWorld();
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  void barrier();
  struct Slot {
    const void* sendbuf = nullptr;
    const std::vector<int>* peers = nullptr;
    const std::vector<i64>* soff = nullptr;
    cudaEvent_t packed = nullptr, copied = nullptr;
    double* red = nullptr;      // pinned host scratch for reductions
    int device = 0;
  };
  std::vector<Slot> slot;
};

struct ThreadComm : Comm {
  ThreadComm(LocalWorld* w, int r) : w(w), r(r) {}
  LocalWorld* w;
  int r;
  int rank() const override { return r; }
  int size() const override { return w->n; }
  void exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff, void* recvbuf,
                const std::vector<i64>& roff, size_t esize, cudaStream_t s) override;
  void allreduce(double* buf, int n, cudaStream_t s) override;
  bool capturable() const override { return false; }
};

// ---------------------------------------------------------------- processes, host-staged
// n ranks as separate processes (any GPUs, e.g. all on one device): a POSIX
// shared-memory segment holds a sense-free generation barrier and one slot per
// rank; an exchange is D2H of the packed send buffer into the own slot (the
// segment is cudaHostRegister'ed), a barrier, H2D of every peer's chunk from the
// peer's slot, a stream synchronise and a second barrier.  Kernels never wait on
// each other; not capturable.  A test transport for the multi-process path on a
// one-GPU machine (bench.py --transport host), not a performance path.
struct HostWorld {
  HostWorld(const char* name, int n, int rank, size_t slot_bytes);
  ~HostWorld();
  int n, rank;
  size_t slot_bytes = 0, total = 0;
  std::string name;
  unsigned char* base = nullptr;
  bool registered = false;
  void barrier();
  // slot q: [directory: n x (offset, count) as i64][payload doubles]
  i64* dir(int q) const { return (i64*)(base + 4096 + (size_t)q * slot_bytes); }
  double* payload(int q) const { return (double*)(base + 4096 + (size_t)q * slot_bytes + 16 * (size_t)n); }
  size_t payload_bytes() const { return slot_bytes - 16 * (size_t)n; }
  size_t payload_cap() const { return payload_bytes() / sizeof(double); }
};

struct HostComm : Comm {
  explicit HostComm(HostWorld* w) : w(w) {}
  HostWorld* w;
  int rank() const override { return w->rank; }
  int size() const override { return w->n; }
  void exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff, void* recvbuf,
                const std::vector<i64>& roff, size_t esize, cudaStream_t s) override;
  void allreduce(double* buf, int n, cudaStream_t s) override;
  bool capturable() const override { return false; }
};

// ---------------------------------------------------------------- NCCL
struct NcclComm : Comm {
  explicit NcclComm(void* comm);
  void* comm;
  int r = 0, n = 1;
  int rank() const override { return r; }
  int size() const override { return n; }
  void exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff, void* recvbuf,
                const std::vector<i64>& roff, size_t esize, cudaStream_t s) override;
  void allreduce(double* buf, int n, cudaStream_t s) override;
  bool capturable() const override { return true; }
};

// NCCL bootstrap helpers (dlopen'ed libnccl)
void nccl_unique_id(char out[128]);
void* nccl_comm_init(const char id[128], int nranks, int rank);
void nccl_comm_destroy(void* comm);

}  // namespace gmg
