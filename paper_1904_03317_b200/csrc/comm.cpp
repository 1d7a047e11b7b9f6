// Communication transports (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>

#include <cstdlib>
#include <string>

namespace gmg {

#define CKC(x)                                                                                  \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) fail(GMG_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));   \
  } while (0)

// ---------------------------------------------------------------- threads
LocalWorld::LocalWorld(int n_) : n(n_), slot(n_) {
  for (auto& s : slot) {
    CKC(cudaEventCreateWithFlags(&s.packed, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
    CKC(cudaMallocHost(&s.red, 4096 * sizeof(double)));
  }
}
LocalWorld::~LocalWorld() {
  for (auto& s : slot) {
    if (s.packed) cudaEventDestroy(s.packed);
    if (s.copied) cudaEventDestroy(s.copied);
    if (s.red) cudaFreeHost(s.red);
  }
}
void LocalWorld::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const long long gen = generation;
  if (++arrived == n) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

void ThreadComm::exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff,
                          void* recvbuf, const std::vector<i64>& roff, size_t esize, cudaStream_t s) {
  auto& me = w->slot[r];
  me.sendbuf = sendbuf;
  me.peers = &peers;
  me.soff = &soff;
  CKC(cudaEventRecord(me.packed, s));
  w->barrier();                       // every rank has packed and published
  for (size_t i = 0; i < peers.size(); ++i) {
    const int q = peers[i];
    const auto& other = w->slot[q];
    const auto& op = *other.peers;
    size_t j = 0;
    while (j < op.size() && op[j] != r) ++j;
    GMG_REQUIRE(j < op.size(), GMG_E_STATE, "asymmetric exchange plan");
    const i64 cnt = (*other.soff)[j + 1] - (*other.soff)[j];
    GMG_REQUIRE(cnt == roff[i + 1] - roff[i], GMG_E_STATE, "exchange count mismatch");
    if (cnt == 0) continue;
    CKC(cudaStreamWaitEvent(s, other.packed, 0));
    CKC(cudaMemcpyAsync((char*)recvbuf + roff[i] * esize, (const char*)other.sendbuf + (*other.soff)[j] * esize,
                        cnt * esize, cudaMemcpyDeviceToDevice, s));
  }
  CKC(cudaEventRecord(me.copied, s));
  w->barrier();                       // every rank has enqueued its copies
  for (int q : peers) CKC(cudaStreamWaitEvent(s, w->slot[q].copied, 0));
  w->barrier();                       // nobody republishes before all waits are enqueued
}

void ThreadComm::allreduce(double* buf, int n, cudaStream_t s) {
  GMG_REQUIRE(n <= 4096, GMG_E_INVALID_ARG, "allreduce size");
  auto& me = w->slot[r];
  CKC(cudaMemcpyAsync(me.red, buf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  w->barrier();
  std::vector<double> sum(n, 0.0);
  for (int q = 0; q < w->n; ++q)           // same order on every rank: identical sums
    for (int i = 0; i < n; ++i) sum[i] += w->slot[q].red[i];
  w->barrier();
  for (int i = 0; i < n; ++i) me.red[i] = sum[i];
  CKC(cudaMemcpyAsync(buf, me.red, n * sizeof(double), cudaMemcpyHostToDevice, s));
  CKC(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- processes (shared memory)
namespace {
struct ShmHdr {                       // zero-initialised by ftruncate: a valid initial state
  std::atomic<long long> arrived;
  std::atomic<long long> generation;
};
}  // namespace

HostWorld::HostWorld(const char* nm, int n_, int r, size_t slot) : n(n_), rank(r), name(nm) {
  GMG_REQUIRE(n_ >= 1 && r >= 0 && r < n_, GMG_E_INVALID_ARG, "host world rank/size");
  GMG_REQUIRE(nm && nm[0] == '/', GMG_E_INVALID_ARG, "host world name must start with '/'");
  slot_bytes = (std::max<size_t>(slot, 1 << 16) + 4095) / 4096 * 4096;
  total = 4096 + slot_bytes * (size_t)n_;
  const int fd = shm_open(nm, O_CREAT | O_RDWR, 0600);
  GMG_REQUIRE(fd >= 0, GMG_E_STATE, std::string("shm_open ") + nm + ": " + std::strerror(errno));
  struct stat st;
  if (fstat(fd, &st) == 0 && (size_t)st.st_size < total && ftruncate(fd, (off_t)total) != 0) {
    close(fd);
    fail(GMG_E_OOM, std::string("ftruncate of the host world: ") + std::strerror(errno));
  }
  void* m = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  GMG_REQUIRE(m != MAP_FAILED, GMG_E_OOM, std::string("mmap of the host world: ") + std::strerror(errno));
  base = (unsigned char*)m;
  registered = cudaHostRegister(base, total, cudaHostRegisterDefault) == cudaSuccess;
  if (!registered) cudaGetLastError();   // fall back to pageable copies
  barrier();                             // every rank has mapped the segment
}

HostWorld::~HostWorld() {
  if (!base) return;
  try {
    barrier();                           // nobody still reads a slot
  } catch (...) {
  }
  if (registered) cudaHostUnregister(base);
  munmap(base, total);
  if (rank == 0) shm_unlink(name.c_str());
}

void HostWorld::barrier() {
  auto* h = (ShmHdr*)base;
  const long long gen = h->generation.load(std::memory_order_acquire);
  if (h->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
    h->arrived.store(0, std::memory_order_relaxed);
    h->generation.fetch_add(1, std::memory_order_release);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  long spins = 0;
  while (h->generation.load(std::memory_order_acquire) == gen) {
    if (++spins > 1000) {
      sched_yield();
      if ((spins & 0xffff) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
        fail(GMG_E_STATE, "host world barrier: a rank did not arrive within 600 s");
    }
  }
}

void HostComm::exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff,
                        void* recvbuf, const std::vector<i64>& roff, size_t esize, cudaStream_t s) {
  const int me = w->rank;
  i64* dir = w->dir(me);
  for (int q = 0; q < w->n; ++q) dir[2 * q] = dir[2 * q + 1] = 0;
  const i64 ns = soff.empty() ? 0 : soff.back();
  GMG_REQUIRE((size_t)ns * esize <= w->payload_bytes(), GMG_E_OOM, "host world slot too small for an exchange");
  for (size_t i = 0; i < peers.size(); ++i) {
    dir[2 * peers[i]] = soff[i];
    dir[2 * peers[i] + 1] = soff[i + 1] - soff[i];
  }
  if (ns) CKC(cudaMemcpyAsync(w->payload(me), sendbuf, ns * esize, cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  w->barrier();                       // every slot is written
  for (size_t i = 0; i < peers.size(); ++i) {
    const int q = peers[i];
    const i64* od = w->dir(q);
    const i64 cnt = od[2 * me + 1];
    GMG_REQUIRE(cnt == roff[i + 1] - roff[i], GMG_E_STATE, "exchange count mismatch");
    if (cnt)
      CKC(cudaMemcpyAsync((char*)recvbuf + roff[i] * esize, (const char*)w->payload(q) + od[2 * me] * esize,
                          cnt * esize, cudaMemcpyHostToDevice, s));
  }
  CKC(cudaStreamSynchronize(s));
  w->barrier();                       // every slot is read: it may be rewritten
}

void HostComm::allreduce(double* buf, int cnt, cudaStream_t s) {
  GMG_REQUIRE((size_t)cnt <= w->payload_cap(), GMG_E_INVALID_ARG, "allreduce size");
  CKC(cudaMemcpyAsync(w->payload(w->rank), buf, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
  CKC(cudaStreamSynchronize(s));
  w->barrier();
  std::vector<double> sum(cnt, 0.0);
  for (int q = 0; q < w->n; ++q)      // same order on every rank: identical sums
    for (int i = 0; i < cnt; ++i) sum[i] += w->payload(q)[i];
  w->barrier();
  CKC(cudaMemcpyAsync(buf, sum.data(), cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  CKC(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef int ncclResult_t;
typedef void* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
constexpr int ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0;
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(ncclComm_t, int*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char* env = std::getenv("GMG_NCCL_LIB");
  const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c) continue;
    api.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  GMG_REQUIRE(api.h, GMG_E_NCCL, "cannot dlopen libnccl.so.2 (set GMG_NCCL_LIB)");
  auto sym = [&](const char* n) {
    void* p = dlsym(api.h, n);
    GMG_REQUIRE(p, GMG_E_NCCL, std::string("libnccl lacks ") + n);
    return p;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.CommCount = (decltype(api.CommCount))sym("ncclCommCount");
  api.CommUserRank = (decltype(api.CommUserRank))sym("ncclCommUserRank");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  return api;
}
void ckn(ncclResult_t r, const char* what) {
  if (r != 0) fail(GMG_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

NcclComm::NcclComm(void* c) : comm(c) {
  ckn(nccl().CommUserRank(comm, &r), "ncclCommUserRank");
  ckn(nccl().CommCount(comm, &n), "ncclCommCount");
}

void NcclComm::exchange(const std::vector<int>& peers, const void* sendbuf, const std::vector<i64>& soff,
                        void* recvbuf, const std::vector<i64>& roff, size_t esize, cudaStream_t s) {
  if (peers.empty()) return;
  auto& a = nccl();
  const int dt = esize == 4 ? ncclFloat32 : ncclFloat64;
  GMG_REQUIRE(esize == 4 || esize == 8, GMG_E_INVALID_ARG, "wire element size");
  ckn(a.GroupStart(), "ncclGroupStart");
  for (size_t i = 0; i < peers.size(); ++i) {
    const i64 sc = soff[i + 1] - soff[i], rc = roff[i + 1] - roff[i];
    if (sc) ckn(a.Send((const char*)sendbuf + soff[i] * esize, (size_t)sc, dt, peers[i], comm, s), "ncclSend");
    if (rc) ckn(a.Recv((char*)recvbuf + roff[i] * esize, (size_t)rc, dt, peers[i], comm, s), "ncclRecv");
  }
  ckn(a.GroupEnd(), "ncclGroupEnd");
}

void NcclComm::allreduce(double* buf, int cnt, cudaStream_t s) {
  ckn(nccl().AllReduce(buf, buf, (size_t)cnt, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
}

void nccl_unique_id(char out[128]) {
  ncclUniqueId id;
  ckn(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}
void* nccl_comm_init(const char id[128], int nranks, int rank) {
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  ckn(nccl().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  return c;
}
void nccl_comm_destroy(void* c) {
  if (c) nccl().CommDestroy(c);
}

}  // namespace gmg
