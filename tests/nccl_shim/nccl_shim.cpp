// Test transport for libtanq's multi-process path: the NCCL calls libtanq makes (unique id,
// comm init/destroy, grouped send/recv, all-reduce sum/max), implemented through host memory
// (an mmap'ed file + process-shared semaphores).  NCCL refuses several ranks on one device
// ("Duplicate GPU detected"); with this shim (TANQ_NCCL_LIB=.../libnccl_shim.so) every rank
// can keep its shard on the same GPU, so the library's own exchange logic -- remap schedule,
// half selection, chunked pack / unpack kernels, bit-map bookkeeping, all-reduced
// probabilities / expectations / state gathers -- runs on hardware (tests/test_gpu_dist.py).
// Test infrastructure only: semantics are NCCL's for the calls used (stream-ordered: every call
// synchronises the caller's stream first, copies on it, and completes before returning);
// nothing is fast.  `g++ -DSHIM_HOST_TEST` builds a CPU variant for the shim's own self-test
// (tests/test_nccl_shim.py).
#include <cuda_runtime.h>
#ifdef SHIM_HOST_TEST  // CPU self-test build (no GPU): "device" buffers are host buffers
static inline cudaError_t shim_memcpy(void* d, const void* s, size_t n, cudaMemcpyKind) {
  __builtin_memcpy(d, s, n);
  return cudaSuccess;
}
static inline cudaError_t shim_memcpy_async(void* d, const void* s, size_t n, cudaMemcpyKind k,
                                            cudaStream_t) {
  return shim_memcpy(d, s, n, k);
}
static inline cudaError_t shim_sync(cudaStream_t) { return cudaSuccess; }
#define cudaMemcpyAsync shim_memcpy_async
#define cudaStreamSynchronize shim_sync
#endif
#include <fcntl.h>
#include <nccl.h>
#include <pthread.h>
#include <semaphore.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr uint32_t kMagic = 0x7a4e5348u;

struct Shared {
  std::atomic<uint32_t> magic;
  int nranks;
  size_t slot;                              // bytes per mailbox
  pthread_barrier_t bar;
  sem_t full[kMaxRanks][kMaxRanks];         // [src][dst]
  sem_t empty[kMaxRanks][kMaxRanks];
  size_t len[kMaxRanks][kMaxRanks];
};

struct Comm {
  Shared* sh = nullptr;
  size_t map_bytes = 0;
  int rank = 0, nranks = 0;
  char* base = nullptr;                      // mailboxes [src][dst], then all-reduce slots [r]
  char path[sizeof(ncclUniqueId) + 1];
  char* box(int src, int dst) { return base + ((size_t)src * kMaxRanks + dst) * sh->slot; }
  char* ar(int r) { return base + ((size_t)kMaxRanks * kMaxRanks + r) * sh->slot; }
};

struct PendingOp {
  bool send;
  char* dev;
  size_t bytes;
  int peer;
  Comm* comm;
  cudaStream_t stream;
};

// Host <-> device copy on the caller's stream, complete on return.  (A plain cudaMemcpy from
// pageable memory may return before its DMA lands, and the caller's non-blocking stream would
// not wait for it.)
cudaError_t copy_sync(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(dst, src, n, kind, st);
  return e != cudaSuccess ? e : cudaStreamSynchronize(st);
}
thread_local int g_group = 0;
thread_local std::vector<PendingOp> g_ops;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t run_ops(std::vector<PendingOp>& ops) {
  // chunk-interleaved so that pairwise exchanges larger than one mailbox cannot deadlock
  size_t maxb = 0;
  for (auto& o : ops) maxb = o.bytes > maxb ? o.bytes : maxb;
  if (ops.empty()) return ncclSuccess;
  const size_t slot = ops[0].comm->sh->slot;
  for (size_t off = 0; off < maxb; off += slot) {
    for (auto& o : ops) {
      if (!o.send || off >= o.bytes) continue;
      Comm* c = o.comm;
      const size_t n = o.bytes - off < slot ? o.bytes - off : slot;
      sem_wait(&c->sh->empty[c->rank][o.peer]);
      if (copy_sync(c->box(c->rank, o.peer), o.dev + off, n, cudaMemcpyDeviceToHost, o.stream) !=
          cudaSuccess)
        return ncclUnhandledCudaError;
      c->sh->len[c->rank][o.peer] = n;
      sem_post(&c->sh->full[c->rank][o.peer]);
    }
    for (auto& o : ops) {
      if (o.send || off >= o.bytes) continue;
      Comm* c = o.comm;
      sem_wait(&c->sh->full[o.peer][c->rank]);
      const size_t n = c->sh->len[o.peer][c->rank];
      if (copy_sync(o.dev + off, c->box(o.peer, c->rank), n, cudaMemcpyHostToDevice, o.stream) !=
          cudaSuccess)
        return ncclUnhandledCudaError;
      sem_post(&c->sh->empty[o.peer][c->rank]);
    }
  }
  ops.clear();
  return ncclSuccess;
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  return r == ncclSuccess ? "success (shim)" : "error (tanq nccl shim)";
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<int> counter{0};
  memset(id, 0, sizeof(*id));
  snprintf(id->internal, sizeof(id->internal), "/tmp/tanq_nccl_shim_%d_%d", (int)getpid(),
           counter.fetch_add(1));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  Comm* c = new Comm;
  c->rank = rank;
  c->nranks = nranks;
  snprintf(c->path, sizeof(c->path), "%s", id.internal);
  const char* mb = getenv("TANQ_SHIM_SLOT_MB");
  const size_t slot = (size_t)(mb ? atoi(mb) : 1) << 20;
  const size_t bytes = 8192 + (size_t)(kMaxRanks * kMaxRanks + kMaxRanks) * slot;
  int fd = -1;
  if (rank == 0) {
    fd = open(c->path, O_RDWR | O_CREAT | O_EXCL, 0600);
    if (fd < 0 || ftruncate(fd, (off_t)bytes) != 0) return ncclSystemError;
  } else {
    for (int i = 0; i < 60000 && fd < 0; ++i) {
      fd = open(c->path, O_RDWR);
      if (fd < 0) usleep(1000);
    }
    if (fd < 0) return ncclSystemError;
    struct stat st;
    for (int i = 0; i < 60000; ++i) {
      if (fstat(fd, &st) == 0 && (size_t)st.st_size >= bytes) break;
      usleep(1000);
    }
  }
  void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) return ncclSystemError;
  c->sh = static_cast<Shared*>(m);
  c->map_bytes = bytes;
  c->base = static_cast<char*>(m) + 8192;
  static_assert(sizeof(Shared) <= 8192, "header pages");
  if (rank == 0) {
    c->sh->nranks = nranks;
    c->sh->slot = slot;
    pthread_barrierattr_t ba;
    pthread_barrierattr_init(&ba);
    pthread_barrierattr_setpshared(&ba, PTHREAD_PROCESS_SHARED);
    pthread_barrier_init(&c->sh->bar, &ba, (unsigned)nranks);
    for (int a = 0; a < kMaxRanks; ++a)
      for (int b = 0; b < kMaxRanks; ++b) {
        sem_init(&c->sh->full[a][b], 1, 0);
        sem_init(&c->sh->empty[a][b], 1, 1);
      }
    c->sh->magic.store(kMagic);
  } else {
    for (int i = 0; i < 60000 && c->sh->magic.load() != kMagic; ++i) usleep(1000);
    if (c->sh->magic.load() != kMagic) return ncclSystemError;
  }
  pthread_barrier_wait(&c->sh->bar);
  if (rank == 0) unlink(c->path);  // every rank has it mapped
  *out = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return ncclSuccess;
  pthread_barrier_wait(&c->sh->bar);
  munmap(c->sh, c->map_bytes);
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_group;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_group > 0 && --g_group == 0) return run_ops(g_ops);
  return ncclSuccess;
}

static ncclResult_t p2p(bool send, const void* buf, size_t count, ncclDataType_t t, int peer,
                        ncclComm_t comm, cudaStream_t stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c || peer < 0 || peer >= c->nranks) return ncclInvalidArgument;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
  g_ops.push_back({send, static_cast<char*>(const_cast<void*>(buf)), count * type_size(t), peer, c,
                   stream});
  return g_group ? ncclSuccess : run_ops(g_ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return p2p(true, buf, count, t, peer, comm, stream);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return p2p(false, buf, count, t, peer, comm, stream);
}

ncclResult_t ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t t,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return ncclInvalidArgument;
  if ((t != ncclFloat64 && t != ncclUint64) || (op != ncclSum && op != ncclMax))
    return ncclInvalidArgument;
  if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
  const size_t bytes = count * 8, slot = c->sh->slot & ~(size_t)7;
  std::vector<char> acc(slot);
  for (size_t off = 0; off < bytes; off += slot) {
    const size_t n = bytes - off < slot ? bytes - off : slot;
    if (copy_sync(c->ar(c->rank), static_cast<const char*>(sendbuf) + off, n,
                  cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return ncclUnhandledCudaError;
    pthread_barrier_wait(&c->sh->bar);
    for (size_t i = 0; i < n / 8; ++i) {  // rank order: deterministic
      if (t == ncclFloat64) {
        double v = 0.0;
        for (int r = 0; r < c->nranks; ++r) {
          const double x = reinterpret_cast<const double*>(c->ar(r))[i];
          v = r == 0 ? x : (op == ncclSum ? v + x : (x > v ? x : v));
        }
        reinterpret_cast<double*>(acc.data())[i] = v;
      } else {
        uint64_t v = 0;
        for (int r = 0; r < c->nranks; ++r) {
          const uint64_t x = reinterpret_cast<const uint64_t*>(c->ar(r))[i];
          v = r == 0 ? x : (op == ncclSum ? v + x : (x > v ? x : v));
        }
        reinterpret_cast<uint64_t*>(acc.data())[i] = v;
      }
    }
    pthread_barrier_wait(&c->sh->bar);  // every rank has read the slots
    if (copy_sync(static_cast<char*>(recvbuf) + off, acc.data(), n, cudaMemcpyHostToDevice,
                  stream) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  return ncclSuccess;
}

}  // extern "C"
