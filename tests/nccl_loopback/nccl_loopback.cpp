// In-process NCCL stand-in for the tests (test infrastructure, not part of the product): the
// ranks of a communicator are host threads of ONE process on ONE device, so the library's
// NCCL code paths (position / permutation broadcasts, slab send/recv transposes, phase-barrier
// and divergence all-reduces, the grid all-reduce mode, the peer-route handle exchange) run
// on a single GPU, where real NCCL refuses two ranks on one device ("Duplicate GPU").
//
// libtfdp.so resolves NCCL with dlopen; TFDP_NCCL_LIB=<this .so> makes it load this one.
// Semantics: every call of a rank enqueues nothing on its stream until all ranks of the
// communicator made the matching call (host rendezvous, calls matched in issue order as NCCL
// requires); the last rank to arrive then makes a private stream wait for every rank's stream
// (an event recorded at its call), moves the data (device copies; reductions on the host),
// synchronises, and every rank's stream waits for that before its next work.  Groups
// (ncclGroupStart/End) collect a rank's calls and rendezvous once at the outermost GroupEnd.
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <vector>

namespace {

enum Kind { kBcast, kAllRed, kSend, kRecv };
struct Op {
  Kind kind;
  const void* send;
  void* recv;
  size_t bytes;
  ncclDataType_t dt;
  ncclRedOp_t red;
  int peer;  // root (broadcast) or peer (send / recv)
};

struct Group;

}  // namespace

struct ncclComm {
  Group* g;
  int rank;
};

namespace {

struct Group {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int joined = 0;
  int live = 0;
  uint64_t gen = 0;
  int arrived = 0;
  std::vector<std::vector<Op>> slots;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t done = nullptr;
  cudaStream_t cs = nullptr;
  ncclResult_t last = ncclSuccess;
};

std::mutex g_reg_m;
std::map<uint64_t, Group*> g_reg;

thread_local int t_depth = 0;
thread_local ncclComm_t t_comm = nullptr;
thread_local cudaStream_t t_stream = nullptr;
thread_local std::vector<Op> t_pending;

size_t dt_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;  // int64, uint64, float64
  }
}

template <class T>
void reduce_into(T* acc, const T* x, size_t n, ncclRedOp_t op) {
  for (size_t i = 0; i < n; ++i) {
    switch (op) {
      case ncclSum: acc[i] = acc[i] + x[i]; break;
      case ncclProd: acc[i] = acc[i] * x[i]; break;
      case ncclMin: acc[i] = x[i] < acc[i] ? x[i] : acc[i]; break;
      case ncclMax: acc[i] = x[i] > acc[i] ? x[i] : acc[i]; break;
      default: break;
    }
  }
}

void reduce_bytes(void* acc, const void* x, size_t bytes, ncclDataType_t t, ncclRedOp_t op) {
  switch (t) {
    case ncclInt8: reduce_into((int8_t*)acc, (const int8_t*)x, bytes, op); break;
    case ncclUint8: reduce_into((uint8_t*)acc, (const uint8_t*)x, bytes, op); break;
    case ncclInt32: reduce_into((int32_t*)acc, (const int32_t*)x, bytes / 4, op); break;
    case ncclUint32: reduce_into((uint32_t*)acc, (const uint32_t*)x, bytes / 4, op); break;
    case ncclInt64: reduce_into((int64_t*)acc, (const int64_t*)x, bytes / 8, op); break;
    case ncclUint64: reduce_into((uint64_t*)acc, (const uint64_t*)x, bytes / 8, op); break;
    case ncclFloat32: reduce_into((float*)acc, (const float*)x, bytes / 4, op); break;
    case ncclFloat64: reduce_into((double*)acc, (const double*)x, bytes / 8, op); break;
    default: break;
  }
}

#define LB_CUDA(x)                          \
  do {                                      \
    if ((x) != cudaSuccess) return ncclUnhandledCudaError; \
  } while (0)

// Executes one matched rendezvous (called by the last rank to arrive, lock held).
ncclResult_t execute(Group& g) {
  for (int r = 0; r < g.n; ++r) LB_CUDA(cudaStreamWaitEvent(g.cs, g.ev[r], 0));
  // collectives: the i-th collective call of every rank belong together
  std::vector<std::vector<const Op*>> coll(g.n);
  for (int r = 0; r < g.n; ++r)
    for (const Op& o : g.slots[r])
      if (o.kind == kBcast || o.kind == kAllRed) coll[r].push_back(&o);
  for (int r = 1; r < g.n; ++r)
    if (coll[r].size() != coll[0].size()) return ncclInvalidUsage;
  for (size_t i = 0; i < coll[0].size(); ++i) {
    const Op& o0 = *coll[0][i];
    for (int r = 1; r < g.n; ++r)
      if (coll[r][i]->kind != o0.kind || coll[r][i]->bytes != o0.bytes) return ncclInvalidUsage;
    if (o0.kind == kBcast) {
      const void* src = coll[o0.peer][i]->send;
      for (int r = 0; r < g.n; ++r)
        if (coll[r][i]->recv != src)
          LB_CUDA(cudaMemcpyAsync(coll[r][i]->recv, src, o0.bytes, cudaMemcpyDeviceToDevice, g.cs));
    } else {
      std::vector<unsigned char> acc(o0.bytes), x(o0.bytes);
      LB_CUDA(cudaMemcpyAsync(acc.data(), coll[0][i]->send, o0.bytes, cudaMemcpyDeviceToHost, g.cs));
      LB_CUDA(cudaStreamSynchronize(g.cs));
      for (int r = 1; r < g.n; ++r) {
        LB_CUDA(cudaMemcpyAsync(x.data(), coll[r][i]->send, o0.bytes, cudaMemcpyDeviceToHost, g.cs));
        LB_CUDA(cudaStreamSynchronize(g.cs));
        reduce_bytes(acc.data(), x.data(), o0.bytes, o0.dt, o0.red);
      }
      for (int r = 0; r < g.n; ++r)
        LB_CUDA(cudaMemcpyAsync(coll[r][i]->recv, acc.data(), o0.bytes, cudaMemcpyHostToDevice, g.cs));
      LB_CUDA(cudaStreamSynchronize(g.cs));
    }
  }
  // point to point: rank s's j-th send to d matches rank d's j-th receive from s
  for (int s = 0; s < g.n; ++s) {
    std::map<int, int> seen;
    for (const Op& o : g.slots[s]) {
      if (o.kind != kSend) continue;
      const int d = o.peer, j = seen[d]++;
      int cnt = 0;
      const Op* match = nullptr;
      for (const Op& q : g.slots[d])
        if (q.kind == kRecv && q.peer == s && cnt++ == j) {
          match = &q;
          break;
        }
      if (!match || match->bytes != o.bytes) return ncclInvalidUsage;
      LB_CUDA(cudaMemcpyAsync(match->recv, o.send, o.bytes, cudaMemcpyDeviceToDevice, g.cs));
    }
  }
  for (int d = 0; d < g.n; ++d) {  // every receive must have been matched by a send
    std::map<int, int> want;
    for (const Op& o : g.slots[d])
      if (o.kind == kRecv) want[o.peer]++;
    for (auto& kv : want) {
      int have = 0;
      for (const Op& o : g.slots[kv.first])
        if (o.kind == kSend && o.peer == d) have++;
      if (have != kv.second) return ncclInvalidUsage;
    }
  }
  LB_CUDA(cudaStreamSynchronize(g.cs));
  LB_CUDA(cudaEventRecord(g.done, g.cs));
  return ncclSuccess;
}

ncclResult_t rendezvous(ncclComm_t c, cudaStream_t s, std::vector<Op> ops) {
  Group& g = *c->g;
  std::unique_lock<std::mutex> lk(g.m);
  const uint64_t my = g.gen;
  if (cudaEventRecord(g.ev[c->rank], s) != cudaSuccess) return ncclUnhandledCudaError;
  g.slots[c->rank] = std::move(ops);
  if (++g.arrived == g.n) {
    g.last = execute(g);
    g.arrived = 0;
    g.gen++;
    g.cv.notify_all();
  } else {
    g.cv.wait(lk, [&] { return g.gen != my; });
  }
  if (g.last != ncclSuccess) return g.last;
  return cudaStreamWaitEvent(s, g.done, 0) == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t submit(ncclComm_t c, cudaStream_t s, const Op& o) {
  if (!c) return ncclInvalidArgument;
  if (t_depth > 0) {
    if (t_comm && t_comm != c) return ncclInvalidUsage;  // (one communicator per group here)
    t_comm = c;
    t_stream = s;
    t_pending.push_back(o);
    return ncclSuccess;
  }
  return rendezvous(c, s, {o});
}

uint64_t key_of(const ncclUniqueId& id) {
  uint64_t k;
  memcpy(&k, id.internal, sizeof k);
  return k;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::mutex m;
  static std::mt19937_64 rng{std::random_device{}()};
  std::lock_guard<std::mutex> lk(m);
  memset(id, 0, sizeof *id);
  const uint64_t k = rng();
  memcpy(id->internal, &k, sizeof k);
  memcpy(id->internal + 8, "LOOPBACK", 8);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  Group* g;
  {
    std::lock_guard<std::mutex> lk(g_reg_m);
    Group*& slot = g_reg[key_of(id)];
    if (!slot) {
      slot = new Group;
      slot->n = nranks;
      slot->slots.resize(nranks);
      slot->ev.resize(nranks, nullptr);
    }
    g = slot;
  }
  if (g->n != nranks) return ncclInvalidUsage;
  std::unique_lock<std::mutex> lk(g->m);
  if (cudaEventCreateWithFlags(&g->ev[rank], cudaEventDisableTiming) != cudaSuccess)
    return ncclUnhandledCudaError;
  g->live++;
  if (++g->joined == nranks) {  // the last rank to join creates the shared resources
    if (cudaStreamCreateWithFlags(&g->cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(g->done, g->cs) != cudaSuccess)
      return ncclUnhandledCudaError;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->joined == g->n; });
  }
  *comm = new ncclComm{g, rank};
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  if (!comm) return ncclInvalidArgument;
  Group* g = comm->g;
  bool last;
  {
    std::lock_guard<std::mutex> lk(g->m);
    last = --g->live == 0;
  }
  if (last) {
    {
      std::lock_guard<std::mutex> lk(g_reg_m);
      for (auto it = g_reg.begin(); it != g_reg.end(); ++it)
        if (it->second == g) {
          g_reg.erase(it);
          break;
        }
    }
    for (cudaEvent_t e : g->ev) cudaEventDestroy(e);
    cudaEventDestroy(g->done);
    cudaStreamDestroy(g->cs);
    delete g;
  }
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  t_depth++;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (t_depth <= 0) return ncclInvalidUsage;
  if (--t_depth > 0 || t_pending.empty()) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(t_pending);
  ncclComm_t c = t_comm;
  t_comm = nullptr;
  return rendezvous(c, t_stream, std::move(ops));
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t dt, int root,
                           ncclComm_t comm, cudaStream_t s) {
  if (!comm || root < 0 || root >= comm->g->n) return ncclInvalidArgument;
  return submit(comm, s, Op{kBcast, send, recv, count * dt_size(dt), dt, ncclSum, root});
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  return submit(comm, s, Op{kAllRed, send, recv, count * dt_size(dt), dt, op, 0});
}

ncclResult_t ncclSend(const void* send, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  if (!comm || peer < 0 || peer >= comm->g->n) return ncclInvalidArgument;
  return submit(comm, s, Op{kSend, send, nullptr, count * dt_size(dt), dt, ncclSum, peer});
}

ncclResult_t ncclRecv(void* recv, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  if (!comm || peer < 0 || peer >= comm->g->n) return ncclInvalidArgument;
  return submit(comm, s, Op{kRecv, nullptr, recv, count * dt_size(dt), dt, ncclSum, peer});
}

const char* ncclGetErrorString(ncclResult_t r) {
  return r == ncclSuccess ? "success (loopback)" : "loopback NCCL stand-in error";
}

}  // extern "C"
