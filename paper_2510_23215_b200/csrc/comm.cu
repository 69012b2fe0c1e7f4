// comm.cu — the exchange steps of the row-partitioned solve (SURVEY §8(a)
// row a11; BASELINE.json configs[4]): halo rows between slab neighbours and
// fp64 all-reduce / all-gather of the small Gram / projection / norm blocks.
//
// Two backends behind one interface (scsf::Comm, comm.cuh):
//  - NCCL over NVLink/NVSwitch, one process per GPU.  libnccl is the one torch
//    already loaded into the process (dlopen by soname, symbols by dlsym), so
//    no link-time dependency; the communicator is built from a 128-byte
//    ncclUniqueId the caller broadcasts (torch.distributed).  All calls are
//    stream-ordered on the solver's stream.
//  - loopback: `world` virtual ranks inside one process on one device, each
//    driven by its own host thread (tests and single-GPU parity of the
//    partitioned path).  Every collective synchronises the caller's stream,
//    meets the other ranks at a host barrier and reduces / copies in rank
//    order, so results are bitwise identical on all ranks.  No kernel ever
//    waits on another rank (B200_PROFILING: never spin across launches).
#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

namespace scsf {

// ------------------------------------------------------------------- NCCL ----
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SCSF_SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
    SCSF_SYM(GetUniqueId);
    SCSF_SYM(CommInitRank);
    SCSF_SYM(CommDestroy);
    SCSF_SYM(AllReduce);
    SCSF_SYM(AllGather);
    SCSF_SYM(Send);
    SCSF_SYM(Recv);
    SCSF_SYM(GroupStart);
    SCSF_SYM(GroupEnd);
    SCSF_SYM(GetErrorString);
#undef SCSF_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
             api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  return api;
}

#define SCSF_NCCL_CHECK(expr)                                                                  \
  do {                                                                                         \
    ncclResult_t r_ = (expr);                                                                  \
    if (r_ != ncclSuccess) {                                                                   \
      set_error("%s: NCCL error %d (%s)", #expr, (int)r_,                                      \
                nccl().GetErrorString ? nccl().GetErrorString(r_) : "?");                      \
      return SCSF_ERR_DEVICE;                                                                  \
    }                                                                                          \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  int allreduce_sum(double* buf, size_t count, cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_NCCL_CHECK(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, s));
    return SCSF_OK;
  }
  int allreduce_max_u64(unsigned long long* buf, size_t count, cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_NCCL_CHECK(nccl().AllReduce(buf, buf, count, ncclUint64, ncclMax, comm, s));
    return SCSF_OK;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    if (world == 1) {
      if (recv != send) SCSF_CUDA_CHECK(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, s));
      return SCSF_OK;
    }
    SCSF_NCCL_CHECK(nccl().AllGather(send, recv, count, ncclFloat64, comm, s));
    return SCSF_OK;
  }
  int halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, size_t count,
           cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_NCCL_CHECK(nccl().GroupStart());
    if (rank > 0) {
      SCSF_NCCL_CHECK(nccl().Send(send_lo, count, ncclFloat64, rank - 1, comm, s));
      SCSF_NCCL_CHECK(nccl().Recv(recv_lo, count, ncclFloat64, rank - 1, comm, s));
    }
    if (rank + 1 < world) {
      SCSF_NCCL_CHECK(nccl().Send(send_hi, count, ncclFloat64, rank + 1, comm, s));
      SCSF_NCCL_CHECK(nccl().Recv(recv_hi, count, ncclFloat64, rank + 1, comm, s));
    }
    SCSF_NCCL_CHECK(nccl().GroupEnd());
    return SCSF_OK;
  }
};
}  // namespace

// --------------------------------------------------------------- loopback ----
namespace {
// Sum of the same slot of `world` buffers in rank order (bitwise identical on every rank).
__global__ void k_sum_ranks(double* const* bufs, int world, size_t count, double* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = bufs[0][i];
    for (int r = 1; r < world; ++r) s += bufs[r][i];
    out[i] = s;
  }
}
__global__ void k_max_ranks(unsigned long long* const* bufs, int world, size_t count, unsigned long long* out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long m = bufs[0][i];
    for (int r = 1; r < world; ++r) m = bufs[r][i] > m ? bufs[r][i] : m;
    out[i] = m;
  }
}

struct LoopGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> slot_a, slot_b;
  void** dev_table = nullptr;        // device copy of slot_a (per collective)
  int refs;
  explicit LoopGroup(int w) : world(w), slot_a(w), slot_b(w), refs(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct LoopComm final : Comm {
  LoopGroup* g = nullptr;
  void** table = nullptr;            // device array of `world` pointers (this rank's copy)
  double* tmp = nullptr;             // device scratch for reductions
  size_t tmp_count = 0;
  ~LoopComm() override {
    if (table) cudaFree(table);
    if (tmp) cudaFree(tmp);
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = (--g->refs == 0);
    }
    if (last) delete g;
  }
  int ensure_tmp(size_t count) {
    if (count <= tmp_count) return SCSF_OK;
    if (tmp) cudaFree(tmp);
    tmp = nullptr;
    SCSF_CUDA_CHECK(cudaMalloc(&tmp, count * sizeof(double)));
    tmp_count = count;
    return SCSF_OK;
  }
  // publish `p`, wait for every rank, copy the table of all ranks' pointers to the device
  int gather_ptrs(const void* p, cudaStream_t s) {
    g->slot_a[rank] = p;
    g->barrier();
    SCSF_CUDA_CHECK(cudaMemcpyAsync(table, g->slot_a.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, s));
    return SCSF_OK;
  }
  int allreduce_sum(double* buf, size_t count, cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_TRY(ensure_tmp(count));
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    SCSF_TRY(gather_ptrs(buf, s));
    k_sum_ranks<<<(int)((count + 255) / 256 < 1024 ? (count + 255) / 256 : 1024), 256, 0, s>>>(
        reinterpret_cast<double* const*>(table), world, count, tmp);
    SCSF_LAUNCH_CHECK();
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->barrier();                      // every rank has read every buffer
    SCSF_CUDA_CHECK(cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return SCSF_OK;
  }
  int allreduce_max_u64(unsigned long long* buf, size_t count, cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_TRY(ensure_tmp(count));
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    SCSF_TRY(gather_ptrs(buf, s));
    k_max_ranks<<<1, 256, 0, s>>>(reinterpret_cast<unsigned long long* const*>(table), world, count,
                                  reinterpret_cast<unsigned long long*>(tmp));
    SCSF_LAUNCH_CHECK();
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->barrier();
    SCSF_CUDA_CHECK(cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return SCSF_OK;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->slot_a[rank] = send;
    g->barrier();
    for (int r = 0; r < world; ++r)
      SCSF_CUDA_CHECK(cudaMemcpyAsync(recv + (size_t)r * count, g->slot_a[r], count * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->barrier();
    return SCSF_OK;
  }
  int halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, size_t count,
           cudaStream_t s) override {
    if (world == 1 || count == 0) return SCSF_OK;
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->slot_a[rank] = send_lo;
    g->slot_b[rank] = send_hi;
    g->barrier();
    // my lower ghosts are the lower neighbour's top boundary rows, and vice versa
    if (rank > 0)
      SCSF_CUDA_CHECK(cudaMemcpyAsync(recv_lo, g->slot_b[rank - 1], count * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    if (rank + 1 < world)
      SCSF_CUDA_CHECK(cudaMemcpyAsync(recv_hi, g->slot_a[rank + 1], count * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    g->barrier();                      // send buffers may be overwritten after this
    return SCSF_OK;
  }
};
}  // namespace

int comm_unique_id(void* id128) {
  if (!nccl().ok) {
    set_error("NCCL not available (libnccl.so.2 could not be loaded)");
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  SCSF_NCCL_CHECK(nccl().GetUniqueId(&id));
  memcpy(id128, &id, sizeof(id));
  return SCSF_OK;
}

int comm_create_nccl(int rank, int world, const void* id128, Comm** out) {
  if (!nccl().ok) {
    set_error("NCCL not available (libnccl.so.2 could not be loaded)");
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  auto* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank failed: %d", (int)r);
    delete c;
    return SCSF_ERR_DEVICE;
  }
  *out = c;
  return SCSF_OK;
}

int comm_create_loopback(int world, Comm** out) {
  auto* g = new LoopGroup(world);
  for (int r = 0; r < world; ++r) {
    auto* c = new LoopComm();
    c->rank = r;
    c->world = world;
    c->g = g;
    if (cudaMalloc(&c->table, sizeof(void*) * world) != cudaSuccess) {
      set_error("loopback comm: cudaMalloc failed");
      return SCSF_ERR_DEVICE;
    }
    out[r] = c;
  }
  return SCSF_OK;
}

}  // namespace scsf
