// comm.cu — the transports of the multi-GPU path (include/vr.h "Multi-GPU"): NCCL
// communicators (one process per GPU, or one process over several GPUs with
// ncclCommInitAll) and an in-process group whose ranks are host threads sharing one GPU.
// Collectives act on device buffers, ordered on the caller's stream.
#include <condition_variable>
#include <cstdlib>
#include <dlfcn.h>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/vr.h"
#include "vr_internal.h"

namespace {

// ------------------------------------------------------------------ NCCL, loaded at first use
// libvr does not link NCCL: a process that also uses torch must keep ONE libnccl.so.2, the one
// torch brings (loading the system copy first breaks torch's import).  The library resolves
// NCCL when the first communicator is made: the already-loaded libnccl.so.2 if any, else
// $VR_NCCL_LIB (the Python binding points it at the wheel torch uses), else libnccl.so.2.
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      const char* env = std::getenv("VR_NCCL_LIB");
      if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommInitAll = (decltype(api.CommInitAll))dlsym(h, "ncclCommInitAll");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommInitAll && api.AllReduce && api.AllGather && api.Broadcast &&
             api.CommDestroy && api.GetErrorString;
  });
  return api;
}
int nccl_missing() {
  vr::set_last_error("NCCL could not be loaded (libnccl.so.2; set VR_NCCL_LIB)");
  return VR_EDEVICE;
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  bool own = true;
};
int nccl_rc(ncclResult_t r) {
  if (r == ncclSuccess) return VR_OK;
  vr::set_last_error(std::string("NCCL: ") + nccl().GetErrorString(r));
  return VR_EDEVICE;
}
int nccl_allreduce(void* ctx, uint64_t* buf, int64_t n, void* stream) {
  if (n <= 0) return VR_OK;
  return nccl_rc(nccl().AllReduce(buf, buf, (size_t)n, ncclUint64, ncclSum, ((NcclCtx*)ctx)->comm, (cudaStream_t)stream));
}
int nccl_allgather(void* ctx, const uint64_t* send, uint64_t* recv, int64_t n_each, void* stream) {
  if (n_each <= 0) return VR_OK;
  return nccl_rc(nccl().AllGather(send, recv, (size_t)n_each, ncclUint64, ((NcclCtx*)ctx)->comm, (cudaStream_t)stream));
}
int nccl_bcast(void* ctx, uint64_t* buf, int64_t n, int32_t root, void* stream) {
  if (n <= 0) return VR_OK;
  return nccl_rc(nccl().Broadcast(buf, buf, (size_t)n, ncclUint64, root, ((NcclCtx*)ctx)->comm, (cudaStream_t)stream));
}
void nccl_destroy(void* ctx) {
  NcclCtx* c = (NcclCtx*)ctx;
  if (c->comm && c->own) nccl().CommDestroy(c->comm);
  delete c;
}
vr_comm* wrap_nccl(ncclComm_t comm, int rank, int world) {
  vr_comm* v = new vr_comm{};
  NcclCtx* c = new NcclCtx();
  c->comm = comm;
  v->ctx = c;
  v->rank = rank;
  v->world = world;
  v->allreduce_sum_u64 = nccl_allreduce;
  v->allgather_u64 = nccl_allgather;
  v->broadcast_u64 = nccl_bcast;
  v->destroy = nccl_destroy;
  return v;
}

// ------------------------------------------------------------------ in-process group
// Ranks are host threads (each with its own stream on the shared device).  A collective:
// every rank stages its device data in a host slot, a barrier, every rank computes its
// result from all slots and copies it back, a barrier before the slots are reused.
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<uint64_t>> slot;
  explicit LocalGroup(int w) : world(w), slot((size_t)w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};
struct LocalCtx {
  std::shared_ptr<LocalGroup> g;
  int rank;
};
int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return VR_OK;
  vr::set_last_error(std::string("CUDA: ") + cudaGetErrorString(e));
  return VR_EDEVICE;
}
int local_allreduce(void* ctx, uint64_t* buf, int64_t n, void* stream) {
  LocalCtx* c = (LocalCtx*)ctx;
  LocalGroup& G = *c->g;
  auto& mine = G.slot[(size_t)c->rank];
  mine.resize((size_t)std::max<int64_t>(n, 0));
  int rc = VR_OK;
  if (n > 0) {
    rc = cuda_rc(cudaMemcpyAsync(mine.data(), buf, (size_t)n * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  G.barrier();
  std::vector<uint64_t> sum((size_t)std::max<int64_t>(n, 0), 0);
  for (int r = 0; r < G.world; ++r)
    for (int64_t i = 0; i < n; ++i) sum[(size_t)i] += G.slot[(size_t)r][(size_t)i];
  G.barrier();
  if (n > 0 && !rc) {
    rc = cuda_rc(cudaMemcpyAsync(buf, sum.data(), (size_t)n * 8, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  return rc;
}
int local_allgather(void* ctx, const uint64_t* send, uint64_t* recv, int64_t n_each, void* stream) {
  LocalCtx* c = (LocalCtx*)ctx;
  LocalGroup& G = *c->g;
  auto& mine = G.slot[(size_t)c->rank];
  mine.resize((size_t)std::max<int64_t>(n_each, 0));
  int rc = VR_OK;
  if (n_each > 0) {
    rc = cuda_rc(cudaMemcpyAsync(mine.data(), send, (size_t)n_each * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  G.barrier();
  if (n_each > 0 && !rc) {
    for (int r = 0; r < G.world && !rc; ++r)
      rc = cuda_rc(cudaMemcpyAsync(recv + (size_t)r * (size_t)n_each, G.slot[(size_t)r].data(), (size_t)n_each * 8,
                                   cudaMemcpyHostToDevice, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  G.barrier();
  return rc;
}
int local_bcast(void* ctx, uint64_t* buf, int64_t n, int32_t root, void* stream) {
  LocalCtx* c = (LocalCtx*)ctx;
  LocalGroup& G = *c->g;
  int rc = VR_OK;
  if (c->rank == root && n > 0) {
    G.slot[(size_t)root].resize((size_t)n);
    rc = cuda_rc(cudaMemcpyAsync(G.slot[(size_t)root].data(), buf, (size_t)n * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  G.barrier();
  if (c->rank != root && n > 0 && !rc) {
    rc = cuda_rc(cudaMemcpyAsync(buf, G.slot[(size_t)root].data(), (size_t)n * 8, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    if (!rc) rc = cuda_rc(cudaStreamSynchronize((cudaStream_t)stream));
  }
  G.barrier();
  return rc;
}
void local_destroy(void* ctx) { delete (LocalCtx*)ctx; }

}  // namespace

namespace vr {
// devices 0..G-1 of this process, ncclCommInitAll (vr_options.num_gpus)
std::vector<vr_comm*> comm_nccl_all(int G) {
  if (!nccl().ok) {
    nccl_missing();
    return {};
  }
  std::vector<ncclComm_t> comms((size_t)G);
  std::vector<int> devs((size_t)G);
  for (int g = 0; g < G; ++g) devs[(size_t)g] = g;
  if (nccl_rc(nccl().CommInitAll(comms.data(), G, devs.data())) != VR_OK) return {};
  std::vector<vr_comm*> out;
  for (int g = 0; g < G; ++g) out.push_back(wrap_nccl(comms[(size_t)g], g, G));
  return out;
}
}  // namespace vr

extern "C" {

int vr_nccl_unique_id(uint8_t id[128]) {
  if (!id) return VR_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  if (!nccl().ok) return nccl_missing();
  ncclUniqueId u;
  const int rc = nccl_rc(nccl().GetUniqueId(&u));
  if (rc) return rc;
  std::memcpy(id, &u, 128);
  return VR_OK;
}

int vr_comm_nccl(const uint8_t id[128], int32_t rank, int32_t world, int32_t device, vr_comm** out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return VR_EINVAL;
  *out = nullptr;
  if (!nccl().ok) return nccl_missing();
  if (int rc = cuda_rc(cudaSetDevice(device))) return rc;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm = nullptr;
  if (int rc = nccl_rc(nccl().CommInitRank(&comm, world, u, rank))) return rc;
  *out = wrap_nccl(comm, rank, world);
  return VR_OK;
}

int vr_comm_local(int32_t world, vr_comm** comms) {
  if (!comms || world < 1) return VR_EINVAL;
  auto g = std::make_shared<LocalGroup>(world);
  for (int r = 0; r < world; ++r) {
    vr_comm* v = new vr_comm{};
    v->ctx = new LocalCtx{g, r};
    v->rank = r;
    v->world = world;
    v->allreduce_sum_u64 = local_allreduce;
    v->allgather_u64 = local_allgather;
    v->broadcast_u64 = local_bcast;
    v->destroy = local_destroy;
    comms[r] = v;
  }
  return VR_OK;
}

void vr_comm_free(vr_comm* c) {
  if (!c) return;
  if (c->destroy) c->destroy(c->ctx);
  delete c;
}

}  // extern "C"
