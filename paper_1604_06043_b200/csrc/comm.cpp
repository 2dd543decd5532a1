// comm.cpp — NCCL and host-callback implementations of comm.h.
#include "comm.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "host_util.h"

namespace mstab_b200 {

namespace {

// ---- NCCL, resolved at run time (no link-time dependency for single-GPU users) ---------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
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
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* s) { return dlsym(api.h, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.Send ||
      !api.Recv || !api.GroupStart || !api.GroupEnd)
    throw Error(MSTAB_E_CUDA, "NCCL (libnccl.so.2) not available");
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(MSTAB_E_CUDA, std::string(what) + ": " +
                                  (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

class NcclComm final : public Comm {
 public:
  NcclComm(int rank, int world, const void* uid, int device) : Comm(rank, world) {
    NcclApi& api = nccl();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    cudaSetDevice(device);
    nccl_ok(api.CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
    // the halo side stream and its fork / join events exist before any stream capture starts
    cuda_ok(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "halo side stream");
    cuda_ok(cudaEventCreateWithFlags(&e0_, cudaEventDisableTiming), "halo event");
    cuda_ok(cudaEventCreateWithFlags(&e1_, cudaEventDisableTiming), "halo event");
  }
  ~NcclComm() override {
    if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
    if (e0_) cudaEventDestroy(e0_);
    if (e1_) cudaEventDestroy(e1_);
    if (side_) cudaStreamDestroy(side_);
  }
  bool capturable() const override { return true; }
  const char* name() const override { return "nccl"; }
  void allreduce_sum(double* dev, int64_t count, cudaStream_t st) override {
    nccl_ok(nccl().AllReduce(dev, dev, (size_t)count, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
  }
  void allgather(const double* in, double* out, int64_t count, cudaStream_t st) override {
    nccl_ok(nccl().AllGather(in, out, (size_t)count, ncclFloat64, comm_, st), "ncclAllGather");
  }
  void halo(double* x, const HaloPlan& plan, cudaStream_t st) override {
    if (plan.empty()) return;
    NcclApi& api = nccl();
    nccl_ok(api.GroupStart(), "ncclGroupStart");
    for (const auto& s : plan.sends)
      nccl_ok(api.Send(x + s.offset, (size_t)s.count, ncclFloat64, s.peer, comm_, st), "ncclSend");
    for (const auto& r : plan.recvs)
      nccl_ok(api.Recv(x + r.offset, (size_t)r.count, ncclFloat64, r.peer, comm_, st), "ncclRecv");
    nccl_ok(api.GroupEnd(), "ncclGroupEnd");
  }
  // The exchange on a side stream forked from (and later joined to) the solver stream with
  // events, so the interior rows of the product run while NVLink moves the halo planes. Inside a
  // stream capture the fork and join become graph edges.
  void halo_begin(double* x, const HaloPlan& plan, cudaStream_t st) override {
    if (plan.empty()) return;
    cuda_ok(cudaEventRecord(e0_, st), "halo fork");
    cuda_ok(cudaStreamWaitEvent(side_, e0_, 0), "halo fork");
    halo(x, plan, side_);
    cuda_ok(cudaEventRecord(e1_, side_), "halo join");
    pending_ = true;
  }
  void halo_end(cudaStream_t st) override {
    if (!pending_) return;
    cuda_ok(cudaStreamWaitEvent(st, e1_, 0), "halo join");
    pending_ = false;
  }

 private:
  static void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(MSTAB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  ncclComm_t comm_ = nullptr;
  cudaStream_t side_ = nullptr;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
  bool pending_ = false;
};

// ---- host callbacks ---------------------------------------------------------------------------
class HostComm final : public Comm {
 public:
  HostComm(int rank, int world, const mstab_host_comm& f) : Comm(rank, world), f_(f) {}
  ~HostComm() override {
    if (pinned_) cudaFreeHost(pinned_);
  }
  bool capturable() const override { return false; }
  const char* name() const override { return "host"; }
  void allreduce_sum(double* dev, int64_t count, cudaStream_t st) override {
    double* h = stage(count);
    copy(h, dev, count, cudaMemcpyDeviceToHost, st);
    sync(st);
    check(f_.allreduce_sum(f_.user, h, count), "allreduce_sum");
    copy(dev, h, count, cudaMemcpyHostToDevice, st);
    sync(st);  // the staging buffer is reused by the next call
  }
  void allgather(const double* in, double* out, int64_t count, cudaStream_t st) override {
    double* h = stage(count * (world_ + 1));
    copy(h, in, count, cudaMemcpyDeviceToHost, st);
    sync(st);
    check(f_.allgather(f_.user, h, h + count, count), "allgather");
    copy(out, h + count, count * world_, cudaMemcpyHostToDevice, st);
    sync(st);
  }
  void halo(double* x, const HaloPlan& plan, cudaStream_t st) override {
    if (plan.empty()) return;
    int64_t total = 0;
    for (const auto& s : plan.sends) total += s.count;
    for (const auto& r : plan.recvs) total += r.count;
    double* h = stage(total);
    std::vector<const double*> sb;
    std::vector<double*> rb;
    std::vector<int32_t> sp, rp;
    std::vector<int64_t> sc, rc;
    double* cur = h;
    for (const auto& s : plan.sends) {
      copy(cur, x + s.offset, s.count, cudaMemcpyDeviceToHost, st);
      sb.push_back(cur);
      sp.push_back(s.peer);
      sc.push_back(s.count);
      cur += s.count;
    }
    for (const auto& r : plan.recvs) {
      rb.push_back(cur);
      rp.push_back(r.peer);
      rc.push_back(r.count);
      cur += r.count;
    }
    sync(st);
    check(f_.halo_exchange(f_.user, (int32_t)sb.size(), sp.data(), sb.data(), sc.data(), (int32_t)rb.size(),
                           rp.data(), rb.data(), rc.data()),
          "halo_exchange");
    for (size_t i = 0; i < plan.recvs.size(); ++i)
      copy(x + plan.recvs[i].offset, rb[i], plan.recvs[i].count, cudaMemcpyHostToDevice, st);
    sync(st);
  }

 private:
  double* stage(int64_t count) {
    if (count > cap_) {
      if (pinned_) cudaFreeHost(pinned_);
      cap_ = std::max<int64_t>(count, 1024);
      if (cudaMallocHost(reinterpret_cast<void**>(&pinned_), sizeof(double) * cap_) != cudaSuccess)
        throw Error(MSTAB_E_CUDA, "host comm: pinned staging allocation failed");
    }
    return pinned_;
  }
  static void copy(void* dst, const void* src, int64_t count, cudaMemcpyKind k, cudaStream_t st) {
    if (count > 0 && cudaMemcpyAsync(dst, src, sizeof(double) * count, k, st) != cudaSuccess)
      throw Error(MSTAB_E_CUDA, "host comm: staging copy failed");
  }
  static void sync(cudaStream_t st) {
    if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(MSTAB_E_CUDA, "host comm: stream sync failed");
  }
  static void check(int rc, const char* what) {
    if (rc != 0) throw Error(MSTAB_E_ERROR, std::string("host comm callback failed: ") + what);
  }
  mstab_host_comm f_;
  double* pinned_ = nullptr;
  int64_t cap_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id, int device) {
  return std::make_unique<NcclComm>(rank, world, unique_id, device);
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  nccl_ok(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

std::unique_ptr<Comm> make_host_comm(int rank, int world, const mstab_host_comm& fns) {
  if (!fns.allreduce_sum || !fns.allgather || !fns.halo_exchange)
    throw Error(MSTAB_E_CONFIG, "host comm: every callback must be set");
  return std::make_unique<HostComm>(rank, world, fns);
}

}  // namespace mstab_b200
