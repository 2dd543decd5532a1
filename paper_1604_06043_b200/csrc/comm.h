// comm.h — cross-rank communication of a row-sharded Mstab solve.
//
// Every operation of the solve loop except the SpMV is row-local (idrstab.cpp:105-191); the SpMV
// needs the halo rows of its input owned by the neighbouring ranks, and every length-N
// reduction (P^H[V|r], the least-squares factor, ||r||, validate's Grams) needs a sum over the
// ranks. The solver therefore needs exactly three primitives, all enqueued on the solver stream:
//
//   allreduce_sum(buf, count)        sum of `count` fp64 over the ranks, result on every rank
//                                    (bit-identical on every rank: the replicated dense steps
//                                    must take identical branches);
//   allgather(in, out, count)        rank-major concatenation (the least-squares R factors are
//                                    merged, not summed);
//   halo(x)                          receive the halo rows of x from their owners, send the owned
//                                    rows the neighbours need (plan: HaloPlan).
//
// Two implementations:
//   * NcclComm  — one process per GPU, NCCL over NVLink/NVSwitch (libnccl loaded at run time);
//                 stream-ordered and CUDA-graph capturable, so the sharded cycle is still one
//                 graph launch per cycle;
//   * HostComm  — caller-supplied host callbacks (include/mstab_b200.h mstab_host_comm): device
//                 buffers are staged through pinned host memory and the caller's runtime (MPI,
//                 gloo, ...) moves them. Not capturable (the solver then launches eagerly). Used
//                 by the tests to run several ranks on one GPU without any kernel waiting on
//                 another rank's kernel.
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mstab_b200.h"

typedef struct CUstream_st* cudaStream_t;

namespace mstab_b200 {

// Halo exchange of one rank: ranges are in elements relative to the owned-rows start of a
// vector (negative = left halo).
struct HaloXfer {
  int peer = 0;
  int64_t offset = 0;
  int64_t count = 0;
};
struct HaloPlan {
  std::vector<HaloXfer> sends;  // owned rows the peer needs
  std::vector<HaloXfer> recvs;  // halo rows owned by the peer
  bool empty() const { return sends.empty() && recvs.empty(); }
};

class Comm {
 public:
  Comm(int rank, int world) : rank_(rank), world_(world) {}
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  virtual bool capturable() const = 0;
  virtual void allreduce_sum(double* dev, int64_t count, cudaStream_t st) = 0;
  virtual void allgather(const double* dev_in, double* dev_out, int64_t count, cudaStream_t st) = 0;
  virtual void halo(double* x_owned, const HaloPlan& plan, cudaStream_t st) = 0;
  // Split form: halo_begin starts the exchange (a communicator that can run it beside the solver
  // stream does: NcclComm forks onto a side stream), halo_end makes `st` wait for it. Work enqueued
  // on `st` between the two must not read the halo rows. Default: the blocking exchange.
  virtual void halo_begin(double* x_owned, const HaloPlan& plan, cudaStream_t st) { halo(x_owned, plan, st); }
  virtual void halo_end(cudaStream_t) {}
  virtual const char* name() const = 0;

 protected:
  int rank_, world_;
};

// NCCL communicator over an id from nccl_unique_id() on rank 0 (distributed by the caller).
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id, int device);
// Fills `out` (128 bytes, ncclUniqueId) on the calling process.
void nccl_unique_id(void* out);
// Host-callback communicator.
std::unique_ptr<Comm> make_host_comm(int rank, int world, const mstab_host_comm& fns);

}  // namespace mstab_b200
