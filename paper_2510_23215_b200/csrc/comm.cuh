// comm.cuh — collective interface of the row-partitioned solve (comm.cu).
#pragma once
#include "common.cuh"

namespace scsf {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // in place, element-wise over ranks; identical bits on every rank
  virtual int allreduce_sum(double* buf, size_t count, cudaStream_t s) = 0;
  virtual int allreduce_max_u64(unsigned long long* buf, size_t count, cudaStream_t s) = 0;
  // recv[r * count + i] = send_of_rank_r[i]
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
  // send_lo -> rank-1 (lands in its recv_hi), send_hi -> rank+1 (lands in its recv_lo)
  virtual int halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, size_t count,
                   cudaStream_t s) = 0;
  // stream-ordered without host participation (NCCL): the collectives may be captured into a
  // CUDA graph; the loopback backend meets at host barriers and is not capturable
  virtual bool capturable() const { return false; }
};

int comm_unique_id(void* id128);
int comm_create_nccl(int rank, int world, const void* id128, Comm** out);
int comm_create_loopback(int world, Comm** out);   // out: array of `world` communicators

}  // namespace scsf
