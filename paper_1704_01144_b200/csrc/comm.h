// Transport for the multi-GPU path: the collectives and halo exchange a
// shard needs, replacing the reference's RankComm and
// GhostExchange over its custom transport (exchange.cpp:126-514,
// transport.cpp). Two implementations:
//   * NcclComm     one process per GPU, NCCL over NVLink/NVSwitch; all calls
//                  are stream-ordered and CUDA-graph capturable;
//   * LoopbackComm R ranks as host threads of one process (one GPU or
//                  several): host barriers + event-ordered device copies, no
//                  device-side waiting (the in-process analogue of the
//                  reference's LoopbackHub, transport.hpp).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

struct tafv_gpu;

struct tafv_comm {
  int rank_count = 1;
  virtual ~tafv_comm() {}
  virtual bool capturable() const = 0;
  virtual int nranks() const { return rank_count; }
  // In-place all-reduces on device buffers, ordered on `st`.
  virtual void allreduce_min_f64(int rank, double* d, int n, cudaStream_t st) = 0;
  virtual void allreduce_max_i32(int rank, int* d, int n, cudaStream_t st) = 0;
  virtual void allreduce_sum_f64(int rank, double* d, int n, cudaStream_t st) = 0;
  virtual void allreduce_sum_i64(int rank, long long* d, int n, cudaStream_t st) = 0;
  // Halo exchange of `bytes_per_row` rows already packed in h.sendbuf (peer
  // segments) into h.recvbuf (peer segments), ordered on `st`. scount /
  // rcount (per peer, in h.peers order; null = whole segments): the leading
  // rows of each segment that move (level-sorted lists).
  virtual void exchange(tafv_gpu& h, int bytes_per_row, cudaStream_t st, const int* scount = nullptr,
                        const int* rcount = nullptr) = 0;
  virtual void attach(int rank, tafv_gpu* h) {}
};

tafv_comm* make_loopback_comm(int nranks);
tafv_comm* make_nccl_comm(const void* unique_id, int rank, int nranks);
int nccl_unique_id(void* out);
