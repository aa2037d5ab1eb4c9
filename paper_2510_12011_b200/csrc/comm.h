// comm.h -- inter-GPU transport of the partitioned PCG (NCCL over NVLink /
// NVSwitch, one process per GPU).  Only NCCL's types come from the system
// header; the library itself is resolved at run time (comm.cpp).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

namespace tcb {

struct HaloMsg {
  int peer;      // rank
  double* ptr;   // device buffer
  size_t count;  // doubles
};

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::string init(int rank, int world, const uint8_t id[128]);
  void destroy();
  std::string allreduce_sum(double* buf, size_t count, cudaStream_t s);
  std::string allgather(const double* send, double* recv, size_t count, cudaStream_t s);
  std::string exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                       cudaStream_t s);
};

std::string nccl_unique_id(uint8_t out[128]);

}  // namespace tcb
