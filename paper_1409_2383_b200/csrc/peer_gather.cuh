// Row all-gather over NVLink peer memory (peer_gather.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ntf {

constexpr int kPeerMaxRanks = 8;
constexpr int kPeerGatherThreads = 256;
constexpr int kPeerGatherTimeout = 6;  // status word value written on a wait timeout
// Peer buffer layout: [arrival counter | seq | pad to 256 B][staging parity 0][staging parity 1]
constexpr size_t kPeerHeaderBytes = 256;

__host__ __device__ inline unsigned int* peer_arrivals(void* base) {
  return static_cast<unsigned int*>(base);
}
__host__ __device__ inline unsigned int* peer_seq(void* base) {
  return static_cast<unsigned int*>(base) + 16;
}
__host__ __device__ inline double* peer_staging(void* base) {
  return reinterpret_cast<double*>(static_cast<char*>(base) + kPeerHeaderBytes);
}

struct PeerGatherArgs {
  int nranks, me, R, ctas;
  int64_t row_offset[kPeerMaxRanks + 1];
  double* full;
  void* base[kPeerMaxRanks];  // rank q's peer buffer, mapped in this process
  int* status;
  int64_t timeout_ns;
};

struct PeerGatherGroup {
  PeerGatherArgs args[kPeerMaxRanks];  // args[q].me == q, one entry per rank
};

cudaError_t peer_gather_launch(const PeerGatherArgs& a, cudaStream_t stream);
// all ranks' gathers as one cooperative launch on the current device
cudaError_t peer_gather_group_launch(const PeerGatherGroup& g, int nranks, cudaStream_t stream);
// co-residency bound on ctas (per rank) for one launch holding ranks_in_launch ranks
int peer_gather_max_ctas(int ranks_in_launch);

}  // namespace ntf
