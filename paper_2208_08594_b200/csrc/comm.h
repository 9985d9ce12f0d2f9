// Communication layer of the z-slab distributed MSP-GMRES.
// Plain device pointers and CUDA streams; two backends:
//   - NCCL (one process per GPU; NCCL over NVLink 5 / NVSwitch): ncclSend/ncclRecv
//     halo exchanges, ncclAllReduce for the Krylov dot products, ncclAllGather of the
//     level-1 right-hand side (coarse levels are replicated on every rank);
//   - loopback (P virtual ranks as host threads of ONE process on ONE GPU, each with
//     its own stream): the same calls implemented with device-to-device copies ordered
//     by CUDA events and host barriers.  No kernel ever waits on another kernel, so it
//     is safe on a single GPU; it exists to test the distributed path without a cluster.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

namespace msp {

// Ghost exchange plan of one vector space (cell space or AMG level 0).  Ghost entries of
// a rank live after its n_own owned entries, grouped by source peer and, inside a peer,
// by color segment; the matching send lists are grouped the same way, so every segment
// is one contiguous send and one contiguous receive.
struct HaloPlan {
  int nseg = 1;                              // color segments
  std::vector<int> peers;                    // peers exchanged with (ascending rank)
  std::vector<std::vector<int>> send_off;    // [peer][nseg+1] offsets into the peer's send block
  std::vector<std::vector<int>> recv_off;    // [peer][nseg+1] offsets into the peer's ghost block
  std::vector<int> send_base, recv_base;     // [peer] block starts (send_idx / ghost index)
  int nsend = 0, nghost = 0;
  int32_t* d_send_idx = nullptr;             // device: owned local index of every send entry
  double* d_sendbuf = nullptr;               // device: nsend * max_width
  int2* d_slots = nullptr;                   // device, per owned entry: its (<= 2) send positions
                                             // (-1 none) -- producer kernels write the send buffer
                                             // themselves (null: a row is sent more than twice)
};

class Comm {
 public:
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // ghost values of vec (width doubles per entry): segment seg of every peer (-1: all)
  // packed: the producer kernel already wrote the send buffer (no pack kernel)
  virtual void halo(cudaStream_t s, const HaloPlan& plan, double* vec, int n_own, int width, int seg,
                    bool packed = false) = 0;
  // in-place sum over ranks (identical result on every rank)
  virtual void allreduce_sum(cudaStream_t s, double* buf, int count) = 0;
  // recv[r*count .. ) = send of rank r
  virtual void allgather(cudaStream_t s, const double* send, double* recv, int count) = 0;
  // buf of every rank = buf of rank `root`
  virtual void broadcast(cudaStream_t s, double* buf, int count, int root) = 0;
  // true if every call only enqueues work on s (no host synchronisation), so the
  // Arnoldi steps that use it can be captured into CUDA graphs
  virtual bool capturable() const { return false; }
};

// pack: sendbuf[k*width + w] = vec[idx[k]*width + w] for k in [k0, k1)
void launch_pack(cudaStream_t s, const int32_t* idx, const double* vec, double* sendbuf, int k0, int k1,
                 int width);

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int nranks, int* err);
int nccl_unique_id(void* out128);

struct LoopbackGroup;
std::shared_ptr<LoopbackGroup> make_loopback_group(int nranks);
std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank);
void loopback_barrier(LoopbackGroup& g);

}  // namespace msp
