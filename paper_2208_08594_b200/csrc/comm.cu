// Communication backends of the z-slab distributed path (see comm.h).
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "comm.h"

namespace msp {

__global__ void pack_kernel(const int32_t* __restrict__ idx, const double* __restrict__ vec,
                            double* __restrict__ buf, int k0, int k1, int width) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = (k1 - k0) * width;
  if (t >= n) return;
  const int k = k0 + t / width, w = t % width;
  buf[(size_t)k * width + w] = vec[(size_t)idx[k] * width + w];
}

void launch_pack(cudaStream_t s, const int32_t* idx, const double* vec, double* sendbuf, int k0, int k1,
                 int width) {
  const int n = (k1 - k0) * width;
  if (n <= 0) return;
  pack_kernel<<<(n + 255) / 256, 256, 0, s>>>(idx, vec, sendbuf, k0, k1, width);
}

static void seg_range(const HaloPlan& P, int pi, int seg, bool send, int& a, int& b) {
  const auto& off = send ? P.send_off[pi] : P.recv_off[pi];
  if (seg < 0) { a = off.front(); b = off.back(); }
  else { a = off[seg]; b = off[seg + 1]; }
}

// ------------------------------------------------------------------------ NCCL
class NcclComm : public Comm {
 public:
  ncclComm_t comm = nullptr;
  int r = 0, p = 1;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  int rank() const override { return r; }
  int size() const override { return p; }
  bool capturable() const override { return true; }   // NCCL operations are stream-capturable
  static void chk(ncclResult_t e, const char* what) {
    if (e != ncclSuccess) throw std::runtime_error(std::string("NCCL ") + what + ": " + ncclGetErrorString(e));
  }
  void halo(cudaStream_t s, const HaloPlan& P, double* vec, int n_own, int width, int seg, bool packed) override {
    for (size_t pi = 0; pi < P.peers.size() && !packed; ++pi) {
      int a, b;
      seg_range(P, (int)pi, seg, true, a, b);
      launch_pack(s, P.d_send_idx, vec, P.d_sendbuf, P.send_base[pi] + a, P.send_base[pi] + b, width);
    }
    chk(ncclGroupStart(), "group start");
    for (size_t pi = 0; pi < P.peers.size(); ++pi) {
      int a, b;
      seg_range(P, (int)pi, seg, true, a, b);
      if (b > a)
        chk(ncclSend(P.d_sendbuf + (size_t)(P.send_base[pi] + a) * width, (size_t)(b - a) * width, ncclDouble,
                     P.peers[pi], comm, s), "send");
      seg_range(P, (int)pi, seg, false, a, b);
      if (b > a)
        chk(ncclRecv(vec + (size_t)(n_own + P.recv_base[pi] + a) * width, (size_t)(b - a) * width, ncclDouble,
                     P.peers[pi], comm, s), "recv");
    }
    chk(ncclGroupEnd(), "group end");
  }
  void allreduce_sum(cudaStream_t s, double* buf, int count) override {
    chk(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm, s), "allreduce");
  }
  void allgather(cudaStream_t s, const double* send, double* recv, int count) override {
    chk(ncclAllGather(send, recv, count, ncclDouble, comm, s), "allgather");
  }
  void broadcast(cudaStream_t s, double* buf, int count, int root) override {
    chk(ncclBroadcast(buf, buf, count, ncclDouble, root, comm, s), "broadcast");
  }
};

int nccl_unique_id(void* out) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return 1;
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

std::unique_ptr<Comm> make_nccl_comm(const void* uid, int rank, int nranks, int* err) {
  std::unique_ptr<NcclComm> c(new NcclComm);
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  c->r = rank;
  c->p = nranks;
  ncclResult_t e = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (e != ncclSuccess) {
    *err = (int)e;
    c->comm = nullptr;
    return nullptr;
  }
  *err = 0;
  return c;
}

// -------------------------------------------------------------------- loopback
__global__ void sum_ranks_kernel(double* const* __restrict__ bufs, int nranks, double* __restrict__ out, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < nranks; ++r) s += bufs[r][i];       // fixed rank order
  out[i] = s;
}

// reusable host barrier (generation counting)
struct HostBarrier {
  std::mutex m;
  std::condition_variable cv;
  int n, count = 0;
  long gen = 0;
  explicit HostBarrier(int n_) : n(n_) {}
  void arrive_and_wait() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopbackGroup {
  int n;
  HostBarrier bar;
  std::vector<const HaloPlan*> plan;
  std::vector<const double*> ptr;
  std::vector<cudaEvent_t> ready, done;
  std::vector<double*> stage;          // per-rank staging for allreduce (device)
  double** d_stage = nullptr;
  explicit LoopbackGroup(int n_) : n(n_), bar(n_), plan(n_), ptr(n_), ready(n_), done(n_), stage(n_) {
    for (int r = 0; r < n; ++r) {
      cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
      cudaMalloc(&stage[r], sizeof(double) * 64);
    }
    cudaMalloc(&d_stage, sizeof(double*) * n);
    cudaMemcpy(d_stage, stage.data(), sizeof(double*) * n, cudaMemcpyHostToDevice);
  }
  ~LoopbackGroup() {
    for (int r = 0; r < n; ++r) {
      cudaEventDestroy(ready[r]);
      cudaEventDestroy(done[r]);
      cudaFree(stage[r]);
    }
    cudaFree(d_stage);
  }
};

std::shared_ptr<LoopbackGroup> make_loopback_group(int nranks) { return std::make_shared<LoopbackGroup>(nranks); }

class LoopbackComm : public Comm {
 public:
  std::shared_ptr<LoopbackGroup> g;
  int r;
  LoopbackComm(std::shared_ptr<LoopbackGroup> g_, int r_) : g(std::move(g_)), r(r_) {}
  int rank() const override { return r; }
  int size() const override { return g->n; }
  // peers must have finished reading our buffers of the previous collective before we
  // overwrite them: wait on their `done` events (recorded before the trailing barrier)
  void wait_peers_done(cudaStream_t s) {
    for (int q = 0; q < g->n; ++q)
      if (q != r) cudaStreamWaitEvent(s, g->done[q], 0);
  }
  void halo(cudaStream_t s, const HaloPlan& P, double* vec, int n_own, int width, int seg, bool packed) override {
    wait_peers_done(s);
    for (size_t pi = 0; pi < P.peers.size() && !packed; ++pi) {
      int a, b;
      seg_range(P, (int)pi, seg, true, a, b);
      launch_pack(s, P.d_send_idx, vec, P.d_sendbuf, P.send_base[pi] + a, P.send_base[pi] + b, width);
    }
    cudaEventRecord(g->ready[r], s);
    g->plan[r] = &P;
    g->bar.arrive_and_wait();
    for (size_t pi = 0; pi < P.peers.size(); ++pi) {
      const int q = P.peers[pi];
      const HaloPlan& Q = *g->plan[q];
      int qi = -1;                                      // my index in q's peer list
      for (size_t k = 0; k < Q.peers.size(); ++k) if (Q.peers[k] == r) qi = (int)k;
      if (qi < 0) continue;
      int a, b, qa, qb;
      seg_range(P, (int)pi, seg, false, a, b);
      seg_range(Q, qi, seg, true, qa, qb);
      if (b - a != qb - qa) throw std::runtime_error("loopback halo: send/recv size mismatch");
      if (b > a) {
        cudaStreamWaitEvent(s, g->ready[q], 0);
        cudaMemcpyAsync(vec + (size_t)(n_own + P.recv_base[pi] + a) * width,
                        Q.d_sendbuf + (size_t)(Q.send_base[qi] + qa) * width, sizeof(double) * (b - a) * width,
                        cudaMemcpyDeviceToDevice, s);
      }
    }
    cudaEventRecord(g->done[r], s);
    g->bar.arrive_and_wait();
    wait_peers_done(s);          // later work on s may overwrite buffers peers read
  }
  void allreduce_sum(cudaStream_t s, double* buf, int count) override {
    if (count > 64) throw std::runtime_error("loopback allreduce: count > 64");
    wait_peers_done(s);
    cudaMemcpyAsync(g->stage[r], buf, sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(g->ready[r], s);
    g->bar.arrive_and_wait();
    for (int q = 0; q < g->n; ++q)
      if (q != r) cudaStreamWaitEvent(s, g->ready[q], 0);
    sum_ranks_kernel<<<1, 64, 0, s>>>(g->d_stage, g->n, buf, count);
    cudaEventRecord(g->done[r], s);
    g->bar.arrive_and_wait();
    wait_peers_done(s);          // later work on s may overwrite buffers peers read
  }
  void allgather(cudaStream_t s, const double* send, double* recv, int count) override {
    wait_peers_done(s);
    cudaEventRecord(g->ready[r], s);
    g->ptr[r] = send;
    g->bar.arrive_and_wait();
    for (int q = 0; q < g->n; ++q) {
      if (q != r) cudaStreamWaitEvent(s, g->ready[q], 0);
      cudaMemcpyAsync(recv + (size_t)q * count, g->ptr[q], sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(g->done[r], s);
    g->bar.arrive_and_wait();
    wait_peers_done(s);          // later work on s may overwrite buffers peers read
  }
  void broadcast(cudaStream_t s, double* buf, int count, int root) override {
    wait_peers_done(s);
    cudaEventRecord(g->ready[r], s);
    if (r == root) g->ptr[root] = buf;
    g->bar.arrive_and_wait();
    if (r != root) {
      cudaStreamWaitEvent(s, g->ready[root], 0);
      cudaMemcpyAsync(buf, g->ptr[root], sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(g->done[r], s);
    g->bar.arrive_and_wait();
    wait_peers_done(s);          // later work on s may overwrite buffers peers read
  }
};

void loopback_barrier(LoopbackGroup& g) { g.bar.arrive_and_wait(); }

std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank) {
  return std::unique_ptr<Comm>(new LoopbackComm(std::move(g), rank));
}

}  // namespace msp
