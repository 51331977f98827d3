// comm.cu — NCCL and loopback implementations of the slab collectives (comm.h).
#include "comm.h"

#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "plan.h"

namespace mg {

struct LoopGroup {
  struct Post {
    char* base = nullptr;
    int owned = 0;
    cudaEvent_t ev = nullptr;
  };
  int P;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<Post> post;
  std::vector<cudaEvent_t> done;
  explicit LoopGroup(int n) : P(n), post(n), done(n, nullptr) {}
  // all P ranks' host threads meet here
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++arrived == P) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LoopGroup* loop_group_create(int nranks) { return nranks >= 1 ? new LoopGroup(nranks) : nullptr; }
void loop_group_destroy(LoopGroup* g) { delete g; }
int loop_group_size(const LoopGroup* g) { return g ? g->P : 0; }

bool comm_active(const mg_solver* s) { return s->pt.P > 1 && (s->comm || s->loop); }

static cudaError_t nccl_err(ncclResult_t r) { return r == ncclSuccess ? cudaSuccess : cudaErrorUnknown; }

// loopback: publish (base, owned, ready event), rendezvous, copy what the peers expose,
// publish "copied", rendezvous, and make this stream wait until the peers have copied
// out of this rank's buffer before it may overwrite it
template <class Copies>
static cudaError_t loop_exchange(mg_solver* s, void* buf, int owned, cudaStream_t st, const std::vector<int>& peers,
                                 Copies copies) {
  LoopGroup* G = s->loop;
  const int rk = s->pt.rank;
  cudaError_t e = cudaEventRecord(s->lb_ready, st);
  if (e != cudaSuccess) return e;
  G->post[rk] = LoopGroup::Post{static_cast<char*>(buf), owned, s->lb_ready};
  G->barrier();
  for (int q : peers) {
    if ((e = cudaStreamWaitEvent(st, G->post[q].ev, 0)) != cudaSuccess) return e;
    if ((e = copies(q, G->post[q])) != cudaSuccess) return e;
  }
  if ((e = cudaEventRecord(s->lb_done, st)) != cudaSuccess) return e;
  G->done[rk] = s->lb_done;
  G->barrier();
  for (int q : peers)
    if ((e = cudaStreamWaitEvent(st, G->done[q], 0)) != cudaSuccess) return e;
  G->barrier();  // nobody re-records its events before every rank has waited on them
  return cudaSuccess;
}

cudaError_t comm_halo(mg_solver* s, void* buf, size_t pbytes, int H, int owned, int h, cudaStream_t st) {
  const int P = s->pt.P, rk = s->pt.rank;
  char* b = static_cast<char*>(buf);
  if (s->comm) {
    ncclResult_t nr = ncclGroupStart();
    if (rk < P - 1 && nr == ncclSuccess) {
      nr = ncclSend(b + (size_t)(H + owned - h) * pbytes, h * pbytes, ncclChar, rk + 1, s->comm, st);
      if (nr == ncclSuccess) nr = ncclRecv(b + (size_t)(H + owned) * pbytes, h * pbytes, ncclChar, rk + 1, s->comm, st);
    }
    if (rk > 0 && nr == ncclSuccess) {
      nr = ncclSend(b + (size_t)H * pbytes, h * pbytes, ncclChar, rk - 1, s->comm, st);
      if (nr == ncclSuccess) nr = ncclRecv(b + (size_t)(H - h) * pbytes, h * pbytes, ncclChar, rk - 1, s->comm, st);
    }
    const ncclResult_t ne = ncclGroupEnd();
    return nr != ncclSuccess ? nccl_err(nr) : nccl_err(ne);
  }
  std::vector<int> peers;
  if (rk < P - 1) peers.push_back(rk + 1);
  if (rk > 0) peers.push_back(rk - 1);
  return loop_exchange(s, buf, owned, st, peers, [&](int q, const LoopGroup::Post& p) {
    if (q == rk + 1)  // my upper halo <- the peer's lowest owned planes
      return cudaMemcpyAsync(b + (size_t)(H + owned) * pbytes, p.base + (size_t)H * pbytes, h * pbytes,
                             cudaMemcpyDeviceToDevice, st);
    // my lower halo <- the peer's highest owned planes
    return cudaMemcpyAsync(b + (size_t)(H - h) * pbytes, p.base + (size_t)(H + p.owned - h) * pbytes, h * pbytes,
                           cudaMemcpyDeviceToDevice, st);
  });
}

cudaError_t comm_allgather(mg_solver* s, void* buf, size_t chunk, cudaStream_t st) {
  const int P = s->pt.P, rk = s->pt.rank;
  char* b = static_cast<char*>(buf);
  if (s->comm) return nccl_err(ncclAllGather(b + (size_t)rk * chunk, b, chunk, ncclChar, s->comm, st));
  std::vector<int> peers;
  for (int q = 0; q < P; q++)
    if (q != rk) peers.push_back(q);
  return loop_exchange(s, buf, 0, st, peers, [&](int q, const LoopGroup::Post& p) {
    return cudaMemcpyAsync(b + (size_t)q * chunk, p.base + (size_t)q * chunk, chunk, cudaMemcpyDeviceToDevice, st);
  });
}

}  // namespace mg
