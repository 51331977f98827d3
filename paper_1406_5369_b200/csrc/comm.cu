// comm.cu — NCCL and loopback implementations of the slab collectives (comm.h).
#include "comm.h"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
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
  explicit LoopGroup(int n) : P(n), post(n), done(n, nullptr), uf_post(n), need(n, 0), ev_end(n, nullptr), ev_in(n, nullptr) {}
  ~LoopGroup() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (cudaEvent_t e : ev_end)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_in)
      if (e) cudaEventDestroy(e);
    if (ev_origin) cudaEventDestroy(ev_origin);
    if (ev_out) cudaEventDestroy(ev_out);
  }
  bool broken = false;  // a rank timed out or failed mid-rendezvous: the group is unusable
  // group graphs (loop_graph_part): key = every rank's (u, f) and the part
  struct Key {
    std::vector<std::pair<const void*, const void*>> uf;
    int part;
    bool operator<(const Key& o) const { return part != o.part ? part < o.part : uf < o.uf; }
  };
  std::vector<std::pair<const void*, const void*>> uf_post;
  std::vector<char> need;
  std::map<Key, cudaGraphExec_t> graphs;
  cudaEvent_t ev_origin = nullptr, ev_out = nullptr;
  std::vector<cudaEvent_t> ev_end, ev_in;
  cudaError_t capture_err = cudaSuccess;
  mg_status capture_st = MG_OK;
  // all P ranks' host threads meet here; false after `timeout_s` without the others (the
  // group is then broken for every rank, as a communicator with a dead peer would be)
  bool barrier(double timeout_s) {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const long g = gen;
    if (++arrived == P) {
      arrived = 0;
      gen++;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
    if (!ok || gen == g) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

LoopGroup* loop_group_create(int nranks) { return nranks >= 1 ? new LoopGroup(nranks) : nullptr; }
void loop_group_destroy(LoopGroup* g) { delete g; }
int loop_group_size(const LoopGroup* g) { return g ? g->P : 0; }

bool comm_active(const mg_solver* s) { return s->pt.P > 1 && (s->comm || s->loop); }

// A communication failure: recorded on the solver (the plan maps it to MG_ERR_NCCL and poisons
// the solver), reported to the caller as a failed call
static cudaError_t comm_fail(mg_solver* s, const std::string& msg) {
  s->comm_failed = true;
  s->comm_msg = msg;
  return cudaErrorUnknown;
}
static cudaError_t nccl_err(mg_solver* s, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return cudaSuccess;
  std::string m = std::string(what) + ": " + ncclGetErrorString(r);
  const char* last = s->comm ? ncclGetLastError(s->comm) : nullptr;
  if (last && *last) m += std::string(" (") + last + ")";
  return comm_fail(s, m);
}

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
  const double to = s->comm_timeout_s;
  if (!G->barrier(to)) return comm_fail(s, "loopback exchange: a peer did not arrive (timeout or failed peer)");
  for (int q : peers) {
    if ((e = cudaStreamWaitEvent(st, G->post[q].ev, 0)) != cudaSuccess) return e;
    if ((e = copies(q, G->post[q])) != cudaSuccess) return e;
  }
  if ((e = cudaEventRecord(s->lb_done, st)) != cudaSuccess) return e;
  G->done[rk] = s->lb_done;
  if (!G->barrier(to)) return comm_fail(s, "loopback exchange: a peer did not arrive (timeout or failed peer)");
  for (int q : peers)
    if ((e = cudaStreamWaitEvent(st, G->done[q], 0)) != cudaSuccess) return e;
  // nobody re-records its events before every rank has waited on them
  if (!G->barrier(to)) return comm_fail(s, "loopback exchange: a peer did not arrive (timeout or failed peer)");
  return cudaSuccess;
}

static cudaError_t comm_halo_impl(mg_solver* s, void* buf, size_t pbytes, int H, int owned, int h, cudaStream_t st);

cudaError_t comm_halo(mg_solver* s, void* buf, size_t pbytes, int H, int owned, int h, cudaStream_t st) {
  const bool fire = s->fault_kind != 0 && --s->fault_count == 0;
  const int kind = fire ? s->fault_kind : 0;
  if (fire) s->fault_kind = 0;
  if (kind == 1) return comm_fail(s, "halo exchange: injected communication failure (mg_fault_inject)");
  cudaError_t e = comm_halo_impl(s, buf, pbytes, H, owned, h, st);
  if (e != cudaSuccess || kind != 2) return e;
  // injected silent corruption: the received halo planes get a wrong finite value
  char* b = static_cast<char*>(buf);
  if (s->pt.rank > 0 && (e = cudaMemsetAsync(b + (size_t)(H - h) * pbytes, 0x40, h * pbytes, st)) != cudaSuccess)
    return e;
  if (s->pt.rank < s->pt.P - 1)
    e = cudaMemsetAsync(b + (size_t)(H + owned) * pbytes, 0x40, h * pbytes, st);
  return e;
}

static cudaError_t comm_halo_impl(mg_solver* s, void* buf, size_t pbytes, int H, int owned, int h, cudaStream_t st) {
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
    return nr != ncclSuccess ? nccl_err(s, nr, "halo exchange") : nccl_err(s, ne, "halo exchange (group end)");
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
  if (s->comm) return nccl_err(s, ncclAllGather(b + (size_t)rk * chunk, b, chunk, ncclChar, s->comm, st), "all-gather");
  std::vector<int> peers;
  for (int q = 0; q < P; q++)
    if (q != rk) peers.push_back(q);
  return loop_exchange(s, buf, 0, st, peers, [&](int q, const LoopGroup::Post& p) {
    return cudaMemcpyAsync(b + (size_t)q * chunk, p.base + (size_t)q * chunk, chunk, cudaMemcpyDeviceToDevice, st);
  });
}

mg_status loop_graph_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st) {
  LoopGroup* G = s->loop;
  const int rk = s->pt.rank, P = G->P;
  const double to = s->comm_timeout_s;
  auto bar = [&]() { return G->barrier(to); };
  auto broken = [&]() { return plan_fail(s, MG_ERR_NCCL, "loopback group graph: a peer did not arrive"); };
  auto cfail = [&](cudaError_t e, const char* what) {
    std::string m = std::string("loopback group graph: ") + what + ": " + cudaGetErrorString(e);
    return plan_fail(s, MG_ERR_CUDA, m.c_str());
  };
  cudaError_t e = cudaSuccess;
  if (!G->ev_end[rk]) {
    if ((e = cudaEventCreateWithFlags(&G->ev_end[rk], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&G->ev_in[rk], cudaEventDisableTiming)) != cudaSuccess)
      return cfail(e, "events");
  }
  if (rk == 0 && !G->ev_origin) {
    if ((e = cudaEventCreateWithFlags(&G->ev_origin, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&G->ev_out, cudaEventDisableTiming)) != cudaSuccess)
      return cfail(e, "events");
  }
  G->uf_post[rk] = {u, f};
  if (!bar()) return broken();
  LoopGroup::Key key{G->uf_post, part};
  const bool have = G->graphs.count(key) > 0;  // read by every rank after the same barrier
  if (!bar()) return broken();
  if (!have) {
    // ---- capture every rank's part into one graph
    if (rk == 0) {
      G->capture_err = cudaSuccess;
      G->capture_st = MG_OK;
      e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeRelaxed);
      if (e == cudaSuccess) e = cudaEventRecord(G->ev_origin, s->cap_stream);
      G->capture_err = e;
    }
    if (!bar()) return broken();
    if (G->capture_err != cudaSuccess) return cfail(G->capture_err, "begin capture");
    if (rk != 0 && (e = cudaStreamWaitEvent(s->cap_stream, G->ev_origin, 0)) != cudaSuccess) G->capture_err = e;
    mg_status r = plan_run_part(s, part, u, f, s->cap_stream);
    if (r != MG_OK) G->capture_st = r;
    if (rk != 0 && (e = cudaEventRecord(G->ev_end[rk], s->cap_stream)) != cudaSuccess) G->capture_err = e;
    if (!bar()) return broken();
    if (rk == 0) {
      for (int q = 1; q < P && e == cudaSuccess; q++) e = cudaStreamWaitEvent(s->cap_stream, G->ev_end[q], 0);
      cudaGraph_t graph = nullptr;
      const cudaError_t ee = cudaStreamEndCapture(s->cap_stream, &graph);
      if (e == cudaSuccess) e = ee;
      cudaGraphExec_t exec = nullptr;
      if (e == cudaSuccess && G->capture_err == cudaSuccess && G->capture_st == MG_OK)
        e = cudaGraphInstantiate(&exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (e != cudaSuccess && G->capture_err == cudaSuccess) G->capture_err = e;
      if (exec) {
        if (G->graphs.size() >= 16) {
          cudaGraphExecDestroy(G->graphs.begin()->second);
          G->graphs.erase(G->graphs.begin());
        }
        G->graphs.emplace(key, exec);
      }
    }
    if (!bar()) return broken();
    if (r != MG_OK) return r;
    if (G->capture_st != MG_OK) return plan_fail(s, G->capture_st, "loopback group graph: a peer's capture failed");
    if (G->capture_err != cudaSuccess) return cfail(G->capture_err, "capture");
  }
  // ---- replay after every rank's stream has reached this point; every stream waits for it
  if ((e = cudaEventRecord(G->ev_in[rk], st)) != cudaSuccess) return cfail(e, "record");
  if (!bar()) return broken();
  if (rk == 0) {
    for (int q = 0; q < P && e == cudaSuccess; q++) e = cudaStreamWaitEvent(st, G->ev_in[q], 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(G->graphs.at(key), st);
    if (e == cudaSuccess) e = cudaEventRecord(G->ev_out, st);
    G->capture_err = e;
  }
  if (!bar()) return broken();
  if (G->capture_err != cudaSuccess) return cfail(G->capture_err, "launch");
  if ((e = cudaStreamWaitEvent(st, G->ev_out, 0)) != cudaSuccess) return cfail(e, "wait");
  if (!bar()) return broken();  // ev_out / ev_in are not re-recorded before every rank has waited
  return MG_OK;
}

mg_status plan_wait(mg_solver* s, cudaStream_t st, const char* what) {
  if (!s->comm) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) return MG_OK;
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    return plan_fail(s, MG_ERR_CUDA, m.c_str());
  }
  cudaEvent_t ev = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, st);
  if (e != cudaSuccess) {
    if (ev) cudaEventDestroy(ev);
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    return plan_fail(s, MG_ERR_CUDA, m.c_str());
  }
  const auto t0 = std::chrono::steady_clock::now();
  std::string fail_msg;
  for (int it = 0;; it++) {
    e = cudaEventQuery(ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      cudaEventDestroy(ev);
      std::string m = std::string(what) + ": " + cudaGetErrorString(e);
      return plan_fail(s, MG_ERR_CUDA, m.c_str());
    }
    ncclResult_t ae = ncclSuccess;
    const ncclResult_t qr = ncclCommGetAsyncError(s->comm, &ae);
    if (qr != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
      fail_msg = std::string(what) + ": NCCL asynchronous error: " + ncclGetErrorString(qr != ncclSuccess ? qr : ae);
      break;
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > s->comm_timeout_s) {
      fail_msg = std::string(what) + ": timed out after " + std::to_string((int)s->comm_timeout_s) +
                 " s waiting on the device (a peer rank is stuck or dead)";
      break;
    }
    if (it > 1000) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  if (fail_msg.empty()) {
    cudaEventDestroy(ev);
    return MG_OK;
  }
  plan_comm_abort(s);  // unblocks the NCCL kernels still queued on the streams
  cudaEventDestroy(ev);
  return plan_fail(s, MG_ERR_NCCL, fail_msg.c_str());
}

void plan_comm_abort(mg_solver* s) {
  if (s->comm) {
    ncclCommAbort(s->comm);
    s->comm = nullptr;
  }
}

}  // namespace mg
