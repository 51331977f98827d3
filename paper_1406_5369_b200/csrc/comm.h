// comm.h — the slab decomposition's two collectives behind one interface:
// NCCL over NVLink (production), or LOOPBACK: the ranks of one process sharing one device,
// each driven by its own host thread, exchanging through device-to-device copies ordered
// by CUDA events and a host rendezvous (tests of the multi-rank path on one GPU; no kernel
// ever waits on another rank's kernel).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "mg.h"

struct mg_solver;

namespace mg {

// true when this rank exchanges with others (nranks > 1, NCCL or loopback)
bool comm_active(const mg_solver* s);
// halo exchange of one level array: my h top owned planes go to rank+1's lower halo,
// my h bottom owned planes to rank-1's upper halo; plane stride `pbytes` bytes, H halo
// planes per side, `owned` owned planes of this rank
cudaError_t comm_halo(mg_solver* s, void* buf, size_t pbytes, int H, int owned, int h, cudaStream_t st);
// in-place all-gather: rank r's chunk of `chunk` bytes sits at buf + r * chunk
cudaError_t comm_allgather(mg_solver* s, void* buf, size_t chunk, cudaStream_t st);

// Loopback ranks with CUDA graphs: all ranks of the group call this concurrently (one host
// thread each) for the same part; ONE graph holding every rank's work of that part is captured
// the first time (rank 0 begins the capture, the others' streams join it through an event, the
// exchanges' cross-rank event edges are then edges of that graph), and replayed after each
// rank's stream has reached the call; every rank's stream waits for the replay.
mg_status loop_graph_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st);

// loopback group (opaque to the ABI: mg_loopback_group_create / _destroy)
struct LoopGroup;
LoopGroup* loop_group_create(int nranks);
void loop_group_destroy(LoopGroup* g);
int loop_group_size(const LoopGroup* g);

}  // namespace mg
