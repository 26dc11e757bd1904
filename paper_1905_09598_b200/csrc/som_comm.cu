// som_comm.cu — host runtime of libsom, part 5: the NCCL communicator
// (SURVEY §8.B som_comm_unique_id / som_comm_init with a shard mode, §8.E).
//  * Document sharding (SOM_SHARD_DOCS): every rank maps its own documents
//    with the unchanged per-document path; som_errors / som_errors_csr sum
//    the fp64 sqrt(D1) total and the int64 counts (non-adjacent pairs,
//    scored rows) over the ranks with ncclAllReduce before dividing, so QE
//    and TE are those of the whole corpus on every rank.
//  * Neuron sharding (SOM_SHARD_NEURONS): the units u = rank + world * l of
//    som_comm_init; the per-step winner is exchanged either in-kernel through
//    peer-memory mailboxes (SOM_XCHG_MAILBOX, som_comm_set_peers_*) or with
//    one ncclAllReduce(u64, min) per step between step kernels
//    (SOM_XCHG_NCCL, train_step.cu; launches captured in CUDA graphs).
#include <nccl.h>

#include "som_host.h"

using namespace som;
using namespace som::host;

namespace som {
cudaError_t launch_step(const TrainArgs& a, unsigned long long* keys, const int* chunk, int K, int64_t t_first, int i,
                        cudaStream_t st);
cudaError_t launch_step_chunk_inc(int* chunk, cudaStream_t st);
}  // namespace som

#define NK(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            h->poisoned = true;                                                               \
            return fail(SOM_ENCCL, "%s: %s", #call, ncclGetErrorString(r_));                \
        }                                                                                     \
    } while (0)

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

namespace som {
namespace host {

som_status doc_allreduce(som_ctx* h, double* s, int64_t* c) {
    if (!h->nccl) return SOM_OK;
    CK(h->nstep.ensure(64, h->stream));
    char* base = (char*)h->nstep.p;
    double* ds = (double*)(base + 32);
    int64_t* dc = (int64_t*)(base + 40);
    CK(cudaMemcpyAsync(ds, s, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(dc, c, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
    ncclComm_t comm = (ncclComm_t)h->nccl;
    NK(ncclGroupStart());
    NK(ncclAllReduce(ds, ds, 1, ncclFloat64, ncclSum, comm, h->stream));
    NK(ncclAllReduce(dc, dc, 2, ncclInt64, ncclSum, comm, h->stream));
    NK(ncclGroupEnd());
    CK(cudaMemcpyAsync(s, ds, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(c, dc, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

// Step-at-a-time training with the NCCL u64-min exchange (train_step.cu).
// Steps are replayed from a CUDA graph of K steps (K % 3 == 0 keeps each
// node's key slot fixed across replays); the remainder and the final flush
// are launched directly.  SOM_NCCL_GRAPH=0 launches every step directly.
som_status train_nccl_steps(som_ctx* h, const TrainArgs& a, int* launches) {
    if (!h->nccl) return fail(SOM_ESTATE, "SOM_XCHG_NCCL needs som_comm_init_nccl");
    ncclComm_t comm = (ncclComm_t)h->nccl;
    CK(h->nstep.ensure(64, h->stream));
    unsigned long long* keys = (unsigned long long*)h->nstep.p;   // [3]
    int* chunk = (int*)((char*)h->nstep.p + 24);
    CK(cudaMemsetAsync(keys, 0xFF, 3 * sizeof(unsigned long long), h->stream));
    CK(cudaMemsetAsync(chunk, 0, sizeof(int), h->stream));
    const int64_t steps = a.t1 - a.t0;
    const int K = 96;
    bool graph = steps >= 4 * K;
    if (const char* e = std::getenv("SOM_NCCL_GRAPH")) graph = graph && std::atoi(e) != 0;
    int64_t done = 0;
    *launches = 0;
    if (graph) {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        cudaStream_t cs = nullptr;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        bool ok = e == cudaSuccess;
        for (int i = 0; ok && i < K; ++i) {
            ok = launch_step(a, keys, chunk, K, a.t0, i, cs) == cudaSuccess;
            if (ok) ok = ncclAllReduce(keys + (a.t0 + i) % 3, keys + (a.t0 + i) % 3, 1, ncclUint64, ncclMin, comm, cs) ==
                         ncclSuccess;
        }
        if (ok) ok = launch_step_chunk_inc(chunk, cs) == cudaSuccess;
        e = cudaStreamEndCapture(cs, &g);
        ok = ok && e == cudaSuccess;
        if (ok) ok = cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
        if (ok) {
            // the graph runs after the memsets on h->stream
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, h->stream));
            CK(cudaStreamWaitEvent(cs, ev, 0));
            const int64_t reps = steps / K;
            for (int64_t r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, cs));
            CK(cudaEventRecord(ev, cs));
            CK(cudaStreamWaitEvent(h->stream, ev, 0));
            CK(cudaEventDestroy(ev));
            done = reps * K;
            *launches += (int)(reps * (K + 1));
        }
        cudaGetLastError();
        if (ge) cudaGraphExecDestroy(ge);
        if (g) cudaGraphDestroy(g);
        CK(cudaStreamSynchronize(cs));
        cudaStreamDestroy(cs);
    }
    for (int64_t t = a.t0 + done; t < a.t1; ++t) {
        CK(launch_step(a, keys, nullptr, 0, t, 0, h->stream));
        NK(ncclAllReduce(keys + t % 3, keys + t % 3, 1, ncclUint64, ncclMin, comm, h->stream));
        ++*launches;
    }
    CK(launch_step(a, keys, nullptr, 0, a.t1, 0, h->stream));   // flush the last update (+ its log entry)
    ++*launches;
    return SOM_OK;
}

}  // namespace host
}  // namespace som

extern "C" {

som_status som_comm_unique_id(uint8_t* id128) {
    if (!id128) return fail(SOM_EINVAL, "null id");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(SOM_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    std::memcpy(id128, &id, sizeof(id));
    return SOM_OK;
}

som_status som_comm_init_nccl(som_ctx* h, int32_t rank, int32_t world, const uint8_t* id128, int32_t shard_mode) {
    CHECK_HANDLE(h);
    if (!id128) return fail(SOM_EINVAL, "null id");
    if (shard_mode != SOM_SHARD_DOCS && shard_mode != SOM_SHARD_NEURONS) return fail(SOM_EINVAL, "unknown shard mode");
    if (world < 1 || rank < 0 || rank >= world) return fail(SOM_EINVAL, "bad rank / world");
    if (shard_mode == SOM_SHARD_NEURONS) {
        som_status st = som_comm_init(h, rank, world);   // neuron partition, mailbox, W re-zeroed
        if (st) return st;
    }
    if (h->nccl) {
        ncclCommDestroy((ncclComm_t)h->nccl);
        h->nccl = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    NK(ncclCommInitRank(&comm, world, id, rank));
    h->nccl = comm;
    h->shard_mode = shard_mode;
    h->nccl_rank = rank;
    h->nccl_world = world;
    return SOM_OK;
}

som_status som_set_exchange(som_ctx* h, int32_t mode) {
    CHECK_HANDLE(h);
    if (mode != SOM_XCHG_MAILBOX && mode != SOM_XCHG_NCCL) return fail(SOM_EINVAL, "unknown exchange mode");
    h->xchg_mode = mode;
    return SOM_OK;
}

}  // extern "C"

// called by som_destroy
void som_comm_release(som_ctx* h) {
    if (h->nccl) ncclCommDestroy((ncclComm_t)h->nccl);
    h->nccl = nullptr;
}
