// som_host.h — internal declarations shared by the host-runtime files of
// libsom: som_api.cu (errors, handle, weights, knobs, sharding plumbing,
// staging and CSR validation), som_train_api.cu (online training),
// som_map_api.cu (mapping, errors, U-matrix), som_extra_api.cu (batch SOM,
// upstream steps).  Product code only.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/som.h"
#include "som_device.cuh"
#include "som_internal.h"

namespace som {
namespace host {

// Record a message for som_last_error() (thread-local) and return st.
som_status fail(som_status st, const char* fmt, ...);

// Grow-only device scratch from the stream-ordered allocator: no
// device-wide synchronisation (a plain cudaMalloc would wait for every
// running kernel, e.g. another rank's persistent grid on the same device).
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaStream_t owner = nullptr;
    cudaError_t ensure(size_t bytes, cudaStream_t st) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, (size_t)256);
        cudaError_t e = cudaMallocAsync(&p, want, st);
        if (e == cudaSuccess) { cap = want; owner = st; }
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace host
}  // namespace som

using som::kMaxRanks;
using som::host::DevBuf;

struct som_ctx {
    int rows = 0, cols = 0, dim = 0, topo = 0, device = 0;
    int N = 0;                // units of the map (global)
    int NL = 0;               // units held by this handle (N unless neuron-sharded)
    int rank = 0, world = 1;  // neuron sharding: units u = rank + world * l
    unsigned long long* mail = nullptr;            // own cross-rank mailbox [2][world]
    unsigned long long* peer_mail[kMaxRanks] = {}; // every rank's mailbox (own included)
    bool peer_ipc[kMaxRanks] = {};                 // opened with cudaIpcOpenMemHandle
    float* W = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int sm_count = 0;
    int max_smem_optin = 0;
    bool poisoned = false;
    int map_precision = SOM_MAP_AUTO;
    int train_mode = SOM_TRAIN_AUTO;
    int train_grid = 0;       // 0 = auto
    int last_grid = 0, last_kernel = -1;
    int64_t last_spec_fallbacks = 0;
    unsigned long long* trace = nullptr;   // caller-owned device buffer (som_set_trace)
    int trace_steps = 0;
    // scratch
    DevBuf xin;      // staged X / CSR
    DevBuf xin2, xin3;
    DevBuf keys;     // mapping top-2 keys
    DevBuf outs;     // staged mapping outputs
    DevBuf red;      // reduction partials
    DevBuf ftab;     // decay table
    DevBuf log;      // staged BMU log
    DevBuf xchg;     // per-CTA exchange slots + abort flag
    DevBuf dense;    // densified CSR chunk
    DevBuf utab;     // unit dealing of the CSR training kernels: [G][S] + counts[G]
    int utab_G = 0, utab_NL = 0, utab_rank = -1, utab_world = 0;
    DevBuf wsplit;   // tensor-core mapping: W hi | W lo | |W|^2 (fp64) | max |w|
    int last_tc_fallbacks = 0;   // documents of the last 3xTF32 mapping that took the exact scan (R20b)
    DevBuf xsplit;   // tensor-core mapping: X chunk hi | lo | |x|^2
    bool w_split_valid = false;
    DevBuf bbuf;     // batch SOM: bmu | order | scratch (int32) | cnt | off | sort temp
    DevBuf bS, bnum; // batch SOM: per-BMU sums S and H S (fp64, N x (d+1))
    DevBuf up, up2;  // upstream steps (TF-IDF / PCA scratch)
    DevBuf wt64;     // sparse mapping: W^T fp64 or fp32 (dim x Np) | |W|^2 fp64 (N)
    DevBuf rflags;   // zero-row flags (n bytes, 1 = the row holds a non-zero value)
    DevBuf rmap;     // ascending list of the non-zero rows (int64) | count | select temp
    // NCCL communicator (som_comm_init_nccl): document sharding reduces the
    // error sums over it; neuron sharding can exchange the per-step winner
    // through it (SOM_XCHG_NCCL) instead of the peer-memory mailboxes
    void* nccl = nullptr;   // ncclComm_t
    int shard_mode = 0;     // 0 none, SOM_SHARD_DOCS, SOM_SHARD_NEURONS
    int nccl_rank = 0, nccl_world = 1;
    int xchg_mode = 0;      // SOM_XCHG_MAILBOX / SOM_XCHG_NCCL
    DevBuf nstep;           // NCCL step path: keys [3] u64 | reduce scratch
    DevBuf tcsr, tcsr2;     // dense rows put in CSR form for the training kernels: cnt | rowptr | temp, col | val
    DevBuf fitx, fitx2, fitx3;   // som_fit: the input staged once per call
    bool wt_valid = false, wt_f32 = false, wt_nonneg = false;
    int wt_J = 0;
    // decay-table cache
    int64_t f_T = -1, f_t0 = -1, f_t1 = -1;
    int f_kind = -1;
    double f_k = 0;
    // timing
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0;
    int64_t last_units = 0;
    int last_launches = 0;
    double last_phase_ms[5] = {};   // som_fit: stage+init, train, map, errors, U-matrix (+ copies)
    double last_train_ms = 0;       // som_fit: the training kernels alone
};

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            h->poisoned = true;                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? SOM_ENOMEM : SOM_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                   \
        }                                                                                     \
    } while (0)


#define CHECK_HANDLE(h)                                                                       \
    do {                                                                                      \
        if (!(h)) return fail(SOM_EINVAL, "null handle");                                    \
        if ((h)->poisoned) return fail(SOM_ESTATE, "handle poisoned by an earlier CUDA failure"); \
        cudaError_t e_ = cudaSetDevice((h)->device);                                          \
        if (e_ != cudaSuccess) {                                                              \
            (h)->poisoned = true;                                                             \
            return fail(SOM_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e_));            \
        }                                                                                     \
    } while (0)

namespace som {
namespace host {

struct CsrIn {
    const int64_t* rowptr;
    const int32_t* col;
    const float* val;
    int maxnnz;
    int64_t nnz;
};

struct OutStage {
    int32_t* b1 = nullptr; int32_t* b2 = nullptr; float* d2 = nullptr;
    bool host1 = false, host2 = false, host3 = false;
};

// som_api.cu
bool is_device_ptr(const void* p);
som_status stage_in(som_ctx* h, DevBuf& buf, const void* src, size_t bytes, const void** dev);
void invalidate_w_caches(som_ctx* h);
void fill_decay(double* out, int64_t t0, int64_t t1, int64_t T, int kind, double k);
som_status ensure_decay_table(som_ctx* h, int64_t T, int kind, double k, int64_t t0, int64_t t1);
som_status stage_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n, CsrIn* out);
// zero rows: flags of the n rows of Xd (or csr) into
// h->rflags, *m = number of non-zero rows; with list != NULL, *list = the
// ascending non-zero rows (h->rmap) when some row is zero, else NULL
som_status scan_rows(som_ctx* h, const float* Xd, const CsrIn* csr, int64_t n, int64_t* m, const int64_t** list);
// document sharding over NCCL: in-place sum of (f64 s, i64 c[2]) over the
// communicator (no-op without one)
som_status doc_allreduce(som_ctx* h, double* s, int64_t* c);
// som_comm.cu: step-at-a-time training with one NCCL u64-min all-reduce per
// step (a: TrainArgs of the call; launches: kernels + collectives issued)
som_status train_nccl_steps(som_ctx* h, const TrainArgs& a, int* launches);
// som_map_api.cu
bool use_tc(const som_ctx* h, int64_t n);
int csr_path(const som_ctx* h, const CsrIn& csr, int64_t n);
som_status map_dense_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches);
som_status map_exact_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches);
som_status map_csr_dev(som_ctx* h, const CsrIn& csr, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches);
som_status stage_outputs(som_ctx* h, int64_t n, int32_t* bmu1, int32_t* bmu2, float* d2, bool need_all, OutStage& o);
som_status copy_back(som_ctx* h, int64_t n, int32_t* bmu1, int32_t* bmu2, float* d2, const OutStage& o);
som_status finish_errors(som_ctx* h, int64_t n, const OutStage& o, int launches, double* qe, double* te, int64_t m);
bool doc_sharded(const som_ctx* h);

}  // namespace host
}  // namespace som
