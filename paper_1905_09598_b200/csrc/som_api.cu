// som_api.cu — host runtime of libsom: validation, residency, staging of
// host buffers, the decay table, launch sizing, timing.  Implements
// include/som.h.  Product code: no oracle, no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/som.h"
#include "som_device.cuh"
#include "som_internal.h"

using namespace som;

namespace {

thread_local std::string g_err;

som_status fail(som_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

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

}  // namespace

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
    DevBuf wsplit;   // tensor-core mapping: W hi | W lo | |W|^2 (fp32)
    DevBuf xsplit;   // tensor-core mapping: X chunk hi | lo | |x|^2
    bool w_split_valid = false;
    DevBuf bbuf;     // batch SOM: bmu | order | scratch (int32) | cnt | off | sort temp
    DevBuf bS, bnum; // batch SOM: per-BMU sums S and H S (fp64, N x (d+1))
    DevBuf up, up2;  // upstream steps (TF-IDF / PCA scratch)
    DevBuf wt64;     // sparse mapping: W^T fp64 or fp32 (dim x Np) | |W|^2 fp64 (N)
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
};

namespace {

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            h->poisoned = true;                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? SOM_ENOMEM : SOM_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                   \
        }                                                                                     \
    } while (0)

// W changed: drop every derived copy (tensor-core split planes, sparse W^T)
void invalidate_w_caches(som_ctx* h) {
    h->w_split_valid = false;
    h->wt_valid = false;
}

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

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Make `src` (count bytes) available on the device: device pointers pass
// through; host pointers are copied into `buf`.
som_status stage_in(som_ctx* h, DevBuf& buf, const void* src, size_t bytes, const void** dev) {
    if (is_device_ptr(src)) {
        *dev = src;
        return SOM_OK;
    }
    CK(buf.ensure(bytes, h->stream));
    CK(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, h->stream));
    *dev = buf.p;
    return SOM_OK;
}

// Decay factor table f_t, t in [t0, t1), of T steps (R1).  Computed on the
// host in fp64 with the same expression order as the definition so the
// device sees exactly the factors the definition gives; cached per
// (T, kind, k, range).
void fill_decay(double* out, int64_t t0, int64_t t1, int64_t T, int kind, double k) {
    const double Td = (double)T;
    const double e_k = std::exp(-k);
    for (int64_t t = t0; t < t1; ++t) {
        const double tau = (double)t / Td;
        double f;
        if (kind == SOM_DECAY_GAUSSIAN) f = std::exp(-k * tau * tau);
        else if (kind == SOM_DECAY_LINEAR) f = 1.0 - (1.0 - e_k) * tau;
        else f = std::exp(-k * tau);
        out[t - t0] = f;
    }
}

som_status ensure_decay_table(som_ctx* h, int64_t T, int kind, double k, int64_t t0, int64_t t1) {
    if (h->f_T == T && h->f_kind == kind && h->f_k == k && h->f_t0 == t0 && h->f_t1 == t1) return SOM_OK;
    const int64_t cnt = t1 - t0;
    std::vector<double> host((size_t)cnt);
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (cnt < 65536) nth = 1;
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nth; ++w) {
        int64_t a = t0 + cnt * w / nth, b = t0 + cnt * (w + 1) / nth;
        th.emplace_back(fill_decay, host.data() + (a - t0), a, b, T, kind, k);
    }
    for (auto& x : th) x.join();
    CK(h->ftab.ensure(sizeof(double) * (size_t)std::max<int64_t>(cnt, 1), h->stream));
    CK(cudaMemcpyAsync(h->ftab.p, host.data(), sizeof(double) * (size_t)cnt, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->f_T = T; h->f_kind = kind; h->f_k = k; h->f_t0 = t0; h->f_t1 = t1;
    return SOM_OK;
}

uint64_t mulhi_host(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

}  // namespace

// ===================================================================== ABI
extern "C" {

const char* som_last_error(void) { return g_err.c_str(); }

const char* som_version(void) { return "libsom 0.2 sm_100a (persistent online SOM; exact fp64 and tcgen05 3xTF32 mapping)"; }

som_status som_schedule_default(som_schedule* s) {
    if (!s) return fail(SOM_EINVAL, "null schedule");
    s->kind = SOM_DECAY_GAUSSIAN;
    s->k = std::log(100.0);
    s->sigma_min = 1.0;
    s->cutoff = 1e-4;
    return SOM_OK;
}

som_status som_create(int32_t rows, int32_t cols, int32_t dim, int32_t topology, int32_t device, som_ctx** out) {
    g_err.clear();
    if (!out) return fail(SOM_EINVAL, "null out");
    *out = nullptr;
    if (rows < 1 || cols < 1 || dim < 1) return fail(SOM_EINVAL, "rows, cols, dim must be >= 1");
    if ((int64_t)rows * cols > kMaxUnits) return fail(SOM_EINVAL, "rows*cols must be < 2^24");
    if (topology != SOM_RECT && topology != SOM_HEX) return fail(SOM_EINVAL, "topology must be SOM_RECT or SOM_HEX");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(SOM_ECUDA, "no CUDA device (%s)", cudaGetErrorString(e));
    }
    if (device < 0 || device >= ndev) return fail(SOM_EINVAL, "device %d out of range", device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(SOM_ECUDA, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(SOM_ECUDA, "libsom is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
    som_ctx* h = new som_ctx();
    h->rows = rows; h->cols = cols; h->dim = dim; h->topo = topology; h->device = device;
    h->N = rows * cols;
    h->NL = h->N;
    h->sm_count = prop.multiProcessorCount;
    h->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
    auto bad = [&](cudaError_t err, const char* what) {
        som_status st = fail(err == cudaErrorMemoryAllocation ? SOM_ENOMEM : SOM_ECUDA, "%s: %s", what,
                             cudaGetErrorString(err));
        som_destroy(h);
        return st;
    };
    if ((e = cudaSetDevice(device)) != cudaSuccess) return bad(e, "cudaSetDevice");
    if ((e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking)) != cudaSuccess) return bad(e, "stream");
    h->stream = h->own_stream;
    if ((e = cudaMalloc(&h->W, sizeof(float) * (size_t)h->N * dim)) != cudaSuccess) return bad(e, "cudaMalloc W");
    if ((e = cudaMemsetAsync(h->W, 0, sizeof(float) * (size_t)h->N * dim, h->stream)) != cudaSuccess) return bad(e, "memset");
    if ((e = cudaEventCreate(&h->ev0)) != cudaSuccess) return bad(e, "event");
    if ((e = cudaEventCreate(&h->ev1)) != cudaSuccess) return bad(e, "event");
    if ((e = cudaStreamSynchronize(h->stream)) != cudaSuccess) return bad(e, "sync");
    *out = h;
    return SOM_OK;
}

void som_destroy(som_ctx* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (DevBuf* b : {&h->xin, &h->xin2, &h->xin3, &h->keys, &h->outs, &h->red, &h->ftab, &h->log, &h->xchg, &h->dense,
                      &h->utab, &h->wsplit, &h->xsplit, &h->wt64, &h->bbuf, &h->bS, &h->bnum, &h->up, &h->up2})
        b->release();
    if (h->W) cudaFree(h->W);
    for (int p = 0; p < kMaxRanks; ++p)
        if (h->peer_ipc[p] && h->peer_mail[p]) cudaIpcCloseMemHandle(h->peer_mail[p]);
    if (h->mail) cudaFree(h->mail);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
}

som_status som_set_stream(som_ctx* h, void* cuda_stream) {
    CHECK_HANDLE(h);
    CK(cudaStreamSynchronize(h->stream));
    h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
    return SOM_OK;
}

// The caller always passes the FULL N x dim map.  A neuron-sharded handle
// keeps rows u = rank + world*l (strided 2-D copies); other rows of the
// caller's buffer are left untouched by som_get_weights.
som_status som_set_weights(som_ctx* h, const float* w) {
    CHECK_HANDLE(h);
    if (!w) return fail(SOM_EINVAL, "null weights");
    invalidate_w_caches(h);
    const size_t rowb = sizeof(float) * (size_t)h->dim;
    CK(cudaMemcpy2DAsync(h->W, rowb, w + (size_t)h->rank * h->dim, rowb * h->world, rowb, (size_t)h->NL,
                         cudaMemcpyDefault, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

som_status som_get_weights(som_ctx* h, float* w) {
    CHECK_HANDLE(h);
    if (!w) return fail(SOM_EINVAL, "null weights");
    const size_t rowb = sizeof(float) * (size_t)h->dim;
    CK(cudaMemcpy2DAsync(w + (size_t)h->rank * h->dim, rowb * h->world, h->W, rowb, rowb, (size_t)h->NL,
                         cudaMemcpyDefault, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

som_status som_init_random(som_ctx* h, const float* X, int64_t n, uint64_t seed) {
    CHECK_HANDLE(h);
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0");
    const int N = h->N;
    invalidate_w_caches(h);
    std::vector<int64_t> idx((size_t)N);
    if (N <= n) {
        // Floyd's sampling without replacement, draws from SplitMix64(seed)
        std::unordered_set<int64_t> taken;
        taken.reserve((size_t)N * 2);
        int64_t draw = 0, o = 0;
        for (int64_t j = n - N; j < n; ++j) {
            int64_t r = (int64_t)mulhi_host(splitmix64_at(seed, draw++), (uint64_t)(j + 1));
            int64_t pick = taken.count(r) ? j : r;
            taken.insert(pick);
            idx[(size_t)o++] = pick;
        }
    } else {
        for (int u = 0; u < N; ++u) idx[(size_t)u] = (int64_t)mulhi_host(splitmix64_at(seed, u), (uint64_t)n);
    }
    // a neuron-sharded handle keeps the draws of its own units
    std::vector<int64_t> mine((size_t)h->NL);
    for (int l = 0; l < h->NL; ++l) mine[(size_t)l] = idx[(size_t)h->rank + (size_t)h->world * l];
    const int NL = h->NL;
    const size_t rowb = sizeof(float) * (size_t)h->dim;
    if (is_device_ptr(X)) {
        CK(h->keys.ensure(sizeof(int64_t) * (size_t)NL, h->stream));
        CK(cudaMemcpyAsync(h->keys.p, mine.data(), sizeof(int64_t) * (size_t)NL, cudaMemcpyHostToDevice, h->stream));
        CK(launch_gather_rows(X, (const int64_t*)h->keys.p, NL, h->dim, h->W, h->stream));
    } else {
        std::vector<float> rowsbuf((size_t)NL * h->dim);
        for (int l = 0; l < NL; ++l)
            std::memcpy(rowsbuf.data() + (size_t)l * h->dim, X + mine[(size_t)l] * h->dim, rowb);
        CK(cudaMemcpyAsync(h->W, rowsbuf.data(), rowb * (size_t)NL, cudaMemcpyHostToDevice, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

namespace {

struct CsrIn {
    const int64_t* rowptr;
    const int32_t* col;
    const float* val;
    int maxnnz;
    int64_t nnz;
};

// shared argument checks of som_train_online / som_train_online_csr; on OK
// *sd holds the schedule and [*t_begin, *t_end) the (resolved) step range
som_status check_train(som_ctx* h, int64_t n, int32_t epochs, double alpha0, double sigma0, const som_schedule* s,
                       som_schedule* sd, int64_t* t_begin, int64_t* t_end) {
    som_schedule_default(sd);
    if (s) *sd = *s;
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: no data to train on");
    if (epochs < 0) return fail(SOM_EINVAL, "epochs must be >= 0");
    if (!(alpha0 >= 0.0 && alpha0 <= 1.0)) return fail(SOM_EINVAL, "alpha0 must be in [0, 1]");
    if (!(sigma0 > 0.0) || !std::isfinite(sigma0)) return fail(SOM_EINVAL, "sigma0 must be > 0");
    if (sd->kind < 0 || sd->kind > 2) return fail(SOM_EINVAL, "unknown decay kind");
    if (!(sd->k > 0.0) || !std::isfinite(sd->k)) return fail(SOM_EINVAL, "decay constant k must be > 0");
    if (!(sd->sigma_min > 0.0)) return fail(SOM_EINVAL, "sigma_min must be > 0");
    if (!(sd->cutoff >= 0.0 && sd->cutoff < 1.0)) return fail(SOM_EINVAL, "cutoff must be in [0, 1)");
    const int64_t T = (int64_t)epochs * n;
    if (*t_end == -1) *t_end = T;
    if (*t_begin < 0 || *t_end < *t_begin || *t_end > T)
        return fail(SOM_EINVAL, "bad t-range [%lld, %lld) for T = %lld", (long long)*t_begin, (long long)*t_end,
                    (long long)T);
    h->last_ms = 0; h->last_units = 0; h->last_launches = 0;
    return SOM_OK;
}

// Unit dealing for the CSR training kernels.  With cyclic dealing (b + s*G)
// the units of one CTA lie on a few long lattice lines, so the disk of units
// a pending update touches gives some CTAs many rows and others none, and the
// step waits for the fullest CTA.  Here unit (i, j) goes to class
// (alpha*i + j) mod G with alpha chosen so that every class is a near-square
// sub-lattice (its shortest vector is maximal), then to the first class with
// room (capacity ceil(NL/G), linear probing): any disk then holds about the
// same number of rows of every CTA, and the all-dense step keeps its balance.
void build_unit_tab(int rows, int cols, int topo, int rank, int world, int NL, int G, std::vector<int>& out) {
    const int S = (NL + G - 1) / G;
    int best_alpha = cols % G;
    double best_len = -1.0;
    for (int al = 1; al < G; ++al) {
        double mn = 1e300;
        for (int di = 0; di < rows && di <= 64; ++di) {
            const int dj0 = (int)((((long long)-al * di) % G + G) % G);
            for (int dj : {dj0, dj0 - G}) {
                if (di == 0 && dj == 0) continue;
                if (dj >= cols || -dj >= cols) continue;   // no such pair of units
                const double len = topo == 0 ? (double)di * di + (double)dj * dj
                                             : (double)dj * dj + 0.75 * (double)di * di;
                mn = std::min(mn, len);
            }
        }
        if (mn > best_len) { best_len = mn; best_alpha = al; }
    }
    out.assign((size_t)G * S + G, -1);
    int* cnt = out.data() + (size_t)G * S;
    for (int b = 0; b < G; ++b) cnt[b] = 0;
    for (int l = 0; l < NL; ++l) {
        const long long u = (long long)rank + (long long)world * l;
        const long long i = u / cols, j = u % cols;
        int k = (int)(((long long)best_alpha * i + j) % G);
        while (cnt[k] >= S) k = (k + 1) % G;
        out[(size_t)k * S + cnt[k]++] = l;
    }
}

// CSR arrays staged to the device and checked there (rowptr from 0 and
// non-decreasing, col strictly increasing within a row and < dim); returns
// the device pointers and the largest row length
som_status stage_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                     CsrIn* out) {
    if (!rowptr || !col || !val) return fail(SOM_EINVAL, "null CSR array");
    int64_t nnz = 0;
    if (is_device_ptr(rowptr)) CK(cudaMemcpy(&nnz, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    else nnz = rowptr[n];
    if (nnz < 0) return fail(SOM_EINVAL, "rowptr[n] < 0");
    const void *rpd, *cd, *vd;
    som_status st = stage_in(h, h->xin, rowptr, sizeof(int64_t) * (size_t)(n + 1), &rpd);
    if (st) return st;
    if ((st = stage_in(h, h->xin2, col, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1), &cd))) return st;
    if ((st = stage_in(h, h->xin3, val, sizeof(float) * (size_t)std::max<int64_t>(nnz, 1), &vd))) return st;
    CK(h->red.ensure(64, h->stream));
    int* chk = (int*)h->red.p;
    CK(launch_csr_check((const int64_t*)rpd, (const int32_t*)cd, n, h->dim, chk, h->stream));
    int res[2] = {0, 0};
    CK(cudaMemcpyAsync(res, chk, sizeof(res), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (res[0] & 1) return fail(SOM_EINVAL, "CSR rowptr must start at 0 and be non-decreasing");
    if (res[0] & 2) return fail(SOM_EINVAL, "CSR column index outside [0, dim)");
    if (res[0] & 4) return fail(SOM_EINVAL, "CSR column indices must be strictly increasing within a row");
    out->rowptr = (const int64_t*)rpd;
    out->col = (const int32_t*)cd;
    out->val = (const float*)vd;
    out->maxnnz = res[1];
    out->nnz = nnz;
    return SOM_OK;
}

som_status train_impl(som_ctx* h, const void* Xd, const CsrIn* csr, int64_t n, int32_t epochs, double alpha0,
                      double sigma0, const som_schedule& sd, uint64_t seed, int64_t t_begin, int64_t t_end,
                      int32_t* bmu_log);

}  // namespace

som_status som_train_online(som_ctx* h, const float* X, int64_t n, int32_t epochs, double alpha0, double sigma0,
                            const som_schedule* s, uint64_t seed, int64_t t_begin, int64_t t_end, int32_t* bmu_log) {
    CHECK_HANDLE(h);
    if (!X) return fail(SOM_EINVAL, "null X");
    som_schedule sd;
    som_status st = check_train(h, n, epochs, alpha0, sigma0, s, &sd, &t_begin, &t_end);
    if (st) return st;
    if (t_end == t_begin) return SOM_OK;   // epochs = 0 or empty range: weights unchanged
    const void* Xd = nullptr;
    if ((st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd))) return st;
    return train_impl(h, Xd, nullptr, n, epochs, alpha0, sigma0, sd, seed, t_begin, t_end, bmu_log);
}

som_status som_train_online_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                                int32_t epochs, double alpha0, double sigma0, const som_schedule* s, uint64_t seed,
                                int64_t t_begin, int64_t t_end, int32_t* bmu_log) {
    CHECK_HANDLE(h);
    som_schedule sd;
    som_status st = check_train(h, n, epochs, alpha0, sigma0, s, &sd, &t_begin, &t_end);
    if (st) return st;
    CsrIn csr{};
    if ((st = stage_csr(h, rowptr, col, val, n, &csr))) return st;
    if (t_end == t_begin) return SOM_OK;
    return train_impl(h, nullptr, &csr, n, epochs, alpha0, sigma0, sd, seed, t_begin, t_end, bmu_log);
}

namespace {

som_status train_impl(som_ctx* h, const void* Xd, const CsrIn* csr, int64_t n, int32_t epochs, double alpha0,
                      double sigma0, const som_schedule& sd, uint64_t seed, int64_t t_begin, int64_t t_end,
                      int32_t* bmu_log) {
    const int64_t T = (int64_t)epochs * n;
    invalidate_w_caches(h);
    som_status st = SOM_OK;
    if ((st = ensure_decay_table(h, T, sd.kind, sd.k, t_begin, t_end))) return st;

    TrainArgs a{};
    a.W = h->W; a.X = (const float*)Xd; a.n = n; a.dim = h->dim; a.dimp = (h->dim + 3) & ~3;
    a.rows = h->rows; a.cols = h->cols; a.topo = h->topo; a.N = h->NL;
    a.rank = h->rank; a.world = h->world;
    for (int p = 0; p < kMaxRanks; ++p) a.mail[p] = h->peer_mail[p];
    if (h->world > 1) {
        for (int p = 0; p < h->world; ++p)
            if (!h->peer_mail[p]) return fail(SOM_ESTATE, "neuron sharding: peer mailboxes not set (som_comm_set_peers_*)");
    }
    a.x_vec4 = (h->dim % 4 == 0) && (csr || (uintptr_t)Xd % 16 == 0);   // densified CSR is aligned
    // launch geometry.  Register-resident kernel when a CTA's share of W fits
    // the register file: G minimises (all-gather latency + fp64 distance
    // time), both measured on B200 (profiles/probe_*_r01.json).  Otherwise
    // one persistent CTA per SM with W in shared or global memory.
    // short prototypes (d <= 128): the lane-group kernel (train_small.cu).
    // G minimises (all-gather latency + per-CTA rounds of work), with the
    // L2 traffic of the streamed variant when the map exceeds 4 rounds.
    bool use_small = false;
    if ((h->train_mode == SOM_TRAIN_AUTO || h->train_mode == SOM_TRAIN_SHORT_ROWS) && a.x_vec4 &&
        train_small_supported(h->dim)) {
        auto xchg_us = [](int G) { return G <= 32 ? 0.65 : G <= 64 ? 0.70 : G <= 128 ? 0.85 : 1.65; };
        const int gmax = std::min(h->NL, h->sm_count);
        double best = 1e30;
        int bestG = 0;
        for (int G : {8, 16, 32, 64, 128, gmax}) {
            if (h->train_grid > 0) G = std::min(h->train_grid, gmax);
            if (G < 1 || G > gmax) continue;
            const int R = small_rounds((h->NL + G - 1) / G, h->dim);
            double est = xchg_us(G) + 0.35 * R;   // ~0.35 us per round (tools/sweep_small.py, d = 64)
            // streamed: read + ~60 % written per step at ~12 TB/s of L2 over 148 SMs, pro rata G
            if (R > 4) est += 2.6 * 4.0 * (double)h->NL * h->dim / (12.0e6 * G / 148.0);
            if (est < best) { best = est; bestG = G; }
        }
        use_small = bestG > 0;
        a.G = bestG;
    }
    if (h->train_mode == SOM_TRAIN_SHORT_ROWS && !use_small)
        return fail(SOM_EUNSUPPORTED, "short-row kernel needs d <= 128 and d %% 4 == 0");
    bool use_reg = false;
    if (!use_small && (h->train_mode == SOM_TRAIN_AUTO || h->train_mode == SOM_TRAIN_W_REGISTERS) && a.x_vec4) {
        // all-gather latency by grid size (profiles/probe_xchg_r01.json) and
        // per-CTA F2F-bound distance time: (S + 1) * d conversions at 16/clk
        // (power-of-two grids measured fastest: 16-64 ~0.6-0.7 us, 128 ~0.8 us,
        // 48/96/100/112/134/148 all slower; tools/sweep_grid.py on c2)
        auto xchg_us = [](int G) { return G <= 32 ? 0.65 : G <= 64 ? 0.70 : G <= 128 ? 0.85 : 1.65; };
        double best = 1e30;
        int bestG = 0;
        const int gmax = std::min(h->NL, h->sm_count);
        std::vector<int> cands = {16, 32, 64, 128};
        if (gmax <= 32) cands.push_back(gmax);
        for (int G : cands) {
            if (h->train_grid > 0) G = std::min(h->train_grid, gmax);
            if (G < 1 || G > gmax) continue;
            const int S = (h->NL + G - 1) / G;
            if (!train_reg_supported(S, h->dim)) continue;
            const double est = xchg_us(G) + (double)(S + 1) * h->dim / (16.0 * 1965.0);
            if (est < best) { best = est; bestG = G; }
        }
        if (bestG > 0) { use_reg = true; a.G = bestG; }
    }
    if (h->train_mode == SOM_TRAIN_W_REGISTERS && !use_reg)
        return fail(SOM_EUNSUPPORTED, "map share per CTA does not fit registers (or d %% 4 != 0)");
    if (!use_reg && !use_small) {
        a.G = std::min(h->NL, h->sm_count);
        if (h->train_grid > 0) a.G = std::min(a.G, h->train_grid);
    }
    a.S = (h->NL + a.G - 1) / a.G;
    a.t0 = t_begin; a.t1 = t_end; a.seed = seed;
    a.f_tab = (const double*)h->ftab.p;
    a.alpha0 = alpha0; a.sigma0 = sigma0; a.sigma_min = sd.sigma_min;
    a.cutoff_on = sd.cutoff > 0.0;
    a.ln_inv_eps = sd.cutoff > 0.0 ? std::log(1.0 / sd.cutoff) : 0.0;
    a.trace = h->trace;
    a.trace_steps = h->trace ? h->trace_steps : 0;
    a.trace_clk = 0;
    if (const char* e = std::getenv("SOM_TRACE_CLOCK")) a.trace_clk = std::atoi(e) != 0;
    size_t smem = train_smem_bytes(a.S, a.dimp, 1);
    a.w_smem = smem <= (size_t)h->max_smem_optin;
    if (h->train_mode == SOM_TRAIN_W_SHARED && !a.w_smem)
        return fail(SOM_EUNSUPPORTED, "W slice (%zu B/CTA) does not fit shared memory", smem);
    if (h->train_mode == SOM_TRAIN_W_GLOBAL) a.w_smem = 0;
    if (!a.w_smem) smem = train_smem_bytes(a.S, a.dimp, 0);
    // maps that do not fit on chip stream from global memory with the
    // pipelined kernel (train_glb.cu) when its layout applies
    const bool use_glb = !use_small && !use_reg && !a.w_smem && a.x_vec4 && train_glb_supported(a.S, h->dim);
    if (use_reg) smem = sizeof(float) * (3 * (size_t)a.dimp + (size_t)a.rows * (a.topo == 0 ? a.cols : 2 * a.cols));
    if (use_glb) smem = sizeof(float) * 2 * (size_t)a.dimp;
    if (use_small) {
        a.w_smem = 0;
        smem = sizeof(float) * 3 * (size_t)a.dimp +
               sizeof(double) * ((size_t)a.dimp + a.rows + (a.topo == 0 ? a.cols : 2 * a.cols));
    }
    // CSR input: the sparse-distance kernel where W streams from global
    // memory; on-chip maps (latency-bound, no gain) and layouts it does not
    // cover train on the densified rows
    bool use_csr = false;
    if (csr) {
        use_csr = !use_small && !use_reg && !a.w_smem && train_csr_supported(a.S, h->dim, csr->maxnnz, h->max_smem_optin);
        if (use_csr) {
            a.rowptr = csr->rowptr; a.col = csr->col; a.val = csr->val;
            a.nz_cap = csr_nz_cap(csr->maxnnz);
            // upper bound of the lattice g2 between any two units (exact for
            // rect; hex bound takes the half-column offset at the full row span)
            const double dr = h->rows - 1, dc = h->cols - 1;
            a.g2max = h->topo == 0 ? dr * dr + dc * dc : 0.25 * (2 * dc + 1) * (2 * dc + 1) + 0.75 * dr * dr;
            if (h->utab_G != a.G || h->utab_NL != h->NL || h->utab_rank != h->rank || h->utab_world != h->world) {
                std::vector<int> tab;
                build_unit_tab(h->rows, h->cols, h->topo, h->rank, h->world, h->NL, a.G, tab);
                CK(h->utab.ensure(sizeof(int) * tab.size(), h->stream));
                CK(cudaMemcpyAsync(h->utab.p, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, h->stream));
                CK(cudaStreamSynchronize(h->stream));
                h->utab_G = a.G; h->utab_NL = h->NL; h->utab_rank = h->rank; h->utab_world = h->world;
            }
            a.utab = (const int*)h->utab.p;
            a.ucnt = a.utab + (size_t)a.G * a.S;
            smem = sizeof(float) * 2 * (size_t)a.dimp + 24 * (size_t)a.nz_cap;
        } else {
            CK(h->dense.ensure(sizeof(float) * (size_t)n * h->dim, h->stream));
            CK(launch_densify(csr->rowptr, csr->col, csr->val, 0, n, h->dim, (float*)h->dense.p, h->stream));
            a.X = (const float*)h->dense.p;
        }
    }
    if (smem > (size_t)h->max_smem_optin)
        return fail(SOM_EUNSUPPORTED, "dim %d too large for the x staging ring (%zu B smem)", h->dim, smem);

    // exchange slots: two parities of G slots, each parity on its own 256-byte
    // lines (a line shared by step t's and step t+1's slots would be written
    // by fast CTAs while slow ones still poll it)
    a.xstride = (a.G + 31) & ~31;
    a.poll_ns = 0;
    if (const char* e = std::getenv("SOM_POLL_NS")) a.poll_ns = std::max(0, std::atoi(e));
    CK(h->xchg.ensure(sizeof(unsigned long long) * 2 * (size_t)a.xstride + 64, h->stream));
    a.xchg = (unsigned long long*)h->xchg.p;
    a.abort_flag = (unsigned*)((char*)h->xchg.p + sizeof(unsigned long long) * 2 * (size_t)a.xstride);
    CK(cudaMemsetAsync(h->xchg.p, 0, sizeof(unsigned long long) * 2 * (size_t)a.xstride + 64, h->stream));

    const int64_t steps = t_end - t_begin;
    bool log_dev = bmu_log && is_device_ptr(bmu_log);
    if (bmu_log && !log_dev) CK(h->log.ensure(sizeof(int32_t) * (size_t)steps, h->stream));
    a.bmu_log = bmu_log ? (log_dev ? bmu_log : (int32_t*)h->log.p) : nullptr;

    // W streamed from global memory every step: keep it resident in L2 with a
    // persisting access-policy window (random X rows stream past it), undone
    // after the launch so the caller's stream is left as it was.
    bool l2_window = false;
    const char* nowin = std::getenv("SOM_NO_L2_WINDOW");
    if (!(nowin && std::atoi(nowin)) && !use_reg && !a.w_smem && (!use_small || small_rounds(a.S, h->dim) > 4)) {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
        const size_t wbytes = sizeof(float) * (size_t)h->NL * h->dim;
        int l2_bytes = 0;
        cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, h->device);
        // only for maps that fit the L2: for a map several times the L2 (c4 on
        // one GPU, 800 MB) the persisting lines of the window crowd out the
        // streamed rest of W and the row writes (measured 664 -> 263 us/step
        // without it)
        if (max_persist > 0 && max_window > 0 && wbytes <= (size_t)l2_bytes) {
            const size_t win = std::min(wbytes, (size_t)max_window);
            const size_t keep = std::min(win, (size_t)max_persist);
            if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, keep) == cudaSuccess) {
                cudaStreamAttrValue at{};
                at.accessPolicyWindow.base_ptr = h->W;
                at.accessPolicyWindow.num_bytes = win;
                at.accessPolicyWindow.hitRatio = (float)((double)keep / (double)win);
                at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                l2_window = cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &at) == cudaSuccess;
            }
            cudaGetLastError();
        }
    }
    CK(cudaEventRecord(h->ev0, h->stream));
    if (use_small) CK(launch_train_small(a, h->stream));
    else if (use_reg) CK(launch_train_reg(a, h->stream));
    else if (use_csr) CK(launch_train_csr(a, h->stream));
    else if (use_glb) CK(launch_train_glb(a, h->stream));
    else CK(launch_train(a, smem, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    if (l2_window) {   // later launches on the caller's stream get no window
        cudaStreamAttrValue at{};
        at.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &at);
        cudaGetLastError();
    }
    h->last_grid = a.G;
    h->last_kernel = use_small ? 5 : use_reg ? 2 : use_csr ? 4 : use_glb ? 3 : (a.w_smem ? 1 : 0);
    if (bmu_log && !log_dev)
        CK(cudaMemcpyAsync(bmu_log, h->log.p, sizeof(int32_t) * (size_t)steps, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (l2_window) {   // the kernel is done: demote its persisting lines and release the set-aside L2
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
    }
    unsigned abort_flag = 0;
    CK(cudaMemcpyAsync(&abort_flag, a.abort_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (abort_flag) {
        h->poisoned = true;
        return fail(SOM_ECUDA, "training exchange timed out (a CTA or rank stopped publishing its BMU candidate)");
    }
    // neuron sharding: clear the own mailbox so the next call's tags cannot
    // match stale entries (callers barrier between sharded calls)
    if (h->world > 1) {
        CK(cudaMemsetAsync(h->mail, 0, sizeof(unsigned long long) * 2 * (size_t)h->world, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = steps; h->last_launches = 1;
    return SOM_OK;
}

}  // namespace

som_status som_comm_init(som_ctx* h, int32_t rank, int32_t world) {
    CHECK_HANDLE(h);
    if (world < 1 || world > kMaxRanks) return fail(SOM_EINVAL, "world must be in [1, %d]", kMaxRanks);
    if (rank < 0 || rank >= world) return fail(SOM_EINVAL, "rank out of range");
    if (world > h->N) return fail(SOM_EINVAL, "more ranks than map units");
    const int NL = (h->N - rank + world - 1) / world;
    CK(cudaStreamSynchronize(h->stream));
    if (h->W) CK(cudaFree(h->W));
    h->W = nullptr;
    CK(cudaMalloc(&h->W, sizeof(float) * (size_t)NL * h->dim));
    CK(cudaMemsetAsync(h->W, 0, sizeof(float) * (size_t)NL * h->dim, h->stream));
    for (int p = 0; p < kMaxRanks; ++p) {
        if (h->peer_ipc[p] && h->peer_mail[p]) cudaIpcCloseMemHandle(h->peer_mail[p]);
        h->peer_ipc[p] = false;
        h->peer_mail[p] = nullptr;
    }
    if (h->mail) CK(cudaFree(h->mail));
    h->mail = nullptr;
    // one 2 MiB-aligned allocation of its own so its IPC handle maps nothing else
    CK(cudaMalloc(&h->mail, 2u << 20));
    CK(cudaMemsetAsync(h->mail, 0, 2u << 20, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    // pre-size the per-call training scratch: ranks that share one device
    // (tests) must not grow the memory pool while a peer grid is spinning
    CK(h->xchg.ensure(sizeof(unsigned long long) * 2 * 1024 + 64, h->stream));
    CK(h->ftab.ensure(sizeof(double) * ((size_t)1 << 20), h->stream));
    CK(h->log.ensure(sizeof(int32_t) * ((size_t)1 << 20), h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->rank = rank;
    h->world = world;
    h->NL = NL;
    h->peer_mail[rank] = h->mail;
    invalidate_w_caches(h);
    return SOM_OK;
}

som_status som_comm_local_units(som_ctx* h, int32_t* n_local) {
    if (!h || !n_local) return fail(SOM_EINVAL, "null argument");
    *n_local = h->NL;
    return SOM_OK;
}

som_status som_comm_mailbox_ipc(som_ctx* h, uint8_t* handle64) {
    CHECK_HANDLE(h);
    if (!handle64) return fail(SOM_EINVAL, "null handle buffer");
    if (!h->mail) return fail(SOM_ESTATE, "som_comm_init first");
    cudaIpcMemHandle_t ih;
    CK(cudaIpcGetMemHandle(&ih, h->mail));
    std::memcpy(handle64, &ih, sizeof(ih));
    return SOM_OK;
}

som_status som_comm_set_peers_ipc(som_ctx* h, const uint8_t* handles) {
    CHECK_HANDLE(h);
    if (!handles) return fail(SOM_EINVAL, "null handles");
    if (!h->mail) return fail(SOM_ESTATE, "som_comm_init first");
    for (int p = 0; p < h->world; ++p) {
        if (p == h->rank) continue;
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, handles + 64 * (size_t)p, sizeof(ih));
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
        h->peer_mail[p] = (unsigned long long*)ptr;
        h->peer_ipc[p] = true;
    }
    return SOM_OK;
}

som_status som_comm_set_peers_dev(som_ctx* h, void* const* mailboxes) {
    CHECK_HANDLE(h);
    if (!mailboxes) return fail(SOM_EINVAL, "null mailboxes");
    if (!h->mail) return fail(SOM_ESTATE, "som_comm_init first");
    for (int p = 0; p < h->world; ++p) {
        if (!mailboxes[p]) return fail(SOM_EINVAL, "null mailbox for rank %d", p);
        h->peer_mail[p] = (unsigned long long*)mailboxes[p];
    }
    return SOM_OK;
}

som_status som_comm_mailbox_ptr(som_ctx* h, void** mailbox) {
    if (!h || !mailbox) return fail(SOM_EINVAL, "null argument");
    *mailbox = h->mail;
    return SOM_OK;
}

som_status som_set_train_mode(som_ctx* h, int32_t mode) {
    CHECK_HANDLE(h);
    if (mode < SOM_TRAIN_AUTO || mode > SOM_TRAIN_SHORT_ROWS) return fail(SOM_EINVAL, "unknown train mode");
    h->train_mode = mode;
    return SOM_OK;
}

som_status som_set_trace(som_ctx* h, void* device_buf, int32_t steps) {
    CHECK_HANDLE(h);
    if (device_buf && (steps < 1 || !is_device_ptr(device_buf)))
        return fail(SOM_EINVAL, "trace buffer must be device memory with steps >= 1");
    h->trace = (unsigned long long*)device_buf;
    h->trace_steps = device_buf ? steps : 0;
    return SOM_OK;
}

som_status som_set_train_grid(som_ctx* h, int32_t grid) {
    CHECK_HANDLE(h);
    if (grid < 0) return fail(SOM_EINVAL, "grid must be >= 0 (0 = auto)");
    h->train_grid = grid;
    return SOM_OK;
}

som_status som_last_train_config(som_ctx* h, int32_t* grid, int32_t* kernel) {
    if (!h) return fail(SOM_EINVAL, "null handle");
    if (grid) *grid = h->last_grid;
    if (kernel) *kernel = h->last_kernel;
    return SOM_OK;
}

som_status som_set_map_precision(som_ctx* h, int32_t precision) {
    CHECK_HANDLE(h);
    if (precision < SOM_MAP_AUTO || precision > SOM_MAP_SPARSE_F64) return fail(SOM_EINVAL, "unknown map precision");
    h->map_precision = precision;
    return SOM_OK;
}

namespace {

// Which mapping path serves a call (som_set_map_precision; AUTO picks the
// tensor cores once the contraction is large enough to amortise the split).
bool use_tc(const som_ctx* h, int64_t n) {
    if (h->map_precision == SOM_MAP_EXACT_F64 || h->map_precision == SOM_MAP_SPARSE_F64) return false;
    if (h->map_precision == SOM_MAP_3XTF32) return true;
    return (double)n * h->N * h->dim >= 1.0e10;
}

// W split for the tensor-core path: hi, lo (N x dp) and |w|^2, cached until W changes.
som_status ensure_w_split(som_ctx* h, const float** whi, const float** wlo, const float** wn) {
    const int dp = tc_padded_dim(h->dim);
    const size_t plane = sizeof(float) * (size_t)h->N * dp;
    if (!h->w_split_valid) {
        CK(h->wsplit.ensure(2 * plane + sizeof(float) * (size_t)h->N, h->stream));
        char* base = (char*)h->wsplit.p;
        CK(launch_split_rows(h->W, h->N, h->dim, (float*)base, (float*)(base + plane), (float*)(base + 2 * plane),
                             h->stream));
        h->w_split_valid = true;
    }
    char* base = (char*)h->wsplit.p;
    *whi = (const float*)base;
    *wlo = (const float*)(base + plane);
    *wn = (const float*)(base + 2 * plane);
    return SOM_OK;
}

// Tensor-core mapping of n documents whose split rows are produced chunk by
// chunk by `fill(r0, m, hi, lo, norm)`; outputs device pointers.
using SplitFill = std::function<cudaError_t(int64_t, int64_t, float*, float*, float*)>;
som_status map_tc_rows(som_ctx* h, int64_t n, const SplitFill& fill, int32_t* b1, int32_t* b2, float* d2,
                       int* launches) {
    const float *whi, *wlo, *wn;
    som_status st = ensure_w_split(h, &whi, &wlo, &wn);
    if (st) return st;
    const int dp = tc_padded_dim(h->dim);
    // split-X chunk: up to 8 GiB of hi/lo planes (large chunks keep B panels hot)
    const int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(n, ((int64_t)8 << 30) / (8 * (int64_t)dp)));
    const size_t plane = sizeof(float) * (size_t)chunk * dp;
    CK(h->xsplit.ensure(2 * plane + sizeof(float) * (size_t)chunk, h->stream));
    char* xb = (char*)h->xsplit.p;
    const int tiles_n = tc_unit_tiles(h->N);
    CK(h->keys.ensure(sizeof(unsigned long long) * 2 * (size_t)tiles_n * (size_t)chunk, h->stream));
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t m = std::min(chunk, n - r0);
        CK(fill(r0, m, (float*)xb, (float*)(xb + plane), (float*)(xb + 2 * plane)));
        CK(launch_map_tc((const float*)xb, (const float*)(xb + plane), (const float*)(xb + 2 * plane), m, whi, wlo,
                         wn, h->N, h->dim, (unsigned long long*)h->keys.p, h->sm_count, h->stream));
        CK(launch_map_merge((const unsigned long long*)h->keys.p, tiles_n, m, b1 + r0, b2 ? b2 + r0 : nullptr,
                            d2 ? d2 + r0 : nullptr, h->stream));
        *launches += 3;
    }
    return SOM_OK;
}

som_status map_exact_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2,
                         int* launches);

// Map n rows of the device matrix Xd into device outputs (all device).
som_status map_dense_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches) {
    if (use_tc(h, n)) {
        auto fill = [&](int64_t r0, int64_t m, float* hi, float* lo, float* nrm) {
            return launch_split_rows(Xd + r0 * h->dim, m, h->dim, hi, lo, nrm, h->stream);
        };
        return map_tc_rows(h, n, fill, b1, b2, d2, launches);
    }
    return map_exact_dev(h, Xd, n, b1, b2, d2, launches);
}

// Exact dense definition (R10) of n device rows.
som_status map_exact_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2,
                         int* launches) {
    const int tiles_m = map_exact_tiles_m(n);
    const int tiles_n = map_exact_tiles_n(h->N);
    int nsplit = std::max(1, std::min(tiles_n, (2 * h->sm_count + tiles_m - 1) / tiles_m));
    CK(h->keys.ensure(sizeof(unsigned long long) * 2 * (size_t)nsplit * (size_t)n, h->stream));
    MapArgs a{h->W, h->N, Xd, n, h->dim, nsplit, (unsigned long long*)h->keys.p};
    CK(launch_map_exact(a, h->stream));
    CK(launch_map_merge(a.keys, nsplit, n, b1, b2, d2, h->stream));
    *launches += 2;
    return SOM_OK;
}

struct OutStage {
    int32_t* b1 = nullptr; int32_t* b2 = nullptr; float* d2 = nullptr;
    bool host1 = false, host2 = false, host3 = false;
};

som_status stage_outputs(som_ctx* h, int64_t n, int32_t* bmu1, int32_t* bmu2, float* d2, bool need_all, OutStage& o) {
    o.host1 = bmu1 && !is_device_ptr(bmu1);
    o.host2 = bmu2 && !is_device_ptr(bmu2);
    o.host3 = d2 && !is_device_ptr(d2);
    const size_t per = sizeof(int32_t) * 2 + sizeof(float);
    CK(h->outs.ensure(per * (size_t)std::max<int64_t>(n, 1), h->stream));
    char* base = (char*)h->outs.p;
    o.b1 = (bmu1 && !o.host1) ? bmu1 : (int32_t*)base;
    o.b2 = (bmu2 && !o.host2) ? bmu2 : ((bmu2 || need_all) ? (int32_t*)(base + sizeof(int32_t) * (size_t)n) : nullptr);
    o.d2 = (d2 && !o.host3) ? d2 : ((d2 || need_all) ? (float*)(base + sizeof(int32_t) * 2 * (size_t)n) : nullptr);
    return SOM_OK;
}

som_status copy_back(som_ctx* h, int64_t n, int32_t* bmu1, int32_t* bmu2, float* d2, const OutStage& o) {
    if (o.host1) CK(cudaMemcpyAsync(bmu1, o.b1, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost, h->stream));
    if (o.host2) CK(cudaMemcpyAsync(bmu2, o.b2, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost, h->stream));
    if (o.host3) CK(cudaMemcpyAsync(d2, o.d2, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost, h->stream));
    return SOM_OK;
}

// W^T (fp64 or fp32) and |w|^2 for the sparse path (map_sparse.cu), cached until W changes.
som_status ensure_wt(som_ctx* h, int J, bool f32, const void** WT, const double** wsq, int* Np, bool* fresh) {
    const int np = sparse_padded_units(h->N, J);
    const size_t plane = (f32 ? sizeof(float) : sizeof(double)) * (size_t)h->dim * np;
    *fresh = !h->wt_valid || h->wt_J != J || h->wt_f32 != f32;
    if (*fresh) {
        CK(h->wt64.ensure(plane + sizeof(double) * (size_t)h->N + 16, h->stream));
        char* base = (char*)h->wt64.p;
        int* flag = (int*)(base + plane + sizeof(double) * (size_t)h->N);
        CK(launch_wt(h->W, h->N, h->dim, np, f32, base, (double*)(base + plane), flag, h->stream));
        int bad = 1;
        CK(cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->wt_nonneg = bad == 0;
        h->wt_valid = true;
        h->wt_J = J;
        h->wt_f32 = f32;
    }
    *WT = h->wt64.p;
    *wsq = (const double*)((const char*)h->wt64.p + plane);
    *Np = np;
    return SOM_OK;
}

// Sparse kernel configuration: tile = 64 J units, W^T storage fp32 or fp64
// (SOM_SPARSE_J / SOM_SPARSE_F32 override, for tuning).
void sparse_cfg(const som_ctx* h, int* J, bool* f32) {
    *f32 = true;
    *J = h->N >= 2048 ? 8 : (h->N >= 512 ? 4 : 2);
    if (const char* e = std::getenv("SOM_SPARSE_F32")) *f32 = std::atoi(e) != 0;
    if (const char* e = std::getenv("SOM_SPARSE_J")) {
        const int j = std::atoi(e);
        if (j == 1 || j == 2 || j == 4 || j == 8) *J = j;
    }
    if (*f32 && *J == 1) *J = 2;
    if (!*f32 && *J == 8) *J = 4;
}

// Which path maps CSR rows: the exact sparse identity (R25) unless the
// caller forces another precision, or AUTO finds the dense contraction
// cheaper (rows with more than ~1.5 % of the terms set).
int csr_path(const som_ctx* h, const CsrIn& csr, int64_t n) {
    if (h->map_precision != SOM_MAP_AUTO) return h->map_precision;
    const double avg_nnz = (double)csr.nnz / (double)n;
    if (avg_nnz <= 0.015 * h->dim) return SOM_MAP_SPARSE_F64;
    return use_tc(h, n) ? SOM_MAP_3XTF32 : SOM_MAP_EXACT_F64;
}

// Map n staged CSR rows into device outputs.
som_status map_csr_dev(som_ctx* h, const CsrIn& csr, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches) {
    const int path = csr_path(h, csr, n);
    if (path == SOM_MAP_SPARSE_F64) {
        int J = 4;
        bool f32 = true, fresh = false;
        sparse_cfg(h, &J, &f32);
        const void* WT;
        const double* wsq;
        int np = 0;
        som_status st = ensure_wt(h, J, f32, &WT, &wsq, &np, &fresh);
        if (st) return st;
        // integer-pipe widening of half the values when W holds only +0 and
        // positive normals (TF-IDF maps); SOM_SPARSE_ICV=0 disables it
        bool icv = f32 && h->wt_nonneg && (J == 4 || J == 8);
        if (const char* e = std::getenv("SOM_SPARSE_ICV")) icv = icv && std::atoi(e) != 0;
        if (fresh) *launches += 2;
        const int tiles = np / sparse_tile_units(J);
        // chunk so the partial keys stay <= 1 GiB
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, ((int64_t)1 << 30) / (16 * (int64_t)tiles)));
        CK(h->keys.ensure(sizeof(unsigned long long) * 2 * (size_t)tiles * (size_t)chunk, h->stream));
        for (int64_t r0 = 0; r0 < n; r0 += chunk) {
            const int64_t m = std::min(chunk, n - r0);
            CK(launch_map_sparse(csr.rowptr, csr.col, csr.val, r0, m, WT, f32, icv, wsq, h->N, np, J,
                                 (unsigned long long*)h->keys.p, h->stream));
            CK(launch_map_merge((const unsigned long long*)h->keys.p, tiles, m, b1 + r0, b2 ? b2 + r0 : nullptr,
                                d2 ? d2 + r0 : nullptr, h->stream));
            *launches += 2;
        }
        return SOM_OK;
    }
    if (path == SOM_MAP_3XTF32) {
        auto fill = [&](int64_t r0, int64_t m, float* hi, float* lo, float* nrm) {
            return launch_split_csr(csr.rowptr, csr.col, csr.val, r0, m, h->dim, hi, lo, nrm, h->stream);
        };
        return map_tc_rows(h, n, fill, b1, b2, d2, launches);
    }
    // exact dense definition: densify in chunks of <= 1 GiB and map each chunk
    const int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(n, ((int64_t)1 << 30) / (4 * (int64_t)h->dim)));
    CK(h->dense.ensure(sizeof(float) * (size_t)chunk * h->dim, h->stream));
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t m = std::min(chunk, n - r0);
        CK(launch_densify(csr.rowptr, csr.col, csr.val, r0, m, h->dim, (float*)h->dense.p, h->stream));
        ++*launches;
        som_status st = map_exact_dev(h, (const float*)h->dense.p, m, b1 + r0, b2 ? b2 + r0 : nullptr,
                                      d2 ? d2 + r0 : nullptr, launches);
        if (st) return st;
    }
    return SOM_OK;
}

// QE/TE sums from device mapping outputs (deterministic two-pass), then
// the call's timing; ev0 was recorded before the mapping.
som_status finish_errors(som_ctx* h, int64_t n, const OutStage& o, int launches, double* qe, double* te) {
    const int nb = (int)std::min<int64_t>(std::max<int64_t>(1, (n + 4095) / 4096), 4 * (int64_t)h->sm_count);
    CK(h->red.ensure((sizeof(double) + sizeof(unsigned long long)) * ((size_t)nb + 2), h->stream));
    double* partial = (double*)h->red.p;
    unsigned long long* pcnt = (unsigned long long*)(partial + nb);
    double* osum = (double*)(pcnt + nb);
    unsigned long long* obad = (unsigned long long*)(osum + 1);
    CK(launch_errors(o.b1, o.b2, o.d2, n, h->rows, h->cols, h->topo, partial, pcnt, nb, osum, obad, h->stream));
    launches += 2;
    CK(cudaEventRecord(h->ev1, h->stream));
    double sum = 0;
    unsigned long long bad = 0;
    CK(cudaMemcpyAsync(&sum, osum, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(&bad, obad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (qe) *qe = sum / (double)n;
    if (te) *te = (double)bad / (double)n;
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = launches;
    return SOM_OK;
}

}  // namespace

som_status som_map(som_ctx* h, const float* X, int64_t n, int32_t* bmu1, int32_t* bmu2, float* d2) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (n < 0) return fail(SOM_EINVAL, "n < 0");
    if (n == 0) return SOM_OK;   // S:240 empty matrix -> empty result
    if (!X || !bmu1) return fail(SOM_EINVAL, "null X or bmu1");
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, bmu1, bmu2, d2, false, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_dense_dev(h, (const float*)Xd, n, o.b1, o.b2, o.d2, &launches))) return st;
    CK(cudaEventRecord(h->ev1, h->stream));
    if ((st = copy_back(h, n, bmu1, bmu2, d2, o))) return st;
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = launches;
    return SOM_OK;
}

som_status som_map_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                       int32_t* bmu1, int32_t* bmu2, float* d2) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (n < 0) return fail(SOM_EINVAL, "n < 0");
    if (n == 0) return SOM_OK;
    if (!bmu1) return fail(SOM_EINVAL, "null bmu1");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, bmu1, bmu2, d2, false, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_csr_dev(h, csr, n, o.b1, o.b2, o.d2, &launches))) return st;
    CK(cudaEventRecord(h->ev1, h->stream));
    if ((st = copy_back(h, n, bmu1, bmu2, d2, o))) return st;
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = launches;
    return SOM_OK;
}

namespace {

// Batch SOM (R27): epochs of map -> bucket -> per-BMU sums -> H S -> divide.
som_status train_batch_impl(som_ctx* h, const float* Xd, const CsrIn* csr, int64_t n, int32_t epochs, double sigma0,
                            const som_schedule* s, int32_t* bmu) {
    som_schedule sd;
    som_schedule_default(&sd);
    if (s) sd = *s;
    if (sd.kind < 0 || sd.kind > 2) return fail(SOM_EINVAL, "unknown decay kind");
    if (!(sd.k > 0.0) || !std::isfinite(sd.k)) return fail(SOM_EINVAL, "decay constant k must be > 0");
    if (!(sd.sigma_min > 0.0)) return fail(SOM_EINVAL, "sigma_min must be > 0");
    if (!(sd.cutoff >= 0.0 && sd.cutoff < 1.0)) return fail(SOM_EINVAL, "cutoff must be in [0, 1)");
    if (n > INT32_MAX) return fail(SOM_EUNSUPPORTED, "batch SOM: n >= 2^31 rows");
    if (h->N > 32768) return fail(SOM_EUNSUPPORTED, "batch SOM: more than 32768 units (N x N contraction)");
    const int N = h->N, d = h->dim;
    const size_t tb = batch_sort_temp_bytes(n, N);
    const size_t ints = 4 * (size_t)n + 2 * (size_t)N;
    CK(h->bbuf.ensure(sizeof(int32_t) * ints + tb + 256, h->stream));
    int32_t* b = (int32_t*)h->bbuf.p;
    int32_t* order = b + n;
    int32_t* scratch = order + n;
    int32_t* cnt = scratch + 2 * n;
    int32_t* off = cnt + N;
    void* temp = (void*)(((uintptr_t)(off + N) + 255) & ~(uintptr_t)255);
    const size_t plane = sizeof(double) * (size_t)N * (d + 1);
    CK(h->bS.ensure(plane, h->stream));
    // CSR: per-entry (unit, column) keys for the segmented per-unit sums
    size_t csr_tb = 0;
    void* csr_temp = nullptr;
    if (csr) {
        if ((uint64_t)N * (uint64_t)d > 0xFFFFFFFFull) return fail(SOM_EUNSUPPORTED, "batch SOM: N * dim >= 2^32");
        if (csr->nnz > INT32_MAX) return fail(SOM_EUNSUPPORTED, "batch SOM: nnz >= 2^31");
        csr_tb = batch_csr_temp_bytes(csr->nnz);
        CK(h->up.ensure(16 * (size_t)csr->nnz + csr_tb + 512, h->stream));
        csr_temp = (void*)(((uintptr_t)((char*)h->up.p + 16 * (size_t)csr->nnz) + 255) & ~(uintptr_t)255);
    }
    CK(h->bnum.ensure(plane, h->stream));
    // exact BMUs: the dense definition (R10), or the sparse identity (R25) for TF-IDF-like CSR rows
    const int saved = h->map_precision;
    if (saved == SOM_MAP_AUTO) h->map_precision = csr ? SOM_MAP_AUTO : SOM_MAP_EXACT_F64;
    if (csr && h->map_precision == SOM_MAP_AUTO && csr_path(h, *csr, n) == SOM_MAP_3XTF32)
        h->map_precision = SOM_MAP_EXACT_F64;
    auto map_all = [&](int* launches) -> som_status {
        return csr ? map_csr_dev(h, *csr, n, b, nullptr, nullptr, launches)
                   : map_dense_dev(h, Xd, n, b, nullptr, nullptr, launches);
    };
    int launches = 0;
    som_status st = SOM_OK;
    CK(cudaEventRecord(h->ev0, h->stream));
    for (int32_t e = 0; e < epochs && st == SOM_OK; ++e) {
        // schedule at tau = e / epochs (R1-R3, R5), host fp64 as for the online decay table
        double f = 0.0;
        fill_decay(&f, e, e + 1, epochs, sd.kind, sd.k);
        double sigma = sigma0 * f;
        if (sigma < sd.sigma_min) sigma = sd.sigma_min;
        const double r2 = sd.cutoff > 0.0 ? 2.0 * sigma * sigma * std::log(1.0 / sd.cutoff) : INFINITY;
        if ((st = map_all(&launches))) break;
        CK(launch_batch_bucket(b, n, N, order, cnt, off, scratch, temp, tb, h->stream));
        if (csr) CK(launch_batch_accumulate_csr(csr->rowptr, csr->col, csr->val, n, csr->nnz, d, b, cnt, N,
                                                (double*)h->bS.p, h->up.p, csr_temp, csr_tb, h->stream));
        else CK(launch_batch_accumulate_dense(Xd, d, order, off, cnt, N, (double*)h->bS.p, h->stream));
        CK(launch_batch_update((const double*)h->bS.p, (double*)h->bnum.p, N, d, h->rows, h->cols, h->topo, sigma,
                               r2, h->W, h->stream));
        invalidate_w_caches(h);
        launches += 7;
    }
    if (st == SOM_OK && bmu) {
        st = map_all(&launches);
        if (st == SOM_OK) {
            if (is_device_ptr(bmu)) CK(cudaMemcpyAsync(bmu, b, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, h->stream));
            else CK(cudaMemcpyAsync(bmu, b, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost, h->stream));
        }
    }
    h->map_precision = saved;
    if (st) return st;
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = (int64_t)epochs * n; h->last_launches = launches;
    return SOM_OK;
}

}  // namespace

som_status som_train_batch(som_ctx* h, const float* X, int64_t n, int32_t epochs, double sigma0,
                           const som_schedule* s, int32_t* bmu) {
    CHECK_HANDLE(h);
    if (h->world > 1) return fail(SOM_EUNSUPPORTED, "batch SOM on a neuron-sharded handle");
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: no data to train on");
    if (epochs < 0) return fail(SOM_EINVAL, "epochs must be >= 0");
    if (!(sigma0 > 0.0) || !std::isfinite(sigma0)) return fail(SOM_EINVAL, "sigma0 must be > 0");
    if (epochs == 0 && !bmu) return SOM_OK;
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    return train_batch_impl(h, (const float*)Xd, nullptr, n, epochs, sigma0, s, bmu);
}

som_status som_train_batch_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                               int32_t epochs, double sigma0, const som_schedule* s, int32_t* bmu) {
    CHECK_HANDLE(h);
    if (h->world > 1) return fail(SOM_EUNSUPPORTED, "batch SOM on a neuron-sharded handle");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: no data to train on");
    if (epochs < 0) return fail(SOM_EINVAL, "epochs must be >= 0");
    if (!(sigma0 > 0.0) || !std::isfinite(sigma0)) return fail(SOM_EINVAL, "sigma0 must be > 0");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    if (epochs == 0 && !bmu) return SOM_OK;
    return train_batch_impl(h, nullptr, &csr, n, epochs, sigma0, s, bmu);
}

som_status som_tfidf_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* counts, int64_t n,
                         float* out, int64_t* zero_rows) {
    CHECK_HANDLE(h);
    if (n < 1) return fail(SOM_EEMPTY, "n = 0");
    if (!out) return fail(SOM_EINVAL, "null out");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, counts, n, &csr);
    if (st) return st;
    const int d = h->dim;
    const int64_t nnz = csr.nnz;
    const bool dev = is_device_ptr(out);
    // scratch: idf (d fp64) | zero-row counter (u64) | df (d int) | staged output (nnz fp32, host out only)
    const size_t off_df = sizeof(double) * ((size_t)d + 1);
    const size_t off_o = (off_df + sizeof(int) * (size_t)d + 15) & ~(size_t)15;
    CK(h->up.ensure(off_o + (dev ? 0 : sizeof(float) * (size_t)nnz) + 16, h->stream));
    char* base = (char*)h->up.p;
    double* idf = (double*)base;
    unsigned long long* zr = (unsigned long long*)(idf + d);
    int* df = (int*)(base + off_df);
    float* o = dev ? out : (float*)(base + off_o);
    CK(cudaEventRecord(h->ev0, h->stream));
    CK(launch_tfidf(csr.rowptr, csr.col, csr.val, n, d, nnz, df, idf, o, zr, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    if (!dev && nnz > 0) CK(cudaMemcpyAsync(out, o, sizeof(float) * (size_t)nnz, cudaMemcpyDeviceToHost, h->stream));
    unsigned long long zh = 0;
    CK(cudaMemcpyAsync(&zh, zr, sizeof(zh), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (zero_rows) *zero_rows = (int64_t)zh;
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = 3;
    return SOM_OK;
}

namespace {

som_status copy_out_f64(som_ctx* h, double* dst, const double* src, size_t count) {
    if (!dst) return SOM_OK;
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * count, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice
                                                                             : cudaMemcpyDeviceToHost, h->stream));
    return SOM_OK;
}

// subspace iteration for the top-2 eigenpairs of the centred covariance (R29)
som_status pca_impl(som_ctx* h, PcaInput x, int64_t nnz, double* mean, double* v1, double* v2, double* pc) {
    const int d = h->dim, PB = kPcaBlock;
    const int64_t n = x.n;
    size_t need = sizeof(double) * ((size_t)d * (2 * PB + 3) + (size_t)n * PB + PB + 8);
    CK(h->up.ensure(need, h->stream));
    double* mu = (double*)h->up.p;
    double* Q = mu + d;
    double* Z = Q + (size_t)d * PB;
    double* V1 = Z + (size_t)d * PB;
    double* V2 = V1 + d;
    double* Y = V2 + d;
    double* out = Y + (size_t)n * PB;
    if (!x.X) {
        const size_t tb = pca_csc_temp_bytes(nnz, d);
        CK(h->up2.ensure(sizeof(int) * ((size_t)d + 1) + sizeof(int32_t) * 4 * (size_t)nnz + tb + 512, h->stream));
        int* cptr = (int*)h->up2.p;
        int32_t* cent = (int32_t*)(cptr + d + 1);
        int32_t* erow = cent + nnz;
        int32_t* scratch = erow + nnz;
        void* temp = (void*)(((uintptr_t)(scratch + 2 * nnz) + 255) & ~(uintptr_t)255);
        CK(launch_pca_csc(x.rowptr, x.col, n, d, nnz, cptr, cent, erow, scratch, temp, tb, h->stream));
        x.cptr = cptr; x.cent = cent; x.erow = erow;
    }
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    CK(launch_pca_mean(x, mu, h->stream));
    CK(launch_pca_init_q(Z, d, 0x5EEDull, h->stream));
    CK(launch_pca_orth(Z, Q, d, h->stream));
    launches += 3;
    double hostout[kPcaBlock + 2] = {0};
    const int maxit = 2000, every = 10;
    for (int it = 1; it <= maxit; ++it) {
        if (it % every == 0) {
            CK(launch_pca_rr(x, mu, Q, Y, Z, out, h->stream));
            launches += 4;
            CK(cudaMemcpyAsync(hostout, out, sizeof(hostout), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            const double th0 = hostout[0];
            if (!(th0 > 0.0)) break;                          // constant data: C = 0
            if (hostout[PB] <= 1e-12 * th0 && hostout[PB + 1] <= 1e-12 * th0) break;
        } else {
            CK(launch_pca_apply(x, mu, Q, Y, Z, 1, h->stream));
            launches += 3;
        }
    }
    CK(launch_pca_extract(Q, d, V1, V2, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    som_status st;
    if ((st = copy_out_f64(h, mean, mu, d)) || (st = copy_out_f64(h, v1, V1, d)) || (st = copy_out_f64(h, v2, V2, d)))
        return st;
    CK(cudaStreamSynchronize(h->stream));
    if (pc) {
        const double p[2] = {std::max(hostout[0], 0.0), std::max(hostout[1], 0.0)};
        if (is_device_ptr(pc)) CK(cudaMemcpy(pc, p, sizeof(p), cudaMemcpyHostToDevice));
        else { pc[0] = p[0]; pc[1] = p[1]; }
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = launches + 1;
    return SOM_OK;
}

}  // namespace

som_status som_pca_top2(som_ctx* h, const float* X, int64_t n, double* mean, double* v1, double* v2, double* pc) {
    CHECK_HANDLE(h);
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 2) return fail(n < 1 ? SOM_EEMPTY : SOM_EINVAL, "PCA needs n >= 2 rows");
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    PcaInput x{(const float*)Xd, nullptr, nullptr, nullptr, n, h->dim, nullptr, nullptr, nullptr};
    return pca_impl(h, x, 0, mean, v1, v2, pc);
}

som_status som_pca_top2_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                            double* mean, double* v1, double* v2, double* pc) {
    CHECK_HANDLE(h);
    if (n < 2) return fail(n < 1 ? SOM_EEMPTY : SOM_EINVAL, "PCA needs n >= 2 rows");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    if (csr.nnz > INT32_MAX) return fail(SOM_EUNSUPPORTED, "PCA: nnz >= 2^31");
    PcaInput x{nullptr, csr.rowptr, csr.col, csr.val, n, h->dim, nullptr, nullptr, nullptr};
    return pca_impl(h, x, csr.nnz, mean, v1, v2, pc);
}

som_status som_init_linear(som_ctx* h, const double* mean, const double* v1, const double* v2, double pc1,
                           double pc2) {
    CHECK_HANDLE(h);
    if (h->world > 1) return fail(SOM_EUNSUPPORTED, "linear init on a neuron-sharded handle");
    if (!mean || !v1 || !v2) return fail(SOM_EINVAL, "null mean / v1 / v2");
    if (!std::isfinite(pc1) || !std::isfinite(pc2)) return fail(SOM_EINVAL, "non-finite eigenvalue");
    const size_t vb = sizeof(double) * (size_t)h->dim;
    const void *m, *a, *b;
    som_status st;
    if ((st = stage_in(h, h->xin, mean, vb, &m)) || (st = stage_in(h, h->xin2, v1, vb, &a)) ||
        (st = stage_in(h, h->xin3, v2, vb, &b)))
        return st;
    invalidate_w_caches(h);
    CK(launch_init_linear(h->W, h->rows, h->cols, h->dim, (const double*)m, (const double*)a, (const double*)b, pc1,
                          pc2, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

som_status som_map_geometry(int64_t m, double pc1, double pc2, int32_t* rows, int32_t* cols, int64_t* num_itr) {
    if (m < 1) return fail(SOM_EINVAL, "m >= 1 records needed");
    if (!(pc1 >= 0.0) || !(pc2 >= 0.0)) return fail(SOM_EINVAL, "eigenvalues must be >= 0");
    const double munits = std::round(5.0 * std::sqrt((double)m));                              // step 2
    const double r = (pc1 == 0.0 || pc2 * munits < pc1) ? 1.0 : std::sqrt(pc1 / pc2);        // steps 5-8
    const int64_t size1 = std::max<int64_t>(1, (int64_t)std::llround(std::min(munits, std::sqrt(munits / (r * std::sqrt(0.75))))));
    const int64_t size2 = (int64_t)munits / size1;                                             // step 10
    const int64_t nr = std::min(size1, size2), nc = std::max(size1, size2);                    // steps 11-12
    const double mpd = (double)(nr * nc) / (double)m;                                          // steps 13-14
    if (rows) *rows = (int32_t)nr;
    if (cols) *cols = (int32_t)nc;
    if (num_itr) *num_itr = (int64_t)std::ceil(50.0 * mpd) * m * 4;                            // step 15
    return SOM_OK;
}

som_status som_errors_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                          double* qe, double* te) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: errors need data");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, nullptr, nullptr, nullptr, true, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_csr_dev(h, csr, n, o.b1, o.b2, o.d2, &launches))) return st;
    return finish_errors(h, n, o, launches, qe, te);
}

som_status som_errors(som_ctx* h, const float* X, int64_t n, double* qe, double* te) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: errors need data");
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, nullptr, nullptr, nullptr, true, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_dense_dev(h, (const float*)Xd, n, o.b1, o.b2, o.d2, &launches))) return st;
    return finish_errors(h, n, o, launches, qe, te);
}

som_status som_qerror(som_ctx* h, const float* X, int64_t n, double* qe) {
    if (!qe) return fail(SOM_EINVAL, "null qe");
    return som_errors(h, X, n, qe, nullptr);
}

som_status som_topographic_error(som_ctx* h, const float* X, int64_t n, double* te) {
    if (!te) return fail(SOM_EINVAL, "null te");
    return som_errors(h, X, n, nullptr, te);
}

som_status som_umatrix(som_ctx* h, float* U) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (!U) return fail(SOM_EINVAL, "null U");
    const bool dev = is_device_ptr(U);
    float* Ud = U;
    if (!dev) {
        CK(h->outs.ensure(sizeof(float) * (size_t)h->N, h->stream));
        Ud = (float*)h->outs.p;
    }
    CK(cudaEventRecord(h->ev0, h->stream));
    CK(launch_umatrix(h->W, h->rows, h->cols, h->topo, h->dim, Ud, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    if (!dev) CK(cudaMemcpyAsync(U, Ud, sizeof(float) * (size_t)h->N, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = h->N; h->last_launches = 1;
    return SOM_OK;
}

som_status som_last_stats(som_ctx* h, double* ms, int64_t* units, int32_t* kernel_launches) {
    if (!h) return fail(SOM_EINVAL, "null handle");
    if (ms) *ms = h->last_ms;
    if (units) *units = h->last_units;
    if (kernel_launches) *kernel_launches = h->last_launches;
    return SOM_OK;
}

}  // extern "C"
