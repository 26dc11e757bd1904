// som_api.cu — host runtime of libsom, part 1: errors, the handle, weights,
// initialisation, knobs, neuron-sharding plumbing and the shared helpers
// (staging of host buffers, the decay table, CSR validation).  Implements
// include/som.h together with som_train_api.cu, som_map_api.cu and
// som_extra_api.cu.  Product code: no oracle, no CPU fallback.
#include <thread>
#include <unordered_set>

#include "som_host.h"

using namespace som;
using namespace som::host;

namespace som {
namespace host {

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

// W changed: drop every derived copy (tensor-core split planes, sparse W^T)
void invalidate_w_caches(som_ctx* h) {
    h->w_split_valid = false;
    h->wt_valid = false;
}

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

// CSR arrays staged to the device and checked there (rowptr from 0 and
// non-decreasing, col strictly increasing within a row and < dim); returns
// the device pointers and the largest row length
som_status stage_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                     CsrIn* out) {
    if (!rowptr || !col || !val) return fail(SOM_EINVAL, "null CSR array");
    int64_t nnz = 0;
    if (is_device_ptr(rowptr)) {   // on the handle's stream: the caller may have produced rowptr on it
        CK(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    } else {
        nnz = rowptr[n];
    }
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

som_status scan_rows(som_ctx* h, const float* Xd, const CsrIn* csr, int64_t n, int64_t* m, const int64_t** list) {
    CK(h->rflags.ensure((size_t)std::max<int64_t>(n, 1), h->stream));
    uint8_t* flags = (uint8_t*)h->rflags.p;
    if (csr) CK(launch_row_flags_csr(csr->rowptr, csr->val, n, flags, h->stream));
    else CK(launch_row_flags_dense(Xd, n, h->dim, flags, h->stream));
    const size_t tb = select_rows_temp_bytes(n);
    const size_t idx_bytes = sizeof(int64_t) * ((size_t)n + 1);
    CK(h->rmap.ensure(idx_bytes + 256 + tb, h->stream));
    int64_t* idx = (int64_t*)h->rmap.p;
    int64_t* cnt = idx + n;
    void* temp = (char*)h->rmap.p + ((idx_bytes + 255) & ~(size_t)255);
    CK(launch_select_rows(flags, n, idx, cnt, temp, tb, h->stream));
    int64_t c = 0;
    CK(cudaMemcpyAsync(&c, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *m = c;
    if (list) *list = c < n ? idx : nullptr;
    return SOM_OK;
}

}  // namespace host
}  // namespace som

void som_comm_release(som_ctx* h);

namespace {
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
    s->sampling = SOM_SAMPLE_REPLACE;
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
    som_comm_release(h);
    for (DevBuf* b : {&h->xin, &h->xin2, &h->xin3, &h->keys, &h->outs, &h->red, &h->ftab, &h->log, &h->xchg, &h->dense,
                      &h->utab, &h->wsplit, &h->xsplit, &h->wt64, &h->bbuf, &h->bS, &h->bnum, &h->up, &h->up2,
                      &h->rflags, &h->rmap, &h->nstep, &h->tcsr, &h->tcsr2, &h->fitx, &h->fitx2, &h->fitx3})
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

}  // extern "C"

namespace {
// R18: the rows of the initial codebook — N draws from SplitMix64(seed),
// without replacement (Floyd) when N <= n; a neuron-sharded handle keeps the
// draws of its own units
std::vector<int64_t> init_indices(const som_ctx* h, int64_t n, uint64_t seed) {
    const int N = h->N;
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
    std::vector<int64_t> mine((size_t)h->NL);
    for (int l = 0; l < h->NL; ++l) mine[(size_t)l] = idx[(size_t)h->rank + (size_t)h->world * l];
    return mine;
}
}  // namespace

extern "C" {

som_status som_init_random(som_ctx* h, const float* X, int64_t n, uint64_t seed) {
    CHECK_HANDLE(h);
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0");
    invalidate_w_caches(h);
    const std::vector<int64_t> mine = init_indices(h, n, seed);
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

som_status som_init_random_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                               uint64_t seed) {
    CHECK_HANDLE(h);
    if (n < 1) return fail(SOM_EEMPTY, "n = 0");
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    invalidate_w_caches(h);
    const std::vector<int64_t> mine = init_indices(h, n, seed);
    CK(h->keys.ensure(sizeof(int64_t) * (size_t)h->NL, h->stream));
    CK(cudaMemcpyAsync(h->keys.p, mine.data(), sizeof(int64_t) * (size_t)h->NL, cudaMemcpyHostToDevice, h->stream));
    CK(launch_gather_csr_rows(csr.rowptr, csr.col, csr.val, (const int64_t*)h->keys.p, h->NL, h->dim, h->W,
                              h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return SOM_OK;
}

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

som_status som_last_spec_fallbacks(som_ctx* h, int64_t* count) {
    if (!h) return fail(SOM_EINVAL, "null handle");
    if (!count) return fail(SOM_EINVAL, "null count");
    *count = h->last_spec_fallbacks;
    return SOM_OK;
}

som_status som_last_map_fallbacks(som_ctx* h, int64_t* count) {
    if (!h) return fail(SOM_EINVAL, "null handle");
    if (!count) return fail(SOM_EINVAL, "null count");
    *count = h->last_tc_fallbacks;
    return SOM_OK;
}

som_status som_set_map_precision(som_ctx* h, int32_t precision) {
    CHECK_HANDLE(h);
    if (precision < SOM_MAP_AUTO || precision > SOM_MAP_SPARSE_F64) return fail(SOM_EINVAL, "unknown map precision");
    h->map_precision = precision;
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
