// som_fit.cu — host runtime of libsom, part 6: one pass of the whole hot
// path in one call (the bench "step"): seeded
// initial codebook (R18), online training over the full schedule (P:104-112,
// P:158-166), mapping of every row, QE / TE from that mapping (R14,
// R15) and the U-matrix (R16) — with the input staged to the device ONCE
// per call (a host X would otherwise be copied by every entry point) and the
// errors taken from the mapping outputs instead of a second mapping pass.
// Pure orchestration of the entry points / device paths of the other host
// files; no arithmetic of its own.
#include "som_host.h"

using namespace som;
using namespace som::host;

namespace {

struct PhaseTimer {
    som_ctx* h;
    cudaEvent_t ev[6] = {};
    int k = 0;
    cudaError_t init() {
        for (auto& e : ev) {
            cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
        }
        return cudaSuccess;
    }
    cudaError_t mark() { return cudaEventRecord(ev[k++], h->stream); }
    ~PhaseTimer() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

// outputs of the mapping phase, errors from them, U-matrix, phase times
som_status fit_tail(som_ctx* h, int64_t n, const OutStage& o, int launches, int32_t* bmu1, int32_t* bmu2, float* d2,
                    double* qe, double* te, float* U, PhaseTimer& pt, const float* Xd, const CsrIn* csr) {
    som_status st;
    int64_t m = 0;
    CK(pt.mark());                                                     // map done
    if ((st = scan_rows(h, Xd, csr, n, &m, nullptr))) return st;
    double q = 0, t = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = finish_errors(h, n, o, launches, &q, &t, m))) return st;
    if (qe) *qe = q;
    if (te) *te = t;
    CK(pt.mark());                                                     // errors done
    // staged host outputs go back before the U-matrix call may grow h->outs
    // (stream-ordered: the copy is enqueued before any free)
    if ((st = copy_back(h, n, bmu1, bmu2, d2, o))) return st;
    if (U && (st = som_umatrix(h, U))) return st;
    CK(pt.mark());                                                     // U-matrix done
    CK(cudaStreamSynchronize(h->stream));
    for (int p = 0; p < 5; ++p) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, pt.ev[p], pt.ev[p + 1]));
        h->last_phase_ms[p] = ms;
    }
    float tot = 0;
    CK(cudaEventElapsedTime(&tot, pt.ev[0], pt.ev[5]));
    h->last_ms = tot;
    h->last_units = n;
    return SOM_OK;
}

}  // namespace

extern "C" {

som_status som_fit(som_ctx* h, const float* X, int64_t n, int32_t epochs, double alpha0, double sigma0,
                   const som_schedule* s, uint64_t seed, uint64_t init_seed, int32_t* bmu1, int32_t* bmu2, float* d2,
                   double* qe, double* te, float* U) {
    CHECK_HANDLE(h);
    if (h->world > 1) return fail(SOM_EUNSUPPORTED, "som_fit serves unsharded handles");
    if (!X) return fail(SOM_EINVAL, "null X");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: nothing to fit");
    PhaseTimer pt{h};
    CK(pt.init());
    CK(pt.mark());
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->fitx, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    const float* Xf = (const float*)Xd;
    if ((st = som_init_random(h, Xf, n, init_seed))) return st;
    CK(pt.mark());                                                     // staged + initialised
    if ((st = som_train_online(h, Xf, n, epochs, alpha0, sigma0, s, seed, 0, -1, nullptr))) return st;
    const double train_ms = h->last_ms;
    const int train_launches = h->last_launches;
    CK(pt.mark());                                                     // trained
    OutStage o;
    if ((st = stage_outputs(h, n, bmu1, bmu2, d2, true, o))) return st;
    int launches = 0;
    if ((st = map_dense_dev(h, Xf, n, o.b1, o.b2, o.d2, &launches))) return st;
    st = fit_tail(h, n, o, launches, bmu1, bmu2, d2, qe, te, U, pt, Xf, nullptr);
    h->last_train_ms = train_ms;
    h->last_launches = train_launches + launches + 5;
    return st;
}

som_status som_fit_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                       int32_t epochs, double alpha0, double sigma0, const som_schedule* s, uint64_t seed,
                       uint64_t init_seed, int32_t* bmu1, int32_t* bmu2, float* d2, double* qe, double* te,
                       float* U) {
    CHECK_HANDLE(h);
    if (h->world > 1) return fail(SOM_EUNSUPPORTED, "som_fit serves unsharded handles");
    if (!rowptr || !col || !val) return fail(SOM_EINVAL, "null CSR array");
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: nothing to fit");
    PhaseTimer pt{h};
    CK(pt.init());
    CK(pt.mark());
    int64_t nnz = 0;
    if (is_device_ptr(rowptr)) {
        CK(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    } else {
        nnz = rowptr[n];
    }
    if (nnz < 0) return fail(SOM_EINVAL, "rowptr[n] < 0");
    const void *rp, *cd, *vd;
    som_status st = stage_in(h, h->fitx, rowptr, sizeof(int64_t) * (size_t)(n + 1), &rp);
    if (st) return st;
    if ((st = stage_in(h, h->fitx2, col, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1), &cd))) return st;
    if ((st = stage_in(h, h->fitx3, val, sizeof(float) * (size_t)std::max<int64_t>(nnz, 1), &vd))) return st;
    const int64_t* R = (const int64_t*)rp;
    const int32_t* Cc = (const int32_t*)cd;
    const float* V = (const float*)vd;
    if ((st = som_init_random_csr(h, R, Cc, V, n, init_seed))) return st;
    CK(pt.mark());                                                     // staged + initialised
    if ((st = som_train_online_csr(h, R, Cc, V, n, epochs, alpha0, sigma0, s, seed, 0, -1, nullptr))) return st;
    const double train_ms = h->last_ms;
    const int train_launches = h->last_launches;
    CK(pt.mark());                                                     // trained
    CsrIn csr{};
    if ((st = stage_csr(h, R, Cc, V, n, &csr))) return st;            // device pointers: validation only
    OutStage o;
    if ((st = stage_outputs(h, n, bmu1, bmu2, d2, true, o))) return st;
    int launches = 0;
    if ((st = map_csr_dev(h, csr, n, o.b1, o.b2, o.d2, &launches))) return st;
    st = fit_tail(h, n, o, launches, bmu1, bmu2, d2, qe, te, U, pt, nullptr, &csr);
    h->last_train_ms = train_ms;
    h->last_launches = train_launches + launches + 6;
    return st;
}

som_status som_last_phases(som_ctx* h, double* ms5, double* train_kernel_ms) {
    if (!h || !ms5) return fail(SOM_EINVAL, "null argument");
    for (int p = 0; p < 5; ++p) ms5[p] = h->last_phase_ms[p];
    if (train_kernel_ms) *train_kernel_ms = h->last_train_ms;
    return SOM_OK;
}

}  // extern "C"
