// som_map_api.cu — host runtime of libsom, part 3: batch mapping (dense
// exact, tcgen05 3xTF32, sparse exact), quantization / topographic error,
// U-matrix.

#include "som_host.h"

using namespace som;
using namespace som::host;

namespace {

// W split for the tensor-core path: hi, lo (N x dp), fp64 |w|^2 and max |w|,
// cached until W changes.
som_status ensure_w_split(som_ctx* h, const float** whi, const float** wlo, const double** wn, const double** wmax) {
    const int dp = tc_padded_dim(h->dim);
    const size_t plane = sizeof(float) * (size_t)h->N * dp;
    if (!h->w_split_valid) {
        CK(h->wsplit.ensure(2 * plane + sizeof(double) * ((size_t)h->N + 1), h->stream));
        char* base = (char*)h->wsplit.p;
        CK(launch_split_rows(h->W, h->N, h->dim, (float*)base, (float*)(base + plane), (double*)(base + 2 * plane),
                             nullptr, h->stream));
        CK(launch_wmax((const double*)(base + 2 * plane), h->N, (double*)(base + 2 * plane) + h->N, h->stream));
        h->w_split_valid = true;
    }
    char* base = (char*)h->wsplit.p;
    *whi = (const float*)base;
    *wlo = (const float*)(base + plane);
    *wn = (const double*)(base + 2 * plane);
    *wmax = *wn + h->N;
    return SOM_OK;
}

// Tensor-core mapping of n documents whose split rows are produced chunk by
// chunk by `fill(r0, m, hi, lo, norm, groups)`, certified and rescored
// exactly against the documents themselves (csr rows, or dense device rows
// Xd); outputs device pointers.
using SplitFill = std::function<cudaError_t(int64_t, int64_t, float*, float*, double*, int*)>;
som_status map_tc_rows(som_ctx* h, int64_t n, const SplitFill& fill, const CsrIn* csr, const float* Xd, int32_t* b1,
                       int32_t* b2, float* d2, int* launches) {
    const float *whi, *wlo;
    const double *wn, *wmax;
    som_status st = ensure_w_split(h, &whi, &wlo, &wn, &wmax);
    if (st) return st;
    const int dp = tc_padded_dim(h->dim);
    // split-X chunk: up to 8 GiB of hi/lo planes (large chunks keep B panels hot)
    const int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(n, ((int64_t)8 << 30) / (8 * (int64_t)dp)));
    const size_t plane = sizeof(float) * (size_t)chunk * dp;
    CK(h->xsplit.ensure(2 * plane + (sizeof(double) + sizeof(int)) * (size_t)chunk + 64, h->stream));
    char* xb = (char*)h->xsplit.p;
    double* xn = (double*)(xb + 2 * plane);
    int* grp = (int*)(xn + chunk);
    const int tiles_n = tc_unit_tiles(h->N);
    CK(h->keys.ensure(sizeof(unsigned long long) * kTcCand * (size_t)tiles_n * (size_t)chunk, h->stream));
    CK(h->red.ensure(64, h->stream));
    int* nfall = (int*)h->red.p;
    CK(cudaMemsetAsync(nfall, 0, sizeof(int), h->stream));
    for (int64_t r0 = 0; r0 < n; r0 += chunk) {
        const int64_t m = std::min(chunk, n - r0);
        CK(fill(r0, m, (float*)xb, (float*)(xb + plane), xn, grp));
        CK(launch_map_tc((const float*)xb, (const float*)(xb + plane), xn, m, whi, wlo, wn, h->N, h->dim,
                         (unsigned long long*)h->keys.p, h->sm_count, h->stream));
        CK(launch_tc_rescore((const unsigned long long*)h->keys.p, m, csr ? csr->rowptr : nullptr,
                             csr ? csr->col : nullptr, csr ? csr->val : nullptr, r0,
                             Xd ? Xd + r0 * (int64_t)h->dim : nullptr, h->W, h->N, h->dim, xn, wn, grp, wmax, b1 + r0,
                             b2 ? b2 + r0 : nullptr, d2 ? d2 + r0 : nullptr, nfall, h->stream));
        *launches += 3;
    }
    int nf = 0;
    CK(cudaMemcpyAsync(&nf, nfall, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->last_tc_fallbacks = nf;
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

}  // namespace

namespace som {
namespace host {

// Which mapping path serves a call (som_set_map_precision; AUTO picks the
// tensor cores once the contraction is large enough to amortise the split).
bool use_tc(const som_ctx* h, int64_t n) {
    if (h->map_precision == SOM_MAP_EXACT_F64 || h->map_precision == SOM_MAP_SPARSE_F64) return false;
    if (!tc_rescore_fits(h->dim)) return false;   // the rescoring holds a document in shared memory
    if (h->map_precision == SOM_MAP_3XTF32) return true;
    return (double)n * h->N * h->dim >= 1.0e10;
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

// Map n rows of the device matrix Xd into device outputs (all device).
som_status map_dense_dev(som_ctx* h, const float* Xd, int64_t n, int32_t* b1, int32_t* b2, float* d2, int* launches) {
    if (h->map_precision == SOM_MAP_SPARSE_F64) {
        // dense rows through the sparse identity (R25): CSR form per chunk of
        // rows (<= 256 MB of dense input), then the sparse path
        const int d = h->dim;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, ((int64_t)256 << 20) / (4 * (int64_t)d)));
        const size_t tb = dense_csr_temp_bytes(chunk);
        const size_t ints = 2 * ((size_t)chunk + 1);                      // cnt | rowptr (int64)
        const size_t ent = (size_t)chunk * d;                              // worst case: every entry non-zero
        CK(h->dense.ensure(sizeof(int64_t) * ints + (sizeof(int32_t) + sizeof(float)) * ent + tb + 512, h->stream));
        char* base = (char*)h->dense.p;
        int64_t* cnt = (int64_t*)base;
        int64_t* rp = cnt + chunk + 1;
        int32_t* col = (int32_t*)(rp + chunk + 1);
        float* val = (float*)(col + ent);
        void* temp = (void*)(((uintptr_t)(val + ent) + 255) & ~(uintptr_t)255);
        for (int64_t r0 = 0; r0 < n; r0 += chunk) {
            const int64_t m = std::min(chunk, n - r0);
            const float* Xc = Xd + r0 * d;
            CK(launch_dense_rowptr(Xc, m, d, cnt, rp, temp, tb, h->stream));
            CK(launch_dense_fill(Xc, m, d, rp, col, val, h->stream));
            *launches += 3;
            int64_t nnz = 0;
            CK(cudaMemcpyAsync(&nnz, rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            CsrIn c{rp, col, val, 0, nnz};
            som_status st = map_csr_dev(h, c, m, b1 + r0, b2 ? b2 + r0 : nullptr, d2 ? d2 + r0 : nullptr, launches);
            if (st) return st;
        }
        return SOM_OK;
    }
    if (use_tc(h, n)) {
        auto fill = [&](int64_t r0, int64_t m, float* hi, float* lo, double* nrm, int* grp) {
            return launch_split_rows(Xd + r0 * h->dim, m, h->dim, hi, lo, nrm, grp, h->stream);
        };
        return map_tc_rows(h, n, fill, nullptr, Xd, b1, b2, d2, launches);
    }
    return map_exact_dev(h, Xd, n, b1, b2, d2, launches);
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
        auto fill = [&](int64_t r0, int64_t m, float* hi, float* lo, double* nrm, int* grp) {
            return launch_split_csr(csr.rowptr, csr.col, csr.val, r0, m, h->dim, hi, lo, nrm, grp, h->stream);
        };
        return map_tc_rows(h, n, fill, &csr, nullptr, b1, b2, d2, launches);
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

// QE/TE sums from device mapping outputs (deterministic two-pass), then
// the call's timing; ev0 was recorded before the mapping.
// Zero rows are not scored: the flags of scan_rows (called
// by the entry point, h->rflags) select the rows, m = their count.  With
// document sharding (som_comm_init_nccl, SOM_SHARD_DOCS) the fp64 sum and
// the integer counts are summed over the ranks before the division, so
// every rank returns the errors of the whole corpus.
bool doc_sharded(const som_ctx* h) { return h->nccl && h->shard_mode == SOM_SHARD_DOCS; }

som_status finish_errors(som_ctx* h, int64_t n, const OutStage& o, int launches, double* qe, double* te, int64_t m) {
    double sum = 0;
    unsigned long long bad = 0;
    if (n > 0) {
        const int nb = (int)std::min<int64_t>(std::max<int64_t>(1, (n + 4095) / 4096), 4 * (int64_t)h->sm_count);
        CK(h->red.ensure((sizeof(double) + sizeof(unsigned long long)) * ((size_t)nb + 2), h->stream));
        double* partial = (double*)h->red.p;
        unsigned long long* pcnt = (unsigned long long*)(partial + nb);
        double* osum = (double*)(pcnt + nb);
        unsigned long long* obad = (unsigned long long*)(osum + 1);
        const uint8_t* keep = m < n ? (const uint8_t*)h->rflags.p : nullptr;
        CK(launch_errors(o.b1, o.b2, o.d2, keep, n, h->rows, h->cols, h->topo, partial, pcnt, nb, osum, obad,
                         h->stream));
        launches += 2;
        CK(cudaMemcpyAsync(&sum, osum, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(&bad, obad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
    }
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    int64_t cnt[2] = {(int64_t)bad, m};
    if (doc_sharded(h)) {
        som_status st = doc_allreduce(h, &sum, cnt);
        if (st) return st;
    }
    if (cnt[1] == 0) return fail(SOM_EEMPTY, "every row is zero: no row to score (S:227)");
    if (qe) *qe = sum / (double)cnt[1];
    if (te) *te = (double)cnt[0] / (double)cnt[1];
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = n; h->last_launches = launches;
    return SOM_OK;
}

}  // namespace host
}  // namespace som

extern "C" {

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

som_status som_errors_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                          double* qe, double* te) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (n < 0) return fail(SOM_EINVAL, "n < 0");
    if (n < 1 && !doc_sharded(h)) return fail(SOM_EEMPTY, "n = 0: errors need data");
    if (n == 0) {   // document sharding: an empty shard still joins the reduction
        OutStage o;
        CK(cudaEventRecord(h->ev0, h->stream));
        return finish_errors(h, 0, o, 0, qe, te, 0);
    }
    CsrIn csr{};
    som_status st = stage_csr(h, rowptr, col, val, n, &csr);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, nullptr, nullptr, nullptr, true, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_csr_dev(h, csr, n, o.b1, o.b2, o.d2, &launches))) return st;
    int64_t m = 0;
    if ((st = scan_rows(h, nullptr, &csr, n, &m, nullptr))) return st;
    return finish_errors(h, n, o, launches + 2, qe, te, m);
}

som_status som_errors(som_ctx* h, const float* X, int64_t n, double* qe, double* te) {
    CHECK_HANDLE(h);
    if (h->world > 1)
        return fail(SOM_EUNSUPPORTED, "neuron-sharded handle: gather W into an unsharded handle to map / score");
    if (n < 0) return fail(SOM_EINVAL, "n < 0");
    if (n < 1 && !doc_sharded(h)) return fail(SOM_EEMPTY, "n = 0: errors need data");
    if (!X && n > 0) return fail(SOM_EINVAL, "null X");
    if (n == 0) {   // document sharding: an empty shard still joins the reduction
        OutStage o;
        CK(cudaEventRecord(h->ev0, h->stream));
        return finish_errors(h, 0, o, 0, qe, te, 0);
    }
    const void* Xd = nullptr;
    som_status st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd);
    if (st) return st;
    OutStage o;
    if ((st = stage_outputs(h, n, nullptr, nullptr, nullptr, true, o))) return st;
    int launches = 0;
    CK(cudaEventRecord(h->ev0, h->stream));
    if ((st = map_dense_dev(h, (const float*)Xd, n, o.b1, o.b2, o.d2, &launches))) return st;
    int64_t m = 0;
    if ((st = scan_rows(h, (const float*)Xd, nullptr, n, &m, nullptr))) return st;
    return finish_errors(h, n, o, launches + 2, qe, te, m);
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

}  // extern "C"
