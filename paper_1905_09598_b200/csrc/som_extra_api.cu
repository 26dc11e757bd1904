// som_extra_api.cu — host runtime of libsom, part 4: batch SOM and the
// upstream steps (TF-IDF, PCA, linear initialisation, Fig. 2 sizing).

#include "som_host.h"

using namespace som;
using namespace som::host;

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

extern "C" {

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

}  // extern "C"
