// upstream.cu — the steps before training, on the GPU:
//   * Eq. 2 TF-IDF weighting + L2 row normalisation (R28);
//   * top-2 principal components of the DTM (Fig. 2 step 3; R29) by
//     subspace iteration on the implicitly centred covariance
//       C Q = (X^T (X Q) - n mu (mu^T Q)) / (n - 1),
//     block of P = 8 vectors, CGS2 orthonormalisation, Rayleigh-Ritz with a
//     Jacobi eigensolver on the P x P projection (one thread);
//   * the PCA-plane linear initialisation of the codebook (R30).
// Every reduction has a fixed order (X^T products go through a column-major
// copy of X built with a stable sort), so results are run-to-run identical.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int PB = kPcaBlock;   // subspace block

// ---------------------------------------------------------------- TF-IDF
__global__ void df_kernel(const int64_t* rowptr, const int32_t* col, const float* cnt, int64_t n, int* df) {
    const int64_t nnz = rowptr[n] - rowptr[0];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        if (cnt[rowptr[0] + p] > 0.0f) atomicAdd(df + col[rowptr[0] + p], 1);   // integer: order-free
}

__global__ void idf_kernel(const int* df, int d, int64_t n, double* idf) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < d; t += gridDim.x * blockDim.x)
        idf[t] = df[t] > 0 ? log((double)n / (double)df[t]) : 0.0;   // Eq. 2, natural log (R28)
}

// one warp per row: fp64 norm of (tf * idf), then RN32(tf idf / norm)
__global__ void tfidf_rows_kernel(const int64_t* rowptr, const int32_t* col, const float* cnt, int64_t n,
                                  const double* idf, float* out, unsigned long long* zero_rows) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t p0 = rowptr[i], p1 = rowptr[i + 1];
        double ss = 0.0;
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const double v = (double)cnt[p] * idf[col[p]];
            ss = fma(v, v, ss);
        }
        ss = warp_sum_f64(ss);
        const double nrm = sqrt(ss);
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const double v = (double)cnt[p] * idf[col[p]];
            out[p] = nrm > 0.0 ? (float)(v / nrm) : 0.0f;
        }
        if (lane == 0 && !(nrm > 0.0)) atomicAdd(zero_rows, 1ull);
    }
}

// ------------------------------------------------------------------- PCA
// column-major copy of a CSR matrix from the stable (col, entry) sort:
// ccol[e] = column of sorted entry e, cent[e] = its original entry index
__global__ void iota64_kernel(int32_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

__global__ void col_count_kernel(const int32_t* col, int64_t nnz, int* cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + col[p], 1);
}

// entry -> row map for the CSC walk
__global__ void entry_row_kernel(const int64_t* rowptr, int64_t n, int32_t* erow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) erow[p - rowptr[0]] = (int32_t)i;
}

// mean of the columns: CSC order (entries of a column in row order)
__global__ void mean_csc_kernel(const int* cptr, const int32_t* cent, const float* val, int64_t base, int d,
                                int64_t n, double* mu) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int e = cptr[k]; e < cptr[k + 1]; ++e) s += (double)val[base + cent[e]];
        mu[k] = s / (double)n;
    }
}

__global__ void mean_dense_kernel(const float* X, int64_t n, int d, double* mu) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += (double)X[i * d + k];
        mu[k] = s / (double)n;
    }
}

// Y = X Q (n x PB), CSR: one thread per row, entries in order
__global__ void xq_csr_kernel(const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                              const double* Q, double* Y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double acc[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[j] = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            const double v = (double)val[p];
            const double* q = Q + (size_t)col[p] * PB;
#pragma unroll
            for (int j = 0; j < PB; ++j) acc[j] = fma(v, q[j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < PB; ++j) Y[i * PB + j] = acc[j];
    }
}

// Y = X Q, dense rows: one warp per row, lanes over k, fixed butterfly order
__global__ void xq_dense_kernel(const float* X, int64_t n, int d, const double* Q, double* Y) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double acc[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[j] = 0.0;
        for (int k = lane; k < d; k += 32) {
            const double v = (double)X[i * d + k];
#pragma unroll
            for (int j = 0; j < PB; ++j) acc[j] = fma(v, Q[(size_t)k * PB + j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < PB; ++j) {
            const double s = warp_sum_f64(acc[j]);
            if (lane == 0) Y[i * PB + j] = s;
        }
    }
}

// Z = X^T Y, CSC: one thread per column, entries in row order
__global__ void xty_csc_kernel(const int* cptr, const int32_t* cent, const int32_t* erow, const float* val,
                               int64_t base, int d, const double* Y, double* Z) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double acc[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[j] = 0.0;
        for (int e = cptr[k]; e < cptr[k + 1]; ++e) {
            const int32_t p = cent[e];
            const double v = (double)val[base + p];
            const double* y = Y + (size_t)erow[p] * PB;
#pragma unroll
            for (int j = 0; j < PB; ++j) acc[j] = fma(v, y[j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < PB; ++j) Z[(size_t)k * PB + j] = acc[j];
    }
}

// Z = X^T Y, dense: one thread per column, rows in order
__global__ void xty_dense_kernel(const float* X, int64_t n, int d, const double* Y, double* Z) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double acc[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[j] = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double v = (double)X[i * d + k];
#pragma unroll
            for (int j = 0; j < PB; ++j) acc[j] = fma(v, Y[i * PB + j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < PB; ++j) Z[(size_t)k * PB + j] = acc[j];
    }
}

// block-wide fp64 sum (fixed order: per-thread strided partials, warp butterflies, warp 0)
constexpr int ONE = 1024;
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_f64(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (warp == 0) {
        s = lane < ONE / 32 ? red[lane] : 0.0;
        s = warp_sum_f64(s);
        if (lane == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// center: Z <- (Z - n mu (mu^T Q)) / (n - 1); orth: Q <- orthonormal basis
// of Z (CGS2, Z overwritten); one CTA of 1024 threads
__global__ void __launch_bounds__(ONE) center_orth_kernel(double* Z, double* Q, const double* mu, int d, int64_t n,
                                                          int center, int orth) {
    __shared__ double red[33];
    __shared__ double mq[PB];
    if (center) {
        for (int j = 0; j < PB; ++j) {
            double s = 0.0;
            for (int k = threadIdx.x; k < d; k += ONE) s = fma(mu[k], Q[(size_t)k * PB + j], s);
            s = block_sum(s, red);
            if (threadIdx.x == 0) mq[j] = s;
        }
        __syncthreads();
        const double inv = 1.0 / (double)(n - 1);
        for (int k = threadIdx.x; k < d; k += ONE)
            for (int j = 0; j < PB; ++j)
                Z[(size_t)k * PB + j] = (Z[(size_t)k * PB + j] - (double)n * mu[k] * mq[j]) * inv;
        __syncthreads();
    }
    if (!orth) return;
    for (int j = 0; j < PB; ++j) {
        for (int pass = 0; pass < 2; ++pass) {
            for (int l = 0; l < j; ++l) {
                double s = 0.0;
                for (int k = threadIdx.x; k < d; k += ONE) s = fma(Z[(size_t)k * PB + l], Z[(size_t)k * PB + j], s);
                s = block_sum(s, red);
                for (int k = threadIdx.x; k < d; k += ONE) Z[(size_t)k * PB + j] -= s * Z[(size_t)k * PB + l];
                __syncthreads();
            }
        }
        double s = 0.0;
        for (int k = threadIdx.x; k < d; k += ONE) s = fma(Z[(size_t)k * PB + j], Z[(size_t)k * PB + j], s);
        s = block_sum(s, red);
        const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
        for (int k = threadIdx.x; k < d; k += ONE) Z[(size_t)k * PB + j] *= inv;
        __syncthreads();
    }
    for (int k = threadIdx.x; k < d; k += ONE)
        for (int j = 0; j < PB; ++j) Q[(size_t)k * PB + j] = Z[(size_t)k * PB + j];
}

// Rayleigh-Ritz: Z = C Q (already centred), H = Q^T Z, eigen(H) by cyclic
// Jacobi (thread 0), Ritz values descending in out[0..PB), Q <- Q V, and the
// residual norms |C v_j - theta_j v_j| of the top two in out[PB], out[PB+1].
__global__ void __launch_bounds__(ONE) rayleigh_ritz_kernel(double* Q, double* Z, int d, double* out) {
    __shared__ double red[33];
    __shared__ double H[PB][PB], V[PB][PB], th[PB];
    __shared__ int ord[PB];
    for (int a = 0; a < PB; ++a)
        for (int b = a; b < PB; ++b) {
            double s = 0.0;
            for (int k = threadIdx.x; k < d; k += ONE) s = fma(Q[(size_t)k * PB + a], Z[(size_t)k * PB + b], s);
            s = block_sum(s, red);
            if (threadIdx.x == 0) { H[a][b] = s; H[b][a] = s; }
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        // symmetrise (Q^T C Q is symmetric up to rounding) and diagonalise
        for (int a = 0; a < PB; ++a)
            for (int b = a + 1; b < PB; ++b) { const double m = 0.5 * (H[a][b] + H[b][a]); H[a][b] = H[b][a] = m; }
        for (int a = 0; a < PB; ++a)
            for (int b = 0; b < PB; ++b) V[a][b] = a == b ? 1.0 : 0.0;
        for (int sweep = 0; sweep < 60; ++sweep) {
            double off = 0.0;
            for (int a = 0; a < PB; ++a)
                for (int b = a + 1; b < PB; ++b) off += H[a][b] * H[a][b];
            if (off < 1e-300) break;
            for (int p = 0; p < PB; ++p)
                for (int q = p + 1; q < PB; ++q) {
                    if (H[p][q] == 0.0) continue;
                    const double tau = (H[q][q] - H[p][p]) / (2.0 * H[p][q]);
                    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                    for (int k = 0; k < PB; ++k) {
                        const double hkp = H[k][p], hkq = H[k][q];
                        H[k][p] = c * hkp - s * hkq;
                        H[k][q] = s * hkp + c * hkq;
                    }
                    for (int k = 0; k < PB; ++k) {
                        const double hpk = H[p][k], hqk = H[q][k];
                        H[p][k] = c * hpk - s * hqk;
                        H[q][k] = s * hpk + c * hqk;
                    }
                    for (int k = 0; k < PB; ++k) {
                        const double vkp = V[k][p], vkq = V[k][q];
                        V[k][p] = c * vkp - s * vkq;
                        V[k][q] = s * vkp + c * vkq;
                    }
                }
        }
        for (int a = 0; a < PB; ++a) { th[a] = H[a][a]; ord[a] = a; }
        for (int a = 0; a < PB; ++a)            // descending, stable
            for (int b = a + 1; b < PB; ++b)
                if (th[ord[b]] > th[ord[a]]) { const int x = ord[a]; ord[a] = ord[b]; ord[b] = x; }
        for (int a = 0; a < PB; ++a) out[a] = th[ord[a]];
    }
    __syncthreads();
    // rotate Q and Z into the Ritz basis (sorted)
    double r0 = 0.0, r1 = 0.0;
    for (int k = threadIdx.x; k < d; k += ONE) {
        double q[PB], z[PB];
        for (int a = 0; a < PB; ++a) { q[a] = Q[(size_t)k * PB + a]; z[a] = Z[(size_t)k * PB + a]; }
        for (int j = 0; j < PB; ++j) {
            double sq = 0.0, sz = 0.0;
            for (int a = 0; a < PB; ++a) { sq = fma(q[a], V[a][ord[j]], sq); sz = fma(z[a], V[a][ord[j]], sz); }
            Q[(size_t)k * PB + j] = sq;
            Z[(size_t)k * PB + j] = sz;
            if (j == 0) { const double e = sz - th[ord[0]] * sq; r0 = fma(e, e, r0); }
            if (j == 1) { const double e = sz - th[ord[1]] * sq; r1 = fma(e, e, r1); }
        }
    }
    r0 = block_sum(r0, red);
    r1 = block_sum(r1, red);
    if (threadIdx.x == 0) { out[PB] = sqrt(r0); out[PB + 1] = sqrt(r1); }
}

// v_j = Q[:, j] (j < 2), signed so that its largest-magnitude component is
// positive, lowest index on ties (R29)
__global__ void __launch_bounds__(ONE) extract_kernel(const double* Q, int d, double* v1, double* v2) {
    __shared__ double bv[ONE];
    __shared__ int bi[ONE];
    for (int j = 0; j < 2; ++j) {
        double best = -1.0;
        int bk = d;
        for (int k = threadIdx.x; k < d; k += ONE) {
            const double a = fabs(Q[(size_t)k * PB + j]);
            if (a > best) { best = a; bk = k; }
        }
        bv[threadIdx.x] = best;
        bi[threadIdx.x] = bk;
        __syncthreads();
        for (int s = ONE / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const double o = bv[threadIdx.x + s];
                const int oi = bi[threadIdx.x + s];
                if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
                    bv[threadIdx.x] = o;
                    bi[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        const double sgn = Q[(size_t)bi[0] * PB + j] < 0.0 ? -1.0 : 1.0;
        double* v = j == 0 ? v1 : v2;
        for (int k = threadIdx.x; k < d; k += ONE) v[k] = sgn * Q[(size_t)k * PB + j];
        __syncthreads();
    }
}

__global__ void init_q_kernel(double* Q, int d, uint64_t seed) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d * PB;
         e += (int64_t)gridDim.x * blockDim.x)
        Q[e] = (double)(splitmix64_at(seed, e) >> 11) * 0x1.0p-53 - 0.5;
}

// R30: W(i, j) = mu + a_j sqrt(pc1) v1 + b_i sqrt(pc2) v2, fp64, RN32
__global__ void init_linear_kernel(float* W, int rows, int cols, int d, const double* mu, const double* v1,
                                   const double* v2, double s1, double s2) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)rows * cols * d;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e / d;
        const int k = (int)(e - u * d);
        const int i = (int)(u / cols), j = (int)(u - (int64_t)i * cols);
        const double a = cols == 1 ? 0.0 : -1.0 + 2.0 * (double)j / (double)(cols - 1);
        const double b = rows == 1 ? 0.0 : -1.0 + 2.0 * (double)i / (double)(rows - 1);
        W[e] = (float)(mu[k] + (a * s1) * v1[k] + (b * s2) * v2[k]);
    }
}

int blocks_for(int64_t n, int per) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 8)); }

}  // namespace

cudaError_t launch_tfidf(const int64_t* rowptr, const int32_t* col, const float* cnt, int64_t n, int d, int64_t nnz,
                         int* df, double* idf, float* out, unsigned long long* zero_rows, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(df, 0, sizeof(int) * (size_t)d, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(zero_rows, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    df_kernel<<<blocks_for(nnz, 256), 256, 0, st>>>(rowptr, col, cnt, n, df);
    idf_kernel<<<blocks_for(d, 256), 256, 0, st>>>(df, d, n, idf);
    tfidf_rows_kernel<<<blocks_for(32 * n, 256), 256, 0, st>>>(rowptr, col, cnt, n, idf, out, zero_rows);
    return cudaGetLastError();
}

size_t pca_csc_temp_bytes(int64_t nnz, int d) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)nnz, 0, 31);
    cub::DeviceScan::InclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, d);
    return std::max(a, b) + 256;
}

// column-major copy of the CSR pattern: cptr (d+1), cent (nnz: entry index
// relative to rowptr[0], entries of a column in row order), erow (nnz: row of each entry)
cudaError_t launch_pca_csc(const int64_t* rowptr, const int32_t* col, int64_t n, int d, int64_t nnz, int* cptr,
                           int32_t* cent, int32_t* erow, int32_t* scratch, void* temp, size_t temp_bytes,
                           cudaStream_t st) {
    int32_t* keys_out = scratch;
    int32_t* vals_in = scratch + nnz;
    int bits = 1;
    while ((1ll << bits) < d) ++bits;
    iota64_kernel<<<blocks_for(nnz, 256), 256, 0, st>>>(vals_in, nnz);
    cudaError_t e = cudaMemsetAsync(cptr, 0, sizeof(int) * ((size_t)d + 1), st);
    if (e != cudaSuccess) return e;
    col_count_kernel<<<blocks_for(nnz, 256), 256, 0, st>>>(col, nnz, cptr + 1);
    size_t tb = temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, col, keys_out, vals_in, cent, (int)nnz, 0, bits, st);
    if (e != cudaSuccess) return e;
    tb = temp_bytes;
    e = cub::DeviceScan::InclusiveSum(temp, tb, cptr + 1, cptr + 1, d, st);
    if (e != cudaSuccess) return e;
    entry_row_kernel<<<blocks_for(n, 256), 256, 0, st>>>(rowptr, n, erow);
    return cudaGetLastError();
}

cudaError_t launch_pca_mean(const PcaInput& x, double* mu, cudaStream_t st) {
    if (x.X) mean_dense_kernel<<<blocks_for(x.d, 128), 128, 0, st>>>(x.X, x.n, x.d, mu);
    else mean_csc_kernel<<<blocks_for(x.d, 128), 128, 0, st>>>(x.cptr, x.cent, x.val, 0, x.d, x.n, mu);
    return cudaGetLastError();
}

cudaError_t launch_pca_init_q(double* Q, int d, uint64_t seed, cudaStream_t st) {
    init_q_kernel<<<blocks_for((int64_t)d * PB, 256), 256, 0, st>>>(Q, d, seed);
    return cudaGetLastError();
}

// Z = C Q (centred and scaled, R29); then Q <- orthonormal basis of Z when orth
cudaError_t launch_pca_apply(const PcaInput& x, const double* mu, double* Q, double* Y, double* Z, int orth,
                             cudaStream_t st) {
    if (x.X) {
        xq_dense_kernel<<<blocks_for(32 * x.n, 256), 256, 0, st>>>(x.X, x.n, x.d, Q, Y);
        xty_dense_kernel<<<blocks_for(x.d, 128), 128, 0, st>>>(x.X, x.n, x.d, Y, Z);
    } else {
        xq_csr_kernel<<<blocks_for(x.n, 128), 128, 0, st>>>(x.rowptr, x.col, x.val, x.n, Q, Y);
        xty_csc_kernel<<<blocks_for(x.d, 128), 128, 0, st>>>(x.cptr, x.cent, x.erow, x.val, 0, x.d, Y, Z);
    }
    center_orth_kernel<<<1, ONE, 0, st>>>(Z, Q, mu, x.d, x.n, 1, orth);
    return cudaGetLastError();
}

// orthonormalise the columns of Z into Q (start vectors)
cudaError_t launch_pca_orth(double* Z, double* Q, int d, cudaStream_t st) {
    center_orth_kernel<<<1, ONE, 0, st>>>(Z, Q, nullptr, d, 2, 0, 1);
    return cudaGetLastError();
}

// Rayleigh-Ritz on Z = C Q: Ritz values (descending) in out[0..PB), residual
// norms of the top two in out[PB..PB+2); Q rotated to the Ritz vectors
cudaError_t launch_pca_rr(const PcaInput& x, const double* mu, double* Q, double* Y, double* Z, double* out,
                          cudaStream_t st) {
    cudaError_t e = launch_pca_apply(x, mu, Q, Y, Z, 0, st);
    if (e != cudaSuccess) return e;
    rayleigh_ritz_kernel<<<1, ONE, 0, st>>>(Q, Z, x.d, out);
    return cudaGetLastError();
}

cudaError_t launch_pca_extract(const double* Q, int d, double* v1, double* v2, cudaStream_t st) {
    extract_kernel<<<1, ONE, 0, st>>>(Q, d, v1, v2);
    return cudaGetLastError();
}

cudaError_t launch_init_linear(float* W, int rows, int cols, int d, const double* mu, const double* v1,
                               const double* v2, double pc1, double pc2, cudaStream_t st) {
    init_linear_kernel<<<blocks_for((int64_t)rows * cols * d, 256), 256, 0, st>>>(
        W, rows, cols, d, mu, v1, v2, sqrt(pc1 > 0.0 ? pc1 : 0.0), sqrt(pc2 > 0.0 ? pc2 : 0.0));
    return cudaGetLastError();
}

}  // namespace som
