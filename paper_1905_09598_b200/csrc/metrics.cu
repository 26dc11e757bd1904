// metrics.cu — quantization error, topographic error and U-matrix kernels,
// plus the row gather used by som_init_random.
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int kRedThreads = 256;

// Pass 1: each CTA sums sqrt((double)d2) (R14) and counts rows whose two
// best units are not adjacent (g2 != 1, R15) over a contiguous row range.
// Pass 2 (one CTA) adds the per-CTA partials in index order, so the result
// does not depend on scheduling.
// Zero rows (keep[i] == 0; keep nullable = every row) are not scored
// (S:227); the count of scored rows comes from the host.
__global__ void errors_partial_kernel(const int32_t* bmu1, const int32_t* bmu2, const float* d2,
                                      const uint8_t* keep, int64_t n, int cols, int topo, double* partial,
                                      unsigned long long* partial_cnt) {
    __shared__ double ssum[kRedThreads / 32];
    __shared__ unsigned long long scnt[kRedThreads / 32];
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(n, r0 + per);
    double s = 0.0;
    unsigned long long c = 0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kRedThreads) {
        if (keep && !keep[i]) continue;
        s += sqrt((double)d2[i]);
        const int b2 = bmu2[i];
        if (b2 >= 0 && lattice_g2(cols, topo, bmu1[i], b2) != 1.0) ++c;
    }
    s = warp_sum_f64(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { ssum[warp] = s; scnt[warp] = c; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long ct = 0;
        for (int w = 0; w < kRedThreads / 32; ++w) { t += ssum[w]; ct += scnt[w]; }
        partial[blockIdx.x] = t;
        partial_cnt[blockIdx.x] = ct;
    }
}

__global__ void errors_final_kernel(const double* partial, const unsigned long long* partial_cnt, int nb,
                                    double* out_sum, unsigned long long* out_bad) {
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long c = 0;
        for (int b = 0; b < nb; ++b) { t += partial[b]; c += partial_cnt[b]; }
        *out_sum = t;
        *out_bad = c;
    }
}

// U-matrix (R16): one CTA per unit u; for each lattice neighbour v (g2 = 1)
// in the 3 x 3 window of rows/cols around u, ascending v: |w_u - w_v| in
// fp64; U_u = mean (fp32), 0 without neighbours (R23).
__global__ void umatrix_kernel(const float* W, int rows, int cols, int topo, int dim, float* U) {
    __shared__ double sred[kRedThreads / 32];
    const int u = blockIdx.x;
    const int iu = u / cols, ju = u - iu * cols;
    const float* wu = W + (int64_t)u * dim;
    double sum = 0.0;
    int cnt = 0;
    for (int di = -1; di <= 1; ++di) {
        for (int dj = -1; dj <= 1; ++dj) {
            const int iv = iu + di, jv = ju + dj;
            if (iv < 0 || iv >= rows || jv < 0 || jv >= cols) continue;
            const int v = iv * cols + jv;
            if (lattice_g2(cols, topo, u, v) != 1.0) continue;
            const float* wv = W + (int64_t)v * dim;
            double a = 0.0;
            for (int k = threadIdx.x; k < dim; k += kRedThreads) {
                double d = (double)wu[k] - (double)wv[k];
                a = fma(d, d, a);
            }
            a = warp_sum_f64(a);
            if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = a;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w = 0; w < kRedThreads / 32; ++w) t += sred[w];
                sum += sqrt(t);
            }
            ++cnt;
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) U[u] = cnt ? (float)(sum / (double)cnt) : 0.0f;
}

__global__ void gather_rows_kernel(const float* X, const int64_t* idx, int dim, float* W) {
    const int u = blockIdx.x;
    const float* src = X + idx[u] * (int64_t)dim;
    float* dst = W + (int64_t)u * dim;
    for (int k = threadIdx.x; k < dim; k += blockDim.x) dst[k] = src[k];
}

// the CSR rows idx[u] densified into W row u
__global__ void gather_csr_rows_kernel(const int64_t* rowptr, const int32_t* col, const float* val,
                                       const int64_t* idx, int dim, float* W) {
    const int u = blockIdx.x;
    float* dst = W + (int64_t)u * dim;
    for (int k = threadIdx.x; k < dim; k += blockDim.x) dst[k] = 0.0f;
    __syncthreads();
    const int64_t i = idx[u];
    for (int64_t p = rowptr[i] + threadIdx.x; p < rowptr[i + 1]; p += blockDim.x) dst[col[p]] = val[p];
}

}  // namespace

cudaError_t launch_gather_csr_rows(const int64_t* rowptr, const int32_t* col, const float* val, const int64_t* idx,
                                   int N, int dim, float* W, cudaStream_t st) {
    gather_csr_rows_kernel<<<N, 256, 0, st>>>(rowptr, col, val, idx, dim, W);
    return cudaGetLastError();
}

cudaError_t launch_errors(const int32_t* bmu1, const int32_t* bmu2, const float* d2, const uint8_t* keep, int64_t n,
                          int rows, int cols, int topo, double* partial, unsigned long long* partial_cnt, int nblocks,
                          double* out_qe_sum, unsigned long long* out_bad, cudaStream_t st) {
    (void)rows;
    errors_partial_kernel<<<nblocks, kRedThreads, 0, st>>>(bmu1, bmu2, d2, keep, n, cols, topo, partial,
                                                           partial_cnt);
    errors_final_kernel<<<1, 32, 0, st>>>(partial, partial_cnt, nblocks, out_qe_sum, out_bad);
    return cudaGetLastError();
}

cudaError_t launch_umatrix(const float* W, int rows, int cols, int topo, int dim, float* U, cudaStream_t st) {
    umatrix_kernel<<<rows * cols, kRedThreads, 0, st>>>(W, rows, cols, topo, dim, U);
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(const float* X, const int64_t* idx, int N, int dim, float* W, cudaStream_t st) {
    gather_rows_kernel<<<N, 256, 0, st>>>(X, idx, dim, W);
    return cudaGetLastError();
}

}  // namespace som
