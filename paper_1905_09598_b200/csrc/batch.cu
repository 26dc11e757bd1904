// batch.cu — batch SOM epoch (reading R27: Kohonen's
// batch map; the variant of [25], [26]).
//
// One epoch with the current W:
//   1. BMUs of all documents (the exact mapping paths, R10 / R25);
//   2. documents bucketed by BMU with a stable radix sort of (c_i, i), so
//      every bucket lists its documents in index order;
//   3. S_c = sum_{i: c_i = c} x_i and n_c in fp64, one CTA per unit adding
//      its documents in index order (deterministic, no atomics);
//   4. num_u = sum_c h(u, c) [S_c | n_c] — an N x N x (d+1) contraction with
//      the lattice kernel generated on the fly from separable tables (R26);
//      tiles whose row span is outside the cutoff radius are skipped;
//   5. W_u = RN32(num_u / den_u) where den_u > 0, else unchanged.
// Regrouping sum_i h(c_i,u) x_i as sum_c h(c,u) S_c is exact in real
// arithmetic; in fp64 the two differ by a few ulp, far below the fp32
// rounding of W.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

__global__ void iota_kernel(int32_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

__global__ void count_kernel(const int32_t* bmu, int64_t n, int32_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + bmu[i], 1);   // integer counts: order-independent
}

// S_c (fp64, stride dp = d + 1, column d = n_c) from dense rows, one CTA per unit
__global__ void accumulate_dense_kernel(const float* __restrict__ X, int d, const int32_t* __restrict__ order,
                                        const int32_t* __restrict__ off, const int32_t* __restrict__ cnt, int dp,
                                        double* __restrict__ S) {
    const int c = blockIdx.x;
    double* row = S + (size_t)c * dp;
    const int o = off[c], m = cnt[c];
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double acc = 0.0;
        for (int q = 0; q < m; ++q) acc += (double)X[(int64_t)order[o + q] * d + k];
        row[k] = acc;
    }
    if (threadIdx.x == 0) row[d] = (double)m;
}

// the same from CSR rows: the row of S is zeroed, then each document's
// non-zeros (distinct columns) are added, documents in index order
__global__ void accumulate_csr_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                      const float* __restrict__ val, int d, const int32_t* __restrict__ order,
                                      const int32_t* __restrict__ off, const int32_t* __restrict__ cnt, int dp,
                                      double* __restrict__ S) {
    const int c = blockIdx.x;
    double* row = S + (size_t)c * dp;
    const int o = off[c], m = cnt[c];
    for (int k = threadIdx.x; k < d; k += blockDim.x) row[k] = 0.0;
    __syncthreads();
    for (int q = 0; q < m; ++q) {
        const int64_t i = order[o + q];
        for (int64_t p = rowptr[i] + threadIdx.x; p < rowptr[i + 1]; p += blockDim.x) row[col[p]] += (double)val[p];
        __syncthreads();
    }
    if (threadIdx.x == 0) row[d] = (double)m;
}

// num[u][k] = sum_c h(u, c) S[c][k]; 64 units x 64 columns per CTA, 16 units
// c per step, 4 x 4 outputs per thread; h from the separable tables (R26).
constexpr int GM = 64, GN = 64, GK = 16, GT = 256;

struct GemmArgs {
    const double* S;   // N x dp
    double* num;       // N x dp
    int N, dp, rows, cols, topo;
    double two_s2, r2;
};

__global__ void __launch_bounds__(GT) batch_gemm_kernel(const GemmArgs a) {
    __shared__ double hs[GK][GM + 1];
    __shared__ double ss[GK][GN];
    extern __shared__ double tabs[];   // Er[rows] | Ec[W2]
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    double* er = tabs;
    double* ec = tabs + a.rows;
    for (int e = threadIdx.x; e < a.rows + W2; e += GT) {
        if (e < a.rows) {
            const double di = (double)e;
            er[e] = exp(-(a.topo == 0 ? di * di : 0.75 * (di * di)) / a.two_s2);
        } else {
            const double dx = (double)(e - a.rows);
            ec[e - a.rows] = exp(-(a.topo == 0 ? dx * dx : 0.25 * (dx * dx)) / a.two_s2);
        }
    }
    __syncthreads();

    const int u0 = blockIdx.y * GM, k0 = blockIdx.x * GN;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    // lattice rows spanned by this unit tile (for the cutoff skip)
    const int ulast = min(a.N, u0 + GM) - 1;
    const int ur0 = u0 / a.cols, ur1 = ulast / a.cols;

    for (int c0 = 0; c0 < a.N; c0 += GK) {
        const int clast = min(a.N, c0 + GK) - 1;
        const int cr0 = c0 / a.cols, cr1 = clast / a.cols;
        const int gap = max(0, max(ur0, cr0) - min(ur1, cr1));   // smallest |di| between the tiles
        const double g2min = a.topo == 0 ? (double)gap * gap : 0.75 * ((double)gap * gap);
        if (g2min > a.r2) continue;   // block-uniform: no pair of the tiles is inside the cutoff
        __syncthreads();
        for (int e = threadIdx.x; e < GK * GM; e += GT) {
            const int cc = e / GM, uu = e - cc * GM;
            const int u = u0 + uu, c = c0 + cc;
            double h = 0.0;
            if (u < a.N && c < a.N) {
                const int iu = u / a.cols, ju = u - iu * a.cols, ic = c / a.cols, jc = c - ic * a.cols;
                const int di = abs(iu - ic);
                int dx;
                double g2;
                if (a.topo == 0) {
                    dx = abs(ju - jc);
                    g2 = (double)di * di + (double)dx * dx;
                } else {
                    dx = abs(2 * (ju - jc) + ((iu & 1) - (ic & 1)));
                    g2 = 0.25 * ((double)dx * dx) + 0.75 * ((double)di * di);
                }
                if (g2 <= a.r2) h = er[di] * ec[dx];
            }
            hs[cc][uu] = h;
        }
        for (int e = threadIdx.x; e < GK * GN; e += GT) {
            const int cc = e / GN, kk = e - cc * GN;
            const int c = c0 + cc, k = k0 + kk;
            ss[cc][kk] = (c < a.N && k < a.dp) ? a.S[(size_t)c * a.dp + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int cc = 0; cc < GK; ++cc) {
            double hv[4], sv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) hv[i] = hs[cc][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) sv[j] = ss[cc][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(hv[i], sv[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int u = u0 + ty + 16 * i;
        if (u >= a.N) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = k0 + tx + 16 * j;
            if (k < a.dp) a.num[(size_t)u * a.dp + k] = acc[i][j];
        }
    }
}

// W_u = RN32(num_u / den_u) where den_u > 0 (den = column d), else unchanged
__global__ void batch_finalize_kernel(const double* __restrict__ num, int N, int d, int dp, float* __restrict__ W) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)N * d;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e / d, k = e - u * d;
        const double den = num[u * dp + d];
        if (den > 0.0) W[e] = (float)(num[u * dp + k] / den);
    }
}

}  // namespace

size_t batch_sort_temp_bytes(int64_t n, int N) {
    size_t a = 0, b = 0;
    int bits = 1;
    while ((1ll << bits) < N) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, bits);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, N);
    return std::max(a, b) + 256;
}

// bucket documents by BMU: order (n) = document indices sorted by (bmu, index),
// cnt (N) = bucket sizes, off (N) = bucket starts.  work: 3 n + 2 N int32
// (keys_out | vals_in | spare) inside `scratch`.
cudaError_t launch_batch_bucket(const int32_t* bmu, int64_t n, int N, int32_t* order, int32_t* cnt, int32_t* off,
                                int32_t* scratch, void* temp, size_t temp_bytes, cudaStream_t st) {
    int32_t* keys_out = scratch;
    int32_t* vals_in = scratch + n;
    int bits = 1;
    while ((1ll << bits) < N) ++bits;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    iota_kernel<<<blocks, 256, 0, st>>>(vals_in, n);
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)N, st);
    if (e != cudaSuccess) return e;
    count_kernel<<<blocks, 256, 0, st>>>(bmu, n, cnt);
    size_t tb = temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, bmu, keys_out, vals_in, order, (int)n, 0, bits, st);
    if (e != cudaSuccess) return e;
    tb = temp_bytes;
    e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, off, N, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_batch_accumulate_dense(const float* X, int d, const int32_t* order, const int32_t* off,
                                          const int32_t* cnt, int N, double* S, cudaStream_t st) {
    accumulate_dense_kernel<<<N, 256, 0, st>>>(X, d, order, off, cnt, d + 1, S);
    return cudaGetLastError();
}

cudaError_t launch_batch_accumulate_csr(const int64_t* rowptr, const int32_t* col, const float* val, int d,
                                        const int32_t* order, const int32_t* off, const int32_t* cnt, int N,
                                        double* S, cudaStream_t st) {
    accumulate_csr_kernel<<<N, 256, 0, st>>>(rowptr, col, val, d, order, off, cnt, d + 1, S);
    return cudaGetLastError();
}

cudaError_t launch_batch_update(const double* S, double* num, int N, int d, int rows, int cols, int topo,
                                double sigma, double r2, float* W, cudaStream_t st) {
    GemmArgs a{S, num, N, d + 1, rows, cols, topo, 2.0 * sigma * sigma, r2};
    const size_t tab = sizeof(double) * ((size_t)rows + (topo == 0 ? cols : 2 * cols));
    cudaError_t e = cudaFuncSetAttribute(batch_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((d + 1 + GN - 1) / GN), (unsigned)((N + GM - 1) / GM));
    batch_gemm_kernel<<<grid, GT, tab, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int blocks = (int)std::min<int64_t>(((int64_t)N * d + 255) / 256, 148 * 16);
    batch_finalize_kernel<<<blocks, 256, 0, st>>>(num, N, d, d + 1, W);
    return cudaGetLastError();
}

}  // namespace som
