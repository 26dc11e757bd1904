// batch.cu — batch SOM epoch (reading R27: Kohonen's
// batch map; the variant of [25], [26]).
//
// One epoch with the current W:
//   1. BMUs of all documents (the exact mapping paths, R10 / R25);
//   2. documents bucketed by BMU with a stable radix sort of (c_i, i), so
//      every bucket lists its documents in index order;
//   3. S_c = sum_{i: c_i = c} x_i and n_c in fp64, in document order
//      (dense rows: one CTA per unit; CSR: entries grouped by (unit, column)
//      with a stable sort, one thread per group) — deterministic, no atomics;
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

// CSR rows: every non-zero gets the key (c_i * d + col); a stable radix
// sort of the keys over the entries (which are in document order) groups
// the entries of one (unit, column) pair, documents ascending, and one
// thread per group adds them in that order (balanced even when one unit
// collects thousands of documents; deterministic).
__global__ void entry_keys_kernel(const int64_t* rowptr, const int32_t* col, int64_t n, const int32_t* bmu, int d,
                                  uint32_t* key, int32_t* idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t base = (uint32_t)bmu[i] * (uint32_t)d;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            key[p] = base + (uint32_t)col[p];
            idx[p] = (int32_t)p;
        }
    }
}

// groups of <= 32 entries: one thread adds them in order; longer groups (a
// frequent term in a crowded unit) go to a list for the warp kernel below
constexpr int kShortGroup = 32;
__global__ void segment_sum_kernel(const uint32_t* key, const int32_t* idx, const float* val, int64_t nnz, int d,
                                   int dp, double* S, int32_t* longs, int* nlong) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[e];
        if (e > 0 && key[e - 1] == k) continue;          // not the first entry of its group
        int64_t f = e + 1;
        while (f < nnz && f - e <= kShortGroup && key[f] == k) ++f;
        if (f - e > kShortGroup) {                       // long group: handled by a warp
            longs[atomicAdd(nlong, 1)] = (int32_t)e;
            continue;
        }
        double s = 0.0;
        for (int64_t g = e; g < f; ++g) s += (double)val[idx[g]];
        S[(size_t)(k / (uint32_t)d) * dp + (k % (uint32_t)d)] = s;
    }
}

// one warp per long group: lane j adds entries j, j+32, ... in order, then a
// fixed xor butterfly (the list order varies run to run, each sum does not)
__global__ void long_segment_kernel(const uint32_t* key, const int32_t* idx, const float* val, int64_t nnz, int d,
                                    int dp, double* S, const int32_t* longs, const int* nlong) {
    const int lane = threadIdx.x & 31;
    const int nl = *nlong;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nl; w += (gridDim.x * blockDim.x) >> 5) {
        const int64_t e = longs[w];
        const uint32_t k = key[e];
        double s = 0.0;
        bool more = true;
        for (int64_t f = e + lane; __any_sync(0xffffffffu, more); f += 32) {
            more = f < nnz && key[f] == k;
            if (more) s += (double)val[idx[f]];
        }
        s = warp_sum_f64(s);
        if (lane == 0) S[(size_t)(k / (uint32_t)d) * dp + (k % (uint32_t)d)] = s;
    }
}

__global__ void counts_col_kernel(const int32_t* cnt, int N, int d, int dp, double* S) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
        S[(size_t)c * dp + d] = (double)cnt[c];
}

// num[u][k] = sum_c h(u, c) S[c][k]; 128 units x 64 columns per CTA, 16
// units c per step, 8 x 4 outputs per thread (12 shared-memory wavefronts per
// 1024 DFMAs, so the FP64 pipe, not shared memory, bounds the loop); h from
// the separable tables (R26).
constexpr int GM = 128, GN = 64, GK = 16, GT = 256, TI = GM / 16, TJ = GN / 16;

struct GemmArgs {
    const double* S;   // N x dp
    double* num;       // N x dp
    int N, dp, rows, cols, topo;
    double two_s2, r2;
};

// K steps whose lattice-row span lies inside the cutoff (block-uniform)
__device__ __forceinline__ bool gemm_step_live(const GemmArgs& a, int c0, int ur0, int ur1) {
    const int clast = min(a.N, c0 + GK) - 1;
    const int cr0 = c0 / a.cols, cr1 = clast / a.cols;
    const int gap = max(0, max(ur0, cr0) - min(ur1, cr1));   // smallest |di| between the tiles
    const double g2min = a.topo == 0 ? (double)gap * gap : 0.75 * ((double)gap * gap);
    return g2min <= a.r2;
}

__device__ __forceinline__ int gemm_next_live(const GemmArgs& a, int c0, int ur0, int ur1) {
    while (c0 < a.N && !gemm_step_live(a, c0, ur0, ur1)) c0 += GK;
    return c0;
}

// Double-buffered: while the FMAs of step k run on buffer k&1, the S tile of
// the next live step streams into the other buffer with cp.async and its h
// tile is generated there; one barrier per step.  Lattice coordinates of all
// units come from a packed (i << 16 | j) table in shared memory.
__global__ void __launch_bounds__(GT) batch_gemm_kernel(const GemmArgs a) {
    extern __shared__ __align__(16) double dyn[];
    double (*hs)[GK][GM + 1] = reinterpret_cast<double (*)[GK][GM + 1]>(dyn);                 // [2]
    double (*ss)[GK][GN] = reinterpret_cast<double (*)[GK][GN]>(dyn + 2 * GK * (GM + 1));     // [2]
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    double* er = dyn + 2 * GK * (GM + 1) + 2 * GK * GN;
    double* ec = er + a.rows;
    int* pij = reinterpret_cast<int*>(ec + W2);                                              // [N]
    for (int e = threadIdx.x; e < a.rows + W2; e += GT) {
        if (e < a.rows) {
            const double di = (double)e;
            er[e] = exp(-(a.topo == 0 ? di * di : 0.75 * (di * di)) / a.two_s2);
        } else {
            const double dx = (double)(e - a.rows);
            ec[e - a.rows] = exp(-(a.topo == 0 ? dx * dx : 0.25 * (dx * dx)) / a.two_s2);
        }
    }
    for (int u = threadIdx.x; u < a.N; u += GT) {
        const int i = u / a.cols;
        pij[u] = (i << 16) | (u - i * a.cols);
    }
    __syncthreads();

    const int u0 = blockIdx.y * GM, k0 = blockIdx.x * GN;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[TI][TJ];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) acc[i][j] = 0.0;
    const int ulast = min(a.N, u0 + GM) - 1;
    const int ur0 = u0 / a.cols, ur1 = ulast / a.cols;

    // stage step c0 into buffer q: S tile by cp.async (zero-filled edges), h tile computed
    auto stage = [&](int c0, int q) {
        for (int e = threadIdx.x; e < GK * GN / 2; e += GT) {      // 16-byte pieces
            const int cc = e / (GN / 2), kk = 2 * (e - cc * (GN / 2));
            const int c = c0 + cc, k = k0 + kk;
            double* dst = &ss[q][cc][kk];
            if (c < a.N && k + 1 < a.dp && (((size_t)c * a.dp + k) & 1) == 0) {
                cp_async16(dst, a.S + (size_t)c * a.dp + k);
            } else {
                dst[0] = (c < a.N && k < a.dp) ? a.S[(size_t)c * a.dp + k] : 0.0;
                dst[1] = (c < a.N && k + 1 < a.dp) ? a.S[(size_t)c * a.dp + k + 1] : 0.0;
            }
        }
        cp_async_commit();
        for (int e = threadIdx.x; e < GK * GM; e += GT) {
            const int cc = e / GM, uu = e - cc * GM;
            const int u = u0 + uu, c = c0 + cc;
            double h = 0.0;
            if (u < a.N && c < a.N) {
                const int pu = pij[u], pc = pij[c];
                const int iu = pu >> 16, ju = pu & 0xFFFF, ic = pc >> 16, jc = pc & 0xFFFF;
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
            hs[q][cc][uu] = h;
        }
    };

    int c0 = gemm_next_live(a, 0, ur0, ur1);
    int q = 0;
    if (c0 < a.N) stage(c0, 0);
    cp_async_wait_all();
    __syncthreads();
    while (c0 < a.N) {
        const int cn = gemm_next_live(a, c0 + GK, ur0, ur1);
        if (cn < a.N) stage(cn, q ^ 1);                         // next step into the other buffer
#pragma unroll
        for (int cc = 0; cc < GK; ++cc) {
            double hv[TI], sv[TJ];
#pragma unroll
            for (int i = 0; i < TI; ++i) hv[i] = hs[q][cc][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < TJ; ++j) sv[j] = ss[q][cc][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < TJ; ++j) acc[i][j] = fma(hv[i], sv[j], acc[i][j]);
        }
        cp_async_wait_all();
        __syncthreads();
        c0 = cn;
        q ^= 1;
    }
#pragma unroll
    for (int i = 0; i < TI; ++i) {
        const int u = u0 + ty + 16 * i;
        if (u >= a.N) continue;
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
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

size_t batch_csr_temp_bytes(int64_t nnz) {
    size_t a = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)nnz, 0, 32);
    return a + 256;
}

// S_c for CSR rows by (unit, column) groups; work: 2 nnz u32 keys + 2 nnz int32 (inside `work`)
cudaError_t launch_batch_accumulate_csr(const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                                        int64_t nnz, int d, const int32_t* bmu, const int32_t* cnt, int N, double* S,
                                        void* work, void* temp, size_t temp_bytes, cudaStream_t st) {
    uint32_t* key_in = (uint32_t*)work;
    uint32_t* key_out = key_in + nnz;
    int32_t* idx_in = (int32_t*)(key_out + nnz);
    int32_t* idx_out = idx_in + nnz;
    const int dp = d + 1;
    cudaError_t e = cudaMemsetAsync(S, 0, sizeof(double) * (size_t)N * dp, st);
    if (e != cudaSuccess) return e;
    if (nnz > 0) {
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
        entry_keys_kernel<<<blocks, 256, 0, st>>>(rowptr, col, n, bmu, d, key_in, idx_in);
        int bits = 1;
        while (bits < 32 && ((uint64_t)1 << bits) < (uint64_t)N * (uint64_t)d) ++bits;
        size_t tb = temp_bytes;
        e = cub::DeviceRadixSort::SortPairs(temp, tb, key_in, key_out, idx_in, idx_out, (int)nnz, 0, bits, st);
        if (e != cudaSuccess) return e;
        int32_t* longs = (int32_t*)key_in;                 // key_in is free after the sort
        int* nlong = (int*)(idx_in);                       // idx_in likewise (first word)
        e = cudaMemsetAsync(nlong, 0, sizeof(int), st);
        if (e != cudaSuccess) return e;
        segment_sum_kernel<<<(int)std::min<int64_t>((nnz + 255) / 256, 148 * 16), 256, 0, st>>>(
            key_out, idx_out, val, nnz, d, dp, S, longs, nlong);
        long_segment_kernel<<<148 * 4, 256, 0, st>>>(key_out, idx_out, val, nnz, d, dp, S, longs, nlong);
    }
    counts_col_kernel<<<(N + 255) / 256, 256, 0, st>>>(cnt, N, d, dp, S);
    return cudaGetLastError();
}

cudaError_t launch_batch_update(const double* S, double* num, int N, int d, int rows, int cols, int topo,
                                double sigma, double r2, float* W, cudaStream_t st) {
    GemmArgs a{S, num, N, d + 1, rows, cols, topo, 2.0 * sigma * sigma, r2};
    const size_t dyn = sizeof(double) * (2 * (size_t)GK * (GM + 1) + 2 * (size_t)GK * GN + (size_t)rows +
                                         (topo == 0 ? cols : 2 * cols)) + sizeof(int) * (size_t)N;
    cudaError_t e = cudaFuncSetAttribute(batch_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((d + 1 + GN - 1) / GN), (unsigned)((N + GM - 1) / GM));
    batch_gemm_kernel<<<grid, GT, dyn, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int blocks = (int)std::min<int64_t>(((int64_t)N * d + 255) / 256, 148 * 16);
    batch_finalize_kernel<<<blocks, 256, 0, st>>>(num, N, d, d + 1, W);
    return cudaGetLastError();
}

}  // namespace som
