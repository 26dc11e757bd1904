// map_exact.cu — exact batch BMU mapping, fp64-accumulated direct
// distances (R10) with a fused top-2 epilogue (R9, R15).  This is the
// SOM_MAP_EXACT_F64 path: every D_u is the same fp32 value the definition
// gives, so bmu1/bmu2/d2 match the oracle bit for bit.  The fast tensor-core
// path (3xTF32, R20) lives in map_tc.cu.
//
// Tiling: a CTA owns BM = 64 documents and one contiguous range of neuron
// tiles (BN = 128 units each); the K loop stages 16-wide slabs of X and W in
// shared memory already converted to fp64 (each element converted once per
// CTA, reused 128x / 64x).  Thread (tx, ty) of a 16 x 16 layout computes
// documents ty + 16 i (i < 4) x units tx + 16 j (j < 8): both smem reads are
// conflict-free (W row: 16 consecutive doubles; X: broadcast).  Per output
// element per k: one DADD + one DFMA.
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int BM = 64, BN = 128, BK = 16, TM = 4, TN = 8, NT = 256;

__device__ __forceinline__ void top2_insert(unsigned long long& k1, unsigned long long& k2,
                                            unsigned long long v) {
    if (v < k1) { k2 = k1; k1 = v; }
    else if (v < k2) { k2 = v; }
}

__device__ __forceinline__ void top2_merge(unsigned long long& k1, unsigned long long& k2,
                                           unsigned long long o1, unsigned long long o2) {
    top2_insert(k1, k2, o1);
    top2_insert(k1, k2, o2);
}

__global__ void __launch_bounds__(NT) map_exact_kernel(const MapArgs a) {
    __shared__ double xs[BK][BM];
    __shared__ double ws[BK][BN];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int ntiles = (a.N + BN - 1) / BN;
    const int per = (ntiles + a.nsplit - 1) / a.nsplit;
    const int nt0 = blockIdx.y * per;
    const int nt1 = min(ntiles, nt0 + per);

    unsigned long long k1[TM], k2[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) { k1[i] = ~0ull; k2[i] = ~0ull; }

    for (int nt = nt0; nt < nt1; ++nt) {
        const int n0 = nt * BN;
        double acc[TM][TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

        for (int k0 = 0; k0 < a.dim; k0 += BK) {
            // stage X slab [BM docs][BK] -> xs[k][m] and W slab [BN][BK] -> ws[k][n]
            for (int e = threadIdx.x; e < BM * BK; e += NT) {
                int m = e / BK, k = e % BK;
                int64_t gm = m0 + m;
                int gk = k0 + k;
                float v = (gm < a.n && gk < a.dim) ? a.X[gm * a.dim + gk] : 0.0f;
                xs[k][m] = (double)v;
            }
            for (int e = threadIdx.x; e < BN * BK; e += NT) {
                int n = e / BK, k = e % BK;
                int gn = n0 + n, gk = k0 + k;
                float v = (gn < a.N && gk < a.dim) ? a.W[(int64_t)gn * a.dim + gk] : 0.0f;
                ws[k][n] = (double)v;
            }
            __syncthreads();
#pragma unroll 4
            for (int k = 0; k < BK; ++k) {
                double xv[TM], wv[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) xv[i] = xs[k][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < TN; ++j) wv[j] = ws[k][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) {
                        double d = xv[i] - wv[j];
                        acc[i][j] = fma(d, d, acc[i][j]);
                    }
            }
            __syncthreads();
        }
        // epilogue: running top-2 per document
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int u = n0 + tx + 16 * j;
            if (u < a.N) {
#pragma unroll
                for (int i = 0; i < TM; ++i) top2_insert(k1[i], k2[i], make_key((float)acc[i][j], u));
            }
        }
    }
    // combine across the 16 threads (tx) sharing each document row
#pragma unroll
    for (int i = 0; i < TM; ++i) {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            unsigned long long o1 = __shfl_xor_sync(0xffffffffu, k1[i], o);
            unsigned long long o2 = __shfl_xor_sync(0xffffffffu, k2[i], o);
            top2_merge(k1[i], k2[i], o1, o2);
        }
        const int64_t gm = m0 + ty + 16 * i;
        if (tx == 0 && gm < a.n) {
            unsigned long long* dst = a.keys + ((size_t)blockIdx.y * a.n + gm) * 2;
            dst[0] = k1[i];
            dst[1] = k2[i];
        }
    }
}

__global__ void map_merge_kernel(const unsigned long long* keys, int nsplit, int64_t n, int32_t* bmu1,
                                 int32_t* bmu2, float* d2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long k1 = ~0ull, k2 = ~0ull;
        for (int s = 0; s < nsplit; ++s) {
            const unsigned long long* p = keys + ((size_t)s * n + i) * 2;
            top2_merge(k1, k2, p[0], p[1]);
        }
        bmu1[i] = key_unit(k1);
        if (bmu2) bmu2[i] = (k2 == ~0ull) ? -1 : key_unit(k2);
        if (d2) d2[i] = key_dist(k1);
    }
}

__global__ void densify_kernel(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0,
                               int64_t nrows, int dim, float* out) {
    // one CTA per row: zero the row, then scatter its nonzeros
    for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
        float* o = out + r * (int64_t)dim;
        for (int k = threadIdx.x; k < dim; k += blockDim.x) o[k] = 0.0f;
        __syncthreads();
        const int64_t p0 = rowptr[r0 + r], p1 = rowptr[r0 + r + 1];
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) o[col[p]] = val[p];
        __syncthreads();
    }
}

}  // namespace

int map_exact_tiles_n(int N) { return (N + BN - 1) / BN; }
int map_exact_tiles_m(int64_t n) { return (int)((n + BM - 1) / BM); }

cudaError_t launch_map_exact(const MapArgs& a, cudaStream_t st) {
    dim3 grid((unsigned)map_exact_tiles_m(a.n), (unsigned)a.nsplit);
    map_exact_kernel<<<grid, NT, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_map_merge(const unsigned long long* keys, int nsplit, int64_t n, int32_t* bmu1,
                             int32_t* bmu2, float* d2, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (blocks < 1) blocks = 1;
    map_merge_kernel<<<blocks, 256, 0, st>>>(keys, nsplit, n, bmu1, bmu2, d2);
    return cudaGetLastError();
}

cudaError_t launch_densify(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0,
                           int64_t nrows, int dim, float* out, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>(nrows, 148 * 16);
    if (blocks < 1) return cudaSuccess;
    densify_kernel<<<blocks, 256, 0, st>>>(rowptr, col, val, r0, nrows, dim, out);
    return cudaGetLastError();
}

}  // namespace som
