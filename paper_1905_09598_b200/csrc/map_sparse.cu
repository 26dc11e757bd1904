// map_sparse.cu — exact batch BMU mapping of sparse (CSR) documents
// (SURVEY §8.F NEXT-1 "SpMM mapping"), the SOM_MAP_SPARSE_F64 path.
//
// TF-IDF rows have ~50 non-zeros out of d = 3k..20k terms, so
// the dense contraction does ~d/nnz times more work than the definition
// needs.  Expanding Eq. (Euclidean distance) over the
// non-zeros of x (reading R25):
//     D_u = RN_fp32( max(0, (|x|^2 - 2 sum_{k in nz(x)} x_k w_uk) + |w_u|^2) )
// with every product and sum in fp64 (fp32 operands are exact in fp64 and
// x_k w_uk is exact too; only the additions round).  This equals the
// definition (R10) exactly in real arithmetic; in fp64 the two differ by a
// few ulp of O(1) values, i.e. the fp32 D is the same unless the exact sum
// lies within ~1e-16 relative of an fp32 rounding boundary.
//
// Data layout: the map is re-laid out once per W change as W^T in fp64,
// WT[k][u] (d x Np, Np = N rounded up to the unit tile), so that for one
// term k the weights of a tile of units are one contiguous, coalesced row
// segment, and the inner loop is one fp64 FMA per (non-zero, unit) with no
// conversion.  |w_u|^2 is kept in fp64 beside it.
//
// Kernel: grid (document blocks, unit tiles); document blocks vary fastest
// so the CTAs resident at any time share one unit tile (its WT slice,
// d x 64 J x 8 B, stays in L2 while every document streams past it).  A
// warp owns one document at a time; lane l owns units u0 + 2 l + 64 j + {0,1}
// (j < J), loaded as double2 through the read-only path (hot terms stay in
// L1 across the documents of the CTA).  Non-zeros are fetched 32 at a time
// (one per lane) and broadcast with shuffles, 4 per iteration so each lane
// has 4 J independent 16-byte loads in flight.  Epilogue: D, key (R9), lane
// top-2, warp butterfly top-2; lane 0 writes the tile's two keys, and the
// exact path's merge kernel combines tiles.
#include <algorithm>
#include <cub/device/device_scan.cuh>
#include <cstdlib>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int SP_THREADS = 512;
constexpr int SP_WARPS = SP_THREADS / 32;

__device__ __forceinline__ void top2_ins(unsigned long long& k1, unsigned long long& k2, unsigned long long v) {
    if (v < k1) { k2 = k1; k1 = v; }
    else if (v < k2) { k2 = v; }
}

// W (N x d fp32, row-major) -> WT (d x Np, fp64 or fp32); columns u >= N
// are zero, -0 becomes +0 (same products), and *flag is set if any value is
// negative, subnormal, infinite or NaN (then the integer widening below may
// not be used).
template <typename T>
__global__ void wt_kernel(const float* __restrict__ W, int N, int d, int Np, T* __restrict__ WT, int* flag) {
    __shared__ float tile[32][33];
    const int u0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    bool bad = false;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int u = u0 + r, k = k0 + threadIdx.x;
        float v = (u < N && k < d) ? W[(int64_t)u * d + k] : 0.0f;
        if (v == 0.0f) v = 0.0f;
        const unsigned bits = __float_as_uint(v);
        const unsigned ex = bits & 0x7F800000u;
        bad |= (bits >> 31) != 0u || ex == 0x7F800000u || (ex == 0u && bits != 0u);
        tile[r][threadIdx.x] = v;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int k = k0 + r, u = u0 + threadIdx.x;
        if (k < d && u < Np) WT[(int64_t)k * Np + u] = (T)tile[threadIdx.x][r];
    }
}

// |w_u|^2 in fp64, one warp per unit (any summation order: R25).
__global__ void row_sqnorm_kernel(const float* __restrict__ W, int N, int d, double* __restrict__ wsq) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= N) return;
    const float* w = W + (int64_t)warp * d;
    double s = 0.0;
    for (int k = lane; k < d; k += 32) {
        const double v = (double)w[k];
        s = fma(v, v, s);
    }
    s = warp_sum_f64(s);
    if (lane == 0) wsq[warp] = s;
}

struct SparseArgs {
    const int64_t* rowptr;  // rows r0 .. r0 + m of the caller's CSR
    const int32_t* col;
    const float* val;
    int64_t r0, m;
    const void* WT;         // d x Np, fp64 or fp32
    const double* wsq;      // N
    int N, Np;
    int docs_per_cta;
    unsigned long long* keys;  // [tiles][m][2]
};

// Loads VEC consecutive W^T entries of one term as fp64 (fp32 storage is
// widened exactly in registers).
template <bool F32> struct WtVec;
template <> struct WtVec<false> {
    static constexpr int VEC = 2;
    __device__ __forceinline__ static void load(const void* base, int64_t off, double (&w)[2]) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(static_cast<const double*>(base) + off));
        w[0] = v.x; w[1] = v.y;
    }
};
template <> struct WtVec<true> {
    static constexpr int VEC = 4;
    __device__ __forceinline__ static void load(const void* base, int64_t off, double (&w)[4]) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(base) + off));
        w[0] = (double)v.x; w[1] = (double)v.y; w[2] = (double)v.z; w[3] = (double)v.w;
    }
};

// Exact fp32 -> fp64 widening on the integer pipe, valid for +0 and positive
// normal floats only (the host checks W^T holds nothing else): sign 0,
// exponent e8 + 896, mantissa m23 << 29.  Used for half of the values so
// that the F2F.F64.F32 pipe (~16/clk/SM) is not the only converter.
__device__ __forceinline__ double widen_nonneg(float f) {
    const unsigned b = __float_as_uint(f);
    const unsigned hi = b ? (b >> 3) + 0x38000000u : 0u;
    return __hiloint2double((int)hi, (int)(b << 29));
}

// Tile = 64 J units; lane l owns units u0 + VEC l + 32 VEC g + c (g < G, c < VEC).
// ICV (fp32 storage only): groups g >= G/2 are widened on the integer pipe.
template <int J, bool F32, bool ICV = false>
__global__ void __launch_bounds__(SP_THREADS, 1) map_sparse_kernel(const SparseArgs a) {
    using L = WtVec<F32>;
    constexpr int VEC = L::VEC;
    constexpr int G = 64 * J / (32 * VEC);
    // non-zeros in flight per iteration: fp32 storage keeps the raw float4 loads
    // (4 registers each) and widens at use, so it affords twice as many
    constexpr int UN = F32 ? 4 : ((G * VEC > 8) ? 2 : 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.y;
    const int u0 = tile * (64 * J);
    const int64_t lbase = u0 + VEC * lane;
    const int64_t dbeg = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t dend = min(a.m, dbeg + a.docs_per_cta);
    __shared__ int next_doc;   // dynamic hand-out: row lengths vary, warps finish unevenly
    if (threadIdx.x == 0) next_doc = SP_WARPS;
    __syncthreads();

    for (int64_t doc = dbeg + warp; doc < dend;) {
        const int64_t p0 = a.rowptr[a.r0 + doc], p1 = a.rowptr[a.r0 + doc + 1];
        double acc[G][VEC];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int c = 0; c < VEC; ++c) acc[g][c] = 0.0;
        double xsq = 0.0;
        for (int64_t pb = p0; pb < p1; pb += 32) {
            const int cnt = (int)((p1 - pb) < 32 ? (p1 - pb) : 32);
            int kk = 0;
            double vv = 0.0;
            if (lane < cnt) {
                kk = __ldg(a.col + pb + lane);
                vv = (double)__ldg(a.val + pb + lane);
            }
            xsq = fma(vv, vv, xsq);
            for (int q = 0; q < cnt; q += UN) {
                int k[UN];
                double v[UN];
#pragma unroll
                for (int e = 0; e < UN; ++e) {
                    k[e] = __shfl_sync(0xffffffffu, kk, q + e);   // lanes >= cnt carry k = 0, v = 0
                    v[e] = __shfl_sync(0xffffffffu, vv, q + e);
                }
                if constexpr (F32) {
                    float4 raw[UN][G];
#pragma unroll
                    for (int e = 0; e < UN; ++e)
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            raw[e][g] = __ldg(reinterpret_cast<const float4*>(
                                static_cast<const float*>(a.WT) + (int64_t)k[e] * a.Np + lbase + 32 * VEC * g));
#pragma unroll
                    for (int e = 0; e < UN; ++e)
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float4 r = raw[e][g];
                            double wv[4];
                            if (ICV && g >= G / 2) {
                                wv[0] = widen_nonneg(r.x); wv[1] = widen_nonneg(r.y);
                                wv[2] = widen_nonneg(r.z); wv[3] = widen_nonneg(r.w);
                            } else {
                                wv[0] = (double)r.x; wv[1] = (double)r.y; wv[2] = (double)r.z; wv[3] = (double)r.w;
                            }
#pragma unroll
                            for (int c = 0; c < VEC; ++c) acc[g][c] = fma(v[e], wv[c], acc[g][c]);
                        }
                } else {
                    double w[UN][G][VEC];
#pragma unroll
                    for (int e = 0; e < UN; ++e)
#pragma unroll
                        for (int g = 0; g < G; ++g) L::load(a.WT, (int64_t)k[e] * a.Np + lbase + 32 * VEC * g, w[e][g]);
#pragma unroll
                    for (int e = 0; e < UN; ++e)
#pragma unroll
                        for (int g = 0; g < G; ++g)
#pragma unroll
                            for (int c = 0; c < VEC; ++c) acc[g][c] = fma(v[e], w[e][g][c], acc[g][c]);
                }
            }
        }
        xsq = warp_sum_f64(xsq);   // xor butterfly: every lane holds the same sum
        unsigned long long k1 = ~0ull, k2 = ~0ull;
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int c = 0; c < VEC; ++c) {
                const int u = (int)lbase + 32 * VEC * g + c;
                if (u < a.N) {
                    double D = fma(-2.0, acc[g][c], xsq) + __ldg(a.wsq + u);
                    D = D > 0.0 ? D : 0.0;
                    top2_ins(k1, k2, make_key((float)D, u));
                }
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, k1, o);
            const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, k2, o);
            top2_ins(k1, k2, o1);
            top2_ins(k1, k2, o2);
        }
        int nd = 0;
        if (lane == 0) {
            unsigned long long* dst = a.keys + ((size_t)tile * a.m + doc) * 2;
            dst[0] = k1;
            dst[1] = k2;
            nd = atomicAdd(&next_doc, 1);
        }
        doc = dbeg + __shfl_sync(0xffffffffu, nd, 0);
    }
}

}  // namespace

// ---------------------------------------------------- dense rows -> CSR
// (SOM_MAP_SPARSE_F64 on dense input): one warp per row counts and then
// writes its non-zeros in column order (ballot + popc), so the sparse path
// sees exactly the CSR form of the rows.
namespace {
__global__ void dense_count_kernel(const float* X, int64_t m, int d, int64_t* cnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int c = 0;
        for (int k = lane; k < d; k += 32) c += X[i * d + k] != 0.0f;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) cnt[i] = c;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[m] = 0;
}

__global__ void dense_fill_kernel(const float* X, int64_t m, int d, const int64_t* rowptr, int32_t* col, float* val) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int64_t o = rowptr[i];
        for (int k0 = 0; k0 < d; k0 += 32) {
            const int k = k0 + lane;
            const float v = k < d ? X[i * d + k] : 0.0f;
            const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0f);
            if (v != 0.0f) {
                const int64_t p = o + __popc(mask & ((1u << lane) - 1u));
                col[p] = k;
                val[p] = v;
            }
            o += __popc(mask);
        }
    }
}
}  // namespace

size_t dense_csr_temp_bytes(int64_t m) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(m + 1));
    return b + 256;
}

// rowptr (m+1) of the CSR form of m dense rows; col/val filled by launch_dense_fill
cudaError_t launch_dense_rowptr(const float* X, int64_t m, int d, int64_t* cnt, int64_t* rowptr, void* temp,
                                size_t temp_bytes, cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>((32 * m + 255) / 256, 148 * 16);
    dense_count_kernel<<<std::max(blocks, 1), 256, 0, st>>>(X, m, d, cnt);
    size_t tb = temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, rowptr, (int)(m + 1), st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_dense_fill(const float* X, int64_t m, int d, const int64_t* rowptr, int32_t* col, float* val,
                              cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>((32 * m + 255) / 256, 148 * 16);
    dense_fill_kernel<<<std::max(blocks, 1), 256, 0, st>>>(X, m, d, rowptr, col, val);
    return cudaGetLastError();
}

int sparse_tile_units(int J) { return 64 * J; }
int sparse_padded_units(int N, int J) { return (N + 64 * J - 1) / (64 * J) * (64 * J); }

cudaError_t launch_wt(const float* W, int N, int d, int Np, bool f32, void* WT, double* wsq, int* flag,
                      cudaStream_t st) {
    dim3 g1((unsigned)((Np + 31) / 32), (unsigned)((d + 31) / 32));
    cudaError_t e0 = cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (e0 != cudaSuccess) return e0;
    if (f32) wt_kernel<float><<<g1, dim3(32, 8), 0, st>>>(W, N, d, Np, (float*)WT, flag);
    else wt_kernel<double><<<g1, dim3(32, 8), 0, st>>>(W, N, d, Np, (double*)WT, flag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    row_sqnorm_kernel<<<(N + 7) / 8, 256, 0, st>>>(W, N, d, wsq);
    return cudaGetLastError();
}

cudaError_t launch_map_sparse(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0, int64_t m,
                              const void* WT, bool f32, bool icv, const double* wsq, int N, int Np, int J,
                              unsigned long long* keys, cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    const int tiles = Np / (64 * J);
    int docs_per_cta = 256;
    if (const char* e = std::getenv("SOM_SPARSE_DPC")) docs_per_cta = std::max(16, std::atoi(e));
    SparseArgs a{rowptr, col, val, r0, m, WT, wsq, N, Np, docs_per_cta, keys};
    dim3 grid((unsigned)((m + docs_per_cta - 1) / docs_per_cta), (unsigned)tiles);
    if (f32 && icv) {
        switch (J) {
            case 4: map_sparse_kernel<4, true, true><<<grid, SP_THREADS, 0, st>>>(a); return cudaGetLastError();
            case 8: map_sparse_kernel<8, true, true><<<grid, SP_THREADS, 0, st>>>(a); return cudaGetLastError();
            default: break;
        }
    }
    const int cfg = J * 2 + (f32 ? 1 : 0);
    switch (cfg) {
        case 2: map_sparse_kernel<1, false><<<grid, SP_THREADS, 0, st>>>(a); break;
        case 4: map_sparse_kernel<2, false><<<grid, SP_THREADS, 0, st>>>(a); break;
        case 8: map_sparse_kernel<4, false><<<grid, SP_THREADS, 0, st>>>(a); break;
        case 5: map_sparse_kernel<2, true><<<grid, SP_THREADS, 0, st>>>(a); break;
        case 9: map_sparse_kernel<4, true><<<grid, SP_THREADS, 0, st>>>(a); break;
        case 17: map_sparse_kernel<8, true><<<grid, SP_THREADS, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace som
