// map_tc.cu — batch BMU mapping on the 5th-gen tensor cores (tcgen05), the
// SOM_MAP_3XTF32 path (P:248 assignment of documents to BMUs; R20).
//
//   D(i, u) = |x_i|^2 - 2 x_i . w_u + |w_u|^2,  bmu1/bmu2 = two smallest (D, u)
//
// x . w is a true documents x units x vocabulary contraction, run as
// 3xTF32: x = x_hi + x_lo, w = w_hi + w_lo with hi = cvt.rna.tf32(v),
// lo = cvt.rna.tf32(v - hi) (split once, in global memory, by split_kernel),
// and x.w ~ x_lo.w_hi + x_hi.w_lo + x_hi.w_hi accumulated in fp32 in TMEM;
// norms are summed in fp64 by the split kernels and D is formed in fp64.
// The GEMM is a filter (R20b): its epilogue keeps the 4 smallest approximate
// D per document and unit tile, a merge keeps the 4 smallest overall, and a
// rescoring kernel computes the exact fp64 D (the dense definition, R10) of
// those candidates and certifies the result against a bound E on the
// approximation error: every other unit has exact D >= (4th approximate D) -
// E; if that exceeds the 2nd exact candidate by more than an fp32 ulp, the
// exact top-2 are among the candidates, else the document is mapped exactly
// over all units in the same kernel.  bmu1, bmu2 and D1 are therefore those
// of the exact definition for every document.
//
// Kernel: persistent CTAs of 6 warps.  warp 0 = TMA producer (4 tiles per
// K-block: A_hi, A_lo 128x32 fp32, B_hi, B_lo BNx32 fp32, 128B swizzle),
// warp 1 = TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN,
// K=8 per instruction, 12 instructions per 32-wide K-block), warps 2-5 =
// epilogue: tcgen05.ld 32 accumulator columns at a time, D in fp32, running
// top-2 (D, u) per document row across all unit tiles of the work item.
// Two TMEM accumulators (2 x BN columns, per buffer) hold the hi.hi products and the
// two small lo products separately (accuracy: see the MMA loop).  A work item is (128-document block, range
// of unit tiles); its partial top-2 keys go to the same merge kernel as the
// exact path.
#include <cuda.h>
#include <cuda_runtime.h>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int TC_BM = 128;
// Unit tile of 128 (3 stages of 64 KB, two accumulator buffers in TMEM: the
// epilogue of tile i overlaps the MMAs of tile i + 1) or (SOM_TC_BN=256)
// 256 (2 stages of 96 KB, one accumulator buffer)
#ifndef SOM_TC_BN
#define SOM_TC_BN 128
#endif
constexpr int TC_BN = SOM_TC_BN;
constexpr int TC_BK = 32;                 // fp32 elements = 128 B = one swizzle atom row
constexpr int TC_STAGES = TC_BN == 128 ? 3 : 2;
constexpr int TC_ACC_BUFS = TC_BN == 128 ? 2 : 1;
constexpr int TC_THREADS = 192;
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;            // 16 KB
constexpr uint32_t B_BYTES = TC_BN * TC_BK * 4;            // 32 KB
constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // 96 KB
constexpr uint32_t TMEM_COLS = 2 * TC_BN * TC_ACC_BUFS;     // hh and lo accumulators per buffer
constexpr int TC_K = 4;                                    // candidates per document (R20b)

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled operand tile: rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address (16 B units)
    d |= (uint64_t)1 << 16;                          // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcArgs {
    int64_t n;        // documents
    int N;            // units
    int kblocks;      // padded d / 32
    int n_tiles;      // ceil(N / BN)
    int m_blocks;     // ceil(n / 128)
    int group;        // unit tiles per raster group (L2 reuse of A and B panels)
    const double* xnorm;  // [n] fp64 |x|^2
    const double* wnorm;  // [N] fp64 |w|^2
    unsigned long long* keys;   // [n_tiles][n][TC_K] partial top-K per unit tile
};

// Work item wi -> (document block, unit tile).  Grouped raster: unit tiles
// are taken `group` at a time and, within a group, consecutive work items
// walk the unit tiles of one document block, so the ~148 concurrently
// running items share a few A panels (documents) and a few B panels (units)
// in L2 instead of streaming every panel from HBM.
__device__ __forceinline__ void work_coords(int wi, const TcArgs& a, int& mb, int& nt) {
    const int per_group = a.m_blocks * a.group;
    const int g = wi / per_group;
    const int r = wi - g * per_group;
    const int gsize = min(a.group, a.n_tiles - g * a.group);
    mb = r / gsize;
    nt = g * a.group + (r - mb * gsize);
}

__global__ void __launch_bounds__(TC_THREADS, 1)
map_tc_kernel(const __grid_constant__ CUtensorMap tm_ahi, const __grid_constant__ CUtensorMap tm_alo,
              const __grid_constant__ CUtensorMap tm_bhi, const __grid_constant__ CUtensorMap tm_blo, const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle atoms
    unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE_BYTES);
    uint64_t* empty = full + TC_STAGES;
    uint64_t* tfull = empty + TC_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int work_items = a.m_blocks * a.n_tiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_ahi); prefetch_tmap(&tm_alo); prefetch_tmap(&tm_bhi); prefetch_tmap(&tm_blo);
    }
    if (warp == 1) tmem_alloc(tmem_base_smem, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_smem;

    if (warp == 0) {
        // ===== TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int wi = blockIdx.x; wi < work_items; wi += gridDim.x) {
                int mb, nt;
                work_coords(wi, a, mb, nt);
                {
                    for (int kb = 0; kb < a.kblocks; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        unsigned char* sb = smem + stage * STAGE_BYTES;
                        mbar_expect_tx(&full[stage], STAGE_BYTES);
                        const int kc = kb * TC_BK;
                        tma_load_2d(sb, &tm_ahi, &full[stage], kc, mb * TC_BM);
                        tma_load_2d(sb + A_BYTES, &tm_alo, &full[stage], kc, mb * TC_BM);
                        tma_load_2d(sb + 2 * A_BYTES, &tm_bhi, &full[stage], kc, nt * TC_BN);
                        tma_load_2d(sb + 2 * A_BYTES + B_BYTES, &tm_blo, &full[stage], kc, nt * TC_BN);
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread)
        const uint32_t idesc = (1u << 4)                          // D format F32
                               | (2u << 7) | (2u << 10)           // A, B format TF32
                               | ((uint32_t)(TC_BN >> 3) << 17)   // N
                               | ((uint32_t)(TC_BM >> 4) << 24);  // M
        int stage = 0;
        uint32_t phase = 0;
        uint32_t tile = 0;
        for (int wi = blockIdx.x; wi < work_items; wi += gridDim.x, ++tile) {
            {
                // accumulator buffer `buf`: hh (x_hi.w_hi) at its column 0 and
                // lo (x_lo.w_hi + x_hi.w_lo) at column BN, so the large
                // accumulator takes K/8 adds instead of 3K/8 (its fp32
                // accumulation is not round-to-nearest)
                const uint32_t buf = tile % TC_ACC_BUFS, tph = (tile / TC_ACC_BUFS) & 1;
                mbar_wait(&tempty[buf], tph ^ 1);
                tc_fence_after();
                const uint32_t acc_hh = tmem_base + buf * 2 * TC_BN, acc_lo = acc_hh + TC_BN;
                for (int kb = 0; kb < a.kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sb = smem_u32(smem + stage * STAGE_BYTES);
                        const uint64_t ahi = make_sdesc(sb), alo = make_sdesc(sb + A_BYTES);
                        const uint64_t bhi = make_sdesc(sb + 2 * A_BYTES), blo = make_sdesc(sb + 2 * A_BYTES + B_BYTES);
#pragma unroll
                        for (int k = 0; k < TC_BK / 8; ++k) {
                            const uint64_t ko = (uint64_t)((k * 32) >> 4);   // +32 B per K=8 step
                            const uint32_t acc0 = (kb | k) != 0;
                            mma_tf32(acc_lo, alo + ko, bhi + ko, idesc, acc0);
                            mma_tf32(acc_lo, ahi + ko, blo + ko, idesc, 1u);
                            mma_tf32(acc_hh, ahi + ko, bhi + ko, idesc, acc0);
                        }
                        mma_commit(&empty[stage]);                   // smem slot free when these MMAs finish
                        if (kb == a.kblocks - 1) mma_commit(&tfull[buf]);
                    }
                    __syncwarp();
                    if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else {
        // ===== epilogue: warps 2..5 own TMEM lane quadrants (warp % 4)
        const int q = warp & 3;
        const int row_in_tile = q * 32 + lane;
        uint32_t tile = 0;
        for (int wi = blockIdx.x; wi < work_items; wi += gridDim.x, ++tile) {
            int mb, nt;
            work_coords(wi, a, mb, nt);
            const int64_t row = (int64_t)mb * TC_BM + row_in_tile;
            const double xn = row < a.n ? a.xnorm[row] : 0.0;
            unsigned long long kk[TC_K];
#pragma unroll
            for (int j = 0; j < TC_K; ++j) kk[j] = ~0ull;
            {
                const uint32_t buf = tile % TC_ACC_BUFS, tph = (tile / TC_ACC_BUFS) & 1;
                mbar_wait(&tfull[buf], tph);
                tc_fence_after();
                const uint32_t taddr = tmem_base + buf * 2 * TC_BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
                for (int c = 0; c < TC_BN / 32; ++c) {
                    float v[32], vl[32];
                    tmem_ld32(taddr + c * 32, v);
                    tmem_ld32(taddr + TC_BN + c * 32, vl);
                    const int u0 = nt * TC_BN + c * 32;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int u = u0 + i;
                        if (u < a.N) {
                            // D = |x|^2 + |w|^2 - 2 x.w in fp64 from the two
                            // fp32 accumulators, clamped >= 0 (R20), rounded
                            // to fp32 for the candidate key
                            const double xw = (double)v[i] + (double)vl[i];
                            const double D = fmax(fma(-2.0, xw, xn + __ldg(a.wnorm + u)), 0.0);
                            unsigned long long k = make_key((float)D, u);
                            // insertion into the sorted top-K
#pragma unroll
                            for (int j = 0; j < TC_K; ++j) {
                                const unsigned long long lo = umin64(kk[j], k), hi = kk[j] < k ? k : kk[j];
                                kk[j] = lo;
                                k = hi;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
            }
            if (row < a.n) {
                unsigned long long* dst = a.keys + ((size_t)nt * a.n + row) * TC_K;
#pragma unroll
                for (int j = 0; j < TC_K; ++j) dst[j] = kk[j];
            }
        }
    }
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem_base, TMEM_COLS);
}

// Split rows of a dense fp32 matrix into tf32 hi / lo parts (K padded to a
// multiple of 32 with zeros), the fp64 squared norm of each row and (groups,
// nullable) the number of 8-wide K groups holding a non-zero (the MMA steps
// whose accumulation can round, R20b).  One warp per row; fixed reduction
// order (deterministic).
__global__ void split_kernel(const float* __restrict__ src, int64_t rows, int d, int dp, float* __restrict__ hi,
                             float* __restrict__ lo, double* __restrict__ norm, int* __restrict__ groups) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = wg; r < rows; r += nw) {
        const float* s = src + r * d;
        float* h = hi + r * dp;
        float* l = lo + r * dp;
        double acc = 0.0;
        int g = 0;
        for (int k = lane; k < dp; k += 32) {
            const float v = k < d ? s[k] : 0.0f;
            uint32_t hb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
            const float hv = __uint_as_float(hb);
            uint32_t lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(v - hv));
            h[k] = hv;
            l[k] = __uint_as_float(lb);
            acc = fma((double)v, (double)v, acc);
            // lanes 8q..8q+7 hold one K group of this 32-wide slab
            const unsigned nzm = __ballot_sync(0xffffffffu, v != 0.0f);
            if (lane == 0) g += ((nzm & 0xFFu) != 0u) + ((nzm & 0xFF00u) != 0u) + ((nzm & 0xFF0000u) != 0u) +
                                ((nzm & 0xFF000000u) != 0u);
        }
        acc = warp_sum_f64(acc);
        if (lane == 0) {
            norm[r] = acc;
            if (groups) groups[r] = g;
        }
    }
}

// CSR rows -> split dense rows (zero + scatter) and norms from the non-zeros.
__global__ void split_csr_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                 const float* __restrict__ val, int64_t r0, int64_t rows, int dp, float* __restrict__ hi,
                                 float* __restrict__ lo, double* __restrict__ norm, int* __restrict__ groups) {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        float* h = hi + r * dp;
        float* l = lo + r * dp;
        for (int k = threadIdx.x; k < dp; k += blockDim.x) { h[k] = 0.0f; l[k] = 0.0f; }
        __syncthreads();
        const int64_t p0 = rowptr[r0 + r], p1 = rowptr[r0 + r + 1];
        double acc = 0.0;
        int g = 0;   // distinct K groups (col >> 3) among the sorted columns
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x)
            g += (p == p0 || (col[p] >> 3) != (col[p - 1] >> 3));
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
            const float v = val[p];
            uint32_t hb, lb;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
            const float hv = __uint_as_float(hb);
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(v - hv));
            h[col[p]] = hv;
            l[col[p]] = __uint_as_float(lb);
            acc = fma((double)v, (double)v, acc);
        }
        // block reduction (fixed order)
        __shared__ double red[32];
        __shared__ int gred[32];
        acc = warp_sum_f64(acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
        if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = acc; gred[threadIdx.x >> 5] = g; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            int gt = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += red[w]; gt += gred[w]; }
            norm[r] = t;
            if (groups) groups[r] = gt;
        }
        __syncthreads();
    }
}

// ------------------------------------------------ certified rescoring (R20b)
// x_i for the rescoring: CSR rows (rowptr/col/val from row r0) or dense rows X
struct XSrc {
    const int64_t* rowptr;
    const int32_t* col;
    const float* val;
    int64_t r0;
    const float* X;
};

__device__ __forceinline__ void top_insert(unsigned long long (&kk)[TC_K], unsigned long long k) {
#pragma unroll
    for (int j = 0; j < TC_K; ++j) {
        const unsigned long long lo = umin64(kk[j], k), hi = kk[j] < k ? k : kk[j];
        kk[j] = lo;
        k = hi;
    }
}

constexpr int RS_THREADS = 256;   // two CTAs (two documents in flight) per SM
constexpr int RS_WARPS = RS_THREADS / 32;

// Block-wide exact fp64 D (the dense definition, R10) of up to TC_K units
// (u < 0: skipped) against the document in shared memory; fixed summation
// order (per thread, warp butterfly, warps in order); result in out[] on
// thread 0.  Loads unrolled 4 x TC_K deep (latency).
__device__ __forceinline__ void exact_k(const float* xs, const float* __restrict__ W, int d, const int (&cu)[TC_K],
                                        double (*part)[TC_K], double (&out)[TC_K]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc[TC_K];
#pragma unroll
    for (int j = 0; j < TC_K; ++j) acc[j] = 0.0;
    int k = tid;
    for (; k + 3 * RS_THREADS < d; k += 4 * RS_THREADS) {
        float wv[4][TC_K];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < TC_K; ++j)
                wv[q][j] = cu[j] >= 0 ? __ldg(W + (int64_t)cu[j] * d + k + q * RS_THREADS) : 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double xv = (double)xs[k + q * RS_THREADS];
#pragma unroll
            for (int j = 0; j < TC_K; ++j) {
                const double e = xv - (double)wv[q][j];
                acc[j] = fma(e, e, acc[j]);
            }
        }
    }
    for (; k < d; k += RS_THREADS) {
        const double xv = (double)xs[k];
#pragma unroll
        for (int j = 0; j < TC_K; ++j) {
            if (cu[j] < 0) continue;
            const double e = xv - (double)__ldg(W + (int64_t)cu[j] * d + k);
            acc[j] = fma(e, e, acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < TC_K; ++j) {
        const double v = warp_sum_f64(acc[j]);
        if (lane == 0) part[warp][j] = v;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int j = 0; j < TC_K; ++j) {
            double t = 0.0;
            for (int w = 0; w < RS_WARPS; ++w) t += part[w][j];
            out[j] = t;
        }
    }
}

// Certificate (thread 0): candidates c[] with exact fp64 D exd[]; every
// other unit has exact D >= lb.  True: (e1, e2) = the exact top-2 (R9 keys).
__device__ __forceinline__ bool certify(const int (&cu)[TC_K], const double (&exd)[TC_K], double lb, int N,
                                        unsigned long long& e1, unsigned long long& e2) {
    e1 = e2 = ~0ull;
    int nv = 0;
#pragma unroll
    for (int j = 0; j < TC_K; ++j) {
        if (cu[j] < 0) continue;
        ++nv;
        const unsigned long long k = make_key((float)exd[j], cu[j]);
        if (k < e1) { e2 = e1; e1 = k; } else if (k < e2) e2 = k;
    }
    if (nv >= N) return true;                 // every unit is a candidate
    if (nv < TC_K || e2 == ~0ull) return false;
    // every other unit's RN32(D) >= RN32(lb) > fp32 D of the 2nd candidate:
    // no unit outside can come before it, not even on an fp32 tie (R9)
    return lb > (double)nextafterf(key_dist(e2), INFINITY);
}

// One CTA per document: merge the per-tile candidates, exact fp64 D of the
// 4 candidates (dense definition, R10), certificate; else (rare) the sparse
// identity (R25) over every unit picks 4 new candidates certified with R25's
// own error bound; else the dense definition over every unit.
// d2 = RN32(exact D of bmu1).
__global__ void __launch_bounds__(RS_THREADS) tc_rescore_kernel(
    const unsigned long long* __restrict__ keys, int n_tiles, int64_t n, const XSrc xs_src, const float* __restrict__ W,
    int N, int d, const double* __restrict__ xnorm, const double* __restrict__ wnorm, const int* __restrict__ groups,
    const double* __restrict__ wmax_p, int32_t* __restrict__ bmu1, int32_t* __restrict__ bmu2, float* __restrict__ d2,
    int* __restrict__ nfall) {
    extern __shared__ __align__(16) float xs[];          // the document, dense (d floats)
    __shared__ unsigned long long cand[TC_K];
    __shared__ unsigned long long wtop[RS_WARPS][TC_K];
    __shared__ double part[RS_WARPS][TC_K];
    __shared__ int s_ok;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double wmax = *wmax_p;
    // block merge of per-thread top-K lists -> cand[] (all threads call)
    auto block_topk = [&](unsigned long long (&kk)[TC_K]) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long other[TC_K];
#pragma unroll
            for (int j = 0; j < TC_K; ++j) other[j] = __shfl_xor_sync(0xffffffffu, kk[j], o);
#pragma unroll
            for (int j = 0; j < TC_K; ++j) top_insert(kk, other[j]);
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < TC_K; ++j) wtop[warp][j] = kk[j];
        }
        __syncthreads();
        if (tid == 0) {
            unsigned long long t[TC_K];
#pragma unroll
            for (int j = 0; j < TC_K; ++j) t[j] = ~0ull;
            for (int w = 0; w < RS_WARPS; ++w)
#pragma unroll
                for (int j = 0; j < TC_K; ++j) top_insert(t, wtop[w][j]);
#pragma unroll
            for (int j = 0; j < TC_K; ++j) cand[j] = t[j];
        }
        __syncthreads();
    };
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        // the document -> shared memory (dense)
        if (xs_src.X) {
            const float* xr = xs_src.X + i * (int64_t)d;
            for (int k = tid; k < d; k += RS_THREADS) xs[k] = xr[k];
        } else {
            for (int k = tid; k < d; k += RS_THREADS) xs[k] = 0.0f;
            __syncthreads();
            const int64_t p0 = xs_src.rowptr[xs_src.r0 + i], p1 = xs_src.rowptr[xs_src.r0 + i + 1];
            for (int64_t p = p0 + tid; p < p1; p += RS_THREADS) xs[xs_src.col[p]] = xs_src.val[p];
        }
        // candidates of the 3xTF32 filter: top-K over the unit tiles
        {
            unsigned long long kk[TC_K];
#pragma unroll
            for (int j = 0; j < TC_K; ++j) kk[j] = ~0ull;
            for (int t = tid; t < n_tiles; t += RS_THREADS) {
                const unsigned long long* p = keys + ((size_t)t * n + i) * TC_K;
#pragma unroll
                for (int j = 0; j < TC_K; ++j) top_insert(kk, p[j]);
            }
            block_topk(kk);   // (its barrier also publishes xs)
        }
        int cu[TC_K];
#pragma unroll
        for (int j = 0; j < TC_K; ++j) cu[j] = cand[j] == ~0ull ? -1 : key_unit(cand[j]);
        double exd[TC_K];
        exact_k(xs, W, d, cu, part, exd);
        const double xn = xnorm[i];
        if (tid == 0) {
            // every other unit v: approximate D >= float(A_K) - ulp, exact
            // D >= that - E, E = 2 (g + 2) 2^-20 |x| max|w| (+ fp64 slop)
            const double E = 2.0 * ((double)groups[i] + 2.0) * 0x1p-20 * sqrt(xn) * wmax + 1e-14 * (xn + wmax * wmax);
            const double lb = cand[TC_K - 1] == ~0ull ? INFINITY
                                                      : (double)nextafterf(key_dist(cand[TC_K - 1]), -INFINITY) - E;
            unsigned long long e1, e2;
            const bool ok = certify(cu, exd, lb, N, e1, e2);
            if (ok) {
                bmu1[i] = key_unit(e1);
                if (bmu2) bmu2[i] = e2 == ~0ull ? -1 : key_unit(e2);
                if (d2) d2[i] = key_dist(e1);
            } else {
                atomicAdd(nfall, 1);
            }
            s_ok = ok ? 1 : 0;
        }
        __syncthreads();
        if (s_ok) continue;
        // ---- fallback A (CSR documents): the sparse identity over every
        // unit (R25), D_u = |w_u|^2 + sum_{k in nz(x)} ((x_k - w_uk)^2 -
        // w_uk^2), thread per unit; its error is <= (d + nnz + 8) 2^-52
        // (|x|^2 + max|w|^2) (fp64 sums of exact products), so its top-K are
        // certified by the same rule after exact rescoring
        if (!xs_src.X) {
            const int64_t p0 = xs_src.rowptr[xs_src.r0 + i], p1 = xs_src.rowptr[xs_src.r0 + i + 1];
            const int nnz = (int)(p1 - p0);
            const int32_t* colp = xs_src.col + p0;
            {
                unsigned long long kk[TC_K];
#pragma unroll
                for (int j = 0; j < TC_K; ++j) kk[j] = ~0ull;
                for (int u = tid; u < N; u += RS_THREADS) {
                    const float* wr = W + (int64_t)u * d;
                    double sv = 0.0;
                    for (int q = 0; q < nnz; ++q) {
                        const int k = __ldg(colp + q);
                        const double wv = (double)__ldg(wr + k);
                        const double e = (double)xs[k] - wv;
                        sv += fma(e, e, -(wv * wv));
                    }
                    const double D = fmax(wnorm[u] + sv, 0.0);
                    top_insert(kk, make_key((float)D, u));
                }
                block_topk(kk);
            }
#pragma unroll
            for (int j = 0; j < TC_K; ++j) cu[j] = cand[j] == ~0ull ? -1 : key_unit(cand[j]);
            exact_k(xs, W, d, cu, part, exd);
            if (tid == 0) {
                const double delta = ((double)d + (double)nnz + 8.0) * 0x1p-52 * (xn + wmax * wmax);
                const double lb = cand[TC_K - 1] == ~0ull
                                      ? INFINITY
                                      : (double)nextafterf(key_dist(cand[TC_K - 1]), -INFINITY) - delta;
                unsigned long long e1, e2;
                const bool ok = certify(cu, exd, lb, N, e1, e2);
                if (ok) {
                    bmu1[i] = key_unit(e1);
                    if (bmu2) bmu2[i] = e2 == ~0ull ? -1 : key_unit(e2);
                    if (d2) d2[i] = key_dist(e1);
                }
                s_ok = ok ? 1 : 0;
            }
            __syncthreads();
            if (s_ok) continue;
        }
        // ---- fallback B: the dense definition over every unit (warp per unit)
        {
            unsigned long long k1 = ~0ull, k2 = ~0ull;
            for (int u = warp; u < N; u += RS_WARPS) {
                const float* wr = W + (int64_t)u * d;
                double a0 = 0.0, a1 = 0.0;
                int k = lane;
                for (; k + 32 < d; k += 64) {
                    const double e0 = (double)xs[k] - (double)__ldg(wr + k);
                    const double e1v = (double)xs[k + 32] - (double)__ldg(wr + k + 32);
                    a0 = fma(e0, e0, a0);
                    a1 = fma(e1v, e1v, a1);
                }
                if (k < d) {
                    const double e0 = (double)xs[k] - (double)__ldg(wr + k);
                    a0 = fma(e0, e0, a0);
                }
                const double t = warp_sum_f64(a0 + a1);
                const unsigned long long kv = make_key((float)t, u);
                if (kv < k1) { k2 = k1; k1 = kv; } else if (kv < k2) k2 = kv;
            }
            if (lane == 0) { wtop[warp][0] = k1; wtop[warp][1] = k2; }
            __syncthreads();
            if (tid == 0) {
                unsigned long long b1 = ~0ull, b2 = ~0ull;
                for (int w = 0; w < RS_WARPS; ++w)
                    for (int j = 0; j < 2; ++j) {
                        const unsigned long long kv = wtop[w][j];
                        if (kv < b1) { b2 = b1; b1 = kv; } else if (kv < b2) b2 = kv;
                    }
                bmu1[i] = key_unit(b1);
                if (bmu2) bmu2[i] = b2 == ~0ull ? -1 : key_unit(b2);
                if (d2) d2[i] = key_dist(b1);
            }
            __syncthreads();
        }
    }
}

// max_u |w_u| from the fp64 squared norms (one CTA)
__global__ void wmax_kernel(const double* __restrict__ wn, int N, double* __restrict__ out) {
    __shared__ double red[32];
    double m = 0.0;
    for (int u = threadIdx.x; u < N; u += blockDim.x) m = fmax(m, wn[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
        *out = sqrt(t);
    }
}

// ------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeFn)p;
    }
    return fn;
}

bool make_map(CUtensorMap* m, const float* base, int64_t rows, int dp, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)dp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)dp * 4};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

int tc_padded_dim(int d) { return (d + TC_BK - 1) / TC_BK * TC_BK; }

cudaError_t launch_split_rows(const float* src, int64_t rows, int d, float* hi, float* lo, double* norm, int* groups,
                              cudaStream_t st) {
    const int dp = tc_padded_dim(d);
    int blocks = (int)std::min<int64_t>((rows + 7) / 8, 148 * 16);
    if (blocks < 1) blocks = 1;
    split_kernel<<<blocks, 256, 0, st>>>(src, rows, d, dp, hi, lo, norm, groups);
    return cudaGetLastError();
}

cudaError_t launch_split_csr(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0, int64_t rows,
                             int d, float* hi, float* lo, double* norm, int* groups, cudaStream_t st) {
    const int dp = tc_padded_dim(d);
    int blocks = (int)std::min<int64_t>(rows, 148 * 16);
    if (blocks < 1) return cudaSuccess;
    split_csr_kernel<<<blocks, 256, 0, st>>>(rowptr, col, val, r0, rows, dp, hi, lo, norm, groups);
    return cudaGetLastError();
}

cudaError_t launch_wmax(const double* wn, int N, double* out, cudaStream_t st) {
    wmax_kernel<<<1, 1024, 0, st>>>(wn, N, out);
    return cudaGetLastError();
}

bool tc_rescore_fits(int d) { return 4 * (size_t)d <= 110 * 1024; }

// rows [0, n) of this chunk: candidates keys[tc_unit_tiles(N)][n][TC_K] ->
// certified exact bmu1 / bmu2 / D1; *nfall (device) counts documents that
// took the exact scan over every unit
cudaError_t launch_tc_rescore(const unsigned long long* keys, int64_t n, const int64_t* rowptr, const int32_t* col,
                              const float* val, int64_t r0, const float* X, const float* W, int N, int d,
                              const double* xnorm, const double* wnorm, const int* groups, const double* wmax,
                              int32_t* bmu1, int32_t* bmu2, float* d2, int* nfall, cudaStream_t st) {
    const size_t smem = 4 * (size_t)d;   // the document
    cudaError_t e = cudaFuncSetAttribute(tc_rescore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    XSrc xs{rowptr, col, val, r0, X};
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n, 148 * 16));
    tc_rescore_kernel<<<grid, RS_THREADS, smem, st>>>(keys, tc_unit_tiles(N), n, xs, W, N, d, xnorm, wnorm, groups,
                                                      wmax, bmu1, bmu2, d2, nfall);
    return cudaGetLastError();
}

int tc_unit_tiles(int N) { return (N + TC_BN - 1) / TC_BN; }
int tc_doc_blocks(int64_t n) { return (int)((n + TC_BM - 1) / TC_BM); }

// Documents [n] split (x_hi, x_lo, xnorm) against units [N] split (w_hi,
// w_lo, wnorm); partial top-K keys into keys[tc_unit_tiles(N)][n][TC_K].
cudaError_t launch_map_tc(const float* xhi, const float* xlo, const double* xnorm, int64_t n, const float* whi,
                          const float* wlo, const double* wnorm, int N, int d, unsigned long long* keys, int sm_count,
                          cudaStream_t st) {
    const int dp = tc_padded_dim(d);
    CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
    if (!make_map(&ma_hi, xhi, n, dp, TC_BM) || !make_map(&ma_lo, xlo, n, dp, TC_BM) ||
        !make_map(&mb_hi, whi, N, dp, TC_BN) || !make_map(&mb_lo, wlo, N, dp, TC_BN))
        return cudaErrorInvalidValue;
    TcArgs a;
    a.n = n; a.N = N; a.kblocks = dp / TC_BK; a.n_tiles = tc_unit_tiles(N); a.m_blocks = tc_doc_blocks(n);
    a.xnorm = xnorm; a.wnorm = wnorm; a.keys = keys;
    // group size: minimise panel re-streaming for ~sm_count concurrent items,
    // (n_tiles/b)|A| + (m_blocks/(sm/b))|B| with |A| ~ n, |B| ~ N
    {
        double best = 1e300;
        a.group = a.n_tiles;
        for (int b = 1; b <= a.n_tiles; ++b) {
            const double conc_m = std::max(1.0, (double)sm_count / b);
            const double cost = (double)a.n_tiles / b * (double)n + (double)a.m_blocks / conc_m * (double)N;
            if (cost < best) { best = cost; a.group = b; }
        }
    }
    const size_t smem = TC_STAGES * STAGE_BYTES + 1024 + 256;
    cudaError_t e = cudaFuncSetAttribute(map_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int work = a.m_blocks * a.n_tiles;
    const int grid = std::max(1, std::min(work, sm_count));
    map_tc_kernel<<<grid, TC_THREADS, smem, st>>>(ma_hi, ma_lo, mb_hi, mb_lo, a);
    return cudaGetLastError();
}

}  // namespace som
