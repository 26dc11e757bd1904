// som_device.cuh — small device helpers of libsom (product side).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace som {

// R8: t-th output of a SplitMix64 stream seeded with `seed` (a
// counter-based draw: no state crosses steps), mapped to [0, n) by the high
// 64 bits of the 128-bit product.
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, int64_t t) {
    uint64_t z = seed + (uint64_t)(t + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t sample_at(uint64_t seed, int64_t t, int64_t n) {
    return (int64_t)__umul64hi(splitmix64_at(seed, t), (uint64_t)n);
}

// R8b (optional per-epoch permutation): epoch e = t / m, position p = t mod
// m; cycle-walk a keyed bijection of [0, 2^b) (b = bit length of m - 1):
// four rounds of add key, xor-shift right by ceil(b/2), multiply by an odd
// constant, all mod 2^b; keys = SplitMix64 outputs 4e + r of a derived seed.
__device__ __forceinline__ int64_t perm_at(uint64_t seed, int64_t t, int64_t m) {
    if (m <= 1) return 0;
    const int64_t e = t / m, p = t - e * m;
    const int b = 64 - __clzll((long long)(m - 1));
    const uint64_t mask = b >= 64 ? ~0ull : ((1ull << b) - 1ull);
    const int sh = (b + 1) / 2;
    uint64_t k[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) k[r] = splitmix64_at(seed ^ 0x5851F42D4C957F2DULL, 4 * e + r);
    uint64_t x = (uint64_t)p;
    do {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            x = (x + k[r]) & mask;
            x ^= x >> sh;
            x = (x * 0x9E3779B97F4A7C15ULL) & mask;
        }
    } while (x >= (uint64_t)m);
    return (int64_t)x;
}

// P:166 / S:164: squared lattice distance, exact (multiples of 1/4).
// rect: di^2 + dj^2; hex (pointy-top, odd rows shifted right by 1/2):
// (dj + ((iu&1) - (iv&1))/2)^2 + 3/4 di^2.
__device__ __forceinline__ double lattice_g2(int cols, int topo, int u, int v) {
    int iu = u / cols, ju = u - iu * cols;
    int iv = v / cols, jv = v - iv * cols;
    double di = (double)(iu - iv);
    if (topo == 0) {
        double dj = (double)(ju - jv);
        return di * di + dj * dj;
    }
    // work in half-units: 2*dx is an integer (all values exact in fp64)
    double dx2 = (double)(2 * (ju - jv) + ((iu & 1) - (iv & 1)));
    return 0.25 * (dx2 * dx2) + 0.75 * (di * di);
}

// BMU key: fp32 distance bits (monotone for D >= 0) | unit index | tag.
// Unsigned min over keys with equal tag = lexicographic min over (D, u),
// i.e. equal distances go to the lowest unit index (R9).
__device__ __forceinline__ unsigned long long make_key(float D, int u) {
    return ((unsigned long long)__float_as_uint(D) << 32) | ((unsigned long long)(unsigned)u << 8);
}
__device__ __forceinline__ int key_unit(unsigned long long k) { return (int)((k >> 8) & 0xFFFFFFu); }
__device__ __forceinline__ float key_dist(unsigned long long k) { return __uint_as_float((unsigned)(k >> 32)); }

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = umin64(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// cp.async global -> shared (L2 only), 16 or 4 bytes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// mbarrier + bulk (non-tensor) TMA copy of one contiguous row, global ->
// shared, completion counted in bytes on the barrier (train_glb.cu,
// train_csr.cu row rings).
__device__ __forceinline__ void mbar_init_g(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_g(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITG_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITG_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const unsigned sb = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"(sb) : "memory");
}

__device__ __forceinline__ float4 eq1u(float h, float4 w, float4 x) {
    // Eq. 1 per element: w + h (x - w) as fmaf(h, RN(x - w), w)  (R11)
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

// Warp sum of SMAX per-lane values with a multi-value butterfly: at each of
// the first log2(SMAX) levels a lane keeps half of its slots and sends the
// other half, so the warp issues 2*(SMAX-1) + 2*(5 - log2 SMAX) shuffles
// instead of 10*SMAX.  Returns the full warp sum of slot `*slot` in lanes
// whose low (5 - log2 SMAX) bits are zero.
template <int SMAX>
__device__ __forceinline__ double butterfly_sum(double (&v)[SMAX], int lane, int* slot) {
    int sl = 0;
#pragma unroll
    for (int width = SMAX, off = 16; width > 1; width >>= 1, off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < width / 2; ++i) {
            const double send = upper ? v[i] : v[i + width / 2];
            const double keep = upper ? v[i + width / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
        sl = sl * 2 + (upper ? 1 : 0);
    }
    double x = v[0];
#pragma unroll
    for (int off = 16 / SMAX; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    *slot = sl;
    return x;
}

}  // namespace som
