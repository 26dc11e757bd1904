// train_onchip.cu — online SOM training with the map
// held on chip: kernel 9.  Same step and arithmetic contract as the CSR
// training kernels (train_csr.cu: pending Eq. 1 update of step t-1 fused
// with step t, R9-R11, sparse identity R25, tagged all-gather exchange), for
// maps whose per-SM share does not fit the register file but largely fits
// the SM's on-chip memories (c3: 50x50 x 10,000 = 100 MB over 148 SMs is
// 17 rows of 40 KB per SM).  Where the rows live, per CTA:
//   * TMEM rows: tcgen05 tensor memory (256 KB per SM, 512 columns x 128
//     lanes of 32 bit) used as plain storage: a row is 16 KJ columns of all
//     128 lanes; data thread (warp w = 1..15, lane i) owns lane 32 (w % 4) + i
//     (the lane quarter its warp may access) and columns ((w - 1) / 4) 4 KJ +
//     4 j + c — exactly its register chunks j (float4 index (tid - 32) +
//     480 j) of the other classes, so tcgen05.ld/st move a
//     thread's own elements (measured 41 elements/clk/SM read-modify-write,
//     profiles/probe_onchip_r02.json, vs 15 for shared memory);
//   * SMEM rows: dynamic shared memory;
//   * GLOBAL rows: W in global memory (L2-resident: only the rest of the map
//     streams), through a TMA bulk-copy ring as in train_csr.cu.
// Warps 1-15 own the data; warp 0 is the control warp (keys, exchange,
// neighbourhood, lists, ring prefill).  Per step t:
//   1. dense pass (data warps) over the units the pending update of t-1
//      touches: w' = fmaf(h, RN(x_{t-1} - w), w) (R11) written back to the
//      unit's storage, |w'|^2 in fp64 and the sparse term
//      S = sum_{k in nz(x_t)} ((x_k - w'_k)^2 - w'_k^2) in fp64 from the
//      owning threads (x_t is in registers);  D = |w'|^2 + S  (R25);
//   2. barrier A; the control warp forms the keys (units outside the
//      update: D = |w|^2 + S from the speculative sums of step 3 of the
//      previous step), exchanges, takes the winner, builds h and the next
//      update list, prefills the ring;  meanwhile the data warps compute S
//      of step t+1 for every unit (speculative: exact for every unit the
//      update of step t does not touch, as in train_csr.cu) — on-chip rows
//      by their owning threads, GLOBAL rows by gathers — and stage x_{t+2};
//   3. barrier B; x_{t+1} into registers.
// All sums have a fixed order (deterministic); at the end of the launch the
// on-chip rows are written back to W.
#include <algorithm>
#include <cstdlib>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int ND = 15;             // data warps 1..15
constexpr int NDT = ND * 32;       // data threads (own the rows' elements)
constexpr int NTH = NDT + 32;      // + the control warp 0 (512 threads: 128 registers)
constexpr int kSlots = 32;         // units per CTA (one control lane each)
constexpr int kCtl = 0;            // control warp index

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_data() { asm volatile("bar.sync 1, %0;" ::"n"(NDT) : "memory"); }

// ---- tcgen05 tensor-memory moves of N consecutive 32-bit columns (32 lanes)
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tm_ld<1>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(ta));
}
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta));
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tm_st<4>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
template <>
__device__ __forceinline__ void tm_st<16>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// a thread's 4 KJ columns of one TMEM row <-> its KJ float4 chunks
// (C = 4 KJ columns: 16-column pieces, then an 8 and a 4 as needed)
template <int KJ>
__device__ __forceinline__ void tm_load_row(uint32_t ta, float4 (&w)[KJ]) {
    constexpr int C = 4 * KJ;
    constexpr int O8 = (C / 16) * 16;
    constexpr int O4 = O8 + (((C - O8) >= 8) ? 8 : 0);
    uint32_t r[C];
    if constexpr (C >= 16) tm_ld<16>(ta, r);
    if constexpr (C >= 32) tm_ld<16>(ta + 16, r + 16);
    if constexpr ((C - O8) >= 8) tm_ld<8>(ta + O8, r + O8);
    if constexpr ((C - O4) >= 4) tm_ld<4>(ta + O4, r + O4);
    tm_wait_ld();
#pragma unroll
    for (int j = 0; j < KJ; ++j)
        w[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                           __uint_as_float(r[4 * j + 3]));
}
template <int KJ>
__device__ __forceinline__ void tm_store_row(uint32_t ta, const float4 (&w)[KJ]) {
    constexpr int C = 4 * KJ;
    constexpr int O8 = (C / 16) * 16;
    constexpr int O4 = O8 + (((C - O8) >= 8) ? 8 : 0);
    uint32_t r[C];
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        r[4 * j] = __float_as_uint(w[j].x); r[4 * j + 1] = __float_as_uint(w[j].y);
        r[4 * j + 2] = __float_as_uint(w[j].z); r[4 * j + 3] = __float_as_uint(w[j].w);
    }
    if constexpr (C >= 16) tm_st<16>(ta, r);
    if constexpr (C >= 32) tm_st<16>(ta + 16, r + 16);
    if constexpr ((C - O8) >= 8) tm_st<8>(ta + O8, r + O8);
    if constexpr ((C - O4) >= 4) tm_st<4>(ta + O4, r + O4);
}

// sparse term of one element (R25): (x - w)^2 - w^2, both products exact-ish in fp64
__device__ __forceinline__ double sterm(float x, float w) {
    const double wd = (double)w;
    const double e = (double)x - wd;
    return fma(e, e, -(wd * wd));
}

// value of column k in the sorted CSR list (cols ci, vals cv, cnt entries); 0 if absent
__device__ __forceinline__ float list_value(const int* ci, const float* cv, int cnt, int k) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < k) lo = mid + 1; else hi = mid;
    }
    return (lo < cnt && ci[lo] == k) ? cv[lo] : 0.0f;
}

template <int KJ>
__global__ void __launch_bounds__(NTH, 1) som_train_onchip_kernel(const TrainArgs a, int ntm, int nsm, int R_max) {
    __shared__ double partn[kSlots][ND];     // |w'|^2 partials of dense-pass rows
    __shared__ double part[kSlots][ND];      // sparse-term partials of dense-pass rows
    __shared__ double saccw[kSlots][ND];     // speculative sparse terms, on-chip rows
    __shared__ double saccg[kSlots];         // speculative sparse terms, GLOBAL rows
    __shared__ double wns[kSlots];           // fp64 |w_u|^2
    __shared__ float hs[kSlots];
    __shared__ unsigned char upd[kSlots];
    __shared__ int lst[kSlots];
    __shared__ int uid[kSlots];
    __shared__ int s_nup, s_ng0, s_abort;
    __shared__ uint32_t s_tmem;
    __shared__ long long nb[3][2];           // CSR bounds of x_t in nb[t % 3]
    __shared__ __align__(8) uint64_t mbar[4];
    extern __shared__ __align__(128) float sm[];
    // sm: ring [R_max][dimp] | smem rows [nsm][dimp] | nzi[3][cap] | nzv[3][cap] | bitmap[2][bmw]

    const int b = blockIdx.x, G = a.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool data = warp != kCtl;
    const int dw = warp - 1;           // data warp index 0..14
    const int dtid = tid - 32;         // data thread index 0..479
    const int Sb = a.utab ? a.ucnt[b] : (a.N - b + G - 1) / G;
    const int non = min(Sb, ntm + nsm);      // on-chip slots [0, non)
    const int R = min(R_max, max(Sb - non, 0));
    const int d4 = a.dimp >> 2;
    const int cap = a.nz_cap;
    const int bmw = (a.dimp >> 5) + 1;
    const uint32_t row_bytes = (uint32_t)a.dim * 4u;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float4* ring4 = reinterpret_cast<float4*>(sm);
    float* smr = sm + (size_t)R_max * a.dimp;
    float4* smr4 = reinterpret_cast<float4*>(smr);
    int* nzi = reinterpret_cast<int*>(sm + (size_t)(R_max + nsm) * a.dimp);
    float* nzv = reinterpret_cast<float*>(nzi + 3 * (size_t)cap);
    uint32_t* bmp = reinterpret_cast<uint32_t*>(nzv + 3 * (size_t)cap);

    // data thread geometry: float4 chunk dtid + 480 j; TMEM lane quarter and column group
    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = data && dtid + j * NDT < d4;
    const uint32_t tm_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t tm_colg = (uint32_t)((dw >> 2) * 4 * KJ);   // quarter q holds warps q (+4, +8, +12)
    auto tm_addr = [&](int s) { return s_tmem + tm_lane + (uint32_t)(s * 16 * KJ) + tm_colg; };

    auto bounds = [&](int64_t t) {
        const int64_t i = train_row(a, t);
        nb[t % 3][0] = a.rowptr[i];
        nb[t % 3][1] = a.rowptr[i + 1];
    };
    auto cnt_of = [&](int64_t t) { return (int)(nb[t % 3][1] - nb[t % 3][0]); };
    auto li_of = [&](int64_t t) { return nzi + (size_t)(t % 3) * cap; };
    auto lv_of = [&](int64_t t) { return nzv + (size_t)(t % 3) * cap; };
    // (col, val) of x_t -> list slot t % 3 (data threads)
    auto stage_list = [&](int64_t t) {
        if (t < a.t1) {
            const int64_t p0 = nb[t % 3][0];
            const int cnt = cnt_of(t);
            int* di = nzi + (size_t)(t % 3) * cap;
            float* dv = nzv + (size_t)(t % 3) * cap;
            for (int p = dtid; p < cnt; p += NDT) {
                cp_async4(di + p, a.col + p0 + p);
                cp_async4(dv + p, a.val + p0 + p);
            }
        }
        cp_async_commit();
    };
    // bitmap of x_t's columns in slot t & 1 (data threads; two data barriers)
    auto build_bitmap = [&](int64_t t) {
        uint32_t* bm = bmp + (size_t)(t & 1) * bmw;
        for (int q = dtid; q < bmw; q += NDT) bm[q] = 0u;
        bar_data();
        const int cnt = cnt_of(t);
        const int* ci = li_of(t);
        for (int p = dtid; p < cnt; p += NDT) atomicOr(bm + (ci[p] >> 5), 1u << (ci[p] & 31));
        bar_data();
    };
    // bit 4 j + c: this thread's element (j, c) is non-zero in x_t
    auto mask_of = [&](int64_t t) {
        const uint32_t* bm = bmp + (size_t)(t & 1) * bmw;
        uint32_t m = 0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            if (!valid[j]) continue;
            const int k0 = 4 * (dtid + j * NDT);
            m |= ((bm[k0 >> 5] >> (k0 & 31)) & 0xFu) << (4 * j);
        }
        return m;
    };
    // this thread's chunks of x_t (values of the set bits from the sorted list)
    auto load_x = [&](int64_t t, uint32_t m, float4 (&x)[KJ]) {
        const int* ci = li_of(t);
        const float* cv = lv_of(t);
        const int cnt = cnt_of(t);
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            x[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            const uint32_t bits = (m >> (4 * j)) & 0xFu;
            if (bits) {
                const int k0 = 4 * (dtid + j * NDT);
                if (bits & 1u) x[j].x = list_value(ci, cv, cnt, k0);
                if (bits & 2u) x[j].y = list_value(ci, cv, cnt, k0 + 1);
                if (bits & 4u) x[j].z = list_value(ci, cv, cnt, k0 + 2);
                if (bits & 8u) x[j].w = list_value(ci, cv, cnt, k0 + 3);
            }
        }
    };
    // speculative sparse terms S_{t'}(u) of every unit with its current row
    // (data warps): on-chip rows by the threads owning the non-zero columns
    // of x_{t'} (TMEM columns loaded warp-wide), GLOBAL rows gathered
    auto sparse_terms = [&](int64_t tq) {
        const int cnt = cnt_of(tq);
        const int* ci = li_of(tq);
        const float* cv = lv_of(tq);
        const uint32_t m = mask_of(tq);
        const uint32_t M = __reduce_or_sync(0xffffffffu, m);
        // two passes of up to 8 slots each (TMEM rows, then shared-memory
        // rows), one multi-value butterfly per pass
#pragma unroll 1
        for (int ph = 0; ph < 2; ++ph) {
            const int s0 = ph == 0 ? 0 : ntm, s1 = ph == 0 ? min(ntm, non) : non;
            if (s1 <= s0) continue;
            if (M) {
                double acc[8];
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) acc[qq] = 0.0;
                uint32_t Mr = M;
                while (Mr) {
                    const int bit = __ffs(Mr) - 1;
                    Mr &= Mr - 1;
                    const bool mine = (m >> bit) & 1u;
                    const int k = 4 * (dtid + (bit >> 2) * NDT) + (bit & 3);
                    const float xe = mine ? list_value(ci, cv, cnt, k) : 0.0f;
                    if (ph == 0) {
                        uint32_t rv[8];
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq)
                            if (qq < s1) tm_ld<1>(tm_addr(qq) + (uint32_t)bit, &rv[qq]);
                        tm_wait_ld();
                        if (mine) {
#pragma unroll
                            for (int qq = 0; qq < 8; ++qq)
                                if (qq < s1) acc[qq] += sterm(xe, __uint_as_float(rv[qq]));
                        }
                    } else if (mine) {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq)
                            if (s0 + qq < s1) acc[qq] += sterm(xe, smr[(size_t)qq * a.dimp + k]);
                    }
                }
                int slot = 0;
                const double tot = butterfly_sum<8>(acc, lane, &slot);
                if ((lane & 3) == 0 && s0 + slot < s1) saccw[s0 + slot][dw] = tot;
            } else if (lane < s1 - s0) {
                saccw[s0 + lane][dw] = 0.0;
            }
        }
        // GLOBAL rows: warps gather, lanes over the non-zeros of x_{t'}
        for (int s = non + dw; s < Sb; s += ND) {
            const float* row = a.W + (int64_t)uid[s] * a.dimp;
            double v = 0.0;
            for (int p = lane; p < cnt; p += 32) v += sterm(cv[p], __ldcg(row + ci[p]));
            v = warp_sum_f64(v);
            if (lane == 0) saccg[s] = v;
        }
    };
    // row of slot s (class storage) -> registers; GLOBAL rows from ring slot buf
    auto load_row = [&](int s, bool glob, int buf, float4 (&w)[KJ]) {
        if (s < ntm) {
            tm_load_row<KJ>(tm_addr(s), w);
        } else {
            const float4* src = glob ? ring4 + (size_t)buf * d4 : smr4 + (size_t)(s - ntm) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) w[j] = valid[j] ? src[dtid + j * NDT] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_row = [&](int s, bool glob, const float4 (&w)[KJ]) {
        if (s < ntm) {
            tm_store_row<KJ>(tm_addr(s), w);
        } else if (!glob) {
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) smr4[(size_t)(s - ntm) * d4 + dtid + j * NDT] = w[j];
        } else {
            float4* row = W4 + (int64_t)uid[s] * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) __stcg(row + dtid + j * NDT, w[j]);
        }
    };

    // ---- prologue
    if (warp == kCtl) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        if (lane == 0) {
            s_abort = 0;
            s_nup = 0;
            s_ng0 = 0;
            for (int r = 0; r < 4; ++r) mbar_init_g(&mbar[r], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            bounds(a.t0);
            if (a.t0 + 1 < a.t1) bounds(a.t0 + 1);
        }
    }
    for (int s = tid; s < kSlots; s += NTH) { hs[s] = 0.0f; upd[s] = 0; lst[s] = s; }
    for (int s = tid; s < Sb; s += NTH) uid[s] = a.utab ? a.utab[(size_t)b * a.S + s] : b + s * G;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float4 xp[KJ];      // x_{t-1} (the pending update's sample)
    uint32_t mc = 0;    // non-zero columns of x_t among this thread's elements
    if (data) {
        stage_list(a.t0);
        stage_list(a.t0 + 1);
        // on-chip rows from W; fp64 norms of every row
        for (int s = 0; s < Sb; ++s) {
            const float4* row = W4 + (int64_t)uid[s] * d4;
            float4 w[KJ];
#pragma unroll
            for (int j = 0; j < KJ; ++j) w[j] = valid[j] ? __ldcg(row + dtid + j * NDT) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (s < non) store_row(s, false, w);
            double n0 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                n0 = fma((double)w[j].x, (double)w[j].x, n0);
                n0 = fma((double)w[j].y, (double)w[j].y, n0);
                n0 = fma((double)w[j].z, (double)w[j].z, n0);
                n0 = fma((double)w[j].w, (double)w[j].w, n0);
            }
            n0 = warp_sum_f64(n0);
            if (lane == 0) partn[s][dw] = n0;
        }
        tm_wait_st();
        cp_async_wait_all();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == kCtl && lane == 0 && a.t0 + 2 < a.t1) bounds(a.t0 + 2);
    if (data) {
        build_bitmap(a.t0);
        mc = mask_of(a.t0);
#pragma unroll
        for (int j = 0; j < KJ; ++j) xp[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        sparse_terms(a.t0);
    } else if (lane < Sb) {
        double tot = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < ND; ++w8) tot += partn[lane][w8];
        wns[lane] = tot;
    }
    __syncthreads();
    int64_t q = 0;   // GLOBAL rows consumed from the ring so far (CTA-uniform)

    for (int64_t t = a.t0; t < a.t1; ++t) {
        const int nup = s_nup, ng0 = s_ng0;
        // ---- 1. dense pass (data warps) over the pending update's rows, in
        // pairs (one multi-value butterfly per pair for |w'|^2 and S)
        if (data) {
            const int* ci = li_of(t);
            const float* cv = lv_of(t);
            const int cnt = cnt_of(t);
            for (int i0 = 0; i0 < nup; i0 += 2) {
                double acc[4];
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    acc[2 * g] = 0.0;
                    acc[2 * g + 1] = 0.0;
                    const int i = i0 + g;
                    if (i >= nup) continue;
                    const int s = lst[i];
                    const float h = hs[s];
                    const bool glob = i >= ng0;
                    int buf = 0;
                    if (glob) {
                        const int64_t qq = q + (i - ng0);
                        buf = (int)(qq % R);
                        mbar_wait_g(&mbar[buf], (uint32_t)((qq / R) & 1));
                    }
                    float4 w[KJ];
                    load_row(s, glob, buf, w);
                    double n0 = 0.0, n1 = 0.0;
#pragma unroll
                    for (int j = 0; j < KJ; ++j) {
                        w[j] = eq1u(h, w[j], xp[j]);
                        const double w0 = w[j].x, w1 = w[j].y, w2 = w[j].z, w3 = w[j].w;
                        n0 = fma(w0, w0, n0);
                        n1 = fma(w1, w1, n1);
                        n0 = fma(w2, w2, n0);
                        n1 = fma(w3, w3, n1);
                    }
                    double sp = 0.0;
                    if (mc) {
#pragma unroll
                        for (int j = 0; j < KJ; ++j) {
                            const uint32_t bj = (mc >> (4 * j)) & 0xFu;
                            if (!bj) continue;
                            const int k0 = 4 * (dtid + j * NDT);
                            if (bj & 1u) sp += sterm(list_value(ci, cv, cnt, k0), w[j].x);
                            if (bj & 2u) sp += sterm(list_value(ci, cv, cnt, k0 + 1), w[j].y);
                            if (bj & 4u) sp += sterm(list_value(ci, cv, cnt, k0 + 2), w[j].z);
                            if (bj & 8u) sp += sterm(list_value(ci, cv, cnt, k0 + 3), w[j].w);
                        }
                    }
                    store_row(s, glob, w);
                    acc[2 * g] = n0 + n1;
                    acc[2 * g + 1] = sp;
                    if (glob) {
                        bar_data();   // ring slot consumed, row written back
                        const int ig = i - ng0;
                        if (dtid == 0 && ig + R < nup - ng0) {
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            bulk_row(ring4 + (size_t)buf * d4, W4 + (int64_t)uid[lst[i + R]] * d4, row_bytes,
                                     &mbar[buf]);
                        }
                    }
                }
                int slot = 0;
                const double tot = butterfly_sum<4>(acc, lane, &slot);
                const int i = i0 + (slot >> 1);
                if ((lane & 7) == 0 && i < nup) {
                    if (slot & 1) part[lst[i]][dw] = tot; else partn[lst[i]][dw] = tot;
                }
            }
            tm_wait_st();
            // streamed rows written back above are read again by the next
            // step's ring prefill (async proxy): order the writes first
            if (ng0 < nup) asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        q += nup - ng0;
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();   // (A) pass done: partials complete, rows stored
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

        const double f = a.f_tab[t - a.t0];
        const double alpha = a.alpha0 * f;
        double sigma = a.sigma0 * f;
        if (sigma < a.sigma_min) sigma = a.sigma_min;
        const double two_s2 = 2.0 * sigma * sigma;
        const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;

        if (!data) {
            // ---- 2. control warp: keys, exchange, winner, next update list
            unsigned long long best = ~0ull;
            if (lane < Sb) {
                const int s = lane;
                double tot;
                if (upd[s]) {
                    double nn = 0.0, sp = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < ND; ++w8) { nn += partn[s][w8]; sp += part[s][w8]; }
                    wns[s] = nn;
                    tot = nn + sp;
                } else if (s < non) {
                    double sp = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < ND; ++w8) sp += saccw[s][w8];
                    tot = wns[s] + sp;
                } else {
                    tot = wns[s] + saccg[s];
                }
                tot = tot > 0.0 ? tot : 0.0;   // R25: the identity can round below 0
                best = make_key((float)tot, global_unit(a, uid[s]));
            }
            best = warp_min_u64(best);
            xchg_publish(a, best, t, b, lane);
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            bool u2 = false;
            if (lane < Sb) {
                const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, uid[lane]), c);
                u2 = g2 <= r2;
                upd[lane] = u2 ? 1 : 0;
                hs[lane] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
            const unsigned mu = __ballot_sync(0xffffffffu, lane < Sb && u2);
            if (lane < Sb && u2) lst[__popc(mu & ((1u << lane) - 1u))] = lane;
            __syncwarp();
            const int n_up = __popc(mu);
            const int n_on = __popc(mu & (non >= 32 ? 0xffffffffu : ((1u << non) - 1u)));
            if (lane == 0) {
                s_nup = n_up;
                s_ng0 = n_on;
                // first GLOBAL rows of the next pass into the ring (none after
                // the last step: the final flush reads rows directly)
                if (!stop && t + 1 < a.t1) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    const int m = min(n_up - n_on, R);
                    for (int i = 0; i < m; ++i) {
                        const int64_t qq = q + i;
                        bulk_row(ring4 + (size_t)(qq % R) * d4, W4 + (int64_t)uid[lst[n_on + i]] * d4, row_bytes,
                                 &mbar[qq % R]);
                    }
                }
            }
        } else {
            // ---- 2'. data warps: bitmap of x_{t+1}, speculative sparse terms
            // of step t+1 (skipped when the radius covers the whole lattice:
            // every unit then takes the dense pass), list of x_{t+2}
            stage_list(t + 2);
            if (t + 1 < a.t1) {
                build_bitmap(t + 1);
                if (!(r2 >= a.g2max)) sparse_terms(t + 1);
            }
            if (dtid == 0 && t + 3 < a.t1) bounds(t + 3);
            cp_async_wait_all();
        }
        __syncthreads();   // (B)
        if (s_abort) break;
        if (data && t + 1 < a.t1) {
            load_x(t, mc, xp);      // x_t becomes the pending update's sample
            mc = mask_of(t + 1);
        }
    }

    // flush the update of the last step (sample x_{t1-1}), then write the
    // on-chip rows back to W
    if (data && a.t1 > a.t0 && !s_abort) {
        load_x(a.t1 - 1, mc, xp);
        const int nup = s_nup, ng0 = s_ng0;
        for (int i = 0; i < nup; ++i) {
            const int s = lst[i];
            const float h = hs[s];
            float4 w[KJ];
            if (i >= ng0) {
                const float4* row = W4 + (int64_t)uid[s] * d4;
#pragma unroll
                for (int j = 0; j < KJ; ++j) w[j] = valid[j] ? __ldcg(row + dtid + j * NDT) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                load_row(s, false, 0, w);
            }
#pragma unroll
            for (int j = 0; j < KJ; ++j) w[j] = eq1u(h, w[j], xp[j]);
            store_row(s, i >= ng0, w);
        }
        tm_wait_st();
    }
    if (data && !s_abort) {
        for (int s = 0; s < non; ++s) {
            float4 w[KJ];
            load_row(s, false, 0, w);
            store_row(s, true, w);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kCtl)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512) : "memory");
}

size_t onchip_smem_bytes(int dimp, int cap, int R, int nsm) {
    return sizeof(float) * (size_t)(R + nsm) * dimp + 24 * (size_t)cap + 8 * (size_t)((dimp >> 5) + 1) + 128;
}

template <int KJ>
cudaError_t launch_onchip_kj(const TrainArgs& a, int ntm, int nsm, int R, cudaStream_t st) {
    const size_t smem = onchip_smem_bytes(a.dimp, a.nz_cap, R, nsm);
    auto fn = som_train_onchip_kernel<KJ>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    int p1 = ntm, p2 = nsm, p3 = R;
    void* params[] = {&args, &p1, &p2, &p3};
    return launch_persistent((const void*)fn, a, NTH, smem, params, st);
}

// static shared memory of the kernel (partials, lists) + headroom
constexpr size_t kOnchipStatic = 3 * kSlots * ND * 8 + 4 * kSlots * 8 + 1024;

}  // namespace

int onchip_kj(int dim) { return ((dim / 4) + NDT - 1) / NDT; }

// Placement: TMEM rows = 512 columns / 16 KJ; shared-memory rows and a ring
// of R rows for the GLOBAL remainder from the shared-memory budget.
bool train_onchip_plan(int S, int dim, int maxnnz, int max_smem_optin, int* ntm, int* nsm, int* R) {
    if (dim % 4 != 0 || S > kSlots || S < 1) return false;
    const int kj = onchip_kj(dim);
    if (kj < 1 || kj > 6) return false;
    const int cap = csr_nz_cap(maxnnz);
    const int t = std::min(std::min(S, 8), 512 / (16 * kj));
    const size_t budget = (size_t)max_smem_optin - kOnchipStatic;
    const size_t row = sizeof(float) * (size_t)dim;
    const size_t fixed = onchip_smem_bytes(dim, cap, 0, 0);
    if (fixed + row > budget) return false;
    int rmax = 2;
    if (const char* e = std::getenv("SOM_ONCHIP_RING")) rmax = std::max(1, std::min(4, std::atoi(e)));
    int best_s = 0, best_r = 0;
    int smax = 8;   // SOM_ONCHIP_NSM caps the shared-memory rows (ring depth vs on-chip rows)
    if (const char* e = std::getenv("SOM_ONCHIP_NSM")) smax = std::max(0, std::min(8, std::atoi(e)));
    // most on-chip rows first, then the deepest ring the rest of the budget allows
    for (int s = std::min(S - t, smax); s >= 0; --s) {
        const int rest = S - t - s;
        const int r = rest > 0 ? 1 : 0;
        if (fixed + (size_t)(s + r) * row <= budget) {
            best_s = s;
            best_r = r;
            while (rest > best_r && best_r < rmax && fixed + (size_t)(s + best_r + 1) * row <= budget) ++best_r;
            break;
        }
    }
    if (t + best_s > 16 || t + best_s < 1) return false;
    *ntm = t;
    *nsm = best_s;
    *R = best_r;
    return true;
}

cudaError_t launch_train_onchip(const TrainArgs& a, int ntm, int nsm, int R, cudaStream_t st) {
    switch (onchip_kj(a.dimp)) {
        case 1: return launch_onchip_kj<1>(a, ntm, nsm, R, st);
        case 2: return launch_onchip_kj<2>(a, ntm, nsm, R, st);
        case 3: return launch_onchip_kj<3>(a, ntm, nsm, R, st);
        case 4: return launch_onchip_kj<4>(a, ntm, nsm, R, st);
        case 5: return launch_onchip_kj<5>(a, ntm, nsm, R, st);
        case 6: return launch_onchip_kj<6>(a, ntm, nsm, R, st);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace som
