// train_tier.cu — online SOM training, kernel 10:
// the map held in the SM's tiers of storage, for maps whose per-SM share
// (c3: 2,500 units x 10,000 terms = 100 MB over 148 SMs, 17 rows of 40 KB
// per SM) exceeds any one of them.  Same step and arithmetic contract as the
// CSR kernels (train_csr.cu): the pending Eq. 1 update of step t-1 fused with
// step t's distances (an exact reorder), R9-R11, the sparse identity R25
// (D_u = |w_u|^2 + sum_{k in nz(x)} ((x_k - w_k)^2 - w_k^2), |w|^2 in fp64),
// the tagged all-gather exchange (som_internal.h).
//
// Where a CTA's rows live (slot s of its S units, in this order):
//   [0, ntm)           tensor memory, used as plain storage: data thread dt
//                      (warp w = 1..NDW, NDW = 12 or 16, NDT = 32 NDW
//                      threads) holds float4 chunks dt + NDT j (j < KJ) of a
//                      row as 4 KJ words of its TMEM lane (lane quarter
//                      w % 4), column group (w - 1) / 4 (512 / (NDW / 4)
//                      columns each), 4 KJ r; moved with tcgen05.ld/st (its
//                      own path beside the shared-memory port); updated rows
//                      are also written through to W (the sparse sums below
//                      gather from W, and only the owning warp can read a
//                      TMEM lane) — while every unit is updated every step
//                      only at x_t's non-zeros, fully once the speculative
//                      sums run (after one catch-up of every TMEM row);
//   [ntm, non)         shared memory, [row][j][dt] float4 (conflict-free);
//   [non, S)           W in global memory (L2-resident: only these rows are
//                      read during the launch), streamed through a ring of
//                      RC chunks (chunk j of a row = float4 [NDT j, NDT j + NDT)
//                      = the thread's chunk j), filled by cp.async.bulk from
//                      the control warp, full/empty mbarriers; updated rows
//                      are written back from registers.
// Warp 0 is the control warp (keys, exchange, neighbourhood, lists, ring
// producer); warps 1..NDW hold the data.  Per step t:
//   1. dense pass (data warps) over the rows of update(t-1), streamed rows
//      alternating with on-chip rows so the ring keeps moving, branch-free:
//      w' = fmaf(h, RN(x_{t-1} - w), w) (R11; x_{t-1} in registers, built
//      once per step from its non-zeros) and |w'|^2 in fp64, per-warp
//      partials by a multi-value butterfly over two rows; then S(x_t) of
//      those rows, one warp per row over x_t's non-zeros (shared-memory rows
//      from shared memory, the others from W); meanwhile the control warp
//      feeds the ring;
//   2. barrier A; control warp: keys (updated units from the partials, the
//      others from the speculative S of step 2' of the previous step), the
//      exchange, the winner, h and the lists of update(t), first ring chunks
//      of step t+1 (one per lane); data warps meanwhile (2'): bitmap of
//      x_{t+1}, speculative S(x_{t+1}) of every unit with its current row
//      (exact for every unit update(t) leaves alone; skipped while the
//      radius covers the lattice), list of x_{t+2};
//   3. barrier B.
// All sums have a fixed order (deterministic run to run).  At the end of the
// launch the update of the last step is applied and the on-chip rows are
// written back to W.
#include <algorithm>
#include <cstdlib>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

// data warps 1..NDW: 12 (3 TMEM column groups of 170) or 16 (4 groups of
// 128; 544 threads at <= 120 registers, chosen where a row needs <= 5 float4
// chunks per thread: c3 22.1 vs 23.0 us/step in the full-coverage window,
// bit-identical, tools/lib_ab.py)
template <int NDW>
struct TierShape {
    static constexpr int ndt = NDW * 32;               // data threads: own the rows' elements
    static constexpr int nth = ndt + 32;               // + control warp 0
    static constexpr int tm_cols = 512 / (NDW / 4);    // TMEM columns per column group
};
constexpr int kSlots = 32;         // units per CTA (one control lane each)
constexpr int kRingMax = 16;       // ring chunks
constexpr int kTmMax = 8;          // TMEM rows (unrolled loops)
constexpr int kSmMax = 4;          // shared-memory rows (unrolled loops)

struct TierPlan {
    int ntm, nsm, rc;              // TMEM rows, shared-memory rows, ring chunks
    int ndw;                       // data warps (12 or 16)
};

template <int NDT>
__device__ __forceinline__ void bar_data_n() { asm volatile("bar.sync 1, %0;" ::"n"(NDT) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---- tcgen05 tensor-memory moves of N consecutive 32-bit columns (32 lanes)
template <int N>
__device__ __forceinline__ void tld(uint32_t ta, uint32_t* r);
template <>
__device__ __forceinline__ void tld<4>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
}
template <>
__device__ __forceinline__ void tld<8>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
}
template <>
__device__ __forceinline__ void tld<16>(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta));
}
template <int N>
__device__ __forceinline__ void tst(uint32_t ta, const uint32_t* r);
template <>
__device__ __forceinline__ void tst<4>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}
template <>
__device__ __forceinline__ void tst<8>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
template <>
__device__ __forceinline__ void tst<16>(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// a thread's 4 KJ words of one TMEM row <-> its KJ float4 chunks
template <int KJ>
__device__ __forceinline__ void tm_load(uint32_t ta, float4 (&w)[KJ]) {
    constexpr int C = 4 * KJ;
    uint32_t r[C];
    int o = 0;
#pragma unroll
    for (int q = 0; q < C / 16; ++q, o += 16) tld<16>(ta + o, r + o);
    if constexpr ((C % 16) >= 8) { tld<8>(ta + o, r + o); o += 8; }
    if constexpr ((C % 8) >= 4) tld<4>(ta + o, r + o);
    twait_ld();
#pragma unroll
    for (int j = 0; j < KJ; ++j)
        w[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                           __uint_as_float(r[4 * j + 3]));
}
template <int KJ>
__device__ __forceinline__ void tm_store(uint32_t ta, const float4 (&w)[KJ]) {
    constexpr int C = 4 * KJ;
    uint32_t r[C];
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        r[4 * j] = __float_as_uint(w[j].x); r[4 * j + 1] = __float_as_uint(w[j].y);
        r[4 * j + 2] = __float_as_uint(w[j].z); r[4 * j + 3] = __float_as_uint(w[j].w);
    }
    int o = 0;
#pragma unroll
    for (int q = 0; q < C / 16; ++q, o += 16) tst<16>(ta + o, r + o);
    if constexpr ((C % 16) >= 8) { tst<8>(ta + o, r + o); o += 8; }
    if constexpr ((C % 8) >= 4) tst<4>(ta + o, r + o);
}

// R25 sparse term of one element: (x - w)^2 - w^2 in fp64 (both squares exact)
__device__ __forceinline__ double sterm(float x, float w) {
    const double wd = (double)w;
    const double e = (double)x - wd;
    return fma(e, e, -(wd * wd));
}

// value of column k in a sorted (col, val) list of cnt entries, 0 if absent
// (out of line: the hot loops only reach it past the 4-entry cache)
__device__ __noinline__ float list_lookup(const int* ci, const float* cv, int cnt, int k) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < k) lo = mid + 1; else hi = mid;
    }
    return (lo < cnt && ci[lo] == k) ? cv[lo] : 0.0f;
}

// position of column k in a sorted column list of cnt entries (-1 if absent)
__device__ __noinline__ int list_pos(const int* ci, int cnt, int k) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < k) lo = mid + 1; else hi = mid;
    }
    return (lo < cnt && ci[lo] == k) ? lo : -1;
}

template <int KJ, int NDW>
__global__ void __launch_bounds__(TierShape<NDW>::nth, 1) som_train_tier_kernel(const TrainArgs a, const TierPlan p) {
    constexpr int NDT = TierShape<NDW>::ndt;
    constexpr int NTH = TierShape<NDW>::nth;
    constexpr int kTmCols = TierShape<NDW>::tm_cols;
    auto bar_data = [] { bar_data_n<NDT>(); };
    __shared__ double pn[kSlots][NDW];        // |w'|^2 partials of dense-pass rows
    __shared__ double sg[2][kSlots];          // speculative S of every row, [parity of the step]
    __shared__ double sgd[kSlots];            // S(x_t) of dense-pass rows
    __shared__ double wns[kSlots];            // fp64 |w_u|^2
    __shared__ float hs[kSlots];              // h of the pending update
    __shared__ int uid[kSlots];               // local unit (W row) of slot s
    __shared__ int ord[kSlots];               // dense-pass order of the pending update's rows
    __shared__ int strm[kSlots];              // its streamed rows, in ring order
    __shared__ int iota[kSlots];              // 0, 1, 2, ... (every slot)
    __shared__ int s_nord, s_nstr, s_abort;
    __shared__ long long nb[4][2];            // CSR bounds of x_t in nb[t & 3]
    __shared__ __align__(8) uint64_t full[kRingMax];
    __shared__ __align__(8) uint64_t empty[kRingMax];
    __shared__ uint32_t s_tmem;
    extern __shared__ __align__(128) float4 sm4[];
    // sm4: ring [rc][NDT] | smem rows [nsm][KJ][NDT] | x cache float[2][2][NDT] | nzi int[3][cap] |
    //      nzv float[3][cap] | bitmap u32[2][bmw]

    const int b = blockIdx.x, G = a.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool data = warp != 0;
    const int dw = warp - 1;            // data warp 0..11
    const int dt = tid - 32;            // data thread 0..383
    const int Sb = a.utab ? a.ucnt[b] : (a.N - b + G - 1) / G;
    const int ntm = p.ntm, nsm = p.nsm, RC = p.rc;
    const int non = min(Sb, ntm + nsm);   // on-chip slots [0, non): TMEM [0, ntm), smem [ntm, non)
    const int d4 = a.dimp >> 2;
    const int cap = a.nz_cap;
    const int bmw = (a.dimp >> 5) + 1;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float4* ring = sm4;
    float4* srows = sm4 + (size_t)RC * NDT;
    // x_t at the thread's first 2 non-zeros: xcs[((t & 1) * 2 + rank) * NDT + dt]
    float* xcs = reinterpret_cast<float*>(srows + (size_t)nsm * KJ * NDT);
    int* nzi = reinterpret_cast<int*>(xcs + 4 * NDT);
    float* nzv = reinterpret_cast<float*>(nzi + 3 * (size_t)cap);
    uint32_t* bmp = reinterpret_cast<uint32_t*>(nzv + 3 * (size_t)cap);
    // chunk KJ-1 is the only one that can run past the row (KJ = ceil(d4 / NDT))
    const bool vlast = data && dt + (KJ - 1) * NDT < d4;
    const uint32_t tm_base_off = ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((dw >> 2) * kTmCols);

    uint32_t mp = 0u, mc = 0u;   // non-zeros of x_{t-1}, x_t among this thread's elements
    bool tm_stale = false;       // some TMEM row's copy in W is partial (full-coverage steps)
    float4 xp[KJ];               // x_{t-1} at this thread's elements (the pending update's sample)
    auto tm_addr = [&](int r) { return s_tmem + tm_base_off + (uint32_t)(r * 4 * KJ); };
    auto bounds = [&](int64_t t) {
        const int64_t i = train_row(a, t);
        nb[t & 3][0] = a.rowptr[i];
        nb[t & 3][1] = a.rowptr[i + 1];
    };
    auto cnt_of = [&](int64_t t) { return (int)(nb[t & 3][1] - nb[t & 3][0]); };
    // (col, val) of x_t -> list slot t % 3 (data threads)
    auto stage_list = [&](int64_t t) {
        if (t < a.t1) {
            const int64_t p0 = nb[t & 3][0];
            const int cnt = cnt_of(t);
            int* di = nzi + (size_t)(t % 3) * cap;
            float* dv = nzv + (size_t)(t % 3) * cap;
            for (int q = dt; q < cnt; q += NDT) {
                cp_async4(di + q, a.col + p0 + q);
                cp_async4(dv + q, a.val + p0 + q);
            }
        }
        cp_async_commit();
    };
    // bitmap of x_t's columns -> slot t & 1 (data threads; two data barriers)
    auto build_bitmap = [&](int64_t t) {
        uint32_t* bm = bmp + (size_t)(t & 1) * bmw;
        for (int q = dt; q < bmw; q += NDT) bm[q] = 0u;
        bar_data();
        const int cnt = cnt_of(t);
        const int* ci = nzi + (size_t)(t % 3) * cap;
        for (int q = dt; q < cnt; q += NDT) atomicOr(bm + (ci[q] >> 5), 1u << (ci[q] & 31));
        bar_data();
    };
    // bit 4 j + c: element (j, c) of this thread is non-zero in x_t
    auto mask_of = [&](int64_t t) {
        const uint32_t* bm = bmp + (size_t)(t & 1) * bmw;
        uint32_t m = 0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            if (j == KJ - 1 && !vlast) continue;
            const int k0 = 4 * (dt + j * NDT);
            m |= ((bm[k0 >> 5] >> (k0 & 31)) & 0xFu) << (4 * j);
        }
        return m;
    };
    // x_t at this thread's element `bit` (set in mask m): the per-step cache
    // holds the first 2 non-zeros in rank order; beyond, the sorted list
    auto elem_k = [&](int bit) { return 4 * (dt + (bit >> 2) * NDT) + (bit & 3); };
    auto xget = [&](int64_t t, uint32_t m, int bit) {
        const int rank = __popc(m & ((1u << bit) - 1u));
        if (rank < 2) return xcs[((int)(t & 1) * 2 + rank) * NDT + dt];
        return nzv[(size_t)(t % 3) * cap + list_pos(nzi + (size_t)(t % 3) * cap, cnt_of(t), elem_k(bit))];
    };
    auto fill_cache = [&](int64_t t, uint32_t m) {
        int rank = 0;
        while (m != 0u && rank < 2) {
            const int bit = __ffs(m) - 1;
            m &= m - 1u;
            const int q = list_pos(nzi + (size_t)(t % 3) * cap, cnt_of(t), elem_k(bit));
            xcs[((int)(t & 1) * 2 + rank) * NDT + dt] = nzv[(size_t)(t % 3) * cap + q];
            ++rank;
        }
    };
    // x_{t-1} into registers (zero off its non-zeros)
    auto build_xp = [&](int64_t tp, uint32_t m) {
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            const uint32_t bits = (m >> (4 * j)) & 0xFu;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bits != 0u) {
                if (bits & 1u) v.x = xget(tp, m, 4 * j);
                if (bits & 2u) v.y = xget(tp, m, 4 * j + 1);
                if (bits & 4u) v.z = xget(tp, m, 4 * j + 2);
                if (bits & 8u) v.w = xget(tp, m, 4 * j + 3);
            }
            xp[j] = v;
        }
    };
    // per-row |w'|^2 -> per-warp partials pn, two rows per multi-value butterfly
    double pv0 = 0.0;
    int pr0 = -1;
    auto push = [&](int s, double n) {
        if (pr0 < 0) { pv0 = n; pr0 = s; return; }
        double v[2] = {pv0, n};
        int sl = 0;
        const double tot = butterfly_sum<2>(v, lane, &sl);
        if ((lane & 15) == 0) pn[sl ? s : pr0][dw] = tot;
        pr0 = -1;
    };
    auto push_flush = [&]() {
        if (pr0 < 0) return;
        const double tot = warp_sum_f64(pv0);
        if (lane == 0) pn[pr0][dw] = tot;
        pr0 = -1;
    };
    // S(x_t) = sum_p (x_p - w_p)^2 - w_p^2 over x_t's non-zeros p, one warp
    // per row, two rows per warp at a time (multi-value butterfly); each row
    // with its current value: shared-memory rows from shared memory, the
    // others from W in global memory (streamed rows are current, TMEM rows
    // are written through)
    auto fetch = [&](int s, int k) {
        if (s >= ntm && s < non) {
            const int e = k >> 2, j = e / NDT, d = e - j * NDT;
            return reinterpret_cast<const float*>(srows + ((size_t)(s - ntm) * KJ + j) * NDT + d)[k & 3];
        }
        return __ldcg(a.W + (int64_t)uid[s] * a.dimp + k);
    };
    auto sparse_rows = [&](int64_t tq, const int* slots, int count, double* dst) {
        const int cnt = cnt_of(tq);
        const int* ci = nzi + (size_t)(tq % 3) * cap;
        const float* cv = nzv + (size_t)(tq % 3) * cap;
        for (int i = dw; i < count; i += 2 * NDW) {
            const bool two = i + NDW < count;
            const int sa = slots[i], sb2 = two ? slots[i + NDW] : sa;
            double va = 0.0, vb = 0.0;
            for (int q = lane; q < cnt; q += 32) {
                const float x = cv[q];
                const int k = ci[q];
                const float wa = fetch(sa, k);
                const float wb = two ? fetch(sb2, k) : 0.f;
                va += sterm(x, wa);
                vb += sterm(x, wb);
            }
            double v2[2] = {va, vb};
            int sl = 0;
            const double tot = butterfly_sum<2>(v2, lane, &sl);
            if ((lane & 15) == 0 && (sl == 0 || two)) dst[sl ? sb2 : sa] = tot;
        }
    };

    // ---- prologue
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&s_tmem)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        if (lane == 0) {
            s_abort = 0;
            s_nord = 0;
            s_nstr = 0;
            for (int r = 0; r < RC; ++r) {
                mbar_init_g(&full[r], 1);
                mbar_init_g(&empty[r], NDW);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            bounds(a.t0);
            if (a.t0 + 1 < a.t1) bounds(a.t0 + 1);
            if (a.t0 + 2 < a.t1) bounds(a.t0 + 2);
        }
    }
    for (int s = tid; s < Sb; s += NTH) uid[s] = a.utab ? a.utab[(size_t)b * a.S + s] : b + s * G;
    for (int s = tid; s < kSlots; s += NTH) { hs[s] = 0.0f; iota[s] = s; }
    tc_before();
    __syncthreads();
    tc_after();
    if (data) {
        stage_list(a.t0);
        stage_list(a.t0 + 1);
        // rows into their tiers; fp64 norms of every row
        for (int s = 0; s < Sb; ++s) {
            const float4* row = W4 + (int64_t)uid[s] * d4 + dt;
            float4 w[KJ];
            double n0 = 0.0, n1 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                w[j] = (j < KJ - 1 || vlast) ? __ldcg(row + j * NDT) : make_float4(0.f, 0.f, 0.f, 0.f);
                const double e0 = w[j].x, e1 = w[j].y, e2 = w[j].z, e3 = w[j].w;
                n0 = fma(e0, e0, n0); n1 = fma(e1, e1, n1); n0 = fma(e2, e2, n0); n1 = fma(e3, e3, n1);
            }
            if (s < ntm) {
                tm_store<KJ>(tm_addr(s), w);
            } else if (s < non) {
                float4* sr = srows + (size_t)(s - ntm) * KJ * NDT + dt;
#pragma unroll
                for (int j = 0; j < KJ; ++j) sr[j * NDT] = w[j];
            }
            push(s, n0 + n1);
        }
        push_flush();
        twait_st();
        cp_async_wait_all();
        bar_data();
        build_bitmap(a.t0);
        mc = mask_of(a.t0);
        fill_cache(a.t0, mc);
        // speculative S(x_t0) of every unit (no update is pending; W is current)
        sparse_rows(a.t0, iota, Sb, sg[a.t0 & 1]);
    }
    tc_before();
    __syncthreads();
    tc_after();
    bool my_upd = false;     // control lane s: unit s is in the pending update
    if (warp == 0 && lane < Sb) {
        double tot = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < NDW; ++w8) tot += pn[lane][w8];
        wns[lane] = tot;
    }
    // ring positions: producer (control lane 0) and consumers (data threads)
    int pslot = 0, pu = 0, issued = 0;
    int cslot = 0, cu = 0;
    auto produce = [&](int c) {   // chunk c of the streamed rows of the pending update
        const int row = strm[c / KJ], j = c % KJ;
        if (pu > 0) mbar_wait_g(&empty[pslot], (uint32_t)((pu - 1) & 1));
        const int nf4 = min(NDT, d4 - j * NDT);
        bulk_row(ring + (size_t)pslot * NDT, W4 + (int64_t)uid[row] * d4 + (size_t)j * NDT, (uint32_t)nf4 * 16u,
                 &full[pslot]);
        if (++pslot == RC) { pslot = 0; ++pu; }
    };
    __syncthreads();

    double f_next = a.t1 > a.t0 ? a.f_tab[0] : 0.0;   // decay factor of the coming step, loaded a step ahead
    for (int64_t t = a.t0; t < a.t1; ++t) {
        // phase trace (som_set_trace): control lane 0 stamps [0] loop top,
        // [3] keys formed, [4] winner known; data thread 0 stamps [1] dense
        // pass done, [2] its sparse sums done, [5] bitmap + x cache of
        // x_{t+1} done, [6] speculative on-chip sums done, [7] phase 2' done
        unsigned long long* tr = nullptr;
        unsigned long long* tr1 = nullptr;
        if (a.trace && t - a.t0 < a.trace_steps) {
            unsigned long long* row = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
            if (tid == 0) tr = row;
            if (tid == 32) tr1 = row;
        }
        if (tr) tr[0] = trace_now(a.trace_clk);
        const double f = f_next;
        const double alpha = a.alpha0 * f;
        double sigma = a.sigma0 * f;
        if (sigma < a.sigma_min) sigma = a.sigma_min;
        const double two_s2 = 2.0 * sigma * sigma;
        const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
        // speculative sums run in 2' of this step unless the radius covers
        // the lattice (every unit then takes the next dense pass)
        const bool spec = !(r2 >= a.g2max);
        // ---- 1. dense pass over update(t-1)'s rows: Eq. 1 with x_{t-1}
        // (registers), |w'|^2 (TMEM rows written through to W); then S(x_t)
        // of those rows
        if (data) {
            const int nord = s_nord;
            if (nord > 0) build_xp(t - 1, mp);
            for (int i = 0; i < nord; ++i) {
                const int s = ord[i];
                const float h = hs[s];
                double n0 = 0.0, n1 = 0.0;
                float4* grow = W4 + (int64_t)uid[s] * d4 + dt;
                if (s < ntm) {
                    float4 w[KJ];
                    tm_load<KJ>(tm_addr(s), w);
#pragma unroll
                    for (int j = 0; j < KJ; ++j) {
                        w[j] = eq1u(h, w[j], xp[j]);
                        if (spec) {
                            if (j < KJ - 1 || vlast) __stcg(grow + j * NDT, w[j]);   // write-through
                        } else {
                            // only x_t's non-zeros: the gathers below read nothing else
                            const uint32_t bits = (mc >> (4 * j)) & 0xFu;
                            if (bits) {
                                float* g = reinterpret_cast<float*>(grow + j * NDT);
                                if (bits & 1u) __stcg(g, w[j].x);
                                if (bits & 2u) __stcg(g + 1, w[j].y);
                                if (bits & 4u) __stcg(g + 2, w[j].z);
                                if (bits & 8u) __stcg(g + 3, w[j].w);
                            }
                        }
                        const double e0 = w[j].x, e1 = w[j].y, e2 = w[j].z, e3 = w[j].w;
                        n0 = fma(e0, e0, n0); n1 = fma(e1, e1, n1); n0 = fma(e2, e2, n0); n1 = fma(e3, e3, n1);
                    }
                    tm_store<KJ>(tm_addr(s), w);
                } else if (s < non) {
                    float4* sr = srows + (size_t)(s - ntm) * KJ * NDT + dt;
#pragma unroll
                    for (int j = 0; j < KJ; ++j) {
                        const float4 w = eq1u(h, sr[j * NDT], xp[j]);
                        sr[j * NDT] = w;
                        const double e0 = w.x, e1 = w.y, e2 = w.z, e3 = w.w;
                        n0 = fma(e0, e0, n0); n1 = fma(e1, e1, n1); n0 = fma(e2, e2, n0); n1 = fma(e3, e3, n1);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < KJ; ++j) {
                        mbar_wait_g(&full[cslot], (uint32_t)(cu & 1));
                        const bool v = j < KJ - 1 || vlast;
                        float4 w = v ? ring[(size_t)cslot * NDT + dt] : make_float4(0.f, 0.f, 0.f, 0.f);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[cslot]);
                        if (++cslot == RC) { cslot = 0; ++cu; }
                        w = eq1u(h, w, xp[j]);
                        if (v) __stcg(grow + j * NDT, w);
                        const double e0 = w.x, e1 = w.y, e2 = w.z, e3 = w.w;
                        n0 = fma(e0, e0, n0); n1 = fma(e1, e1, n1); n0 = fma(e2, e2, n0); n1 = fma(e3, e3, n1);
                    }
                }
                push(s, n0 + n1);
            }
            push_flush();
            if (!spec && nord > 0 && ntm > 0) tm_stale = true;
            if (spec && tm_stale) {
                // TMEM rows were written through partially (full-coverage
                // steps): W catches up once before the speculative gathers
                twait_st();
                for (int s2 = 0; s2 < ntm && s2 < Sb; ++s2) {
                    float4 w[KJ];
                    tm_load<KJ>(tm_addr(s2), w);
                    float4* grow = W4 + (int64_t)uid[s2] * d4 + dt;
#pragma unroll
                    for (int j = 0; j < KJ; ++j)
                        if (j < KJ - 1 || vlast) __stcg(grow + j * NDT, w[j]);
                }
                tm_stale = false;
            }
            twait_st();
            if (tr1) tr1[1] = trace_now(a.trace_clk);
            if (nord > 0) {
                // rows written above: visible to the gathers below (generic)
                // and to the next ring fill (async proxy)
                asm volatile("fence.proxy.async.global;" ::: "memory");
                bar_data();
                sparse_rows(t, ord, nord, sgd);
            }
            if (tr1) tr1[2] = trace_now(a.trace_clk);
        } else {
            // ring producer (lane 0): the rest of this step's streamed chunks
            if (lane == 0) {
                const int total = s_nstr * KJ;
                for (int c = issued; c < total; ++c) produce(c);
            }
            issued = 0;
            pslot = __shfl_sync(0xffffffffu, pslot, 0);
            pu = __shfl_sync(0xffffffffu, pu, 0);
        }
        tc_before();
        __syncthreads();   // (A) pass done: partials complete, rows stored
        tc_after();

        if (t + 1 < a.t1) f_next = a.f_tab[t + 1 - a.t0];

        if (!data) {
            // ---- 2. control warp: keys, exchange, winner, lists of update(t)
            unsigned long long best = ~0ull;
            if (lane < Sb) {
                double tot;
                if (my_upd) {
                    double nn = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < NDW; ++w8) nn += pn[lane][w8];
                    wns[lane] = nn;
                    tot = nn + sgd[lane];
                } else {
                    tot = wns[lane] + sg[t & 1][lane];
                }
                tot = tot > 0.0 ? tot : 0.0;   // R25: the identity can round below 0
                best = make_key((float)tot, global_unit(a, uid[lane]));
            }
            best = warp_min_u64(best);
            if (tr) tr[3] = trace_now(a.trace_clk);
            xchg_publish(a, best, t, b, lane);
            // the data warps start 2' only now: beside the keys above it
            // slowed them down on the step's critical path
            asm volatile("bar.arrive 3, %0;" ::"n"(NTH) : "memory");
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (tr) tr[4] = trace_now(a.trace_clk);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            bool u2 = false;
            if (lane < Sb) {
                const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, uid[lane]), c);
                u2 = g2 <= r2;
                hs[lane] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
            my_upd = u2;
            const unsigned mu = __ballot_sync(0xffffffffu, u2);
            const unsigned lo_non = non >= 32 ? 0xffffffffu : ((1u << non) - 1u);
            const unsigned onm = mu & lo_non;
            const unsigned stm = mu & ~lo_non;
            const int ns = __popc(stm), no = __popc(onm), m = min(ns, no);
            const unsigned lt = (1u << lane) - 1u;
            // dense-pass order: streamed and on-chip rows alternate (the ring
            // refills while on-chip rows are processed)
            if ((stm >> lane) & 1u) {
                const int i = __popc(stm & lt);
                strm[i] = lane;
                ord[i < m ? 2 * i : m + i] = lane;
            }
            if ((onm >> lane) & 1u) {
                const int k = __popc(onm & lt);
                ord[k < m ? 2 * k + 1 : m + k] = lane;
            }
            __syncwarp();
            if (lane == 0) {
                s_nord = ns + no;
                s_nstr = ns;
            }
            // first chunks of the next pass into the ring, one per lane (none
            // after the last step: the flush reads streamed rows directly)
            if (!stop && t + 1 < a.t1) {
                const int first = min(RC, ns * KJ);
                if (lane < first) {
                    int slot = pslot + lane, u = pu;
                    if (slot >= RC) { slot -= RC; ++u; }
                    const int row = strm[lane / KJ], j = lane % KJ;
                    if (u > 0) mbar_wait_g(&empty[slot], (uint32_t)((u - 1) & 1));
                    const int nf4 = min(NDT, d4 - j * NDT);
                    bulk_row(ring + (size_t)slot * NDT, W4 + (int64_t)uid[row] * d4 + (size_t)j * NDT,
                             (uint32_t)nf4 * 16u, &full[slot]);
                }
                pslot += first;
                if (pslot >= RC) { pslot -= RC; ++pu; }
                issued = first;
            }
        } else {
            // ---- 2'. data warps: list of x_{t+2}, bounds of x_{t+3}, bitmap
            // of x_{t+1}, speculative S(x_{t+1}) of every unit (skipped when
            // the radius covers the whole lattice: every unit then takes the
            // dense pass), once the control warp has published
            asm volatile("bar.sync 3, %0;" ::"n"(NTH) : "memory");
            stage_list(t + 2);
            if (dt == 0 && t + 3 < a.t1) bounds(t + 3);
            uint32_t mn = 0u;
            if (t + 1 < a.t1) {
                build_bitmap(t + 1);
                mn = mask_of(t + 1);
                fill_cache(t + 1, mn);
                if (tr1) tr1[5] = trace_now(a.trace_clk);
                if (spec) sparse_rows(t + 1, iota, Sb, sg[(t + 1) & 1]);
                if (tr1) tr1[6] = trace_now(a.trace_clk);
            }
            cp_async_wait_all();
            mp = mc;
            mc = mn;
            if (tr1) tr1[7] = trace_now(a.trace_clk);
        }
        tc_before();
        __syncthreads();   // (B)
        tc_after();
        if (s_abort) break;
    }

    // flush the update of the last step (sample x_{t1-1}) into the rows'
    // storage, then write every on-chip row back to W
    if (data && a.t1 > a.t0 && !s_abort) {
        const int nord = s_nord;
        if (nord > 0) build_xp(a.t1 - 1, mp);
        for (int i = 0; i < nord; ++i) {
            const int s = ord[i];
            const float h = hs[s];
            if (s < ntm) {
                float4 w[KJ];
                tm_load<KJ>(tm_addr(s), w);
#pragma unroll
                for (int j = 0; j < KJ; ++j) w[j] = eq1u(h, w[j], xp[j]);
                tm_store<KJ>(tm_addr(s), w);
            } else if (s < non) {
                float4* sr = srows + (size_t)(s - ntm) * KJ * NDT + dt;
#pragma unroll
                for (int j = 0; j < KJ; ++j) sr[j * NDT] = eq1u(h, sr[j * NDT], xp[j]);
            } else {
                float4* grow = W4 + (int64_t)uid[s] * d4 + dt;
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (j < KJ - 1 || vlast) __stcg(grow + j * NDT, eq1u(h, __ldcg(grow + j * NDT), xp[j]));
            }
        }
        twait_st();
        for (int s = 0; s < non; ++s) {
            float4 w[KJ];
            if (s < ntm) {
                tm_load<KJ>(tm_addr(s), w);
            } else {
                const float4* sr = srows + (size_t)(s - ntm) * KJ * NDT + dt;
#pragma unroll
                for (int j = 0; j < KJ; ++j) w[j] = sr[j * NDT];
            }
            float4* grow = W4 + (int64_t)uid[s] * d4 + dt;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (j < KJ - 1 || vlast) __stcg(grow + j * NDT, w[j]);
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512) : "memory");
}

constexpr size_t tier_static(int ndw) { return (size_t)kSlots * ndw * 8 + 4 * kSlots * 8 + 5 * kSlots * 4 + 1024 + 512; }

size_t tier_smem_bytes(int /*S*/, int kj, int dimp, int cap, const TierPlan& p) {
    const size_t ndt = 32 * (size_t)p.ndw;
    return sizeof(float4) * ndt * ((size_t)p.rc + (size_t)p.nsm * kj) + 4 * 4 * ndt + 24 * (size_t)cap +
           8 * (size_t)((dimp >> 5) + 1) + 128;
}

template <int KJ, int NDW>
cudaError_t launch_tier_kj(const TrainArgs& a, const TierPlan& p, cudaStream_t st) {
    const size_t smem = tier_smem_bytes(a.S, KJ, a.dimp, a.nz_cap, p);
    auto fn = som_train_tier_kernel<KJ, NDW>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    TierPlan pp = p;
    void* params[] = {&args, &pp};
    return launch_persistent((const void*)fn, a, TierShape<NDW>::nth, smem, params, st);
}

int tier_kj(int dimp, int ndw) { return ((dimp / 4) + 32 * ndw - 1) / (32 * ndw); }

bool tier_plan(int S, int dimp, int maxnnz, int max_smem_optin, TierPlan* out) {
    if (dimp % 4 != 0 || S < 1 || S > kSlots) return false;
    TierPlan p{};
    p.ndw = 16;
    if (const char* e = std::getenv("SOM_TIER_NDW")) p.ndw = std::atoi(e) == 12 ? 12 : 16;
    // 16 warps spill above 5 chunks per thread; below 4 the row is short enough for 12
    if (tier_kj(dimp, p.ndw) > 5 || tier_kj(dimp, p.ndw) < 4) p.ndw = 12;
    const int kj = tier_kj(dimp, p.ndw);
    if (kj < 4 || kj > 8) return false;
    const int tm_cols = 512 / (p.ndw / 4);
    p.ntm = std::min(kTmMax, tm_cols / (4 * kj));
    p.ntm = std::max(0, std::min(p.ntm, S));
    const int cap = csr_nz_cap(maxnnz);
    const size_t budget = (size_t)max_smem_optin - tier_static(p.ndw);
    int rc_min = 8, rc_max = kRingMax;
    if (const char* e = std::getenv("SOM_TIER_RING")) rc_max = std::max(2, std::min(kRingMax, std::atoi(e))), rc_min = std::min(rc_min, rc_max);
    int smax = kSmMax;
    if (const char* e = std::getenv("SOM_TIER_NSM")) smax = std::max(0, std::min(kSmMax, std::atoi(e)));
    const int rest = S - p.ntm;
    p.nsm = std::max(0, std::min(smax, rest));
    p.rc = rest > p.nsm ? rc_min : 2;
    while (p.nsm > 0 && tier_smem_bytes(S, kj, dimp, cap, p) > budget) --p.nsm;
    if (S - p.ntm - p.nsm > 0) p.rc = rc_min;
    if (tier_smem_bytes(S, kj, dimp, cap, p) > budget) return false;
    while (p.rc < rc_max && S - p.ntm - p.nsm > 0) {
        TierPlan q = p;
        ++q.rc;
        if (tier_smem_bytes(S, kj, dimp, cap, q) > budget) break;
        p = q;
    }
    *out = p;
    return true;
}

}  // namespace

bool train_tier_supported(int S, int dim, int maxnnz, int max_smem_optin) {
    TierPlan p;
    return tier_plan(S, dim, maxnnz, max_smem_optin, &p);
}

cudaError_t launch_train_tier(const TrainArgs& a, int max_smem_optin, cudaStream_t st) {
    TierPlan p;
    if (!tier_plan(a.S, a.dimp, a.nz_cap, max_smem_optin, &p)) return cudaErrorInvalidConfiguration;
    if (p.ndw == 16) {
        switch (tier_kj(a.dimp, 16)) {
            case 4: return launch_tier_kj<4, 16>(a, p, st);
            case 5: return launch_tier_kj<5, 16>(a, p, st);
            default: return cudaErrorInvalidConfiguration;
        }
    }
    switch (tier_kj(a.dimp, 12)) {
        case 4: return launch_tier_kj<4, 12>(a, p, st);
        case 5: return launch_tier_kj<5, 12>(a, p, st);
        case 6: return launch_tier_kj<6, 12>(a, p, st);
        case 7: return launch_tier_kj<7, 12>(a, p, st);
        case 8: return launch_tier_kj<8, 12>(a, p, st);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace som
