// train_small.cu — persistent online-SOM training for short prototypes and
// large maps (d <= 128, d % 4 == 0), the shape of the paper's map-size
// study (Table 3: weight length 64, maps 16x16 ... 512x512).
//
// The step is the one of train.cu / train_reg.cu (pending Eq. 1 update of
// step t-1 fused with the fp64 distance pass of step t, packed (D, u) keys,
// tagged all-gather of per-CTA minima, R9-R11).  What changes is
// the work split: a prototype of d <= 128 floats is only d/4 <= 32 float4
// chunks, so instead of spreading one unit over the whole CTA, a group of
// L lanes (L = d/16 rounded up to a power of two: 4 for d = 64) owns one
// unit, lane `sub` holding the 4 chunks sub + c*L; a warp handles 32/L
// units per round and the D_u partials are combined with log2(L) in-group
// shuffles, no shared memory and no barrier per unit.  CTA b owns units
// l = b + s*G (cyclic), slot s = r*(16*32/L) + warp*(32/L) + group in round
// r.  The step is issue-bound (ncu: ~45-60 % issue active), so per-unit
// overheads are amortised over 16 elements per lane and the neighbourhood
// of each unit is computed once per step by one lane and passed to its
// group with a shuffle.  x_t is kept in shared memory in fp64 (converted
// once per step during the exchange), x_{t-1} as the fp32 ring slot.
//
// W placement: registers (up to 4 rounds of 16 floats per lane) when the
// CTA's share fits, else streamed from global memory every step (the 67 MB
// of a 512x512x64 map stays in the 126 MB L2).
//
// Neighbourhood (R4, R5, R26): per step the kernel needs h for up to N =
// 262,144 units; one fp64 exp per unit and step would dominate.  g2 splits
// into a row part a(di) and a column part b(dx) (rect: di^2 + dj^2; hex:
// 3/4 di^2 + 1/4 dx2^2, both exact), so while warp 0 waits on the exchange
// warps 1-15 tabulate Er[di] = exp(-a/2sigma^2) and Ec[dx] = exp(-b/2sigma^2)
// (rows + 2 cols values) and each unit takes h = RN32(alpha * (Er * Ec)).
// This equals the oracle's RN32(alpha * exp(-g2/2sigma^2)) in real
// arithmetic; the fp64 values differ by a few ulp (R26).  The
// cutoff test g2 <= r2 uses the exact g2.
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;
constexpr int kSC = 4;    // float4 chunks per lane of the default layout: L lanes cover 16 L floats

__device__ __forceinline__ float4 eq1s(float h, float4 w, float4 x) {
    // Eq. 1 per element: w + h (x - w) as fmaf(h, RN(x - w), w)  (R11)
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

struct Sched {
    double alpha, two_s2, r2;
};

__device__ __forceinline__ Sched sched_at(const TrainArgs& a, int64_t t) {
    const double f = a.f_tab[t - a.t0];
    Sched s;
    s.alpha = a.alpha0 * f;
    double sigma = a.sigma0 * f;
    if (sigma < a.sigma_min) sigma = a.sigma_min;
    s.two_s2 = 2.0 * sigma * sigma;
    s.r2 = a.cutoff_on ? s.two_s2 * a.ln_inv_eps : INFINITY;
    return s;
}

// h of the unit at lattice (iu, ju) for winner (ic, jc), or -1 outside the cutoff
__device__ __forceinline__ float h_of(const TrainArgs& a, int iu, int ju, int ic, int jc, const Sched& sc,
                                      const double* er, const double* ec) {
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
    if (!(g2 <= sc.r2)) return -1.0f;
    return (float)(sc.alpha * (er[di] * ec[dx]));
}

// SC float4 chunks per lane (kSC by default; 2 or 1 spread a CTA's units
// over more lanes when they all fit one round: shorter per-lane chains)
template <int L, int SC, int R, bool GLB>
__global__ void __launch_bounds__(NT, 1) som_train_small_kernel(const TrainArgs a) {
    constexpr int GPW = 32 / L;            // units per warp per round
    constexpr int UPR = NW * GPW;          // units per CTA per round
    __shared__ unsigned long long wmin[NW];
    __shared__ int s_c, s_abort;
    // [3][dimp] fp32 x ring | x_t in fp64 [dimp] | Er[rows] | Ec[W2] (fp64)
    extern __shared__ __align__(16) float xring[];

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / L, sub = lane % L;
    const int Sb = (a.N - b + G - 1) / G;
    const int rounds = GLB ? (Sb + UPR - 1) / UPR : R;
    const int d4 = a.dimp >> 2;
    const float4* ring4 = reinterpret_cast<const float4*>(xring);
    double* x64 = reinterpret_cast<double*>(xring + 3 * (size_t)a.dimp);
    const double2* x64v = reinterpret_cast<const double2*>(x64);
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    double* er = x64 + a.dimp;
    double* ec = er + a.rows;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    bool cv[SC];
#pragma unroll
    for (int c = 0; c < SC; ++c) cv[c] = sub + c * L < d4;

    // register-resident prototypes: round r, chunk c = float4 (sub + c*L) of unit slot r*UPR + warp*GPW + grp
    float4 w[GLB ? 1 : R][SC];
    if (!GLB) {
#pragma unroll
        for (int r = 0; r < (GLB ? 1 : R); ++r) {
            const int s = r * UPR + warp * GPW + grp;
#pragma unroll
            for (int c = 0; c < SC; ++c) {
                w[r][c] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (s < Sb && cv[c]) w[r][c] = W4[(int64_t)(b + s * G) * d4 + sub + c * L];
            }
        }
    }
    if (threadIdx.x == 0) s_abort = 0;

    // x ring: threads 0..d4-1 stage whole rows with cp.async one step ahead
    auto issue_x = [&](int64_t t) {
        if (threadIdx.x < d4 && t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + train_row(a, t) * (int64_t)a.dim);
            cp_async16((void*)(ring4 + (size_t)(t % 3) * d4 + threadIdx.x), src + threadIdx.x);
            cp_async_commit();
        }
    };
    auto land_x = [&]() {
        if (threadIdx.x < d4) asm volatile("cp.async.wait_group 0;" ::: "memory");
    };
    // x_t (landed, after a barrier) -> fp64 copy, threads lo.. of the CTA
    auto convert_x = [&](int64_t t, int lo) {
        const float* src = xring + (size_t)(t % 3) * a.dimp;
        for (int k = threadIdx.x - lo; k < a.dimp; k += NT - lo) x64[k] = (double)src[k];
    };

    if (a.t1 > a.t0) {
        issue_x(a.t0);
        land_x();
        __syncthreads();
        convert_x(a.t0, 0);
        issue_x(a.t0 + 1);
    }
    __syncthreads();

    bool pending = false;     // update of step t-1 not yet applied
    int icp = 0, jcp = 0;     // its winner
    Sched scp{0.0, 1.0, -1.0};

    // h of this lane's unit in a batch of L rounds starting at r0: lane k
    // serves round r0 + k / GPW, group k % GPW (one neighbourhood per unit)
    auto batch_h = [&](int r0) -> float {
        const int rr = r0 + lane / GPW;
        const int s = rr * UPR + warp * GPW + (lane % GPW);
        if (rr >= rounds || s >= Sb) return -1.0f;
        const int u = global_unit(a, b + s * G);
        const int iu = u / a.cols;
        return h_of(a, iu, u - iu * a.cols, icp, jcp, scp, er, ec);
    };

    for (int64_t t = a.t0; t < a.t1; ++t) {
        // optional phase trace (som_set_trace): thread 0 records loop top,
        // fused pass done, barrier A, key published, winner known, barrier B;
        // thread 32 records the end of the table build (phase 5)
        unsigned long long* tr = nullptr;
        if (a.trace && (threadIdx.x == 0 || threadIdx.x == 32) && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
#define TRACE(p) do { if (tr) tr[p] = trace_now(a.trace_clk); } while (0)
        if (threadIdx.x == 0) TRACE(0);
        const float4* xp4 = ring4 + (size_t)((t + 2) % 3) * d4;   // x_{t-1}
        // ---- fused pass: pending update (t-1), then D_u(x_t), per-lane min key
        unsigned long long kmin = ~0ull;
        float hb = -1.0f;
#pragma unroll(GLB ? 2 : R)
        for (int r = 0; r < rounds; ++r) {
            const int s = r * UPR + warp * GPW + grp;
            const bool valid = s < Sb;
            const int l = b + s * G;
            if (pending && (r % L) == 0) hb = batch_h(r);
            const float h = __shfl_sync(0xffffffffu, hb, (r % L) * GPW + grp);
            float4 wv[SC];
#pragma unroll
            for (int c = 0; c < SC; ++c) {
                if (GLB) wv[c] = (valid && cv[c]) ? __ldcg(W4 + (int64_t)l * d4 + sub + c * L)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                else wv[c] = w[r][c];
            }
            if (pending && valid && h >= 0.0f) {
#pragma unroll
                for (int c = 0; c < SC; ++c) {
                    if (cv[c]) {
                        wv[c] = eq1s(h, wv[c], xp4[sub + c * L]);
                        if (GLB) __stcg(W4 + (int64_t)l * d4 + sub + c * L, wv[c]);
                    }
                }
            }
            // R10: (double)x - (double)w, squared and summed in fp64
            double p0 = 0.0, p1 = 0.0;
#pragma unroll
            for (int c = 0; c < SC; ++c) {
                if (!GLB) w[r][c] = wv[c];
                if (cv[c]) {
                    const double2 xa = x64v[2 * (sub + c * L)], xb = x64v[2 * (sub + c * L) + 1];
                    const double e0 = xa.x - (double)wv[c].x, e1 = xa.y - (double)wv[c].y;
                    const double e2 = xb.x - (double)wv[c].z, e3 = xb.y - (double)wv[c].w;
                    p0 = fma(e0, e0, p0);
                    p1 = fma(e1, e1, p1);
                    p0 = fma(e2, e2, p0);
                    p1 = fma(e3, e3, p1);
                }
            }
            double p = p0 + p1;
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (valid) kmin = umin64(kmin, make_key((float)p, global_unit(a, l)));
        }
        kmin = warp_min_u64(kmin);
        if (lane == 0) wmin[warp] = kmin;
        if (threadIdx.x == 0) TRACE(1);
        land_x();          // x_{t+1} (issued a step ago) has landed
        __syncthreads();   // A: per-warp minima ready, x_{t+1} visible, x_t / x_{t-1} reads done
        if (threadIdx.x == 0) TRACE(2);

        const Sched sc = sched_at(a, t);
        issue_x(t + 2);    // into the slot of x_{t-1}
        if (warp == 0) {
            unsigned long long key = lane < NW ? wmin[lane] : ~0ull;
            key = warp_min_u64(key);
            xchg_publish(a, key, t, b, lane);
            if (threadIdx.x == 0) TRACE(3);
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (threadIdx.x == 0) TRACE(4);
            if (lane == 0) {
                const int c = key_unit(gmin);
                s_c = c;
                if (stop) s_abort = 1;
                if (b == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            }
        } else {
            if (t + 1 < a.t1) convert_x(t + 1, 32);
            // separable neighbourhood tables of step t (R26), built during the exchange
            for (int e = threadIdx.x - 32; e < a.rows + W2; e += NT - 32) {
                if (e < a.rows) {
                    const double di = (double)e;
                    const double part = a.topo == 0 ? di * di : 0.75 * (di * di);
                    er[e] = exp(-part / sc.two_s2);
                } else {
                    const double dx = (double)(e - a.rows);
                    const double part = a.topo == 0 ? dx * dx : 0.25 * (dx * dx);
                    ec[e - a.rows] = exp(-part / sc.two_s2);
                }
            }
            if (threadIdx.x == 32) TRACE(5);
        }
        __syncthreads();   // B: winner, tables and x_{t+1} in fp64 ready
        if (threadIdx.x == 0) { TRACE(6); TRACE(7); }
#undef TRACE
        if (s_abort) break;
        const int c = s_c;
        icp = c / a.cols;
        jcp = c - icp * a.cols;
        scp = sc;
        pending = true;
    }

    // flush the update of the last step (x_{t1-1} is ring slot (t1-1) % 3)
    if (a.t1 > a.t0 && !s_abort) {
        const float4* xl4 = ring4 + (size_t)((a.t1 - 1) % 3) * d4;
        float hb = -1.0f;
        for (int r = 0; r < rounds; ++r) {
            const int s = r * UPR + warp * GPW + grp;
            if ((r % L) == 0) hb = batch_h(r);
            const float h = __shfl_sync(0xffffffffu, hb, (r % L) * GPW + grp);
            if (s >= Sb || h < 0.0f) continue;
            const int l = b + s * G;
#pragma unroll
            for (int c = 0; c < SC; ++c) {
                if (!cv[c]) continue;
                if (GLB) {
                    float4* p = W4 + (int64_t)l * d4 + sub + c * L;
                    __stcg(p, eq1s(h, __ldcg(p), xl4[sub + c * L]));
                } else {
#pragma unroll
                    for (int rr = 0; rr < (GLB ? 1 : R); ++rr)
                        if (rr == r) w[rr][c] = eq1s(h, w[rr][c], xl4[sub + c * L]);
                }
            }
        }
    }
    land_x();
    if (!GLB && !s_abort) {
#pragma unroll
        for (int r = 0; r < (GLB ? 1 : R); ++r) {
            const int s = r * UPR + warp * GPW + grp;
#pragma unroll
            for (int c = 0; c < SC; ++c)
                if (s < Sb && cv[c]) W4[(int64_t)(b + s * G) * d4 + sub + c * L] = w[r][c];
        }
    }
}

size_t small_smem_bytes(const TrainArgs& a) {
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    return sizeof(float) * 3 * (size_t)a.dimp + sizeof(double) * ((size_t)a.dimp + a.rows + W2);
}

template <int L, int SC, int R, bool GLB>
cudaError_t launch_small_one(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = small_smem_bytes(a);
    cudaError_t e = cudaFuncSetAttribute(som_train_small_kernel<L, SC, R, GLB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)som_train_small_kernel<L, SC, R, GLB>, a, NT, smem, params, st);
}

template <int L>
cudaError_t launch_small_L(const TrainArgs& a, int rounds, cudaStream_t st) {
    if (rounds <= 1) {
        // one round: widen the lane groups while the CTA's units still fit it
        const int S = a.S;
        if (L * 4 <= 32 && S <= kTrainWarps * (32 / (L * 4))) return launch_small_one<(L * 4 <= 32 ? L * 4 : 32), 1, 1, false>(a, st);
        if (L * 2 <= 32 && S <= kTrainWarps * (32 / (L * 2))) return launch_small_one<(L * 2 <= 32 ? L * 2 : 32), 2, 1, false>(a, st);
        return launch_small_one<L, kSC, 1, false>(a, st);
    }
    if (rounds <= 2) return launch_small_one<L, kSC, 2, false>(a, st);
    if (rounds <= 4) return launch_small_one<L, kSC, 4, false>(a, st);
    return launch_small_one<L, kSC, 1, true>(a, st);
}

}  // namespace

// lanes per unit of the default layout: kSC float4 chunks per lane, L a power of two
int small_lanes(int dim) {
    const int d4 = (dim + 3) / 4;
    int L = 1;
    while (L * kSC < d4) L <<= 1;
    return L;
}

bool train_small_supported(int dim) { return dim % 4 == 0 && dim <= 128; }

// rounds of 16*32/L units per CTA for S units (> 4: the streamed variant)
int small_rounds(int S, int dim) {
    const int upr = kTrainWarps * (32 / small_lanes(dim));
    return (S + upr - 1) / upr;
}

cudaError_t launch_train_small(const TrainArgs& a, cudaStream_t st) {
    const int L = small_lanes(a.dim);
    const int rounds = small_rounds(a.S, a.dim);
    switch (L) {
        case 1: return launch_small_L<1>(a, rounds, st);
        case 2: return launch_small_L<2>(a, rounds, st);
        case 4: return launch_small_L<4>(a, rounds, st);
        case 8: return launch_small_L<8>(a, rounds, st);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace som
