// train_spec.cu — register-resident online-SOM training with the winner
// exchange of step t overlapped with the distance pass of step t+1.
//
// Same result as train_reg.cu (exact R10 distances, lowest-index argmin R9,
// Eq. 1 update R11; every BMU and weight identical), different schedule.
// In train_reg.cu the exchange of step t can only start once the pass over
// the registers (update t-1, distances t) is done, and the pass of t+1 only
// once the winner c_t is back: pass and exchange add up.  Here the pass of
// step t+1 runs while the exchange of step t is in flight, on weights that
// do not yet carry the update of step t, and the distance of t+1 is
// completed afterwards from per-unit sums.
//
// Per unit u, before c_{t-1} is known (w = W^{(t-1)}, a = x_t - w,
// dx = x_{t-1} - x_t, all in fp64 from fp32 inputs, exact):
//   A_u = sum a^2,  P_u = sum a dx            (one pass, registers)
//   Delta_t = sum dx^2,  X2_t = sum x_t^2     (per step, from the x ring)
// The update of step t-1 with coefficient s (= alpha h, Eq. 1) moves w to
// w' = w + s (x_{t-1} - w) + e, e the fp32 rounding of R11, so
//   D_t(u) = sum (x_t - w')^2 = Q - 2 sum (r a - s dx) e + sum e^2,
//   Q = r^2 A - 2 s r P + s^2 Delta,  r = 1 - s.
// With |e_k| <= 2^-24 (s |b_k| + |w'_k|) + 2^-150 and ||w'|| <= ||x_t|| +
// sqrt(Q), every D_t(u) lies in [Q - E_u, Q + E_u] (E_u below, including the
// fp64 rounding of the sums); units the update did not touch (s < 0) have
// D_t(u) = A_u exactly.  Each CTA publishes its smallest lower-bound key,
// the upper bound of that unit and its second-smallest lower bound; when the
// global winner's upper bound is below every other unit's lower bound (in
// RN32, so the fp32 comparison of R10 cannot flip), it is the exact BMU.
// Otherwise (rare near-ties) the step falls back to the exact pass on the
// updated registers and a second exchange.  DESIGN.md R32.
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;
constexpr int kSpecMaxG = 128;            // exchange slots held per lane <= 4
constexpr int kSpecPass = 32 * (NW - NW / 4);   // pass threads per CTA

__device__ __forceinline__ unsigned long long* spec_slot_a(const TrainArgs& a, uint32_t q) {
    return a.xchg + (size_t)(q & 1) * a.xstride;
}
__device__ __forceinline__ unsigned long long* spec_slot_b(const TrainArgs& a, uint32_t q) {
    return a.xchg + (size_t)(2 + (q & 1)) * a.xstride;
}

// Wait for exchange q; with_b: the B words carry (upper bound | 2nd lower
// bound).  Returns the global min A word; *hb_w, *m2_w: the winner CTA's B
// fields; *sec: the smallest A distance bits of the other CTAs.
__device__ __forceinline__ unsigned long long spec_wait(const TrainArgs& a, uint32_t q, int lane, bool with_b,
                                                        unsigned* hb_w, unsigned* m2_w, unsigned* sec, int* stop,
                                                        unsigned long long* tr = nullptr) {
    const unsigned long long tag = xchg_tag(q);
    const unsigned long long* sa = spec_slot_a(a, q);
    const unsigned long long* sb = spec_slot_b(a, q);
    unsigned long long va[kSpecMaxG / 32], vb[kSpecMaxG / 32];
    Spin spins;
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < kSpecMaxG / 32; ++k) {
            const int j = lane + 32 * k;
            va[k] = ~0ull;
            vb[k] = ~0ull;
            if (j < a.G) {
                va[k] = ld_relaxed_u64(sa + j);
                ok &= (va[k] & 0xFFull) == tag;
                if (with_b) {
                    vb[k] = ld_relaxed_u64(sb + j);
                    ok &= (vb[k] & 0xFFull) == tag;
                }
            }
        }
        if (__all_sync(0xffffffffu, ok)) break;
        if (spins.n == 0 && tr) tr[5] = trace_now(a.trace_clk);
        if (xchg_should_stop(a, spins, lane)) { *stop = 1; return 0; }
        if (a.poll_ns > 0) __nanosleep(a.poll_ns);
    }
    if (tr) { tr[6] = trace_now(a.trace_clk); tr[4] = spins.n; }
    unsigned long long m = ~0ull;
#pragma unroll
    for (int k = 0; k < kSpecMaxG / 32; ++k) m = umin64(m, va[k]);
    // warp min of the 64-bit words as two 32-bit reductions (high, then low among equals)
    const unsigned mh = __reduce_min_sync(0xffffffffu, (unsigned)(m >> 32));
    const unsigned ml = __reduce_min_sync(0xffffffffu, (unsigned)(m >> 32) == mh ? (unsigned)m : 0xFFFFFFFFu);
    const unsigned long long gmin = ((unsigned long long)mh << 32) | ml;
    if (with_b) {
        unsigned hb = 0, m2 = 0, s2 = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < kSpecMaxG / 32; ++k) {
            if (lane + 32 * k >= a.G) continue;
            if (va[k] == gmin) {
                hb = (unsigned)(vb[k] >> 32);
                m2 = (unsigned)vb[k] & ~0xFFu;
            } else {
                s2 = min(s2, (unsigned)(va[k] >> 32));
            }
        }
        *hb_w = __reduce_max_sync(0xffffffffu, hb);   // exactly one slot holds gmin
        *m2_w = __reduce_max_sync(0xffffffffu, m2);
        *sec = __reduce_min_sync(0xffffffffu, s2);
    }
    return gmin;
}

template <int SMAX, int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_spec_kernel(const TrainArgs a) {
    constexpr int NV = 2 * SMAX;             // per unit: A, P
    // pass threads: every warp except those of sub-partition 0 (warps 0, 4,
    // 8, 12), so that the control warp has its scheduler to itself
    constexpr int NPW = NW - NW / 4;
    constexpr int NP = 32 * NPW;
    static_assert(NP == kSpecPass, "pass thread count");
    __shared__ double part[2][NW][NV + 2];   // per-warp partials of the pass (+ Delta, ||x||^2), by step parity
    __shared__ double partx[NW][SMAX];       // per-warp partials of the exact (fallback) pass
    __shared__ float s_h[2][SMAX];           // h of this CTA's units for the update of step t (parity t)
    __shared__ double s_u[2][SMAX][3];       // per unit: A, P, sqrt(A) of the next step (parity of that step)
    __shared__ double s_x[2][3];             // Delta, sqrt(Delta), ||x|| of the next step
    __shared__ int s_fb[2], s_abort;
    extern __shared__ __align__(16) float xring[];   // [3][dimp] x ring

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pw = (warp & 3) ? warp - (warp >> 2) - 1 : -1;   // pass warp index (< 0: control / idle)
    const int pt = pw >= 0 ? pw * 32 + lane : -1;
    const int Sb = (a.N - b + G - 1) / G;
    const int d4 = a.dimp >> 2;
    const float4* W4 = reinterpret_cast<const float4*>(a.W);
    float4* ring4 = reinterpret_cast<float4*>(xring);

    // pass threads own float4 chunks pt + j * NP of every unit of the CTA
    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = pt >= 0 && pt + j * NP < d4;

    float4 w[SMAX][KJ];
    float4 xm[KJ], xc[KJ], xn[KJ];          // x_{t-1}, x_t, x_{t+1} (own chunks, fp32)
    float hh[SMAX];                          // pending update of each unit (s, or < 0: none)
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s < Sb && valid[j]) v = W4[(int64_t)(b + s * G) * d4 + pt + j * NP];
            w[s][j] = v;
        }
        hh[s] = -1.0f;
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j) xm[j] = xc[j] = xn[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) { s_abort = 0; s_fb[0] = s_fb[1] = 0; }

    auto issue_x = [&](int64_t t) {
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + train_row(a, t) * (int64_t)a.dim);
            float4* dst = ring4 + (size_t)(t % 3) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) cp_async16(dst + pt + j * NP, src + pt + j * NP);
        }
        cp_async_commit();
    };
    auto load_x = [&](int64_t t) {           // own chunks of ring slot t % 3
        const float4* src = ring4 + (size_t)(t % 3) * d4;
#pragma unroll
        for (int j = 0; j < KJ; ++j)
            if (valid[j]) xn[j] = src[pt + j * NP];
    };
    // pass (warps 1..15): pending update (s = hh) on the registers, then
    // A_u = sum (x_{t+1} - w)^2, P_u = sum (x_{t+1} - w)(x_t - x_{t+1}),
    // Delta = sum (x_t - x_{t+1})^2, X2 = sum x_{t+1}^2
    auto spec_pass = [&](int par) {
        double v[NV], xv[2] = {0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = 0.0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            if (!valid[j]) continue;
            const double n0 = xn[j].x, n1 = xn[j].y, n2 = xn[j].z, n3 = xn[j].w;
            const double d0 = (double)xc[j].x - n0, d1 = (double)xc[j].y - n1;
            const double d2 = (double)xc[j].z - n2, d3 = (double)xc[j].w - n3;
            xv[0] = fma(d0, d0, fma(d1, d1, fma(d2, d2, fma(d3, d3, xv[0]))));
            xv[1] = fma(n0, n0, fma(n1, n1, fma(n2, n2, fma(n3, n3, xv[1]))));
#pragma unroll
            for (int s = 0; s < SMAX; ++s) {
                if (s >= Sb) continue;
                if (hh[s] >= 0.0f) w[s][j] = eq1u(hh[s], w[s][j], xm[j]);
                const double w0 = w[s][j].x, w1 = w[s][j].y, w2 = w[s][j].z, w3 = w[s][j].w;
                const double a0 = n0 - w0, a1 = n1 - w1;
                const double a2 = n2 - w2, a3 = n3 - w3;
                v[s] = fma(a0, a0, fma(a1, a1, fma(a2, a2, fma(a3, a3, v[s]))));
                v[SMAX + s] = fma(a0, d0, fma(a1, d1, fma(a2, d2, fma(a3, d3, v[SMAX + s]))));
            }
        }
        int slot;
        const double r = butterfly_sum<NV>(v, lane, &slot);
        if ((lane & (32 / NV - 1)) == 0) part[par][pw][slot] = r;
        const double rx = butterfly_sum<2>(xv, lane, &slot);
        if ((lane & 15) == 0) part[par][pw][NV + slot] = rx;
    };
    // control warp, lane l: sums of unit l & (SMAX-1): uA = A, uP = P,
    // usA = sqrt(A); the step's Delta, sqrt(Delta), ||x|| (sqrt bounds
    // inflated by 1e-12)
    const int su = lane & (SMAX - 1);
    const int uid = global_unit(a, b + su * G);
    const int iu = uid / a.cols, ju = uid - iu * a.cols;
    // warp 1, after the pass warps' named barrier: CTA totals of the pass
    // partials, per unit and per step, into s_u / s_x; then signals warp 0
    // (barrier 2: warp 1 arrives, warp 0 waits)
    auto totals_w1 = [&](int par, bool signal) {
        asm volatile("bar.sync 1, %0;" ::"n"(NP) : "memory");
        if (warp == 1) {
            double tot = 0.0;
            if (lane < NV + 2) {
#pragma unroll
                for (int w8 = 0; w8 < NPW; ++w8) tot += part[par][w8][lane];
            }
            const double A = __shfl_sync(0xffffffffu, tot, su);
            const double P = __shfl_sync(0xffffffffu, tot, SMAX + su);
            const double Dx = __shfl_sync(0xffffffffu, tot, NV);
            const double X2 = __shfl_sync(0xffffffffu, tot, NV + 1);
            if (lane < SMAX) {
                s_u[par][lane][0] = A;
                s_u[par][lane][1] = P;
                s_u[par][lane][2] = sqrt(A) * (1.0 + 1e-12);
            }
            if (lane == 0) {
                s_x[par][0] = Dx;
                s_x[par][1] = sqrt(Dx) * (1.0 + 1e-12);
                s_x[par][2] = sqrt(X2) * (1.0 + 1e-12);
            }
            if (signal) asm volatile("bar.arrive 2, 64;" ::: "memory");
        }
    };
    float hs = -1.0f;                        // control warp lane s < SMAX: h of unit s, pending
    // control warp: schedule of step t (R1-R3, R5), read before the wait so
    // that only the exp remains between the winner and the barrier
    double alpha_t = 0.0, two_s2_t = 1.0, r2_t = 0.0;
    auto sched = [&](int64_t t) {
        const double f = a.f_tab[t - a.t0];
        alpha_t = a.alpha0 * f;
        double sigma = a.sigma0 * f;
        if (sigma < a.sigma_min) sigma = a.sigma_min;
        two_s2_t = 2.0 * sigma * sigma;
        r2_t = a.cutoff_on ? two_s2_t * a.ln_inv_eps : INFINITY;
    };
    // control warp: h of this CTA's units for winner c at step t (R4, R5)
    auto unit_h = [&](int c, int64_t t) {
        if (lane < SMAX) {
            float h = -1.0f;
            if (lane < Sb) {
                const int ic = c / a.cols, jc = c - ic * a.cols;
                const double di = (double)abs(iu - ic);
                double g2;
                if (a.topo == 0) {
                    const double dj = (double)abs(ju - jc);
                    g2 = di * di + dj * dj;
                } else {
                    const double dx = (double)abs(2 * (ju - jc) + ((iu & 1) - (ic & 1)));
                    g2 = 0.25 * (dx * dx) + 0.75 * (di * di);
                }
                if (g2 <= r2_t) h = (float)(alpha_t * exp(-g2 / two_s2_t));
            }
            s_h[t & 1][lane] = h;
            hs = h;
        }
    };

    issue_x(a.t0);
    issue_x(a.t0 + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    if (pt >= 0) {
        load_x(a.t0);                        // xn = x_{t0}; no pending update: A_u = D_{t0}(u)
        spec_pass(a.t0 & 1);
        totals_w1(a.t0 & 1, a.t1 > a.t0);
    }
    uint32_t q = 0;                          // exchange sequence number (same in every CTA)

    for (int64_t t = a.t0; t < a.t1; ++t) {
        const int par = (int)(t & 1);
        unsigned long long* tr = nullptr;    // optional phase trace (som_set_trace)
        if (a.trace && (threadIdx.x == 0 || threadIdx.x == 32) && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
#define TRACE(p) do { if (tr) tr[p] = trace_now(a.trace_clk); } while (0)
        if (warp == 0) {
            TRACE(0);
            // ---- bounds of D_t from the sums, keys, publish exchange q
            asm volatile("bar.sync 2, 64;" ::: "memory");   // sums of step t (warp 1)
            const double uA = s_u[par][su][0], uP = s_u[par][su][1], usA = s_u[par][su][2];
            const double wDx = s_x[par][0], wSdx = s_x[par][1], wSx = s_x[par][2];
            const float hcur = __shfl_sync(0xffffffffu, hs, su);
            double L = uA, U = uA;
            if (hcur >= 0.0f) {
                const double s = hcur, r = 1.0 - s;
                const double Q = r * r * uA - 2.0 * s * r * uP + s * s * wDx;
                // fp64 rounding of the sums (depth <= 4 KJ + 21 terms) and of Q,
                // plus that of the exact pass the result must agree with
                const double Ef = 6e-14 * (r * r * uA + s * r * (uA + wDx) + s * s * wDx);
                // sqrt(Q) <= r ||a|| + s ||dx||;  ||x_{t-1} - w|| <= ||a|| + ||dx||
                const double sq = (r * usA + s * wSdx) * (1.0 + 1e-12);
                // ||e|| <= 2^-24 (s ||x_{t-1} - w|| + ||x_t|| + sqrt(Q)) + 2^-150 sqrt(d)
                const double R = 6e-8 * (s * (usA + wSdx) + wSx + sq) + 1e-37;
                const double E = 1.001 * (2.0 * sq * R + R * R) + Ef;
                L = fmax(Q - E, 0.0);
                U = Q + E;
            }
            const bool mine = lane < SMAX && lane < Sb;
            // CTA: smallest lower-bound key (D bits, then unit), its upper
            // bound, and the second-smallest lower bound (D bits)
            const unsigned lb = mine ? __float_as_uint((float)L) : 0xFFFFFFFFu;
            const unsigned ub = mine ? __float_as_uint((float)U) : 0xFFFFFFFFu;
            const unsigned md = __reduce_min_sync(0xffffffffu, lb);
            const unsigned mu = __reduce_min_sync(0xffffffffu, lb == md ? (unsigned)uid : 0xFFFFFFFFu);
            const bool win = lb == md && (unsigned)uid == mu;
            const unsigned h1 = __reduce_min_sync(0xffffffffu, win ? ub : 0xFFFFFFFFu);
            const unsigned m2 = __reduce_min_sync(0xffffffffu, win ? 0xFFFFFFFFu : lb);
            if (lane == 0) {
                const unsigned long long m1 = ((unsigned long long)md << 32) | ((unsigned long long)mu << 8);
                st_relaxed_u64(spec_slot_b(a, q) + b,
                               ((unsigned long long)h1 << 32) | (unsigned long long)(m2 & ~0xFFu) | xchg_tag(q));
                st_relaxed_u64(spec_slot_a(a, q) + b, m1 | xchg_tag(q));
            }
            TRACE(1);
            sched(t);
            // ---- wait for the winner (the pass runs meanwhile on warps 1..15)
            int stop = 0;
            unsigned hbw = 0, m2w = 0, sec = 0;
            const unsigned long long gmin = spec_wait(a, q, lane, true, &hbw, &m2w, &sec, &stop, tr);
            ++q;
            const bool safe = hbw < min(sec, m2w);
            if (safe && !stop) {
                const int c = key_unit(gmin);
                unit_h(c, t);
                if (lane == 0 && b == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            }
            if (lane == 0) {
                s_fb[par] = safe ? 0 : 1;
                if (stop) s_abort = 1;
            }
            TRACE(2);
        } else if (pt >= 0) {
            // ---- pass: update t-1, sums of step t+1 (overlaps the exchange)
#pragma unroll
            for (int j = 0; j < KJ; ++j) { xm[j] = xc[j]; xc[j] = xn[j]; }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            if (t + 1 < a.t1) load_x(t + 1);
            issue_x(t + 2);
            spec_pass((t + 1) & 1);
            TRACE(3);
            totals_w1((t + 1) & 1, t + 1 < a.t1);
        }
        __syncthreads();   // A: winner (or fallback flag), h, partials of step t+1
        if (s_abort) break;
        if (s_fb[par]) {
            // near-tie: exact distances of step t on the updated registers
            if (pt >= 0) {
                double v[SMAX];
#pragma unroll
                for (int s = 0; s < SMAX; ++s) v[s] = 0.0;
#pragma unroll
                for (int j = 0; j < KJ; ++j) {
                    if (!valid[j]) continue;
                    const double c0 = xc[j].x, c1 = xc[j].y, c2 = xc[j].z, c3 = xc[j].w;
#pragma unroll
                    for (int s = 0; s < SMAX; ++s) {
                        if (s >= Sb) continue;
                        const double e0 = c0 - (double)w[s][j].x, e1 = c1 - (double)w[s][j].y;
                        const double e2 = c2 - (double)w[s][j].z, e3 = c3 - (double)w[s][j].w;
                        v[s] = fma(e0, e0, fma(e1, e1, fma(e2, e2, fma(e3, e3, v[s]))));
                    }
                }
                int slot;
                const double r = butterfly_sum<SMAX>(v, lane, &slot);
                if ((lane & (32 / SMAX - 1)) == 0) partx[pw][slot] = r;
            }
            __syncthreads();
            if (warp == 0) {
                unsigned long long key = ~0ull;
                if (lane < SMAX && lane < Sb) {
                    double d = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < NPW; ++w8) d += partx[w8][lane];
                    key = make_key((float)d, uid);
                }
                key = warp_min_u64(key);
                if (lane == 0) st_relaxed_u64(spec_slot_a(a, q) + b, (key & ~0xFFull) | xchg_tag(q));
                int stop = 0;
                unsigned hbw, m2w, sec;
                const unsigned long long gmin = spec_wait(a, q, lane, false, &hbw, &m2w, &sec, &stop);
                ++q;
                const int c = key_unit(gmin);
                if (!stop) unit_h(c, t);
                if (lane == 0) {
                    if (b == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
                    if (b == 0 && a.spec_fallbacks) atomicAdd(a.spec_fallbacks, 1ull);
                    if (stop) s_abort = 1;
                }
            }
            __syncthreads();
            if (s_abort) break;
        }
#pragma unroll
        for (int s = 0; s < SMAX; ++s) hh[s] = s_h[par][s];
#undef TRACE
    }

    if (a.t1 > a.t0 && !s_abort && pt >= 0) {
        // flush the update of the last step (x_{t1-1} is in xc)
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            if (s < Sb && hh[s] >= 0.0f) {
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (valid[j]) w[s][j] = eq1u(hh[s], w[s][j], xc[j]);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (!s_abort) {
        float4* Wo = reinterpret_cast<float4*>(a.W);
#pragma unroll
        for (int s = 0; s < SMAX; ++s)
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (s < Sb && valid[j]) Wo[(int64_t)(b + s * G) * d4 + pt + j * NP] = w[s][j];
    }
}

template <int SMAX, int KJ>
cudaError_t launch_one(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * 3 * (size_t)a.dimp;
    cudaError_t e = cudaFuncSetAttribute(som_train_spec_kernel<SMAX, KJ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)som_train_spec_kernel<SMAX, KJ>, a, NT, smem, params, st);
}

int smax_of(int S) { return S <= 1 ? 1 : S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : 99; }

}  // namespace

// Same register budget as train_reg.cu; one GPU (the neuron-sharded
// exchange stays in train_reg.cu), G <= 128.
bool train_spec_supported(int S, int dim, int G, int world) {
    if (world != 1 || G > kSpecMaxG || dim % 4 != 0) return false;
    const int kj = ((dim / 4) + kSpecPass - 1) / kSpecPass;
    const int sm = smax_of(S);
    return kj <= 4 && sm <= 8 && sm * kj <= (kj == 4 ? 4 : 8);
}

cudaError_t launch_train_spec(const TrainArgs& a, cudaStream_t st) {
    const int kj = ((a.dimp / 4) + kSpecPass - 1) / kSpecPass;
    const int sm = smax_of(a.S);
#define TRY(SM, K) if (sm == SM && kj == K) return launch_one<SM, K>(a, st)
    TRY(1, 1); TRY(2, 1); TRY(4, 1); TRY(8, 1);
    TRY(1, 2); TRY(2, 2); TRY(4, 2);
    TRY(1, 3); TRY(2, 3);
    TRY(1, 4);
#undef TRY
    return cudaErrorInvalidConfiguration;
}

}  // namespace som
