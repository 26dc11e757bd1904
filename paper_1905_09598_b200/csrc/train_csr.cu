// train_csr.cu — online SOM training on CSR (sparse TF-IDF) input with a
// sparse distance path (the data are sparse TF-IDF
// vectors, and the paper's future work names hashed TF-IDF,
// P:321).  Same step, exchange and arithmetic contract as train_glb.cu
// (pending Eq. 1 update of t-1 fused with the distance of t, packed keys,
// tagged all-gather, R9-R11), for maps that stream from global
// memory (c3/c4).  What changes:
//  * x_t arrives as a CSR row: its (col, val) list is staged into shared
//    memory with cp.async two steps ahead and scattered into a dense fp32
//    buffer (the update still needs every x_k; x_k = 0 off the pattern);
//  * units that the pending update touches (inside the cutoff radius of the
//    previous winner, R5) take the dense pass: update, fp64 distance and
//    the fp64 squared norm |w_u|^2 of the new row, all from one read;
//  * every other unit skips its dense row: D_u = |w_u|^2 +
//    sum_{k in nz(x_t)} ((x_k - w_uk)^2 - w_uk^2)   (R25) — the same real
//    number as the definition, summed in fp64 and rounded once to fp32, so
//    the BMU sequence is that of the dense oracle (R10's argument), while the
//    bytes read fall from 4 d to ~32 nnz(x_t) per unit (one sector a term).
// Units are dealt cyclically (u = b + s*G) as in train_glb.cu.
#include <algorithm>
#include <cstdlib>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;
constexpr int kMaxSlotsC = 128;   // units per CTA (smem bookkeeping)

__device__ __forceinline__ float4 eq1c(float h, float4 w, float4 x) {
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

// ---------------------------------------------------------------------------
// CSR validation (one warp per row): rowptr[0] = 0, rowptr non-decreasing,
// col strictly increasing within a row and inside [0, dim).  out[0]: error
// bits (1 rowptr, 2 col range, 4 col order), out[1]: max nonzeros per row.
__global__ void csr_check_kernel(const int64_t* rowptr, const int32_t* col, int64_t n, int dim, int* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int err = 0, mx = 0;
    if (w0 == 0 && lane == 0 && rowptr[0] != 0) err |= 1;
    for (int64_t r = w0; r < n; r += nw) {
        const int64_t p0 = rowptr[r], p1 = rowptr[r + 1];
        if (p1 < p0) { err |= 1; continue; }
        if (p1 - p0 > 0x7FFFFFFF) { err |= 1; continue; }
        mx = max(mx, (int)(p1 - p0));
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            const int c = col[p];
            if (c < 0 || c >= dim) err |= 2;
            if (p + 1 < p1 && col[p + 1] <= c) err |= 4;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        err |= __shfl_xor_sync(0xffffffffu, err, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        if (err) atomicOr(out, err);
        atomicMax(out + 1, mx);
    }
}

// ---------------------------------------------------------------------------
template <int KJ, bool CACHE_X>
__global__ void __launch_bounds__(NT, 1) som_train_csr_kernel(const TrainArgs a) {
    __shared__ double part[kMaxSlotsC][NW];    // D partials of dense-pass rows
    __shared__ double partn[kMaxSlotsC][NW];   // |w|^2 partials of dense-pass rows
    __shared__ double wns[kMaxSlotsC];         // fp64 |w_u|^2 of this CTA's units
    __shared__ double dsp[kMaxSlotsC];         // D of sparse-path units
    __shared__ float hs[kMaxSlotsC];
    __shared__ unsigned char upd[kMaxSlotsC];
    __shared__ int lst[kMaxSlotsC];            // [0, nup): updated slots, [nup, Sb): the others
    __shared__ int uid[kMaxSlotsC];            // local unit (W row) of slot s
    __shared__ int s_nup, s_abort;
    __shared__ long long nb[3][2];             // CSR bounds of x_t in nb[t % 3]
    extern __shared__ __align__(16) float sm[];
    // sm: xbuf[2][dimp] (x_t dense in slot t & 1), nzi[3][cap], nzv[3][cap]

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = a.utab ? a.ucnt[b] : (a.N - b + G - 1) / G;
    const int d4 = a.dimp >> 2;
    const int cap = a.nz_cap;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float* xbuf = sm;
    int* nzi = reinterpret_cast<int*>(sm + 2 * (size_t)a.dimp);
    float* nzv = reinterpret_cast<float*>(nzi + 3 * (size_t)cap);

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    auto bounds = [&](int64_t t) {   // CSR range of sample i_t
        const int64_t i = train_row(a, t);
        nb[t % 3][0] = a.rowptr[i];
        nb[t % 3][1] = a.rowptr[i + 1];
    };
    auto stage_list = [&](int64_t t) {   // (col, val) of x_t -> list slot t % 3
        if (t < a.t1) {
            const int64_t p0 = nb[t % 3][0];
            const int cnt = (int)(nb[t % 3][1] - p0);
            int* di = nzi + (size_t)(t % 3) * cap;
            float* dv = nzv + (size_t)(t % 3) * cap;
            for (int p = threadIdx.x; p < cnt; p += NT) {
                cp_async4(di + p, a.col + p0 + p);
                cp_async4(dv + p, a.val + p0 + p);
            }
        }
        cp_async_commit();
    };
    auto scatter = [&](int64_t t) {   // list slot t % 3 -> dense slot t & 1 (zeroed)
        if (t < a.t1) {
            const int cnt = (int)(nb[t % 3][1] - nb[t % 3][0]);
            const int* si = nzi + (size_t)(t % 3) * cap;
            const float* sv = nzv + (size_t)(t % 3) * cap;
            float* dst = xbuf + (size_t)(t & 1) * a.dimp;
            for (int p = threadIdx.x; p < cnt; p += NT) dst[si[p]] = sv[p];
        }
    };

    // ---- prologue: zero both dense slots, stage x_t0, bounds of x_t0+1,
    // fp64 row norms of this CTA's units
    for (int k = threadIdx.x; k < 2 * a.dimp; k += NT) xbuf[k] = 0.0f;
    for (int s = threadIdx.x; s < kMaxSlotsC; s += NT) { hs[s] = 0.0f; upd[s] = 0; lst[s] = s; }
    for (int s = threadIdx.x; s < Sb; s += NT) uid[s] = a.utab ? a.utab[(size_t)b * a.S + s] : b + s * G;
    if (threadIdx.x == 0) {
        s_abort = 0;
        s_nup = 0;
        bounds(a.t0);
        if (a.t0 + 1 < a.t1) bounds(a.t0 + 1);
        nb[(a.t0 + 2) % 3][0] = 0;   // x_{t0-1} does not exist: empty list
        nb[(a.t0 + 2) % 3][1] = 0;
    }
    __syncthreads();
    stage_list(a.t0);
    for (int s = 0; s < Sb; ++s) {
        const float4* row = W4 + (int64_t)uid[s] * d4;
        double n0 = 0.0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            if (!valid[j]) continue;
            const float4 w = __ldcg(row + threadIdx.x + j * NT);
            n0 = fma((double)w.x, (double)w.x, n0);
            n0 = fma((double)w.y, (double)w.y, n0);
            n0 = fma((double)w.z, (double)w.z, n0);
            n0 = fma((double)w.w, (double)w.w, n0);
        }
        n0 = warp_sum_f64(n0);
        if (lane == 0) partn[s][warp] = n0;
    }
    cp_async_wait_all();
    __syncthreads();
    scatter(a.t0);
    for (int s = threadIdx.x; s < Sb; s += NT) {
        double tot = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < NW; ++w8) tot += partn[s][w8];
        wns[s] = tot;
    }
    __syncthreads();

    for (int64_t t = a.t0; t < a.t1; ++t) {
        unsigned long long* tr = nullptr;   // optional phase trace (som_set_trace)
        if (a.trace && threadIdx.x == 0 && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
        if (tr) tr[0] = trace_now(a.trace_clk);
        const float4* xc4 = reinterpret_cast<const float4*>(xbuf + (size_t)(t & 1) * a.dimp);         // x_t
        const float4* xp4 = reinterpret_cast<const float4*>(xbuf + (size_t)((t + 1) & 1) * a.dimp);   // x_{t-1}
        const int nup = s_nup;
        const int cnt = (int)(nb[t % 3][1] - nb[t % 3][0]);
        const int* li = nzi + (size_t)(t % 3) * cap;
        const float* lv = nzv + (size_t)(t % 3) * cap;
        // x_{t-1}'s pattern, read now: its bounds slot is rewritten after barrier A
        const int cntp = (int)(nb[(t + 2) % 3][1] - nb[(t + 2) % 3][0]);
        const int* lip = nzi + (size_t)((t + 2) % 3) * cap;

        double xd[CACHE_X ? KJ : 1][4];
        if (CACHE_X) {
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                const float4 x = valid[j] ? xc4[threadIdx.x + j * NT] : make_float4(0.f, 0.f, 0.f, 0.f);
                xd[j][0] = (double)x.x; xd[j][1] = (double)x.y; xd[j][2] = (double)x.z; xd[j][3] = (double)x.w;
            }
        }

        // first dense-pass row in flight while the sparse units are gathered
        float4 cur[KJ], nxt[KJ];
        if (nup > 0) {
            const float4* r0 = W4 + (int64_t)uid[lst[0]] * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) cur[j] = valid[j] ? __ldcg(r0 + threadIdx.x + j * NT) : make_float4(0, 0, 0, 0);
        }

        // ---- sparse path: one warp per untouched unit, lanes over nz(x_t)
        for (int i = nup + warp; i < Sb; i += NW) {
            const int s = lst[i];
            const float* row = a.W + (int64_t)uid[s] * a.dimp;
            double acc = 0.0;
            for (int p = lane; p < cnt; p += 32) {
                const double w = (double)__ldcg(row + li[p]);
                const double e = (double)lv[p] - w;
                acc += fma(e, e, -(w * w));   // w*w exact in fp64
            }
            acc = warp_sum_f64(acc);
            if (lane == 0) dsp[s] = wns[s] + acc;
        }
        if (tr) tr[1] = trace_now(a.trace_clk);

        // ---- dense path: pending Eq. 1 update + distance + new |w|^2
        for (int i = 0; i < nup; ++i) {
            if (i + 1 < nup) {
                const float4* rn = W4 + (int64_t)uid[lst[i + 1]] * d4;
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    nxt[j] = valid[j] ? __ldcg(rn + threadIdx.x + j * NT) : make_float4(0, 0, 0, 0);
            }
            const int s = lst[i];
            const float h = hs[s];
            float4* row = W4 + (int64_t)uid[s] * d4;
            double a0 = 0.0, a1 = 0.0, n0 = 0.0, n1 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                const float4 w = eq1c(h, cur[j], xp4[c]);
                __stcg(row + c, w);
                double x0, x1, x2, x3;
                if (CACHE_X) {
                    x0 = xd[j][0]; x1 = xd[j][1]; x2 = xd[j][2]; x3 = xd[j][3];
                } else {
                    const float4 x = xc4[c];
                    x0 = x.x; x1 = x.y; x2 = x.z; x3 = x.w;
                }
                const double w0 = w.x, w1 = w.y, w2 = w.z, w3 = w.w;
                const double e0 = x0 - w0, e1 = x1 - w1, e2 = x2 - w2, e3 = x3 - w3;
                a0 = fma(e0, e0, a0);
                a1 = fma(e1, e1, a1);
                a0 = fma(e2, e2, a0);
                a1 = fma(e3, e3, a1);
                n0 = fma(w0, w0, n0);
                n1 = fma(w1, w1, n1);
                n0 = fma(w2, w2, n0);
                n1 = fma(w3, w3, n1);
            }
            const double acc = warp_sum_f64(a0 + a1);
            const double nrm = warp_sum_f64(n0 + n1);
            if (lane == 0) { part[s][warp] = acc; partn[s][warp] = nrm; }
#pragma unroll
            for (int j = 0; j < KJ; ++j) cur[j] = nxt[j];
        }
        __syncthreads();   // (A) pass done: x_{t-1} free, partials complete
        if (tr) tr[2] = trace_now(a.trace_clk);

        // x_{t-1}'s dense slot -> zeros; x_{t+1}'s list in flight; bounds of x_{t+2}
        {
            float* xz = xbuf + (size_t)((t + 1) & 1) * a.dimp;
            for (int p = threadIdx.x; p < cntp; p += NT) xz[lip[p]] = 0.0f;
        }
        stage_list(t + 1);
        if (warp == 1 && lane == 0 && t + 2 < a.t1) bounds(t + 2);

        if (warp == 0) {
            unsigned long long best = ~0ull;
            for (int s = lane; s < Sb; s += 32) {
                double tot;
                if (upd[s]) {
                    tot = 0.0;
                    double nn = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < NW; ++w8) { tot += part[s][w8]; nn += partn[s][w8]; }
                    wns[s] = nn;
                } else {
                    tot = dsp[s] > 0.0 ? dsp[s] : 0.0;   // R25: the identity can round below 0
                }
                best = umin64(best, make_key((float)tot, global_unit(a, uid[s])));
            }
            best = warp_min_u64(best);
            if (tr) tr[3] = trace_now(a.trace_clk);
            xchg_publish(a, best, t, b, lane);
            if (tr) tr[4] = trace_now(a.trace_clk);
            const double f = a.f_tab[t - a.t0];
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            if (tr) tr[5] = trace_now(a.trace_clk);
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            const double alpha = a.alpha0 * f;
            double sigma = a.sigma0 * f;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            // neighbourhood of winner c and the slot lists of the next pass
            int n_up = 0, n_no = 0;
            for (int s0 = 0; s0 < Sb; s0 += 32) {
                const int s = s0 + lane;
                bool u2 = false;
                if (s < Sb) {
                    const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, uid[s]), c);
                    u2 = g2 <= r2;
                    upd[s] = u2 ? 1 : 0;
                    hs[s] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
                }
                const unsigned lt = (1u << lane) - 1u;
                const unsigned mu = __ballot_sync(0xffffffffu, s < Sb && u2);
                const unsigned mn = __ballot_sync(0xffffffffu, s < Sb && !u2);
                if (s < Sb) {
                    if (u2) lst[n_up + __popc(mu & lt)] = s;
                    else lst[Sb - 1 - (n_no + __popc(mn & lt))] = s;
                }
                n_up += __popc(mu);
                n_no += __popc(mn);
            }
            if (lane == 0) s_nup = n_up;
            if (tr) tr[6] = trace_now(a.trace_clk);
        }
        cp_async_wait_all();
        __syncthreads();   // (B) list of x_{t+1} landed, x_{t-1} slot zeroed
        if (s_abort) break;
        scatter(t + 1);
        __syncthreads();   // (C) x_{t+1} dense
        if (tr) tr[7] = trace_now(a.trace_clk);
    }

    // flush the update of the last step (x_{t1-1} in dense slot (t1-1) & 1)
    if (a.t1 > a.t0 && !s_abort) {
        const float4* xl4 = reinterpret_cast<const float4*>(xbuf + (size_t)((a.t1 - 1) & 1) * a.dimp);
        const int nup = s_nup;
        for (int i = 0; i < nup; ++i) {
            const int s = lst[i];
            const float h = hs[s];
            float4* row = W4 + (int64_t)uid[s] * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                __stcg(row + c, eq1c(h, __ldcg(row + c), xl4[c]));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// TMA-ring variant (d <= 12288): x_t lives in registers (fp32 + fp64 copies
// of the thread's chunks, scattered through one zeroed smem row), the rows of
// the pending update stream through a ring of R smem buffers filled by
// cp.async.bulk as soon as the winner is known, and the sparse distances of
// step t+1 are computed for every unit by warps 1-15 WHILE warp 0 runs the
// exchange of step t — speculatively: a unit the next pending update touches
// takes the dense pass instead and its sparse value is ignored.  A unit that
// stays untouched keeps its row between that gather and its use, so the
// speculative value is exact.  The sparse path then costs no step time.
template <int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_csr_tma_kernel(const TrainArgs a, int R_max) {
    __shared__ double part[kMaxSlotsC][NW];    // D partials of dense-pass rows
    __shared__ double partn[kMaxSlotsC][NW];   // |w|^2 partials of dense-pass rows
    __shared__ double wns[kMaxSlotsC];         // fp64 |w_u|^2 of this CTA's units
    __shared__ double sacc[2][kMaxSlotsC];     // sum_{nz(x_t)} (e^2 - w^2) in sacc[t & 1]
    __shared__ float hs[kMaxSlotsC];
    __shared__ unsigned char upd[kMaxSlotsC];
    __shared__ int lst[kMaxSlotsC];            // [0, nup): slots of the pending update
    __shared__ int uid[kMaxSlotsC];            // local unit (W row) of slot s
    __shared__ int s_nup[2], s_abort;   // s_nup by step parity: no barrier A when a step updates nothing
    __shared__ long long nb[3][2];             // CSR bounds of x_t in nb[t % 3]
    __shared__ __align__(8) uint64_t mbar[8];
    extern __shared__ __align__(128) float sm[];
    // sm: R ring rows [R][dimp] | xs[dimp] (scatter row, zero between uses) | nzi[2][cap] | nzv[2][cap]

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = a.utab ? a.ucnt[b] : (a.N - b + G - 1) / G;
    const int R = Sb < R_max ? Sb : R_max;
    const int d4 = a.dimp >> 2;
    const int cap = a.nz_cap;
    const uint32_t row_bytes = (uint32_t)a.dim * 4u;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float4* rows4 = reinterpret_cast<float4*>(sm);
    float* xs = sm + (size_t)R_max * a.dimp;
    float4* xs4 = reinterpret_cast<float4*>(xs);
    int* nzi = reinterpret_cast<int*>(xs + a.dimp);
    float* nzv = reinterpret_cast<float*>(nzi + 2 * (size_t)cap);

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    auto bounds = [&](int64_t t) {
        const int64_t i = train_row(a, t);
        nb[t % 3][0] = a.rowptr[i];
        nb[t % 3][1] = a.rowptr[i + 1];
    };
    // (col, val) of x_t -> list slot t & 1 by threads [tb, tb + nth)
    auto stage_list = [&](int64_t t, int tid, int nth) {
        if (t < a.t1) {
            const int64_t p0 = nb[t % 3][0];
            const int cnt = (int)(nb[t % 3][1] - p0);
            int* di = nzi + (size_t)(t & 1) * cap;
            float* dv = nzv + (size_t)(t & 1) * cap;
            for (int p = tid; p < cnt; p += nth) {
                cp_async4(di + p, a.col + p0 + p);
                cp_async4(dv + p, a.val + p0 + p);
            }
        }
        cp_async_commit();
    };
    auto scatter = [&](int64_t t) {   // list slot t & 1 -> xs (zero)
        if (t < a.t1) {
            const int cnt = (int)(nb[t % 3][1] - nb[t % 3][0]);
            const int* si = nzi + (size_t)(t & 1) * cap;
            const float* sv = nzv + (size_t)(t & 1) * cap;
            for (int p = threadIdx.x; p < cnt; p += NT) xs[si[p]] = sv[p];
        }
    };
    // sparse sums of slots [s_begin, Sb) step s_step, list of x_t, warp-wide
    auto sparse_sums = [&](int64_t t, int w_index, int w_count) {
        if (t >= a.t1) return;
        const int cnt = (int)(nb[t % 3][1] - nb[t % 3][0]);
        const int* li = nzi + (size_t)(t & 1) * cap;
        const float* lv = nzv + (size_t)(t & 1) * cap;
        for (int s = w_index; s < Sb; s += w_count) {
            const float* row = a.W + (int64_t)uid[s] * a.dimp;
            double acc = 0.0;
            for (int p = lane; p < cnt; p += 32) {
                const double w = (double)__ldcg(row + li[p]);
                const double e = (double)lv[p] - w;
                acc += fma(e, e, -(w * w));   // w*w exact in fp64
            }
            acc = warp_sum_f64(acc);
            if (lane == 0) sacc[t & 1][s] = acc;
        }
    };

    // ---- prologue
    for (int k = threadIdx.x; k < a.dimp; k += NT) xs[k] = 0.0f;
    for (int s = threadIdx.x; s < kMaxSlotsC; s += NT) { hs[s] = 0.0f; upd[s] = 0; lst[s] = s; }
    for (int s = threadIdx.x; s < Sb; s += NT) uid[s] = a.utab ? a.utab[(size_t)b * a.S + s] : b + s * G;
    if (threadIdx.x == 0) {
        s_abort = 0;
        s_nup[a.t0 & 1] = 0;
        for (int r = 0; r < R_max; ++r) mbar_init_g(&mbar[r], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        bounds(a.t0);
        if (a.t0 + 1 < a.t1) bounds(a.t0 + 1);
    }
    __syncthreads();
    stage_list(a.t0, threadIdx.x, NT);
    stage_list(a.t0 + 1, threadIdx.x, NT);
    for (int s = 0; s < Sb; ++s) {   // fp64 row norms
        const float4* row = W4 + (int64_t)uid[s] * d4;
        double n0 = 0.0;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            if (!valid[j]) continue;
            const float4 w = __ldcg(row + threadIdx.x + j * NT);
            n0 = fma((double)w.x, (double)w.x, n0);
            n0 = fma((double)w.y, (double)w.y, n0);
            n0 = fma((double)w.z, (double)w.z, n0);
            n0 = fma((double)w.w, (double)w.w, n0);
        }
        n0 = warp_sum_f64(n0);
        if (lane == 0) partn[s][warp] = n0;
    }
    cp_async_wait_all();
    __syncthreads();
    if (threadIdx.x == 0 && a.t0 + 2 < a.t1) bounds(a.t0 + 2);
    scatter(a.t0);
    sparse_sums(a.t0, warp, NW);
    for (int s = threadIdx.x; s < Sb; s += NT) {
        double tot = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < NW; ++w8) tot += partn[s][w8];
        wns[s] = tot;
    }
    __syncthreads();
    float4 xp[KJ], xc[KJ];
    double xd[KJ][4];
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        xp[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        xc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid[j]) {
            xc[j] = xs4[threadIdx.x + j * NT];
            xs4[threadIdx.x + j * NT] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        xd[j][0] = xc[j].x; xd[j][1] = xc[j].y; xd[j][2] = xc[j].z; xd[j][3] = xc[j].w;
    }
    int64_t q = 0;   // rows consumed from the ring so far (CTA-uniform)
    double f_next = a.t1 > a.t0 ? a.f_tab[0] : 0.0;   // decay factor of the coming step, loaded a step ahead

    for (int64_t t = a.t0; t < a.t1; ++t) {
        unsigned long long* tr = nullptr;   // optional phase trace (som_set_trace)
        if (a.trace && threadIdx.x == 0 && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
        if (tr) tr[0] = trace_now(a.trace_clk);
        const int nup = s_nup[t & 1];

        // ---- dense pass over the pending update's rows (ring, issued by
        // thread 0 when the winner of t-1 was known)
        for (int i = 0; i < nup; ++i) {
            const int64_t qq = q + i;
            const int buf = (int)(qq % R);
            mbar_wait_g(&mbar[buf], (uint32_t)((qq / R) & 1));
            const float4* rbuf = rows4 + (size_t)buf * d4;
            const int s = lst[i];
            const float h = hs[s];
            float4* row = W4 + (int64_t)uid[s] * d4;
            double a0 = 0.0, a1 = 0.0, n0 = 0.0, n1 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                const float4 w = eq1c(h, rbuf[c], xp[j]);
                __stcg(row + c, w);
                const double w0 = w.x, w1 = w.y, w2 = w.z, w3 = w.w;
                const double e0 = xd[j][0] - w0, e1 = xd[j][1] - w1, e2 = xd[j][2] - w2, e3 = xd[j][3] - w3;
                a0 = fma(e0, e0, a0);
                a1 = fma(e1, e1, a1);
                a0 = fma(e2, e2, a0);
                a1 = fma(e3, e3, a1);
                n0 = fma(w0, w0, n0);
                n1 = fma(w1, w1, n1);
                n0 = fma(w2, w2, n0);
                n1 = fma(w3, w3, n1);
            }
            const double acc = warp_sum_f64(a0 + a1);
            const double nrm = warp_sum_f64(n0 + n1);
            if (lane == 0) { part[s][warp] = acc; partn[s][warp] = nrm; }
            __syncthreads();   // buffer consumed, row written back
            if (threadIdx.x == 0 && i + R < nup) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                bulk_row(rows4 + (size_t)buf * d4, W4 + (int64_t)uid[lst[i + R]] * d4, row_bytes, &mbar[buf]);
            }
        }
        q += nup;   // the last row's barrier is barrier A (keys need every partial)
        if (tr) tr[1] = trace_now(a.trace_clk);

        const double f = f_next;
        const double alpha = a.alpha0 * f;
        double sigma = a.sigma0 * f;
        if (sigma < a.sigma_min) sigma = a.sigma_min;
        const double two_s2 = 2.0 * sigma * sigma;
        const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;

        if (warp == 0) {
            unsigned long long best = ~0ull;
            for (int s = lane; s < Sb; s += 32) {
                double tot;
                if (upd[s]) {
                    tot = 0.0;
                    double nn = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < NW; ++w8) { tot += part[s][w8]; nn += partn[s][w8]; }
                    wns[s] = nn;
                } else {
                    tot = wns[s] + sacc[t & 1][s];
                    tot = tot > 0.0 ? tot : 0.0;   // R25: the identity can round below 0
                }
                best = umin64(best, make_key((float)tot, global_unit(a, uid[s])));
            }
            best = warp_min_u64(best);
            if (tr) tr[2] = trace_now(a.trace_clk);
            xchg_publish(a, best, t, b, lane);
            // the data warps start their speculative sums only now: run
            // beside the keys above they slowed them down (shared
            // sub-partition and conversion pipe) on the step's critical path
            asm volatile("bar.arrive 3, %0;" ::"n"(NT) : "memory");
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            if (tr) tr[3] = trace_now(a.trace_clk);
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            int n_up = 0, n_no = 0;
            for (int s0 = 0; s0 < Sb; s0 += 32) {
                const int s = s0 + lane;
                bool u2 = false;
                if (s < Sb) {
                    const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, uid[s]), c);
                    u2 = g2 <= r2;
                    upd[s] = u2 ? 1 : 0;
                    hs[s] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
                }
                const unsigned lt = (1u << lane) - 1u;
                const unsigned mu = __ballot_sync(0xffffffffu, s < Sb && u2);
                const unsigned mn = __ballot_sync(0xffffffffu, s < Sb && !u2);
                if (s < Sb) {
                    if (u2) lst[n_up + __popc(mu & lt)] = s;
                    else lst[Sb - 1 - (n_no + __popc(mn & lt))] = s;
                }
                n_up += __popc(mu);
                n_no += __popc(mn);
            }
            __syncwarp();
            if (tr) tr[7] = trace_now(a.trace_clk);
            if (lane == 0) {
                s_nup[(t + 1) & 1] = n_up;
                // first rows of the next pass into the ring (none after the
                // last step: the final flush reads rows directly)
                if (!stop && t + 1 < a.t1) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    const int m = n_up < R ? n_up : R;
                    for (int i = 0; i < m; ++i) {
                        const int64_t qq = q + i;
                        bulk_row(rows4 + (size_t)(qq % R) * d4, W4 + (int64_t)uid[lst[i]] * d4, row_bytes,
                                 &mbar[qq % R]);
                    }
                }
            }
            if (tr) tr[4] = trace_now(a.trace_clk);
        } else {
            // warps 1-15, once warp 0 has published: list of x_{t+2}, bounds
            // of x_{t+3}, and the speculative sparse sums of step t+1
            // (skipped when the radius covers the whole lattice: every unit
            // takes the dense pass)
            asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory");
            // only the 12 warps off warp 0's sub-partition (warp % 4 != 0):
            // warps 4, 8, 12 stay idle so the exchange poll keeps its issue
            // slot and pipes
            if ((warp & 3) != 0) {
                const int hid = warp - 1 - (warp >> 2);   // 0..11
                stage_list(t + 2, hid * 32 + lane, 12 * 32);
                if (warp == 1 && lane == 0 && t + 3 < a.t1) bounds(t + 3);
                if (!(r2 >= a.g2max)) sparse_sums(t + 1, hid, 12);
            }
        }
        cp_async_wait_all();
        __syncthreads();   // (B) lists, ring issue, sparse sums of t+1
        if (tr) tr[5] = trace_now(a.trace_clk);
        if (s_abort) break;
        if (t + 1 < a.t1) f_next = a.f_tab[t + 1 - a.t0];
        scatter(t + 1);
        __syncthreads();   // (C) x_{t+1} in xs
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            xp[j] = xc[j];
            if (valid[j]) {
                xc[j] = xs4[threadIdx.x + j * NT];
                xs4[threadIdx.x + j * NT] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            xd[j][0] = xc[j].x; xd[j][1] = xc[j].y; xd[j][2] = xc[j].z; xd[j][3] = xc[j].w;
        }
        if (tr) tr[6] = trace_now(a.trace_clk);
    }

    // flush the update of the last step (x_{t1-1} is now in xp)
    if (a.t1 > a.t0 && !s_abort) {
        const int nup = s_nup[a.t1 & 1];
        for (int i = 0; i < nup; ++i) {
            const int s = lst[i];
            const float h = hs[s];
            float4* row = W4 + (int64_t)uid[s] * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                __stcg(row + c, eq1c(h, __ldcg(row + c), xp[j]));
            }
        }
    }
}

size_t csr_smem_bytes(int dimp, int cap) { return sizeof(float) * 2 * (size_t)dimp + 8 * 3 * (size_t)cap; }

template <int KJ, bool CX>
cudaError_t launch_csr(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = csr_smem_bytes(a.dimp, a.nz_cap);
    auto fn = som_train_csr_kernel<KJ, CX>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)fn, a, NT, smem, params, st);
}

size_t csr_tma_smem_bytes(int dimp, int cap, int R) {
    return sizeof(float) * (size_t)(R + 1) * dimp + 16 * (size_t)cap + 128;
}

template <int KJ>
cudaError_t launch_csr_tma(const TrainArgs& a, int R, cudaStream_t st) {
    const size_t smem = csr_tma_smem_bytes(a.dimp, a.nz_cap, R);
    auto fn = som_train_csr_tma_kernel<KJ>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    int r = R;
    void* params[] = {&args, &r};
    return launch_persistent((const void*)fn, a, NT, smem, params, st);
}

}  // namespace

int csr_nz_cap(int maxnnz) { return std::max(4, (maxnnz + 3) & ~3); }

bool train_csr_supported(int S, int dim, int maxnnz, int max_smem_optin) {
    if (dim % 4 != 0 || S > kMaxSlotsC) return false;
    const int kj = ((dim / 4) + NT - 1) / NT;
    if (kj > 12) return false;
    const size_t stat = 40 * 1024;   // static smem (partials, norms, lists) headroom
    return csr_smem_bytes(dim, csr_nz_cap(maxnnz)) + stat <= (size_t)max_smem_optin;
}

cudaError_t launch_train_csr(const TrainArgs& a, cudaStream_t st) {
    const int kj = ((a.dimp / 4) + NT - 1) / NT;
    {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const size_t stat = 40 * 1024;   // static smem headroom
        int R = 0;
        for (int r = 4; r >= 2; --r)
            if (csr_tma_smem_bytes(a.dimp, a.nz_cap, r) + stat <= (size_t)optin) { R = r; break; }
        R = std::min(R, a.S);
        if (kj <= 6 && R >= 1 && getenv("SOM_NO_TMA_RING") == nullptr) {
            switch (kj) {
                case 1: return launch_csr_tma<1>(a, R, st);
                case 2: return launch_csr_tma<2>(a, R, st);
                case 3: return launch_csr_tma<3>(a, R, st);
                case 4: return launch_csr_tma<4>(a, R, st);
                case 5: return launch_csr_tma<5>(a, R, st);
                case 6: return launch_csr_tma<6>(a, R, st);
            }
        }
    }
    switch (kj) {
        case 1: return launch_csr<1, true>(a, st);
        case 2: return launch_csr<2, true>(a, st);
        case 3: return launch_csr<3, true>(a, st);
        case 4: return launch_csr<4, true>(a, st);
        case 5: return launch_csr<5, true>(a, st);
        case 6: return launch_csr<6, false>(a, st);
        case 7: return launch_csr<7, false>(a, st);
        case 8: return launch_csr<8, false>(a, st);
        case 9: return launch_csr<9, false>(a, st);
        case 10: return launch_csr<10, false>(a, st);
        case 11: return launch_csr<11, false>(a, st);
        case 12: return launch_csr<12, false>(a, st);
        default: return cudaErrorInvalidConfiguration;
    }
}

cudaError_t launch_csr_check(const int64_t* rowptr, const int32_t* col, int64_t n, int dim, int* out,
                             cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(int), st);
    if (e != cudaSuccess) return e;
    const int64_t warps = std::max<int64_t>(1, std::min<int64_t>(n, 148 * 64));
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    csr_check_kernel<<<blocks, 256, 0, st>>>(rowptr, col, n, dim, out);
    return cudaGetLastError();
}

}  // namespace som
