// train.cu — persistent cooperative online-SOM training kernel (sm_100a).
//
// One launch runs the whole step range [t0, t1) ("data and map
// structures" stay device-resident; "weights are copied to the main
// memory only after all the iterations").  The paper's three kernels per
// iteration — getDistances, reduceMin, updateWeights
// — become one loop body per step:
//
//   fused pass   for every unit u this CTA owns: apply the pending Eq. 1
//                update of step t-1 (R11) and, from the updated
//                prototype, accumulate D_u(x_t) in fp64 (R10).  Reading W
//                once per step serves both.
//   local argmin (D_u, u) packed into a u64 key (R9), warp + block min.
//   exchange     each CTA publishes its key (tagged with t) into its own
//                slot; every CTA polls all G slots and takes the min — the
//                per-step global argmin without a second kernel or atomics.
//   neighbourhood h_u for the CTA's own units from the winner c_t (R4, R5).
//
// Units are dealt cyclically (u = b + s*G) so the shrinking neighbourhood
// late in training stays spread over all CTAs.  A CTA's prototypes live in
// shared memory when they fit (w_smem), else they stream from global
// memory (L2-resident when the map fits the 126 MB L2).  x_{t+1} is
// prefetched with cp.async while the exchange is in flight.
#include <cooperative_groups.h>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {


struct Smem {
    float* xs;        // [2][dimp] x ring (t even / odd)
    float* ws;        // [S][dimp] (w_smem only)
    double* part;     // [S][kTrainWarps] fp64 partial distances
    float* hs;        // [S] neighbourhood weight of the pending update
    int* upd;         // [S] 1 if the unit adapts in the pending update
};

__device__ __forceinline__ Smem carve(unsigned char* base, int S, int dimp, int w_smem) {
    Smem s;
    size_t off = 0;
    s.xs = reinterpret_cast<float*>(base + off);
    off += sizeof(float) * 2 * (size_t)dimp;
    s.ws = reinterpret_cast<float*>(base + off);
    if (w_smem) off += sizeof(float) * (size_t)S * dimp;
    s.part = reinterpret_cast<double*>(base + off);
    off += sizeof(double) * (size_t)S * kTrainWarps;
    s.hs = reinterpret_cast<float*>(base + off);
    off += sizeof(float) * (size_t)S;
    s.upd = reinterpret_cast<int*>(base + off);
    return s;
}

// Stage x_t = X[i_t] into one ring slot (cp.async; caller commits/waits).
__device__ __forceinline__ void stage_x(const TrainArgs& a, float* dst, int64_t t) {
    const int64_t i = train_row(a, t);
    const float* src = a.X + i * (int64_t)a.dim;
    if (a.x_vec4) {
        const int d4 = a.dim >> 2;
        for (int k4 = threadIdx.x; k4 < d4; k4 += kTrainThreads) cp_async16(dst + 4 * k4, src + 4 * k4);
    } else {
        for (int k = threadIdx.x; k < a.dim; k += kTrainThreads) cp_async4(dst + k, src + k);
    }
}

__device__ __forceinline__ float4 eq1_update4(float h, float4 w, float4 x) {
    // Eq. 1 per element: w + h (x - w) as fmaf(h, RN(x - w), w)  (R11)
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

__device__ __forceinline__ void dist_acc4(double& a0, double& a1, float4 x, float4 w) {
    // R10: difference of the fp32 operands formed in fp64, summed in fp64
    double d0 = (double)x.x - (double)w.x;
    double d1 = (double)x.y - (double)w.y;
    double d2 = (double)x.z - (double)w.z;
    double d3 = (double)x.w - (double)w.w;
    a0 = fma(d0, d0, a0);
    a1 = fma(d1, d1, a1);
    a0 = fma(d2, d2, a0);
    a1 = fma(d3, d3, a1);
}

// Fused pass over one unit whose prototype is a float4 row (smem, or a
// 16-byte-aligned global row).  Returns this thread's fp64 partial sum.
template <bool kGlobal>
__device__ __forceinline__ double fused_row4(float* wrow, const float* xp, const float* xc, int d4,
                                             float h, bool up, bool want_dist) {
    float4* w4 = reinterpret_cast<float4*>(wrow);
    const float4* xp4 = reinterpret_cast<const float4*>(xp);
    const float4* xc4 = reinterpret_cast<const float4*>(xc);
    double a0 = 0.0, a1 = 0.0;
    int k4 = threadIdx.x;
    if (kGlobal) {
        // 2x unrolled so two independent L2 loads are in flight per thread
        for (; k4 + kTrainThreads < d4; k4 += 2 * kTrainThreads) {
            float4 w0 = __ldcg(w4 + k4);
            float4 w1 = __ldcg(w4 + k4 + kTrainThreads);
            if (up) {
                w0 = eq1_update4(h, w0, xp4[k4]);
                w1 = eq1_update4(h, w1, xp4[k4 + kTrainThreads]);
                __stcg(w4 + k4, w0);
                __stcg(w4 + k4 + kTrainThreads, w1);
            }
            if (want_dist) {
                dist_acc4(a0, a1, xc4[k4], w0);
                dist_acc4(a0, a1, xc4[k4 + kTrainThreads], w1);
            }
        }
    }
    for (; k4 < d4; k4 += kTrainThreads) {
        float4 w = kGlobal ? __ldcg(w4 + k4) : w4[k4];
        if (up) {
            w = eq1_update4(h, w, xp4[k4]);
            if (kGlobal) __stcg(w4 + k4, w); else w4[k4] = w;
        }
        if (want_dist) dist_acc4(a0, a1, xc4[k4], w);
    }
    return a0 + a1;
}

// Scalar variant for global rows that are not 16-byte aligned (d % 4 != 0).
__device__ __forceinline__ double fused_row1(float* w, const float* xp, const float* xc, int d,
                                             float h, bool up, bool want_dist) {
    double a0 = 0.0;
    for (int k = threadIdx.x; k < d; k += kTrainThreads) {
        float wk = __ldcg(w + k);
        if (up) {
            wk = fmaf(h, xp[k] - wk, wk);
            __stcg(w + k, wk);
        }
        if (want_dist) {
            double dd = (double)xc[k] - (double)wk;
            a0 = fma(dd, dd, a0);
        }
    }
    return a0;
}

__global__ void __launch_bounds__(kTrainThreads, 1) som_train_kernel(const TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_abort;
    const int b = blockIdx.x;
    const int G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = (a.N - b + G - 1) / G;     // units owned: u = b + s*G, s < Sb
    Smem sm = carve(smem_raw, a.S, a.dimp, a.w_smem);
    const int d4 = a.dimp >> 2;
    const bool rows4 = a.w_smem || a.x_vec4;  // prototype rows addressable as float4

    // zero the x ring padding and load the resident prototypes
    for (int k = threadIdx.x; k < 2 * a.dimp; k += kTrainThreads) sm.xs[k] = 0.0f;
    if (a.w_smem) {
        for (int s = 0; s < Sb; ++s) {
            const float* src = a.W + (int64_t)(b + s * G) * a.dim;
            float* dst = sm.ws + (size_t)s * a.dimp;
            for (int k = threadIdx.x; k < a.dimp; k += kTrainThreads) dst[k] = k < a.dim ? src[k] : 0.0f;
        }
    }
    for (int s = threadIdx.x; s < a.S; s += kTrainThreads) { sm.hs[s] = 0.0f; sm.upd[s] = 0; }
    if (threadIdx.x == 0) s_abort = 0;
    __syncthreads();

    if (a.t1 > a.t0) {
        stage_x(a, sm.xs + (a.t0 & 1) * a.dimp, a.t0);
        cp_async_commit();
        cp_async_wait_all();
    }
    __syncthreads();

    int c_last = 0;
    for (int64_t t = a.t0; t < a.t1; ++t) {
        const float* xc = sm.xs + (t & 1) * a.dimp;          // x_t
        const float* xp = sm.xs + ((t + 1) & 1) * a.dimp;    // x_{t-1} (pending update)

        // ---- fused pass: pending update (t-1) + distance D_u(x_t)
        for (int s = 0; s < Sb; ++s) {
            const float h = sm.hs[s];
            const bool up = sm.upd[s] != 0;
            double acc;
            if (a.w_smem) {
                acc = fused_row4<false>(sm.ws + (size_t)s * a.dimp, xp, xc, d4, h, up, true);
            } else if (rows4) {
                acc = fused_row4<true>(a.W + (int64_t)(b + s * G) * a.dim, xp, xc, d4, h, up, true);
            } else {
                acc = fused_row1(a.W + (int64_t)(b + s * G) * a.dim, xp, xc, a.dim, h, up, true);
            }
            acc = warp_sum_f64(acc);
            if (lane == 0) sm.part[s * kTrainWarps + warp] = acc;
        }
        __syncthreads();

        // ---- prefetch x_{t+1} into the slot x_{t-1} just vacated
        if (t + 1 < a.t1) stage_x(a, sm.xs + ((t + 1) & 1) * a.dimp, t + 1);
        cp_async_commit();

        if (warp == 0) {
            // local argmin over this CTA's units (lanes over units)
            unsigned long long best = ~0ull;
            for (int s = lane; s < Sb; s += 32) {
                double tot = 0.0;
#pragma unroll
                for (int w = 0; w < kTrainWarps; ++w) tot += sm.part[s * kTrainWarps + w];
                best = umin64(best, make_key((float)tot, global_unit(a, b + s * G)));
            }
            best = warp_min_u64(best);

            // exchange (in-GPU all-gather, then across ranks when sharded)
            xchg_publish(a, best, t, b, lane);
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            c_last = c;
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;

            // neighbourhood of step t for this CTA's units (R1-R5)
            const double f = a.f_tab[t - a.t0];
            const double alpha = a.alpha0 * f;
            double sigma = a.sigma0 * f;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            for (int s = lane; s < Sb; s += 32) {
                const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, b + s * G), c);
                const bool up = g2 <= r2;
                sm.upd[s] = up ? 1 : 0;
                sm.hs[s] = up ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        if (s_abort) break;   // block-uniform: written by warp 0 before the barrier
    }
    (void)c_last;

    // ---- flush: the update of the last step, then write resident rows back
    if (a.t1 > a.t0 && !s_abort) {
        const float* xl = sm.xs + ((a.t1 - 1) & 1) * a.dimp;   // x_{t1-1}
        for (int s = 0; s < Sb; ++s) {
            const float h = sm.hs[s];
            if (!sm.upd[s]) continue;
            if (a.w_smem) fused_row4<false>(sm.ws + (size_t)s * a.dimp, xl, xl, d4, h, true, false);
            else if (rows4) fused_row4<true>(a.W + (int64_t)(b + s * G) * a.dim, xl, xl, d4, h, true, false);
            else fused_row1(a.W + (int64_t)(b + s * G) * a.dim, xl, xl, a.dim, h, true, false);
        }
    }
    if (a.w_smem) {
        __syncthreads();
        for (int s = 0; s < Sb; ++s) {
            float* dst = a.W + (int64_t)(b + s * G) * a.dim;
            const float* src = sm.ws + (size_t)s * a.dimp;
            for (int k = threadIdx.x; k < a.dim; k += kTrainThreads) dst[k] = src[k];
        }
    }
}

}  // namespace

size_t train_smem_bytes(int S, int dimp, int w_smem) {
    size_t b = sizeof(float) * 2 * (size_t)dimp;
    if (w_smem) b += sizeof(float) * (size_t)S * dimp;
    b += sizeof(double) * (size_t)S * kTrainWarps;
    b += (sizeof(float) + sizeof(int)) * (size_t)S;
    return (b + 15) & ~(size_t)15;
}

cudaError_t launch_train(const TrainArgs& a, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(som_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)som_train_kernel, a, kTrainThreads, smem, params, st);
}

}  // namespace som
