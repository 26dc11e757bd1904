// train_glb.cu — persistent online-SOM training for maps that live in global
// memory (L2-resident up to ~100 MB: c3; HBM beyond: c4), the bandwidth-bound
// regime of the step (4 N d bytes read + 4 H_t d written per
// sample).
//
// Same step and exchange as train_reg.cu / train.cu (pending Eq. 1 update of
// t-1 fused with the fp64 distance of t, packed keys, tagged all-gather;
// P:162-166, R9-R11).  Differences that make it stream:
//  * thread tid owns float4 chunks c = tid + j*512 (j < KJ) of every row, so
//    a row is KJ independent 16-byte loads per thread, all issued at once;
//  * the next unit's row is loaded into a second register set while the
//    current one is updated and measured (cross-row software pipelining);
//  * x_t is converted to fp64 once per step into registers (CACHE_X), so
//    each prototype element costs one F2F.F64.F32 (the ~16/clk/SM pipe);
//  * updated rows are written back with st.global.cg (L2).
// Units are dealt cyclically (u = b + s*G); s runs over this CTA's units.
#include <algorithm>
#include <cstdlib>

#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;
constexpr int kMaxSlotsG = 128;   // units per CTA (smem bookkeeping)

__device__ __forceinline__ float4 eq1g(float h, float4 w, float4 x) {
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

template <int KJ, bool CACHE_X>
__global__ void __launch_bounds__(NT, 1) som_train_glb_kernel(const TrainArgs a) {
    __shared__ double part[kMaxSlotsG][NW];
    __shared__ float hs[kMaxSlotsG];
    __shared__ int upd[kMaxSlotsG];
    __shared__ int s_abort;
    extern __shared__ __align__(16) float xring[];   // [2][dimp]

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = (a.N - b + G - 1) / G;
    const int d4 = a.dimp >> 2;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float4* ring4 = reinterpret_cast<float4*>(xring);

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    for (int k = threadIdx.x; k < 2 * a.dimp; k += NT) xring[k] = 0.0f;
    for (int s = threadIdx.x; s < kMaxSlotsG; s += NT) { hs[s] = 0.0f; upd[s] = 0; }
    if (threadIdx.x == 0) s_abort = 0;
    __syncthreads();

    auto stage = [&](int64_t t) {   // x_t -> ring[t & 1] (cp.async, own chunks)
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + train_row(a, t) * (int64_t)a.dim);
            float4* dst = ring4 + (size_t)(t & 1) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) cp_async16(dst + threadIdx.x + j * NT, src + threadIdx.x + j * NT);
        }
        cp_async_commit();
    };
    stage(a.t0);
    cp_async_wait_all();
    __syncthreads();

    for (int64_t t = a.t0; t < a.t1; ++t) {
        const float4* xc4 = ring4 + (size_t)(t & 1) * d4;          // x_t
        const float4* xp4 = ring4 + (size_t)((t + 1) & 1) * d4;    // x_{t-1}
        double xd[CACHE_X ? KJ : 1][4];
        if (CACHE_X) {
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                const float4 x = valid[j] ? xc4[threadIdx.x + j * NT] : make_float4(0.f, 0.f, 0.f, 0.f);
                xd[j][0] = (double)x.x; xd[j][1] = (double)x.y; xd[j][2] = (double)x.z; xd[j][3] = (double)x.w;
            }
        }

        // ---- fused pass over this CTA's rows, next row's loads in flight
        float4 cur[KJ], nxt[KJ];
        if (Sb > 0) {
            const float4* r0 = W4 + (int64_t)b * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) cur[j] = valid[j] ? __ldcg(r0 + threadIdx.x + j * NT) : make_float4(0, 0, 0, 0);
        }
        for (int s = 0; s < Sb; ++s) {
            if (s + 1 < Sb) {
                const float4* rn = W4 + (int64_t)(b + (s + 1) * G) * d4;
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    nxt[j] = valid[j] ? __ldcg(rn + threadIdx.x + j * NT) : make_float4(0, 0, 0, 0);
            }
            const bool up = upd[s] != 0;
            const float h = hs[s];
            float4* row = W4 + (int64_t)(b + s * G) * d4;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                float4 w = cur[j];
                if (up) {
                    w = eq1g(h, w, xp4[threadIdx.x + j * NT]);
                    __stcg(row + threadIdx.x + j * NT, w);
                }
                double x0, x1, x2, x3;
                if (CACHE_X) {
                    x0 = xd[j][0]; x1 = xd[j][1]; x2 = xd[j][2]; x3 = xd[j][3];
                } else {
                    const float4 x = xc4[threadIdx.x + j * NT];
                    x0 = x.x; x1 = x.y; x2 = x.z; x3 = x.w;
                }
                // R10: (double)x - (double)w squared and summed in fp64
                const double e0 = x0 - (double)w.x, e1 = x1 - (double)w.y;
                const double e2 = x2 - (double)w.z, e3 = x3 - (double)w.w;
                a0 = fma(e0, e0, a0);
                a1 = fma(e1, e1, a1);
                a0 = fma(e2, e2, a0);
                a1 = fma(e3, e3, a1);
            }
            const double acc = warp_sum_f64(a0 + a1);
            if (lane == 0) part[s][warp] = acc;
#pragma unroll
            for (int j = 0; j < KJ; ++j) cur[j] = nxt[j];
        }
        __syncthreads();

        stage(t + 1);      // x_{t+1} into the slot x_{t-1} vacated

        if (warp == 0) {
            unsigned long long best = ~0ull;
            for (int s = lane; s < Sb; s += 32) {
                double tot = 0.0;
#pragma unroll
                for (int w8 = 0; w8 < NW; ++w8) tot += part[s][w8];
                best = umin64(best, make_key((float)tot, global_unit(a, b + s * G)));
            }
            best = warp_min_u64(best);
            xchg_publish(a, best, t, b, lane);
            const double f = a.f_tab[t - a.t0];
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            const double alpha = a.alpha0 * f;
            double sigma = a.sigma0 * f;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            for (int s = lane; s < Sb; s += 32) {
                const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, b + s * G), c);
                const bool u2 = g2 <= r2;
                upd[s] = u2 ? 1 : 0;
                hs[s] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        if (s_abort) break;
    }

    // flush the update of the last step (x_{t1-1} in ring[(t1-1) & 1])
    if (a.t1 > a.t0 && !s_abort) {
        const float4* xl4 = ring4 + (size_t)((a.t1 - 1) & 1) * d4;
        for (int s = 0; s < Sb; ++s) {
            if (!upd[s]) continue;
            const float h = hs[s];
            float4* row = W4 + (int64_t)(b + s * G) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                __stcg(row + c, eq1g(h, __ldcg(row + c), xl4[c]));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// TMA row-ring variant (d <= 12288): thread 0 keeps R rows in flight with
// cp.async.bulk (global -> shared, completion on one mbarrier per buffer),
// continuing into the next step's first rows while the exchange runs, so
// the loop is not exposed to L2/HBM latency row by row.  Rows are consumed
// from shared memory; updated rows go back with st.global.cg.  Row q of the
// CTA's sequence (q = step * Sb + s) lives in buffer q % R; the refill of
// buffer q % R with row q + R is issued only after row q was processed and
// written back (R <= Sb, so row q + R is final at that point).
template <int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_tma_kernel(const TrainArgs a, int R_max) {
    __shared__ double part[kMaxSlotsG][NW];
    __shared__ float hs[kMaxSlotsG];
    __shared__ int upd[kMaxSlotsG];
    __shared__ int s_abort;
    __shared__ __align__(8) uint64_t mbar[8];
    extern __shared__ __align__(128) float sm[];   // [dimp] x staging, then R rows of dimp

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = (a.N - b + G - 1) / G;
    const int R = Sb < R_max ? Sb : R_max;   // ring depth of this CTA (R <= Sb keeps refills final)
    const int d4 = a.dimp >> 2;
    const uint32_t row_bytes = (uint32_t)a.dim * 4u;
    float4* W4 = reinterpret_cast<float4*>(a.W);
    float4* xs4 = reinterpret_cast<float4*>(sm);
    float4* rows4 = reinterpret_cast<float4*>(sm + a.dimp);
    const int64_t nsteps = a.t1 - a.t0;
    const int64_t total_rows = nsteps * Sb;

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    for (int s = threadIdx.x; s < kMaxSlotsG; s += NT) { hs[s] = 0.0f; upd[s] = 0; }
    if (threadIdx.x == 0) {
        s_abort = 0;
        for (int r = 0; r < R_max; ++r) mbar_init_g(&mbar[r], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int64_t q = 0; q < R && q < total_rows; ++q)
            bulk_row(rows4 + (size_t)q * d4, W4 + (int64_t)(b + (int)(q % Sb) * G) * d4, row_bytes, &mbar[q]);
    }

    auto stage = [&](int64_t t) {
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + train_row(a, t) * (int64_t)a.dim);
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) cp_async16(xs4 + threadIdx.x + j * NT, src + threadIdx.x + j * NT);
        }
        cp_async_commit();
    };
    float4 xp[KJ], xc[KJ];
    double xd[KJ][4];
    stage(a.t0);
    cp_async_wait_all();
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        xp[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        xc[j] = valid[j] ? xs4[threadIdx.x + j * NT] : make_float4(0.f, 0.f, 0.f, 0.f);
        xd[j][0] = xc[j].x; xd[j][1] = xc[j].y; xd[j][2] = xc[j].z; xd[j][3] = xc[j].w;
    }
    __syncthreads();

    for (int64_t t = a.t0; t < a.t1; ++t) {
        const int64_t qbase = (t - a.t0) * Sb;
        for (int s = 0; s < Sb; ++s) {
            const int64_t q = qbase + s;
            const int buf = (int)(q % R);
            mbar_wait_g(&mbar[buf], (uint32_t)((q / R) & 1));
            const float4* rbuf = rows4 + (size_t)buf * d4;
            const bool up = upd[s] != 0;
            const float h = hs[s];
            float4* row = W4 + (int64_t)(b + s * G) * d4;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                float4 w = rbuf[c];
                if (up) {
                    w = eq1g(h, w, xp[j]);
                    __stcg(row + c, w);
                }
                const double e0 = xd[j][0] - (double)w.x, e1 = xd[j][1] - (double)w.y;
                const double e2 = xd[j][2] - (double)w.z, e3 = xd[j][3] - (double)w.w;
                a0 = fma(e0, e0, a0);
                a1 = fma(e1, e1, a1);
                a0 = fma(e2, e2, a0);
                a1 = fma(e3, e3, a1);
            }
            const double acc = warp_sum_f64(a0 + a1);
            if (lane == 0) part[s][warp] = acc;
            __syncthreads();   // buffer consumed, row written back
            if (threadIdx.x == 0 && q + R < total_rows) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const int rn = (int)((q + R) % Sb);
                bulk_row(rows4 + (size_t)buf * d4, W4 + (int64_t)(b + rn * G) * d4, row_bytes, &mbar[buf]);
            }
        }

        stage(t + 1);      // x_{t+1} into the staging buffer (consumed at the step start)

        if (warp == 0) {
            unsigned long long best = ~0ull;
            for (int s = lane; s < Sb; s += 32) {
                double tot = 0.0;
#pragma unroll
                for (int w8 = 0; w8 < NW; ++w8) tot += part[s][w8];
                best = umin64(best, make_key((float)tot, global_unit(a, b + s * G)));
            }
            best = warp_min_u64(best);
            xchg_publish(a, best, t, b, lane);
            const double f = a.f_tab[t - a.t0];
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            const double alpha = a.alpha0 * f;
            double sigma = a.sigma0 * f;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            for (int s = lane; s < Sb; s += 32) {
                const double g2 = lattice_g2(a.cols, a.topo, global_unit(a, b + s * G), c);
                const bool u2 = g2 <= r2;
                upd[s] = u2 ? 1 : 0;
                hs[s] = u2 ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
        }
        cp_async_wait_all();
        __syncthreads();
        if (s_abort) break;
        // x_{t-1} <- x_t, x_t <- x_{t+1} (own chunks)
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            xp[j] = xc[j];
            if (valid[j]) {
                xc[j] = xs4[threadIdx.x + j * NT];
                xd[j][0] = xc[j].x; xd[j][1] = xc[j].y; xd[j][2] = xc[j].z; xd[j][3] = xc[j].w;
            }
        }
        __syncthreads();   // staging buffer free for the next cp.async
    }

    if (a.t1 > a.t0 && !s_abort) {
        // flush the update of the last step (x_{t1-1} is now in xp)
        for (int s = 0; s < Sb; ++s) {
            if (!upd[s]) continue;
            const float h = hs[s];
            float4* row = W4 + (int64_t)(b + s * G) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                if (!valid[j]) continue;
                const int c = threadIdx.x + j * NT;
                __stcg(row + c, eq1g(h, __ldcg(row + c), xp[j]));
            }
        }
    }
}

template <int KJ>
cudaError_t launch_tma(const TrainArgs& a, int R, cudaStream_t st) {
    const size_t smem = sizeof(float) * (size_t)a.dimp * (1 + R) + 128;
    auto fn = som_train_tma_kernel<KJ>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    int r = R;
    void* params[] = {&args, &r};
    return launch_persistent((const void*)fn, a, NT, smem, params, st);
}

template <int KJ, bool CX>
cudaError_t launch_glb(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * 2 * (size_t)a.dimp;
    auto fn = som_train_glb_kernel<KJ, CX>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)fn, a, NT, smem, params, st);
}

}  // namespace

// Global-memory variant: d % 4 == 0, rows up to 40 float4 chunks per thread
// (d <= 81,920), at most kMaxSlotsG units per CTA.
bool train_glb_supported(int S, int dim) {
    if (dim % 4 != 0 || S > kMaxSlotsG) return false;
    const int kj = ((dim / 4) + NT - 1) / NT;
    return kj <= 12;
}

cudaError_t launch_train_glb(const TrainArgs& a, cudaStream_t st) {
    const int kj = ((a.dimp / 4) + NT - 1) / NT;
    // TMA row ring when R >= 2 rows of the CTA fit next to the x staging buffer
    {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const size_t rowb = sizeof(float) * (size_t)a.dimp;
        const size_t stat = 20 * 1024;   // static smem (part/hs/upd) headroom
        int R = (int)std::min<size_t>(4, ((size_t)optin - stat) / rowb - 1);
        R = std::min(R, a.S);
        if (kj <= 6 && R >= 2 && a.dim % 4 == 0 && getenv("SOM_NO_TMA_RING") == nullptr) {
            switch (kj) {
                case 1: return launch_tma<1>(a, R, st);
                case 2: return launch_tma<2>(a, R, st);
                case 3: return launch_tma<3>(a, R, st);
                case 4: return launch_tma<4>(a, R, st);
                case 5: return launch_tma<5>(a, R, st);
                case 6: return launch_tma<6>(a, R, st);
            }
        }
    }
    switch (kj) {
        case 1: return launch_glb<1, true>(a, st);
        case 2: return launch_glb<2, true>(a, st);
        case 3: return launch_glb<3, true>(a, st);
        case 4: return launch_glb<4, true>(a, st);
        case 5: return launch_glb<5, true>(a, st);
        case 6: return launch_glb<6, false>(a, st);
        case 7: return launch_glb<7, false>(a, st);
        case 8: return launch_glb<8, false>(a, st);
        case 9: return launch_glb<9, false>(a, st);
        case 10: return launch_glb<10, false>(a, st);
        case 11: return launch_glb<11, false>(a, st);
        case 12: return launch_glb<12, false>(a, st);
        default: return cudaErrorInvalidConfiguration;
    }
}

}  // namespace som
