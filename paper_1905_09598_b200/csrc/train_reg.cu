// train_reg.cu — register-resident persistent online-SOM training kernel.
//
// Same step as train.cu (pending Eq. 1 update of step t-1 fused with the
// fp64 distance pass of step t, packed (D, u) keys, tagged all-gather of
// per-CTA minima, R9-R11), specialised for maps whose per-CTA
// share fits the register file.  Thread `tid` owns the float4 chunks
// c = tid + j*512 (j < KJ) of every one of its CTA's units (s < SMAX): the
// prototypes never leave registers between steps.
//
// Costs that shape it (measured on B200, profiles/*_r01.*):
//  * fp32 -> fp64 conversion (F2F.F64.F32) issues at ~16/clk/SM, 4x slower
//    than the DADD/DFMA that follow, so x_t is converted once per step and
//    kept in registers as fp64; each prototype element costs one F2F.
//  * the tagged all-gather costs ~0.7-0.8 us at G <= 128 CTAs but ~1.6 us at
//    G = 148, so the host picks G <= 128.
//  * after the barrier that ends the fused pass, warp 0 alone is on the
//    critical path (key, publish, poll, neighbourhood): everything it does
//    there is kept short (per-lane unit sums, precomputed lattice
//    coordinates, x shift hidden behind the poll).
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;

__device__ __forceinline__ float4 eq1u(float h, float4 w, float4 x) {
    // Eq. 1 per element: w + h (x - w) as fmaf(h, RN(x - w), w)  (R11)
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

template <int SMAX, int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_reg_kernel(const TrainArgs a) {
    __shared__ double part[NW][SMAX];        // per-warp partial distance of each unit
    __shared__ float hs[SMAX];
    __shared__ int upd[SMAX];
    __shared__ int s_abort;
    extern __shared__ __align__(16) float xring[];   // [3][dimp]

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = (a.N - b + G - 1) / G;
    const int d4 = a.dimp >> 2;
    const float4* W4 = reinterpret_cast<const float4*>(a.W);
    float4* ring4 = reinterpret_cast<float4*>(xring);

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    float4 w[SMAX][KJ];
    float4 xp[KJ], xc[KJ];
    double xd[KJ][4];
#pragma unroll
    for (int s = 0; s < SMAX; ++s)
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s < Sb && valid[j]) v = W4[(int64_t)(b + s * G) * d4 + threadIdx.x + j * NT];
            w[s][j] = v;
        }
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        xp[j] = xc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        xd[j][0] = xd[j][1] = xd[j][2] = xd[j][3] = 0.0;
    }
    if (threadIdx.x < SMAX) { hs[threadIdx.x] = 0.0f; upd[threadIdx.x] = 0; }
    if (threadIdx.x == 0) s_abort = 0;
    // lattice coordinates of unit s = lane (warp 0, lanes < Sb)
    int my_i = 0, my_j = 0;
    if (lane < SMAX && lane < Sb) {
        const int u = global_unit(a, b + lane * G);
        my_i = u / a.cols;
        my_j = u - my_i * a.cols;
    }

    auto issue_x = [&](int64_t t) {
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + sample_at(a.seed, t, a.n) * (int64_t)a.dim);
            float4* dst = ring4 + (size_t)(t % 3) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (valid[j]) cp_async16(dst + threadIdx.x + j * NT, src + threadIdx.x + j * NT);
        }
        cp_async_commit();   // always one group per call (possibly empty)
    };
    // x_{t-1} <- x_t; x_t <- ring[t+1] (own chunks, landed: issued two steps ago)
    auto shift_x = [&](int64_t tnext) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        const float4* src = ring4 + (size_t)(tnext % 3) * d4;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            xp[j] = xc[j];
            if (valid[j]) {
                xc[j] = src[threadIdx.x + j * NT];
                xd[j][0] = (double)xc[j].x; xd[j][1] = (double)xc[j].y;
                xd[j][2] = (double)xc[j].z; xd[j][3] = (double)xc[j].w;
            }
        }
    };

    issue_x(a.t0);
    issue_x(a.t0 + 1);
    shift_x(a.t0);            // xc = x_{t0}, xd = fp64(x_{t0})
    __syncthreads();

    double f_cur = 0.0;
    for (int64_t t = a.t0; t < a.t1; ++t) {
        unsigned long long* tr = nullptr;   // optional phase trace (som_set_trace)
        if (a.trace && threadIdx.x == 0 && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
#define TRACE(p) do { if (tr) tr[p] = globaltimer_ns(); } while (0)
        TRACE(0);
        if (warp == 0) f_cur = a.f_tab[t - a.t0];   // consumed after the exchange

        // ---- fused pass on registers: pending update (t-1), then D_u(x_t)
        double acc[SMAX];
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            acc[s] = 0.0;
            if (s < Sb) {
                const float h = hs[s];
                const bool up = upd[s] != 0;
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int j = 0; j < KJ; ++j) {
                    if (valid[j]) {
                        if (up) w[s][j] = eq1u(h, w[s][j], xp[j]);
                        // R10: (double)x - (double)w, squared and summed in fp64
                        const double e0 = xd[j][0] - (double)w[s][j].x;
                        const double e1 = xd[j][1] - (double)w[s][j].y;
                        const double e2 = xd[j][2] - (double)w[s][j].z;
                        const double e3 = xd[j][3] - (double)w[s][j].w;
                        a0 = fma(e0, e0, a0);
                        a1 = fma(e1, e1, a1);
                        a0 = fma(e2, e2, a0);
                        a1 = fma(e3, e3, a1);
                    }
                }
                acc[s] = a0 + a1;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int s = 0; s < SMAX; ++s) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], o);
        if (lane == 0) {
#pragma unroll
            for (int s = 0; s < SMAX; ++s) part[warp][s] = acc[s];
        }
        TRACE(1);
        issue_x(t + 2);
        __syncthreads();   // A: partial distances ready
        TRACE(2);

        if (warp == 0) {
            // lane s sums its unit's 16 warp partials (fixed order), keys, min
            unsigned long long key = ~0ull;
            if (lane < SMAX && lane < Sb) {
                double tot = 0.0;
#pragma unroll
                for (int w8 = 0; w8 < NW; ++w8) tot += part[w8][lane];
                key = make_key((float)tot, global_unit(a, b + lane * G));
            }
#pragma unroll
            for (int o = SMAX / 2; o > 0; o >>= 1) key = umin64(key, __shfl_xor_sync(0xffffffffu, key, o));
            key = __shfl_sync(0xffffffffu, key, 0);

            xchg_publish(a, key, t, b, lane);
            TRACE(3);
            shift_x(t + 1);                       // hidden behind the poll
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            if (stop && lane == 0) s_abort = 1;
            const int c = key_unit(gmin);
            TRACE(4);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            if (lane < SMAX && lane < Sb) {
                // schedule (R1-R3) and neighbourhood of step t (R4, R5)
                const double alpha = a.alpha0 * f_cur;
                double sigma = a.sigma0 * f_cur;
                if (sigma < a.sigma_min) sigma = a.sigma_min;
                const double two_s2 = 2.0 * sigma * sigma;
                const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
                const int ic = c / a.cols, jc = c - ic * a.cols;
                const double di = (double)(my_i - ic);
                double g2;
                if (a.topo == 0) {
                    const double dj = (double)(my_j - jc);
                    g2 = di * di + dj * dj;
                } else {
                    const double dx2 = (double)(2 * (my_j - jc) + ((my_i & 1) - (ic & 1)));
                    g2 = 0.25 * (dx2 * dx2) + 0.75 * (di * di);
                }
                const bool up = g2 <= r2;
                upd[lane] = up ? 1 : 0;
                hs[lane] = up ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
            __syncwarp();
            TRACE(5);
        } else {
            shift_x(t + 1);
        }
        TRACE(6);
        __syncthreads();   // B: winner's neighbourhood ready
        TRACE(7);
#undef TRACE
        if (s_abort) break;
    }

    if (a.t1 > a.t0 && !s_abort) {
        // flush the update of the last step (x_{t1-1} is in xp)
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            if (s < Sb && upd[s]) {
                const float h = hs[s];
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (valid[j]) w[s][j] = eq1u(h, w[s][j], xp[j]);
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
                if (s < Sb && valid[j]) Wo[(int64_t)(b + s * G) * d4 + threadIdx.x + j * NT] = w[s][j];
    }
}

template <int SMAX, int KJ>
cudaError_t launch_one(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * 3 * (size_t)a.dimp;
    cudaError_t e = cudaFuncSetAttribute(som_train_reg_kernel<SMAX, KJ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    TrainArgs args = a;
    void* params[] = {&args};
    return launch_persistent((const void*)som_train_reg_kernel<SMAX, KJ>, a, NT, smem, params, st);
}

int smax_of(int S) { return S <= 1 ? 1 : S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : 99; }

}  // namespace

// Register budget (spill-free at 128 registers/thread): SMAX*KJ <= 8 float4
// prototype chunks plus x_{t-1}, x_t (fp32) and x_t (fp64) per chunk.
bool train_reg_supported(int S, int dim) {
    if (dim % 4 != 0) return false;
    const int kj = ((dim / 4) + NT - 1) / NT;
    return kj <= 4 && smax_of(S) * kj <= (kj == 4 ? 4 : 8);
}

cudaError_t launch_train_reg(const TrainArgs& a, cudaStream_t st) {
    const int kj = ((a.dimp / 4) + NT - 1) / NT;
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
