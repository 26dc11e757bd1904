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

template <int SMAX, int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_reg_kernel(const TrainArgs a) {
    __shared__ double part[NW][SMAX];        // per-warp partial distance of each unit
    __shared__ int s_c, s_ic, s_jc;          // winner of the current step, its lattice row / column
    __shared__ int s_abort;
    extern __shared__ __align__(16) float xring[];   // [3][dimp] x ring, then the h table

    const int b = blockIdx.x, G = a.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int Sb = (a.N - b + G - 1) / G;
    const int d4 = a.dimp >> 2;
    const float4* W4 = reinterpret_cast<const float4*>(a.W);
    float4* ring4 = reinterpret_cast<float4*>(xring);
    // neighbourhood table of the step: h for every lattice offset
    // (|di|, |dj| rect or |2 dx| hex), -1 outside the cutoff (R4, R5)
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    const int HT = a.rows * W2;
    float* htab = xring + 3 * (size_t)a.dimp;

    bool valid[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) valid[j] = threadIdx.x + j * NT < d4;

    float4 w[SMAX][KJ];
    float4 xp[KJ], xc[KJ];
    double xd[KJ][4];
    float hh[SMAX];          // pending update of each unit (h, or < 0: none)
    int ui[SMAX], uj[SMAX];  // lattice coordinates of this CTA's units
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s < Sb && valid[j]) v = W4[(int64_t)(b + s * G) * d4 + threadIdx.x + j * NT];
            w[s][j] = v;
        }
        hh[s] = -1.0f;
        const int u = global_unit(a, b + s * G);
        ui[s] = u / a.cols;
        uj[s] = u - ui[s] * a.cols;
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        xp[j] = xc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        xd[j][0] = xd[j][1] = xd[j][2] = xd[j][3] = 0.0;
    }
    if (threadIdx.x == 0) s_abort = 0;

    auto issue_x = [&](int64_t t) {
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + train_row(a, t) * (int64_t)a.dim);
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

    for (int64_t t = a.t0; t < a.t1; ++t) {
        unsigned long long* tr = nullptr;   // optional phase trace (som_set_trace)
        if (a.trace && threadIdx.x == 0 && t - a.t0 < a.trace_steps)
            tr = a.trace + ((size_t)b * a.trace_steps + (size_t)(t - a.t0)) * kTracePhases;
#define TRACE(p) do { if (tr) tr[p] = trace_now(a.trace_clk); } while (0)
        TRACE(0);

        // ---- fused pass on registers: pending update (t-1), then D_u(x_t)
        double acc[SMAX];
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            acc[s] = 0.0;
            if (s < Sb) {
                const float h = hh[s];
                const bool up = h >= 0.0f;
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
        {
            int slot;
            const double v = butterfly_sum<SMAX>(acc, lane, &slot);
            if ((lane & (32 / SMAX - 1)) == 0) part[warp][slot] = v;
        }
        TRACE(1);
        issue_x(t + 2);
        __syncthreads();   // A: partial distances ready
        TRACE(2);

        if (warp == 0) {
            unsigned long long key = ~0ull;
            if constexpr (SMAX * 8 <= 32 && NW == 16) {
                // 8 lanes per unit, two warp partials each, a 3-level
                // butterfly (fixed order), then the min over the units
                const int su = lane >> 3, pi = (lane & 7) * 2;
                double v = 0.0;
                if (su < SMAX) v = part[pi][su] + part[pi + 1][su];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((lane & 7) == 0 && su < SMAX && su < Sb) key = make_key((float)v, global_unit(a, b + su * G));
#pragma unroll
                for (int o = 8; o < 8 * SMAX; o <<= 1) key = umin64(key, __shfl_xor_sync(0xffffffffu, key, o));
            } else {
                // lane s sums its unit's warp partials (fixed order), keys, min
                if (lane < SMAX && lane < Sb) {
                    double tot = 0.0;
#pragma unroll
                    for (int w8 = 0; w8 < NW; ++w8) tot += part[w8][lane];
                    key = make_key((float)tot, global_unit(a, b + lane * G));
                }
#pragma unroll
                for (int o = SMAX / 2; o > 0; o >>= 1) key = umin64(key, __shfl_xor_sync(0xffffffffu, key, o));
            }
            key = __shfl_sync(0xffffffffu, key, 0);

            xchg_publish(a, key, t, b, lane);
            // warps 1-15 start the neighbourhood table only now: beside the
            // key above it slowed it down on the step's critical path
            asm volatile("bar.arrive 3, %0;" ::"n"(NT) : "memory");
            TRACE(3);
            shift_x(t + 1);                       // hidden behind the poll
            int stop = 0;
            const unsigned long long gmin = xchg_wait(a, t, b, lane, &stop);
            const int c = key_unit(gmin);
            TRACE(4);
            if (lane == 0) {
                s_c = c;
                s_ic = c / a.cols;
                s_jc = c - s_ic * a.cols;
                if (stop) s_abort = 1;
                if (b == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            }
            TRACE(5);
        } else {
            asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory");   // warp 0 has published
            shift_x(t + 1);
            // neighbourhood table of step t (schedule R1-R3, kernel R4, cutoff
            // R5), built while warp 0 waits on the exchange
            const double f = a.f_tab[t - a.t0];
            const double alpha = a.alpha0 * f;
            double sigma = a.sigma0 * f;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            for (int e = threadIdx.x - 32; e < HT; e += NT - 32) {
                const int di = e / W2, dx = e - di * W2;
                const double ddi = (double)di, ddx = (double)dx;
                const double g2 = a.topo == 0 ? ddi * ddi + ddx * ddx : 0.25 * (ddx * ddx) + 0.75 * (ddi * ddi);
                htab[e] = g2 <= r2 ? (float)(alpha * exp(-g2 / two_s2)) : -1.0f;
            }
        }
        TRACE(6);
        __syncthreads();   // B: winner and neighbourhood table ready
        TRACE(7);
#undef TRACE
        if (s_abort) break;
        {
            // every thread looks up h for its CTA's units (exact g2 offsets)
            const int ic = s_ic, jc = s_jc;
#pragma unroll
            for (int s = 0; s < SMAX; ++s) {
                const int di = abs(ui[s] - ic);
                const int dx = a.topo == 0 ? abs(uj[s] - jc) : abs(2 * (uj[s] - jc) + ((ui[s] & 1) - (ic & 1)));
                hh[s] = s < Sb ? htab[di * W2 + dx] : -1.0f;
            }
        }
    }

    if (a.t1 > a.t0 && !s_abort) {
        // flush the update of the last step (x_{t1-1} is in xp)
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            if (s < Sb && hh[s] >= 0.0f) {
                const float h = hh[s];
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

size_t reg_smem_bytes(const TrainArgs& a) {
    const int W2 = a.topo == 0 ? a.cols : 2 * a.cols;
    return sizeof(float) * (3 * (size_t)a.dimp + (size_t)a.rows * W2);
}

template <int SMAX, int KJ>
cudaError_t launch_one(const TrainArgs& a, cudaStream_t st) {
    const size_t smem = reg_smem_bytes(a);
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
