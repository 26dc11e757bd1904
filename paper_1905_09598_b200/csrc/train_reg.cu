// train_reg.cu — register-resident persistent online-SOM training kernel.
//
// Same step as train.cu (pending Eq. 1 update of step t-1 fused with the
// fp64 distance pass of step t, packed (D, u) keys, tagged all-gather of
// per-CTA minima, R9-R11), specialised for maps whose per-CTA
// share fits the register file: each thread owns the float4 chunks
// c = tid + j*512 (j < KJ) of every one of its CTA's units (s < SMAX), so
// the prototypes never leave registers between steps and x_t / x_{t-1} are
// per-thread registers too.  x_{t+2} is prefetched with cp.async (each
// thread copies exactly the chunks it later reads, so no barrier is needed
// for x).  Grid size G is chosen on the host: the all-gather costs ~0.6 us
// at G <= 64 but ~1.6 us at G = 148 (profiles/probe_xchg_r01.json), so for
// small maps fewer, fuller CTAs win.
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr unsigned kSpinLimitR = 1u << 24;
constexpr int NT = kTrainThreads;
constexpr int NW = kTrainWarps;

__device__ __forceinline__ float4 eq1u(float h, float4 w, float4 x) {
    w.x = fmaf(h, x.x - w.x, w.x);
    w.y = fmaf(h, x.y - w.y, w.y);
    w.z = fmaf(h, x.z - w.z, w.z);
    w.w = fmaf(h, x.w - w.w, w.w);
    return w;
}

__device__ __forceinline__ double dist4(float4 x, float4 w) {
    double d0 = (double)x.x - (double)w.x;
    double d1 = (double)x.y - (double)w.y;
    double d2 = (double)x.z - (double)w.z;
    double d3 = (double)x.w - (double)w.w;
    double a = d0 * d0;          // exact square would also be fine; keep fma chain short
    a = fma(d1, d1, a);
    double b = d2 * d2;
    b = fma(d3, d3, b);
    return a + b;
}

template <int SMAX, int KJ>
__global__ void __launch_bounds__(NT, 1) som_train_reg_kernel(const TrainArgs a) {
    __shared__ double part[SMAX][NW];
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

    float4 w[SMAX][KJ];
    float4 xp[KJ], xc[KJ];
#pragma unroll
    for (int s = 0; s < SMAX; ++s)
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            const int c = threadIdx.x + j * NT;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s < Sb && c < d4) v = W4[(int64_t)(b + s * G) * d4 + c];
            w[s][j] = v;
        }
#pragma unroll
    for (int j = 0; j < KJ; ++j) xp[j] = xc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x < SMAX) { hs[threadIdx.x] = 0.0f; upd[threadIdx.x] = 0; }
    if (threadIdx.x == 0) s_abort = 0;

    auto issue_x = [&](int64_t t) {
        if (t < a.t1) {
            const float4* src = reinterpret_cast<const float4*>(a.X + sample_at(a.seed, t, a.n) * (int64_t)a.dim);
            float4* dst = ring4 + (size_t)(t % 3) * d4;
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                const int c = threadIdx.x + j * NT;
                if (c < d4) cp_async16(dst + c, src + c);
            }
        }
        cp_async_commit();   // always one group per call (possibly empty)
    };
    auto read_x = [&](int64_t t) {
        const float4* src = ring4 + (size_t)(t % 3) * d4;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            const int c = threadIdx.x + j * NT;
            xc[j] = c < d4 ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };

    issue_x(a.t0);
    issue_x(a.t0 + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    read_x(a.t0);
    __syncthreads();

    double f_cur = 0.0;
    for (int64_t t = a.t0; t < a.t1; ++t) {
        if (warp == 0) f_cur = a.f_tab[t - a.t0];   // off the critical path

        // ---- fused pass on registers: update (t-1) + D_u(x_t)
        double acc[SMAX];
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            acc[s] = 0.0;
            if (s < Sb) {
                const float h = hs[s];
                const bool up = upd[s] != 0;
#pragma unroll
                for (int j = 0; j < KJ; ++j) {
                    if (up) w[s][j] = eq1u(h, w[s][j], xp[j]);
                    acc[s] += dist4(xc[j], w[s][j]);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int s = 0; s < SMAX; ++s) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], o);
        if (lane == 0) {
#pragma unroll
            for (int s = 0; s < SMAX; ++s) part[s][warp] = acc[s];
        }
        issue_x(t + 2);
        __syncthreads();   // A: partial distances ready

        if (warp == 0) {
            // lanes over (unit, half of the warps): 16 partials per unit
            unsigned long long best = ~0ull;
#pragma unroll
            for (int s0 = 0; s0 < SMAX; s0 += 2) {
                const int s = s0 + (lane >> 4);
                double v = (s < Sb && s < SMAX) ? part[s < SMAX ? s : 0][lane & 15] : 0.0;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if ((lane & 15) == 0 && s < Sb) best = umin64(best, make_key((float)v, b + s * G));
            }
            best = warp_min_u64(best);

            const unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* slots = a.xchg + (size_t)(t & 1) * G;
            if (lane == 0) st_relaxed_u64(slots + b, (best & ~0xFFull) | tag);
            unsigned long long gmin = 0;
            unsigned spins = 0;
            for (;;) {
                unsigned long long m = ~0ull;
                bool ok = true;
                for (int j = lane; j < G; j += 32) {
                    unsigned long long v = ld_relaxed_u64(slots + j);
                    ok &= (v & 0xFFull) == tag;
                    m = umin64(m, v);
                }
                if (__all_sync(0xffffffffu, ok)) { gmin = warp_min_u64(m); break; }
                if ((++spins & 255u) == 0u) {
                    bool stop = spins > kSpinLimitR || ld_relaxed_u32(a.abort_flag) != 0u;
                    if (__any_sync(0xffffffffu, stop)) {
                        if (lane == 0) { atomicExch(a.abort_flag, 1u); s_abort = 1; }
                        break;
                    }
                }
            }
            const int c = key_unit(gmin);
            if (b == 0 && lane == 0 && a.bmu_log) a.bmu_log[t - a.t0] = c;
            const double alpha = a.alpha0 * f_cur;
            double sigma = a.sigma0 * f_cur;
            if (sigma < a.sigma_min) sigma = a.sigma_min;
            const double two_s2 = 2.0 * sigma * sigma;
            const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
            if (lane < SMAX && lane < Sb) {
                const double g2 = lattice_g2(a.cols, a.topo, b + lane * G, c);
                const bool up = g2 <= r2;
                upd[lane] = up ? 1 : 0;
                hs[lane] = up ? (float)(alpha * exp(-g2 / two_s2)) : 0.0f;
            }
        }
        // x_{t-1} <- x_t, x_t <- x_{t+1} (own chunks; landed two steps after issue)
#pragma unroll
        for (int j = 0; j < KJ; ++j) xp[j] = xc[j];
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        read_x(t + 1);
        __syncthreads();   // B: winner's neighbourhood ready
        if (s_abort) break;
    }

    if (a.t1 > a.t0 && !s_abort) {
        // flush the update of the last step (x_{t1-1} is in xp)
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            if (s < Sb && upd[s]) {
                const float h = hs[s];
#pragma unroll
                for (int j = 0; j < KJ; ++j) w[s][j] = eq1u(h, w[s][j], xp[j]);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (!s_abort) {
        float4* Wo = reinterpret_cast<float4*>(a.W);
#pragma unroll
        for (int s = 0; s < SMAX; ++s)
#pragma unroll
            for (int j = 0; j < KJ; ++j) {
                const int c = threadIdx.x + j * NT;
                if (s < Sb && c < d4) Wo[(int64_t)(b + s * G) * d4 + c] = w[s][j];
            }
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
    return cudaLaunchCooperativeKernel((const void*)som_train_reg_kernel<SMAX, KJ>, dim3(a.G), dim3(NT), params,
                                       smem, st);
}

}  // namespace

// Register budget: SMAX*KJ float4 prototypes (<= 64 floats per thread).
bool train_reg_supported(int S, int dim) {
    if (dim % 4 != 0) return false;
    const int kj = ((dim / 4) + NT - 1) / NT;
    if (kj > 4) return false;
    if (kj == 4 && S > 2) return false;   // keep the register tile spill-free
    const int smax = S <= 1 ? 1 : S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 99;
    return smax * kj <= 16;
}

cudaError_t launch_train_reg(const TrainArgs& a, cudaStream_t st) {
    const int kj = ((a.dimp / 4) + NT - 1) / NT;
    const int S = a.S;
#define TRY(SM, K) if (S <= SM && kj == K) return launch_one<SM, K>(a, st)
    TRY(1, 1); TRY(2, 1); TRY(4, 1); TRY(8, 1); TRY(16, 1);
    TRY(1, 2); TRY(2, 2); TRY(4, 2); TRY(8, 2);
    TRY(1, 3); TRY(2, 3); TRY(4, 3);
    TRY(1, 4); TRY(2, 4);
#undef TRY
    return cudaErrorInvalidConfiguration;
}

}  // namespace som
