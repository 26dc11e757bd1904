// train_step.cu — the step-at-a-time training path whose per-step winner
// exchange is an NCCL all-reduce (SURVEY §8.E "baseline exchange":
// ncclAllReduce(key, 1, ncclUint64, ncclMin), host-driven per step, the
// launches captured in CUDA graphs).  It is the reference point the in-kernel
// peer-memory mailbox of the persistent kernels is measured against, and it
// serves neuron-sharded handles that have an NCCL communicator but no peer
// mailboxes.  Same arithmetic as every other training kernel (Eq. 1 P:108,
// R4, R5, R9-R11), one CTA per local unit:
//   kernel(t): pending Eq. 1 update of step t-1 with the winner of t-1 (the
//              reduced key of slot (t-1) % 3), then D_u(x_t) in fp64 (R10),
//              CTA argmin, atomicMin into slot t % 3;
//   all-reduce(slot t % 3, min) over the ranks;
//   kernel(t+1) ...
// The slot of t+1 is reset by kernel t (nobody reads it during step t).
#include "som_device.cuh"
#include "som_internal.h"

namespace som {

namespace {

constexpr int kStepThreads = 256;

struct StepArgs {
    TrainArgs a;
    unsigned long long* keys;   // [3]
    const int* chunk;           // graph replays: t = t_first + (*chunk) * K + i (nullptr: t = t_first + i)
    int K;
};

__device__ __forceinline__ int64_t step_t(const StepArgs& s, int64_t t_first, int i) {
    return t_first + (s.chunk ? (int64_t)(*s.chunk) * s.K : 0) + i;
}

// update of step t-1 (if t > t0) fused with the distance of step t (if t < t1)
__global__ void __launch_bounds__(kStepThreads) som_step_kernel(const StepArgs s, int64_t t_first, int i) {
    __shared__ double red[kStepThreads / 32];
    __shared__ int s_c;
    const TrainArgs& a = s.a;
    const int64_t t = step_t(s, t_first, i);
    const int l = blockIdx.x;
    const int u = global_unit(a, l);
    float* w = a.W + (int64_t)l * a.dim;
    float h = 0.0f;
    bool upd = false;
    const float* xp = nullptr;
    if (t > a.t0) {
        if (threadIdx.x == 0) s_c = key_unit(s.keys[(t - 1) % 3]);
        __syncthreads();
        const int c = s_c;
        if (l == 0 && threadIdx.x == 0 && a.bmu_log) a.bmu_log[t - 1 - a.t0] = c;
        const double f = a.f_tab[t - 1 - a.t0];
        const double alpha = a.alpha0 * f;
        double sigma = a.sigma0 * f;
        if (sigma < a.sigma_min) sigma = a.sigma_min;
        const double two_s2 = 2.0 * sigma * sigma;
        const double r2 = a.cutoff_on ? two_s2 * a.ln_inv_eps : INFINITY;
        const double g2 = lattice_g2(a.cols, a.topo, u, c);
        upd = g2 <= r2;
        if (upd) h = (float)(alpha * exp(-g2 / two_s2));
        xp = a.X + train_row(a, t - 1) * (int64_t)a.dim;
    }
    if (t < a.t1) {
        if (l == 0 && threadIdx.x == 0) s.keys[(t + 1) % 3] = ~0ull;   // slot of step t+1 (read by nobody now)
        const float* xt = a.X + train_row(a, t) * (int64_t)a.dim;
        double acc = 0.0;
        for (int k = threadIdx.x; k < a.dim; k += kStepThreads) {
            float wk = w[k];
            if (upd) {
                wk = fmaf(h, xp[k] - wk, wk);
                w[k] = wk;
            }
            const double e = (double)xt[k] - (double)wk;
            acc = fma(e, e, acc);
        }
        acc = warp_sum_f64(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int q = 0; q < kStepThreads / 32; ++q) tot += red[q];
            atomicMin(s.keys + t % 3, make_key((float)tot, u));
        }
    } else if (upd) {   // final flush: the update of the last step only
        for (int k = threadIdx.x; k < a.dim; k += kStepThreads) w[k] = fmaf(h, xp[k] - w[k], w[k]);
    }
}

__global__ void step_chunk_inc_kernel(int* chunk) { ++*chunk; }

}  // namespace

cudaError_t launch_step(const TrainArgs& a, unsigned long long* keys, const int* chunk, int K, int64_t t_first, int i,
                        cudaStream_t st) {
    StepArgs s{a, keys, chunk, K};
    som_step_kernel<<<a.N, kStepThreads, 0, st>>>(s, t_first, i);
    return cudaGetLastError();
}

cudaError_t launch_step_chunk_inc(int* chunk, cudaStream_t st) {
    step_chunk_inc_kernel<<<1, 1, 0, st>>>(chunk);
    return cudaGetLastError();
}

}  // namespace som
