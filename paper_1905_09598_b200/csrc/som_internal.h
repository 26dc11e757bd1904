// som_internal.h — shared declarations between the libsom host runtime
// (som_api.cu) and its sm_100a kernels.  Product code: never includes or
// links anything under oracle/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace som {

constexpr int kTrainThreads = 512;                 // 16 warps per persistent CTA
constexpr int kTrainWarps = kTrainThreads / 32;
constexpr int kMaxUnits = (1 << 24) - 1;           // u fits the 24-bit key field

// Arguments of the persistent online-training kernel (train.cu).
struct TrainArgs {
    float* W;                  // N x dim, row-major, device
    const float* X;            // n x dim, row-major, device
    int64_t n;
    int dim;                   // vector length d
    int dimp;                  // d rounded up to a multiple of 4 (smem row stride)
    int rows, cols, topo;
    int N;                     // rows * cols
    int G;                     // grid size (co-resident CTAs)
    int S;                     // max units per CTA = ceil(N / G)
    int64_t t0, t1;            // step range
    uint64_t seed;
    const double* f_tab;       // decay factor f_t for t in [t0, t1)
    double alpha0, sigma0, sigma_min, ln_inv_eps;
    int cutoff_on;             // 0: every unit adapts (eps = 0)
    unsigned long long* xchg;  // [2][G] per-CTA BMU candidate slots
    unsigned int* abort_flag;  // set on exchange timeout
    int32_t* bmu_log;          // nullable, (t1 - t0) entries, device
    int w_smem;                // 1: the CTA's W rows live in shared memory
    int x_vec4;                // 1: X rows are 16-byte aligned (d % 4 == 0)
    unsigned long long* trace; // nullable: [G][trace_steps][kTracePhases] globaltimer (ns) per CTA
    int trace_steps;
};

constexpr int kTracePhases = 8;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

size_t train_smem_bytes(int S, int dimp, int w_smem);
cudaError_t launch_train(const TrainArgs& a, size_t smem, cudaStream_t st);
// register-resident variant (train_reg.cu): needs d % 4 == 0 and a small
// per-CTA share of W (S units x ceil(d/2048) float4 chunks per thread).
bool train_reg_supported(int S, int dim);
cudaError_t launch_train_reg(const TrainArgs& a, cudaStream_t st);

// Exact (fp64-accumulated) batch mapping: partial top-2 keys per doc per
// neuron split, then merged.  keys: [nsplit][n][2] u64 scratch.
struct MapArgs {
    const float* W; int N;
    const float* X; int64_t n; int dim;
    int nsplit;                // neuron ranges processed by separate CTAs
    unsigned long long* keys;  // [nsplit][n][2]
};
cudaError_t launch_map_exact(const MapArgs& a, cudaStream_t st);
cudaError_t launch_map_merge(const unsigned long long* keys, int nsplit, int64_t n,
                             int32_t* bmu1, int32_t* bmu2, float* d2, cudaStream_t st);
int map_exact_tiles_n(int N);
int map_exact_tiles_m(int64_t n);

// Tensor-core (tcgen05, 3xTF32) mapping, map_tc.cu.  Operands are split into
// tf32 hi/lo planes with K padded to tc_padded_dim(d); norms fp64 -> fp32.
int tc_padded_dim(int d);
int tc_unit_tiles(int N);
int tc_doc_blocks(int64_t n);
cudaError_t launch_split_rows(const float* src, int64_t rows, int d, float* hi, float* lo, float* norm, cudaStream_t st);
cudaError_t launch_split_csr(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0, int64_t rows,
                             int d, float* hi, float* lo, float* norm, cudaStream_t st);
cudaError_t launch_map_tc(const float* xhi, const float* xlo, const float* xnorm, int64_t n, const float* whi,
                          const float* wlo, const float* wnorm, int N, int d, unsigned long long* keys, int sm_count,
                          cudaStream_t st);

// CSR -> dense chunk (zero-filled) for the dense mapping paths.
cudaError_t launch_densify(const int64_t* rowptr, const int32_t* col, const float* val,
                           int64_t r0, int64_t nrows, int dim, float* out, cudaStream_t st);

// QE / TE partial sums (deterministic two-pass) and U-matrix.
cudaError_t launch_errors(const int32_t* bmu1, const int32_t* bmu2, const float* d2,
                          int64_t n, int rows, int cols, int topo, double* partial,
                          unsigned long long* partial_cnt, int nblocks, double* out_qe_sum,
                          unsigned long long* out_bad, cudaStream_t st);
cudaError_t launch_umatrix(const float* W, int rows, int cols, int topo, int dim, float* U,
                           cudaStream_t st);
cudaError_t launch_gather_rows(const float* X, const int64_t* idx, int N, int dim, float* W,
                               cudaStream_t st);

}  // namespace som
