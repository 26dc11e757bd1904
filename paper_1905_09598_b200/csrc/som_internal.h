// som_internal.h — shared declarations between the libsom host runtime
// (som_api.cu) and its sm_100a kernels.  Product code: never includes or
// links anything under oracle/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "som_device.cuh"

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
    int xstride;               // slots per exchange parity: G rounded up to 32 (parities on separate lines)
    int poll_ns;               // back-off between exchange polls (0: spin)
    unsigned long long spin_ns;   // exchange wait bound (globaltimer ns) before the abort
    int S;                     // max units per CTA = ceil(N / G)
    int64_t t0, t1;            // step range
    uint64_t seed;
    const double* f_tab;       // decay factor f_t for t in [t0, t1)
    // zero rows: draws go to rowmap[i] for i uniform over
    // [0, n_draw) (the non-zero rows, ascending); rowmap = NULL: no zero
    // row, draws uniform over [0, n)
    const int64_t* rowmap;
    int64_t n_draw;
    int sampling;              // 0: R8 (uniform with replacement), 1: R8b (per-epoch permutation)
    double alpha0, sigma0, sigma_min, ln_inv_eps;
    int cutoff_on;             // 0: every unit adapts (eps = 0)
    unsigned long long* xchg;  // [2][G] per-CTA BMU candidate slots
    unsigned int* abort_flag;  // set on exchange timeout
    int32_t* bmu_log;          // nullable, (t1 - t0) entries, device
    int w_smem;                // 1: the CTA's W rows live in shared memory
    int x_vec4;                // 1: X rows are 16-byte aligned (d % 4 == 0)
    unsigned long long* trace; // nullable: [G][trace_steps][kTracePhases] globaltimer (ns) per CTA
    int trace_steps;
    int trace_clk;             // 1: trace in SM cycles (clock64) instead of globaltimer ns
    // neuron sharding: this launch holds the N local units
    // l = 0..N-1 of global units u = rank + world * l; after the in-GPU
    // exchange, CTA 0 publishes the local winner into mail[p][t&1][rank] of
    // every rank p (peer memory over NVLink) and all CTAs poll mail[rank].
    int rank, world;
    unsigned long long* mail[8];
    // CSR input (train_csr.cu): x_t = row sample_at(t) of (rowptr, col, val)
    const int64_t* rowptr;
    const int32_t* col;
    const float* val;
    int nz_cap;                // per-step (col, val) list capacity in smem
    double g2max;              // largest lattice g2 between two units of the map
    // optional unit dealing (train_csr.cu): CTA b owns local units
    // utab[b * S + s], s < ucnt[b]; NULL = cyclic (b + s * G)
    const int* utab;
    const int* ucnt;
    // train_spec.cu: count of steps that took the exact fallback (nullable)
    unsigned long long* spec_fallbacks;
    // in-GPU exchange (xchg_publish / xchg_wait below): 0 = tagged
    // all-gather, 1 = one atomic max + an arrival counter, 2 = the tagged
    // all-gather read once a relaxed arrival counter says it is complete
    int xchg_atomic;
};

constexpr int kTracePhases = 8;
constexpr int kMaxRanks = 8;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// bounded exchange spin: checked every 256 polls against %globaltimer
struct Spin {
    unsigned n = 0;
    unsigned long long t0 = 0;
};

__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Per-step global argmin (warp 0 of every CTA; R9), in two calls so
// the caller can overlap work with the wait.  key: this CTA's min (D bits |
// global unit << 8).  Level 1: tagged all-gather over the G CTAs of this GPU
// (slots double-buffered by t&1: a CTA can only overwrite parity p after
// every CTA published the step in between, i.e. after all reads of parity
// p).  Level 2 (world > 1): CTA 0 forwards the GPU winner to every rank's
// mailbox (system-scope stores into peer memory); all CTAs poll their own
// mailbox.  Bounded spins: on timeout or a raised abort flag the wait
// returns with *stop = 1 (the host reports SOM_ECUDA, never hangs).
__device__ __forceinline__ unsigned long long xchg_tag(int64_t t) { return 0x80ull | (unsigned long long)(t & 0x7F); }

// Atomic variant (a.xchg_atomic): words [2 xstride, 2 xstride + 64) of the
// exchange buffer (zeroed before every launch) hold an arrival counter C
// (line 0) and three step words M[k] (lines 1..3).  Step t uses
// M[(t - t0) % 3]: every CTA does red.max(M, ~key) then
// red.add.release(C, 1); the wait polls C with acquire loads until it
// reaches G (t - t0 + 1), then reads M (its max of complemented keys is the
// min key: lowest (D, u), R9).  CTA 0 clears M[(t - 1 - t0) % 3] after the
// wait of step t: every CTA read it before arriving at step t, and nobody
// writes it again before step t + 2, whose writes follow CTA 0's arrival at
// step t + 1 (release) in every CTA's acquire order.
__device__ __forceinline__ unsigned long long* xa_count(const TrainArgs& a) { return a.xchg + 2 * (size_t)a.xstride; }
__device__ __forceinline__ unsigned long long* xa_word(const TrainArgs& a, int64_t t) {
    return a.xchg + 2 * (size_t)a.xstride + 16 * (1 + (int)((t - a.t0) % 3));
}

__device__ __forceinline__ void xchg_publish(const TrainArgs& a, unsigned long long key, int64_t t, int b, int lane) {
    if (a.xchg_atomic == 2) {   // tagged slot + relaxed arrival count (a polling hint)
        if (lane == 0) {
            st_relaxed_u64(a.xchg + (size_t)(t & 1) * a.xstride + b, (key & ~0xFFull) | xchg_tag(t));
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(xa_count(a)) : "memory");
        }
        return;
    }
    if (a.xchg_atomic) {
        if (lane == 0) {
            asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(xa_word(a, t)), "l"(~(key | 0xFFull)) : "memory");
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(xa_count(a)) : "memory");
        }
        return;
    }
    if (lane == 0) st_relaxed_u64(a.xchg + (size_t)(t & 1) * a.xstride + b, (key & ~0xFFull) | xchg_tag(t));
}

__device__ __forceinline__ bool xchg_should_stop(const TrainArgs& a, Spin& spins, int lane) {
    if ((++spins.n & 255u) != 0u) return false;
    const unsigned long long now = globaltimer_ns();
    if (spins.t0 == 0) spins.t0 = now;
    const bool s = now - spins.t0 > a.spin_ns || ld_relaxed_u32(a.abort_flag) != 0u;
    if (__any_sync(0xffffffffu, s)) {
        if (lane == 0) atomicExch(a.abort_flag, 1u);
        return true;
    }
    return false;
}

__device__ __forceinline__ unsigned long long xchg_wait(const TrainArgs& a, int64_t t, int b, int lane, int* stop) {
    const unsigned long long tag = xchg_tag(t);
    const unsigned long long* slots = a.xchg + (size_t)(t & 1) * a.xstride;
    unsigned long long gmin = 0;
    Spin spins;
    if (a.xchg_atomic == 2) {   // wait for the count, then read (and validate) the tagged slots
        const unsigned long long want = (unsigned long long)a.G * (unsigned long long)(t - a.t0 + 1);
        for (;;) {
            const unsigned long long c = __shfl_sync(0xffffffffu, ld_relaxed_u64(xa_count(a)), 0);
            if (c >= want) break;
            if (xchg_should_stop(a, spins, lane)) { *stop = 1; return 0; }
            if (a.poll_ns > 0) __nanosleep(a.poll_ns);
        }
    } else if (a.xchg_atomic) {
        const unsigned long long want = (unsigned long long)a.G * (unsigned long long)(t - a.t0 + 1);
        for (;;) {
            unsigned long long c;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(xa_count(a)) : "memory");
            if (__shfl_sync(0xffffffffu, c, 0) >= want) break;
            if (xchg_should_stop(a, spins, lane)) { *stop = 1; return 0; }
            if (a.poll_ns > 0) __nanosleep(a.poll_ns);
        }
        gmin = (~ld_relaxed_u64(xa_word(a, t)) & ~0xFFull) | tag;
        if (b == 0 && lane == 0 && t > a.t0) st_relaxed_u64(xa_word(a, t - 1), 0ull);
    }
    for (; a.xchg_atomic != 1;) {
        unsigned long long m = ~0ull;
        bool ok = true;
        for (int j = lane; j < a.G; j += 32) {
            const unsigned long long v = ld_relaxed_u64(slots + j);
            ok &= (v & 0xFFull) == tag;
            m = umin64(m, v);
        }
        if (__all_sync(0xffffffffu, ok)) { gmin = warp_min_u64(m); break; }
        if (xchg_should_stop(a, spins, lane)) { *stop = 1; return 0; }
        if (a.poll_ns > 0) __nanosleep(a.poll_ns);
    }
    if (a.world <= 1) return gmin;
    const size_t par = (size_t)(t & 1) * a.world;
    if (b == 0 && lane < a.world) st_relaxed_sys_u64(a.mail[lane] + par + a.rank, gmin);
    const unsigned long long* mine = a.mail[a.rank] + par;
    spins = Spin{};
    for (;;) {
        unsigned long long v = ~0ull;
        bool ok = true;
        if (lane < a.world) { v = ld_relaxed_sys_u64(mine + lane); ok = (v & 0xFFull) == tag; }
        if (__all_sync(0xffffffffu, ok)) return warp_min_u64(v);
        if (xchg_should_stop(a, spins, lane)) { *stop = 1; return 0; }
    }
}

// Launch a persistent training grid.  Single rank: cooperative launch (the
// driver guarantees all G CTAs are co-resident).  Neuron-sharded: a plain
// launch after checking that G CTAs fit at once (one per SM), so that ranks
// emulated on one device (tests) can run their grids concurrently; each
// rank of a real multi-GPU run owns its device.
inline cudaError_t launch_persistent(const void* fn, const TrainArgs& a, int threads, size_t smem, void** params,
                                     cudaStream_t st) {
    if (a.world <= 1) return cudaLaunchCooperativeKernel(fn, dim3(a.G), dim3(threads), params, smem, st);
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    if (e != cudaSuccess) return e;
    if (a.G > sms * per_sm) return cudaErrorCooperativeLaunchTooLarge;
    return cudaLaunchKernel(fn, dim3(a.G), dim3(threads), params, smem, st);
}

// R8 + S:218: the row drawn at step t (uniform over the non-zero rows)
__device__ __forceinline__ int64_t train_row(const TrainArgs& a, int64_t t) {
    const int64_t m = a.rowmap ? a.n_draw : a.n;
    const int64_t j = a.sampling == 1 ? perm_at(a.seed, t, m) : sample_at(a.seed, t, m);
    return a.rowmap ? __ldg(a.rowmap + j) : j;
}

// global unit index of local unit l
__device__ __forceinline__ int global_unit(const TrainArgs& a, int l) { return a.rank + a.world * l; }
// trace clock: %globaltimer (ns, comparable across SMs, coarse) or, with
// SOM_TRACE_CLOCK=1, the SM cycle counter (fine, per-SM only)
__device__ __forceinline__ unsigned long long trace_now(int clk) {
    if (clk) {
        unsigned long long c;
        asm volatile("mov.u64 %0, %clock64;" : "=l"(c));
        return c;
    }
    return globaltimer_ns();
}

size_t train_smem_bytes(int S, int dimp, int w_smem);
cudaError_t launch_train(const TrainArgs& a, size_t smem, cudaStream_t st);
// register-resident variant (train_reg.cu): needs d % 4 == 0 and a small
// per-CTA share of W (S units x ceil(d/2048) float4 chunks per thread).
bool train_reg_supported(int S, int dim);
cudaError_t launch_train_reg(const TrainArgs& a, cudaStream_t st);
bool train_spec_supported(int S, int dim, int G, int world);
cudaError_t launch_train_spec(const TrainArgs& a, cudaStream_t st);
// pipelined global-memory variant (train_glb.cu) for maps that do not fit on chip
bool train_glb_supported(int S, int dim);
cudaError_t launch_train_glb(const TrainArgs& a, cudaStream_t st);

// short-prototype variant (train_small.cu): d <= 128, d % 4 == 0; a group
// of small_lanes(d) lanes per unit (4 float4 per lane); W in registers for
// up to 4 rounds of 16*32/L units per CTA, else streamed from global memory
bool train_small_supported(int dim);
int small_lanes(int dim);
int small_rounds(int S, int dim);
cudaError_t launch_train_small(const TrainArgs& a, cudaStream_t st);

// CSR-input variant with the sparse distance path (train_csr.cu)
int csr_nz_cap(int maxnnz);
bool train_csr_supported(int S, int dim, int maxnnz, int max_smem_optin);
cudaError_t launch_train_csr(const TrainArgs& a, cudaStream_t st);
// tiered-storage variant (train_tier.cu, kernel 10): rows in registers,
// TMEM, shared memory, the rest streamed through a chunked TMA ring
bool train_tier_supported(int S, int dim, int maxnnz, int max_smem_optin);
cudaError_t launch_train_tier(const TrainArgs& a, int max_smem_optin, cudaStream_t st);
// CSR validation: out[0] error bits (1 rowptr, 2 col range, 4 col order),
// out[1] max nonzeros per row (device ints)
cudaError_t launch_csr_check(const int64_t* rowptr, const int32_t* col, int64_t n, int dim, int* out,
                             cudaStream_t st);

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
// tf32 hi/lo planes with K padded to tc_padded_dim(d); fp64 norms and the
// count of 8-wide K groups holding a non-zero (groups nullable).
int tc_padded_dim(int d);
int tc_unit_tiles(int N);
int tc_doc_blocks(int64_t n);
constexpr int kTcCand = 4;   // candidates per document of the certified rescoring (R20b)
cudaError_t launch_split_rows(const float* src, int64_t rows, int d, float* hi, float* lo, double* norm, int* groups,
                              cudaStream_t st);
cudaError_t launch_split_csr(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0, int64_t rows,
                             int d, float* hi, float* lo, double* norm, int* groups, cudaStream_t st);
cudaError_t launch_map_tc(const float* xhi, const float* xlo, const double* xnorm, int64_t n, const float* whi,
                          const float* wlo, const double* wnorm, int N, int d, unsigned long long* keys, int sm_count,
                          cudaStream_t st);
cudaError_t launch_wmax(const double* wn, int N, double* out, cudaStream_t st);
bool tc_rescore_fits(int d);
cudaError_t launch_tc_rescore(const unsigned long long* keys, int64_t n, const int64_t* rowptr, const int32_t* col,
                              const float* val, int64_t r0, const float* X, const float* W, int N, int d,
                              const double* xnorm, const double* wnorm, const int* groups, const double* wmax,
                              int32_t* bmu1, int32_t* bmu2, float* d2, int* nfall, cudaStream_t st);

// Exact sparse mapping (map_sparse.cu, R25): W^T (dim x Np, Np = N padded
// to the 64 J-unit tile; fp64, or fp32 widened exactly in registers) +
// |w|^2 fp64; partial top-2 keys [Np / (64 J)][m][2] per chunk of m CSR
// rows starting at r0, merged by launch_map_merge.  (J, f32) in
// {1,2,4} x fp64, {2,4,8} x fp32.
int sparse_tile_units(int J);
int sparse_padded_units(int N, int J);
// *flag (device int) is set when W holds a negative, subnormal, infinite or
// NaN value; otherwise the fp32 variants may widen half of the values on the
// integer pipe (icv).
cudaError_t launch_wt(const float* W, int N, int d, int Np, bool f32, void* WT, double* wsq, int* flag,
                      cudaStream_t st);
cudaError_t launch_map_sparse(const int64_t* rowptr, const int32_t* col, const float* val, int64_t r0, int64_t m,
                              const void* WT, bool f32, bool icv, const double* wsq, int N, int Np, int J,
                              unsigned long long* keys, cudaStream_t st);

// Batch SOM epoch pieces (batch.cu, R27): bucket documents by BMU (stable
// radix sort; scratch 2 n int32), per-BMU fp64 sums S (N x (d+1), column d
// = count), then num = H S with the separable lattice kernel and
// W = RN32(num / den) where den > 0.
size_t batch_sort_temp_bytes(int64_t n, int N);
cudaError_t launch_batch_bucket(const int32_t* bmu, int64_t n, int N, int32_t* order, int32_t* cnt, int32_t* off,
                                int32_t* scratch, void* temp, size_t temp_bytes, cudaStream_t st);
cudaError_t launch_batch_accumulate_dense(const float* X, int d, const int32_t* order, const int32_t* off,
                                          const int32_t* cnt, int N, double* S, cudaStream_t st);
size_t batch_csr_temp_bytes(int64_t nnz);
cudaError_t launch_batch_accumulate_csr(const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                                        int64_t nnz, int d, const int32_t* bmu, const int32_t* cnt, int N, double* S,
                                        void* work, void* temp, size_t temp_bytes, cudaStream_t st);
cudaError_t launch_batch_update(const double* S, double* num, int N, int d, int rows, int cols, int topo,
                                double sigma, double r2, float* W, cudaStream_t st);

// Upstream steps (upstream.cu, R28-R30): TF-IDF + L2 rows; top-2 PCA by
// subspace iteration (block kPcaBlock) on the implicitly centred covariance;
// PCA-plane linear init.
constexpr int kPcaBlock = 8;
cudaError_t launch_tfidf(const int64_t* rowptr, const int32_t* col, const float* cnt, int64_t n, int d, int64_t nnz,
                         int* df, double* idf, float* out, unsigned long long* zero_rows, cudaStream_t st);
struct PcaInput {
    const float* X;          // dense n x d rows, or null for CSR
    const int64_t* rowptr;   // CSR (rowptr[0] == 0)
    const int32_t* col;
    const float* val;
    int64_t n;
    int d;
    const int* cptr;         // column-major copy: d + 1 offsets
    const int32_t* cent;     // entries in column order (rows ascending within a column)
    const int32_t* erow;     // row of each entry
};
size_t pca_csc_temp_bytes(int64_t nnz, int d);
cudaError_t launch_pca_csc(const int64_t* rowptr, const int32_t* col, int64_t n, int d, int64_t nnz, int* cptr,
                           int32_t* cent, int32_t* erow, int32_t* scratch, void* temp, size_t temp_bytes,
                           cudaStream_t st);
cudaError_t launch_pca_mean(const PcaInput& x, double* mu, cudaStream_t st);
cudaError_t launch_pca_init_q(double* Q, int d, uint64_t seed, cudaStream_t st);
cudaError_t launch_pca_apply(const PcaInput& x, const double* mu, double* Q, double* Y, double* Z, int orth,
                             cudaStream_t st);
cudaError_t launch_pca_orth(double* Z, double* Q, int d, cudaStream_t st);
cudaError_t launch_pca_rr(const PcaInput& x, const double* mu, double* Q, double* Y, double* Z, double* out,
                          cudaStream_t st);
cudaError_t launch_pca_extract(const double* Q, int d, double* v1, double* v2, cudaStream_t st);
cudaError_t launch_init_linear(float* W, int rows, int cols, int d, const double* mu, const double* v1,
                               const double* v2, double pc1, double pc2, cudaStream_t st);

// dense rows -> CSR (column order), for SOM_MAP_SPARSE_F64 on dense input:
// rowptr from per-row counts (cnt: m + 1 int64 scratch), then col / val
size_t dense_csr_temp_bytes(int64_t m);
cudaError_t launch_dense_rowptr(const float* X, int64_t m, int d, int64_t* cnt, int64_t* rowptr, void* temp,
                                size_t temp_bytes, cudaStream_t st);
cudaError_t launch_dense_fill(const float* X, int64_t m, int d, const int64_t* rowptr, int32_t* col, float* val,
                              cudaStream_t st);

// CSR -> dense chunk (zero-filled) for the dense mapping paths.
cudaError_t launch_densify(const int64_t* rowptr, const int32_t* col, const float* val,
                           int64_t r0, int64_t nrows, int dim, float* out, cudaStream_t st);

// QE / TE partial sums (deterministic two-pass) over the rows with
// keep[i] != 0 (keep nullable = every row), and U-matrix.
cudaError_t launch_errors(const int32_t* bmu1, const int32_t* bmu2, const float* d2, const uint8_t* keep,
                          int64_t n, int rows, int cols, int topo, double* partial,
                          unsigned long long* partial_cnt, int nblocks, double* out_qe_sum,
                          unsigned long long* out_bad, cudaStream_t st);

// zero rows (rows.cu): flags[i] = row i holds a non-zero value; the
// ascending list of flagged rows (CUB select, temp from
// select_rows_temp_bytes) and its length (device int64)
cudaError_t launch_row_flags_dense(const float* X, int64_t n, int dim, uint8_t* flags, cudaStream_t st);
cudaError_t launch_row_flags_csr(const int64_t* rowptr, const float* val, int64_t n, uint8_t* flags,
                                 cudaStream_t st);
size_t select_rows_temp_bytes(int64_t n);
cudaError_t launch_select_rows(const uint8_t* flags, int64_t n, int64_t* idx, int64_t* count, void* temp,
                               size_t temp_bytes, cudaStream_t st);
cudaError_t launch_umatrix(const float* W, int rows, int cols, int topo, int dim, float* U,
                           cudaStream_t st);
cudaError_t launch_gather_rows(const float* X, const int64_t* idx, int N, int dim, float* W,
                               cudaStream_t st);
cudaError_t launch_gather_csr_rows(const int64_t* rowptr, const int32_t* col, const float* val, const int64_t* idx,
                                   int N, int dim, float* W, cudaStream_t st);

}  // namespace som
