/*
 * som.h — C ABI of libsom, the B200 (sm_100a) implementation of the CUDASOM
 * hot path (Gavval et al., arXiv 1905.09598): online Kohonen SOM training
 * (distance -> argmin BMU -> Gaussian-neighbourhood update, Eq. 1), batch
 * BMU mapping, quantization / topographic error and the U-matrix.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rn = reading n in
 * DESIGN.md §3 (where the paper is silent, ambiguous or garbled).
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Plain C: no C++ types, no exceptions, no torch types.  Every call
 *    returns a som_status; SOM_OK = 0.  A human-readable message for the
 *    last failure on the calling thread is returned by som_last_error().
 *  - Ownership: the handle owns the map W (rows*cols x dim fp32, row-major,
 *    unit u = i*cols + j) and all device scratch.  Inputs X and
 *    all outputs are caller-owned and may be HOST or DEVICE pointers (device
 *    memory of the handle's device; detected per pointer).  Host buffers are
 *    staged through device scratch inside the call.  The library keeps no
 *    caller pointer after a call returns.
 *  - Layout: X is n x dim fp32 row-major (one L2-normalised TF-IDF document
 *    per row).  CSR inputs use int64 rowptr[n+1], int32
 *    col[nnz] and fp32 val[nnz].
 *  - Synchrony: calls run on the handle's stream (som_set_stream; default a
 *    stream the handle creates) and return after that work completes.
 *  - Validation happens before any side effect: SOM_EINVAL for bad sizes or
 *    parameters, SOM_EEMPTY for n = 0 where data is required.
 *  - A CUDA failure returns SOM_ECUDA and poisons the handle: every later
 *    call except som_destroy returns SOM_ESTATE.
 *  - Thread safety: one handle must not be used concurrently; distinct
 *    handles are independent.
 *  - Determinism: identical inputs and seed give bit-identical W, BMU log
 *    and mapping outputs on every run.
 *  - There is no CPU fallback: without a usable sm_100a device som_create
 *    fails with SOM_ECUDA.
 *  - Tuning / diagnostic environment variables (read per call; results do
 *    not depend on them unless stated): SOM_SPARSE_J (1|2|4|8: unit tile
 *    64 J of the sparse mapping), SOM_SPARSE_F32 (0: fp64 W^T),
 *    SOM_SPARSE_ICV (0: no integer-pipe widening), SOM_SPARSE_DPC
 *    (documents per CTA), SOM_NO_TMA_RING (1: register-pipelined streamed
 *    training kernel), SOM_NO_L2_WINDOW (1: no persisting L2 window),
 *    SOM_POLL_NS (back-off between exchange polls), SOM_TRACE_CLOCK (1:
 *    som_set_trace records SM cycles), SOM_XCHG_ATOMIC (in-GPU winner
 *    exchange: 0 tagged all-gather, 1 atomic max + arrival counter, 2 the
 *    all-gather read once a relaxed arrival counter is complete; default 2
 *    from 96 CTAs, else 0), SOM_TIER_NDW (12|16: kernel 10's data warps),
 *    SOM_TIER_COVER (kernel 10 -> 4 hand-over coverage, default 0.4),
 *    SOM_DENSE_COVER (kernel 3 -> 4 hand-over coverage of kernel 12,
 *    default 0.6; 0 = kernel 4 throughout).
 *    Every variant they select is covered by the parity tests.
 */
#ifndef SOM_H
#define SOM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct som_ctx som_ctx; /* opaque handle */

typedef enum {
    SOM_OK = 0,
    SOM_EINVAL = 1,      /* bad size / parameter / t-range                     */
    SOM_EDIM = 2,        /* dimension mismatch                 */
    SOM_EEMPTY = 3,      /* n = 0 where data is required              */
    SOM_ENOMEM = 4,      /* device or host allocation failed                  */
    SOM_ECUDA = 5,       /* CUDA runtime/launch failure (handle poisoned)     */
    SOM_ENCCL = 6,       /* NCCL failure (handle poisoned)                    */
    SOM_ESTATE = 7,      /* handle poisoned by an earlier failure             */
    SOM_EUNSUPPORTED = 8 /* valid request this build/device cannot serve      */
} som_status;

typedef enum { SOM_RECT = 0, SOM_HEX = 1 } som_topology; /* P:166 hex; rect BJ:7 */

typedef enum {
    SOM_DECAY_GAUSSIAN = 0, /* f = exp(-k tau^2)   (R1, "Gaussian decay") */
    SOM_DECAY_LINEAR = 1,   /* f = 1 - (1 - e^-k) tau                          */
    SOM_DECAY_EXP = 2       /* f = exp(-k tau)                                 */
} som_decay_kind;

/* Decay schedule (R1-R6): tau = t/T, alpha_t = alpha0 f,
 * sigma_t = max(sigma_min, sigma0 f); only units with lattice distance^2
 * g2 <= 2 sigma_t^2 ln(1/cutoff) adapt (R5; cutoff = 0: every unit). */
/* Sample draw of step t ("an input sample is randomly selected"):
 * SOM_SAMPLE_REPLACE (R8): uniform with replacement, i_t = mulhi64(
 * SplitMix64 output t of the seed, m); SOM_SAMPLE_PERMUTE (R8b):
 * a keyed pseudo-random permutation of the m drawable rows per epoch of m
 * steps (every row exactly once per epoch).  Both are counter-based (no
 * state crosses calls: t-ranges resume exactly). */
typedef enum { SOM_SAMPLE_REPLACE = 0, SOM_SAMPLE_PERMUTE = 1 } som_sampling;

typedef struct {
    int32_t kind;      /* som_decay_kind; default SOM_DECAY_GAUSSIAN */
    double k;          /* decay constant; default ln(100)            */
    double sigma_min;  /* radius floor; default 1.0 (R3)              */
    double cutoff;     /* epsilon; default 1e-4 (R5); 0 = no cutoff  */
    int32_t sampling;  /* som_sampling; default SOM_SAMPLE_REPLACE    */
} som_schedule;

typedef enum {
    SOM_MAP_AUTO = 0,      /* fastest path available on the device          */
    SOM_MAP_EXACT_F64 = 1, /* fp64-accumulated direct distances (= oracle)   */
    SOM_MAP_3XTF32 = 2,    /* tcgen05 3xTF32 GEMM |x|^2 - 2 x.w + |w|^2 (R20) */
    SOM_MAP_SPARSE_F64 = 3 /* fp64 sparse identity over the non-zeros of x
                              (R25); dense rows are first put in CSR form on
                              the device */
} som_map_precision;

/* Fill *s with the defaults above. */
som_status som_schedule_default(som_schedule *s);

/* Create a rows x cols map of dim-dimensional prototypes on CUDA device
 * `device` ("a three dimensional data structure is used to represent
 * the map along with its weight vectors", flattened).  Weights start at 0.
 * rows, cols, dim >= 1; rows*cols < 2^24; topology in som_topology. */
som_status som_create(int32_t rows, int32_t cols, int32_t dim, int32_t topology,
                      int32_t device, som_ctx **out);
void som_destroy(som_ctx *h);

/* Copy N*dim fp32 weights in (set) / out (get).  Host or device pointer. */
som_status som_set_weights(som_ctx *h, const float *w);
som_status som_get_weights(som_ctx *h, float *w);

/* Seeded initial codebook: the rows X[j_0..j_{N-1}] with the j drawn from
 * SplitMix64(seed) without replacement when N <= n, with replacement
 * otherwise (R18; the paper's PCA-plane init, is NEXT-3). */
som_status som_init_random(som_ctx *h, const float *X, int64_t n, uint64_t seed);

/* som_init_random on CSR rows (the drawn rows densified into W). */
som_status som_init_random_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col, const float *val,
                               int64_t n, uint64_t seed);

/* Online ("standard") SOM training: for each step
 * t in [t_begin, t_end) of T = epochs * n steps (R7):
 *   i_t   = sample index: t-th SplitMix64(seed) output mapped to [0,m) (R8)
 *           over the m non-zero rows (all-zero rows are never drawn, S:104,
 *           S:218; SOM_EEMPTY when every row is zero)
 *   c_t   = argmin_u (RN_fp32(sum_k (x_k - w_uk)^2 in fp64), u)  (R9, R10)
 *   w_u  <- fmaf(h_u, x - w_u, w_u) for units within the cutoff   (Eq. 1, R11)
 *   h_u   = RN_fp32(alpha_t exp(-g2(u,c_t) / (2 sigma_t^2)))      (R4)
 * t_end = -1 means T.  epochs = 0 is a valid no-op.  bmu_log
 * (nullable, host or device, t_end - t_begin int32) receives c_t.
 * Resuming with a later t-range continues bit-exactly.  alpha0 in [0,1],
 * sigma0 > 0; s may be NULL (defaults). */
som_status som_train_online(som_ctx *h, const float *X, int64_t n, int32_t epochs,
                            double alpha0, double sigma0, const som_schedule *s,
                            uint64_t seed, int64_t t_begin, int64_t t_end,
                            int32_t *bmu_log);

/* som_train_online on CSR input (int64 rowptr[n+1] from 0, non-decreasing;
 * int32 col strictly increasing within a row, in [0, dim); fp32 val — the
 * sparse TF-IDF rows of P:148-154).  Same steps, same
 * results as som_train_online on the dense rows: identical BMU log and
 * weights (the dense oracle is the parity reference).  Where W streams from
 * global memory (kernel 4 in som_last_train_config), units outside the
 * cutoff radius of the pending update get
 *   D_u = |w_u|^2 + sum_{k in nz(x)} ((x_k - w_uk)^2 - w_uk^2)
 * in fp64 (R25) instead of a dense pass, with |w_u|^2 kept in fp64 by the
 * update pass; smaller maps train on the densified rows.  A malformed CSR
 * returns SOM_EINVAL before any side effect (checked on the device). */
som_status som_train_online_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col,
                                const float *val, int64_t n, int32_t epochs, double alpha0,
                                double sigma0, const som_schedule *s, uint64_t seed,
                                int64_t t_begin, int64_t t_end, int32_t *bmu_log);

/* Where som_train_online keeps each CTA's prototypes between steps:
 * AUTO picks shared memory when a CTA's share of W fits (else global
 * memory, L2-resident when W fits the L2); REGISTERS keeps each CTA's share
 * in registers (small maps, d % 4 == 0); SHORT_ROWS is the kernel for short
 * prototypes (d <= 128, d % 4 == 0; Table 3's d = 64): one group of
 * d/4 lanes per unit, W in registers or streamed from L2, neighbourhood
 * from separable tables (R26).  AUTO picks SHORT_ROWS whenever it applies.
 * Forcing a placement that does not fit returns SOM_EUNSUPPORTED from
 * som_train_online. */
typedef enum {
    SOM_TRAIN_AUTO = 0, SOM_TRAIN_W_SHARED = 1, SOM_TRAIN_W_GLOBAL = 2, SOM_TRAIN_W_REGISTERS = 3,
    SOM_TRAIN_SHORT_ROWS = 4
} som_train_mode;
som_status som_set_train_mode(som_ctx *h, int32_t mode);

/* Number of persistent CTAs som_train_online uses (0 = automatic: a model
 * of the per-step all-gather latency vs the per-CTA distance work).  Values
 * above min(N, #SMs) are clamped.  Results do not depend on it. */
som_status som_set_train_grid(som_ctx *h, int32_t grid);

/* Grid and kernel variant of the last som_train_online call:
 * kernel 0 = W in global memory (generic), 1 = W in shared memory,
 * 2 = W in registers, 3 = W in global memory (pipelined, d % 4 == 0),
 * 4 = W in global memory with the sparse distance path (CSR input),
 * 5 = short-row kernel (SOM_TRAIN_SHORT_ROWS),
 * 6 = W in registers with the winner exchange of step t overlapped with the
 *     distance pass of step t+1 (train_spec.cu, R32; the same
 *     BMU log and weights as kernel 2 unless two units' exact distances
 *     round to fp32 values closer than the certificate's margin — the
 *     probability argument of R10),
 * 7 = kernel 6 for the steps whose neighbourhood still covers >= 70 % of
 *     the map (SOM_SPEC_COVER), then kernel 2 (two launches in one call).
 * Where kernel 2 applies on one GPU the environment variable SOM_TRAIN_SPEC
 * selects: unset or 0 = kernel 2 (default), 1 = kernel 6 for the whole
 * range, 2 = kernel 7 (needs >= 8192 prototype elements per CTA and no
 * forced mode or grid).  Kernel 8 = the NCCL step path (som_set_exchange).
 * Kernel 10 = CSR input (or sparse dense rows, converted on the device) in
 * AUTO mode where W does not fit the SMs' shared memory: the map held in
 * tensor memory and shared memory, the rest streamed through a TMA ring
 * (train_tier.cu).  It runs while the cutoff disk holds >= 40 % of the
 * units on average over winner positions and kernel 4 after (kernel 11 =
 * both, two launches in one call;
 * SOM_TIER_HANDOVER=0 keeps kernel 10, SOM_TRAIN_TIER=0 selects kernel 4
 * throughout).  Kernel 12 = CSR rows too long for kernel 4's TMA row ring
 * (> 6 float4 per thread, e.g. d = 20,000) on one GPU in AUTO mode: the
 * dense pipelined kernel 3 on the dense rows (densified on the device when
 * it has room) while the cutoff disk holds >= 60 % of the units on average
 * (SOM_DENSE_COVER), then kernel 4 (two launches in one call).
 * All follow the same arithmetic contract (R9-R11). */
som_status som_last_train_config(som_ctx *h, int32_t *grid, int32_t *kernel);

/* Kernel 6 only: number of steps of the last som_train_online call whose
 * speculative winner could not be certified (near-tie) and that took the
 * exact fallback pass (0 for other kernels).  *count >= 0. */
som_status som_last_spec_fallbacks(som_ctx *h, int64_t *count);

/* SOM_MAP_3XTF32 only (R20b): number of documents of the last mapping call
 * whose 4 tensor-core candidates could not be certified and that were mapped
 * by the exact definition over every unit instead (0 after other paths).
 * Every document's bmu1 / bmu2 / D1 are exact either way. */
som_status som_last_map_fallbacks(som_ctx *h, int64_t *count);

/* ---- Neuron sharding: online training of one map across
 * `world` GPUs (one process or handle per rank).  Rank r holds the units
 * u = r + world*l (cyclic, so the shrinking neighbourhood stays spread);
 * every rank passes the same full X and seed (the sampler is counter-based,
 * so x_t needs no communication).  Each step, after the in-GPU argmin, the
 * rank's winner (8 bytes) is written into every rank's mailbox in peer
 * memory (NVLink) by the training kernel itself and the global minimum
 * taken — results are identical to world = 1.
 *   som_comm_init           switch the handle to rank/world (W re-zeroed;
 *                           set/get/init weights keep using the FULL map,
 *                           only this rank's rows are read/written)
 *   som_comm_mailbox_ipc    64-byte cudaIpcMemHandle of this rank's mailbox
 *   som_comm_set_peers_ipc  world x 64 bytes of handles (all ranks; own
 *                           entry ignored), opened with cudaIpcOpenMemHandle
 *   som_comm_set_peers_dev  world device pointers (same-process ranks)
 * Sharded som_train_online calls are collective: every rank calls with the
 * same arguments, and callers barrier between consecutive calls (the
 * mailbox is cleared at the end of each call).  Mapping, errors and the
 * U-matrix are not served by a sharded handle (SOM_EUNSUPPORTED). */
som_status som_comm_init(som_ctx *h, int32_t rank, int32_t world);
som_status som_comm_local_units(som_ctx *h, int32_t *n_local);
som_status som_comm_mailbox_ipc(som_ctx *h, uint8_t *handle64);
som_status som_comm_set_peers_ipc(som_ctx *h, const uint8_t *handles);
som_status som_comm_set_peers_dev(som_ctx *h, void *const *mailboxes);
som_status som_comm_mailbox_ptr(som_ctx *h, void **mailbox);

/* ---- NCCL communicator.  som_comm_unique_id on rank 0
 * fills a 128-byte ncclUniqueId (broadcast it to the other ranks, e.g. with
 * torch.distributed); every rank then calls som_comm_init_nccl with its
 * rank, the world size, the id and the shard mode.  The call is collective
 * (ncclCommInitRank) and binds the communicator to the handle's device.
 *   SOM_SHARD_DOCS    each rank maps / scores its own documents ("we
 *                     assigned each document vector"); som_errors and
 *                     som_errors_csr sum the fp64 sqrt(D1) total and the
 *                     int64 counts (non-adjacent pairs, non-zero rows) over
 *                     the ranks before dividing, so every rank returns QE
 *                     and TE of the whole corpus.  Errors calls are then
 *                     collective; a rank with no documents passes n = 0.
 *                     Per-document outputs equal those of one GPU.
 *   SOM_SHARD_NEURONS som_comm_init(h, rank, world) (units u = rank +
 *                     world * l) plus the communicator, so the per-step
 *                     winner can be exchanged with NCCL (som_set_exchange).
 * Errors: SOM_EINVAL (bad rank/world/mode), SOM_ENCCL (NCCL failure;
 * handle poisoned). */
typedef enum { SOM_SHARD_DOCS = 1, SOM_SHARD_NEURONS = 2 } som_shard_mode;
som_status som_comm_unique_id(uint8_t *id128);
som_status som_comm_init_nccl(som_ctx *h, int32_t rank, int32_t world, const uint8_t *id128, int32_t shard_mode);

/* Per-step winner exchange of neuron-sharded training (§8.E):
 *   SOM_XCHG_MAILBOX (default) in-kernel, through the peer-memory mailboxes
 *                    of som_comm_set_peers_* (one persistent launch);
 *   SOM_XCHG_NCCL    the baseline: one step kernel per step (pending Eq. 1
 *                    update + fp64 distance, one CTA per unit) followed by
 *                    ncclAllReduce(u64 key, min) on the handle's stream,
 *                    replayed from CUDA graphs (kernel id 8 in
 *                    som_last_train_config).  Needs som_comm_init_nccl (any
 *                    world, including 1).  Same results as the mailbox
 *                    path (identical per-unit arithmetic, exact integer
 *                    min). */
typedef enum { SOM_XCHG_MAILBOX = 0, SOM_XCHG_NCCL = 1 } som_exchange;
som_status som_set_exchange(som_ctx *h, int32_t mode);

/* Phase trace of the register-resident training kernel (profiling aid):
 * device_buf (device memory, 148 * steps * 8 uint64, layout [CTA][step][8])
 * receives %globaltimer (ns) at 8 phase boundaries of the first `steps`
 * steps of every CTA (loop top, fused pass done, partials ready, key
 * published, winner known, neighbourhood ready, x staged, step end).
 * NULL disables. */
som_status som_set_trace(som_ctx *h, void *device_buf, int32_t steps);

/* ---- Upstream steps: from a raw document-term matrix to an
 * initialised map, on the device. */

/* Eq. 2 TF-IDF + L2 row normalisation, reading R28:
 * idf_t = ln(n / df_t), df_t = #rows with a positive count of t; out[p] =
 * RN32(counts[p] idf_t / ||row||), products and norm in fp64; the CSR
 * pattern is kept; rows whose norm is 0 stay 0 and are counted in
 * *zero_rows (nullable).  Columns index [0, dim) of the handle's map.
 * out: nnz floats, host or device. */
som_status som_tfidf_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col, const float *counts,
                         int64_t n, float *out, int64_t *zero_rows);

/* Top-2 principal components of the rows (Fig. 2 step 3),
 * reading R29: eigenpairs of the sample covariance (1/(n-1)) sum_i
 * (x_i - mu)(x_i - mu)^T by subspace iteration on the implicitly centred
 * covariance (never formed); each eigenvector signed so that its largest-
 * magnitude component is positive.  Outputs (host or device, fp64): mean
 * (dim), v1, v2 (dim), pc[2] = (pc1, pc2).  n >= 2. */
som_status som_pca_top2(som_ctx *h, const float *X, int64_t n, double *mean, double *v1, double *v2,
                        double *pc);
som_status som_pca_top2_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col, const float *val,
                            int64_t n, double *mean, double *v1, double *v2, double *pc);

/* PCA-plane linear initialisation ("a regular, two-dimensional
 * sequence of vectors taken along a hyperplane spanned by the two largest
 * principal components"), reading R30: unit (i, j) = mean + a_j sqrt(pc1) v1
 * + b_i sqrt(pc2) v2, a_j = -1 + 2j/(cols-1), b_i = -1 + 2i/(rows-1) (0 for
 * one column / row), fp64, RN32.  Inputs fp64, host or device. */
som_status som_init_linear(som_ctx *h, const double *mean, const double *v1, const double *v2, double pc1,
                           double pc2);

/* Fig. 2, reading R31: map rows <= cols and the iteration count
 * numItr = ceil(50 nn/m) m 4 for m records with top eigenvalues pc1 >= pc2.
 * Pure host arithmetic; m >= 1. */
som_status som_map_geometry(int64_t m, double pc1, double pc2, int32_t *rows, int32_t *cols,
                            int64_t *num_itr);

/* Batch SOM (R27: Kohonen's batch map; the variant of the
 * GPU SOMs the paper reviews).  Per epoch e in [0, epochs),
 * with the current W: c_i = BMU of every row (exact mapping, R10 / R25),
 * then W_u = RN32(sum_i h(c_i,u) x_i / sum_i h(c_i,u)) where the sum is
 * > 0 (else W_u is kept), h = exp(-g2 / 2 sigma_e^2) inside the cutoff
 * (R4, R5, no learning rate), sigma_e from the schedule at tau = e/epochs
 * (R1-R3).  X as in som_train_online; epochs = 0 is a no-op.  bmu
 * (nullable, n int32, host or device) receives the BMUs under the final W.
 * Deterministic: documents are bucketed by BMU in index order. */
som_status som_train_batch(som_ctx *h, const float *X, int64_t n, int32_t epochs, double sigma0,
                           const som_schedule *schedule, int32_t *bmu);
som_status som_train_batch_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col,
                               const float *val, int64_t n, int32_t epochs, double sigma0,
                               const som_schedule *schedule, int32_t *bmu);

/* Batch mapping ("assigned each document vector to the best matching
 * vector on the trained map"): for each row, bmu1 = argmin (D,u),
 * bmu2 = argmin over u != bmu1 (-1 if N = 1), d2 = D at bmu1 (squared
 * Euclidean, fp32).  bmu2, d2 nullable.  Precision per som_set_map_precision. */
som_status som_map(som_ctx *h, const float *X, int64_t n, int32_t *bmu1, int32_t *bmu2,
                   float *d2);
/* som_map_csr: CSR rows as in som_train_online_csr (validated on the
 * device, SOM_EINVAL when malformed). */
som_status som_map_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col,
                       const float *val, int64_t n, int32_t *bmu1, int32_t *bmu2,
                       float *d2);
/* Precision / algorithm of the mapping calls (som_map_precision).  AUTO:
 * CSR rows with <= 1.5 % of the terms set take SOM_MAP_SPARSE_F64; other
 * inputs take EXACT_F64, or 3XTF32 once n*N*dim >= 1e10. */
som_status som_set_map_precision(som_ctx *h, int32_t precision);

/* Quantization error (R14; Table 2): mean over the
 * non-zero rows of sqrt(D at the BMU), summed in fp64.
 * n >= 1; SOM_EEMPTY when every row is zero.  Document-sharded handles
 * (som_comm_init_nccl) reduce over the ranks (collective). */
som_status som_qerror(som_ctx *h, const float *X, int64_t n, double *qe);
/* Topographic error (R15; BJ:5): fraction of the non-zero rows whose two
 * best units are not lattice-adjacent (g2 != 1; 0 for a 1-unit map).
 * n >= 1 (as som_qerror). */
som_status som_topographic_error(som_ctx *h, const float *X, int64_t n, double *te);
/* Both errors from one mapping pass.  qe, te nullable. */
som_status som_errors(som_ctx *h, const float *X, int64_t n, double *qe, double *te);
/* The same for CSR rows (validated as in som_map_csr). */
som_status som_errors_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col,
                          const float *val, int64_t n, double *qe, double *te);

/* U-matrix (R16; BJ:5): U_u = mean over lattice-adjacent v (g2 = 1) of
 * |w_u - w_v|_2 (fp64 accumulation, fp32 result), 0 with no neighbour.
 * U: N floats, host or device. */
som_status som_umatrix(som_ctx *h, float *U);

/* The whole hot path in one call: som_init_random
 * (init_seed, R18) + som_train_online over the full schedule [0, epochs*n)
 * + mapping of all n rows (som_map) + QE / TE from those mapping outputs
 * (som_errors, no second mapping pass) + som_umatrix.  The input is staged
 * to the device once per call.  bmu1, bmu2, d2 (n), qe, te, U (N): nullable
 * outputs, host or device.  Same results as the individual calls.
 * som_last_stats reports the whole call; som_last_phases the split. */
som_status som_fit(som_ctx *h, const float *X, int64_t n, int32_t epochs, double alpha0, double sigma0,
                   const som_schedule *s, uint64_t seed, uint64_t init_seed, int32_t *bmu1, int32_t *bmu2,
                   float *d2, double *qe, double *te, float *U);
som_status som_fit_csr(som_ctx *h, const int64_t *rowptr, const int32_t *col, const float *val, int64_t n,
                       int32_t epochs, double alpha0, double sigma0, const som_schedule *s, uint64_t seed,
                       uint64_t init_seed, int32_t *bmu1, int32_t *bmu2, float *d2, double *qe, double *te,
                       float *U);
/* Device time (ms) of the phases of the last som_fit call: [0] staging +
 * init, [1] training, [2] mapping, [3] QE/TE, [4] U-matrix and output
 * copies; *train_kernel_ms (nullable) = the training kernels alone. */
som_status som_last_phases(som_ctx *h, double *ms5, double *train_kernel_ms);

/* Use the caller's CUDA stream (cudaStream_t as void*; NULL = the
 * handle's own stream).  The caller keeps ownership of the stream. */
som_status som_set_stream(som_ctx *h, void *cuda_stream);

/* Device-side duration (CUDA events) of the main kernel(s) of the last
 * call and how many steps or documents it processed. */
som_status som_last_stats(som_ctx *h, double *ms, int64_t *units, int32_t *kernel_launches);

/* Message for the last failure on this thread ("" if none). */
const char *som_last_error(void);

/* Build/version string, e.g. "libsom 0.1 sm_100a". */
const char *som_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SOM_H */
