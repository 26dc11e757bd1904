/*
 * som_oracle.c — ORACLE for the CUDASOM hot path (arXiv 1905.09598).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_1905_09598_b200/, libsom.so) never links, imports or
 * calls it, and it shares no code, header or table with the product: the
 * only things both sides agree on are the definitions written out below and
 * in DESIGN.md ("Readings").
 *
 * This is a plain, slow, obviously-correct CPU implementation of what the
 * method computes.  Each function cites the passage it follows:
 *   P:n  = /root/reference/PAPER.md line n,   S:n = SPEC.md line n,
 *   Rn   = reading n of DESIGN.md §3 (where the paper is silent/garbled).
 * Floating point: fp64 for every accumulation (R10), fp32 for the stored
 * map weights and the update of Eq. 1 (R11).  Build with
 *   gcc -O2 -ffp-contract=off -fno-fast-math
 * so `acc += d * d` stays a rounded multiply followed by a rounded add.
 *
 * Parity pins (tests/test_oracle_pins.py) fix every function against
 * something other than itself: the worked 2x2 example of Eq. 1 computed by
 * hand in exact rational arithmetic, the SplitMix64 published outputs,
 * SPEC lattice examples, closed forms of the schedule, brute force on tiny
 * maps, invariants (alpha=0, symmetry, neighbour counts, fixed point).
 * "parity unpinned" items are listed in DESIGN.md §3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- sampler */
/* R8 ("an input sample is randomly selected on the host"): sample
 * index i_t is the t-th output (t = 0,1,...) of a SplitMix64 stream seeded
 * with `seed`, mapped to [0,n) by the high half of the 128-bit product. */
uint64_t or_splitmix64(uint64_t seed, int64_t t)
{
    /* state after t+1 increments of the Weyl sequence */
    uint64_t z = seed + (uint64_t)(t + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

int64_t or_sample_index(uint64_t seed, int64_t t, int64_t n)
{
    unsigned __int128 p = (unsigned __int128)or_splitmix64(seed, t) * (uint64_t)n;
    return (int64_t)(p >> 64);
}

/* R8b (per-epoch permutation as an option to R8): epoch
 * e = t / m, position p = t mod m, i_t = pi_e(p) with pi_e the permutation
 * of [0, m) obtained by cycle-walking a keyed bijection of [0, 2^b),
 * b = bit length of m - 1: four rounds of (add key r, xor with itself
 * shifted right by ceil(b/2), multiply by 0x9E3779B97F4A7C15), every
 * operation mod 2^b, keys k_r = or_splitmix64(seed ^ 0x5851F42D4C957F2D,
 * 4e + r).  Every index appears exactly once per epoch. */
int64_t or_perm_index(uint64_t seed, int64_t t, int64_t m)
{
    if (m <= 1) return 0;
    int64_t e = t / m, p = t % m;
    int b = 64 - __builtin_clzll((uint64_t)(m - 1));
    uint64_t mask = b >= 64 ? ~0ULL : ((1ULL << b) - 1ULL);
    int sh = (b + 1) / 2;
    uint64_t k[4];
    for (int r = 0; r < 4; ++r) k[r] = or_splitmix64(seed ^ 0x5851F42D4C957F2DULL, 4 * e + r);
    uint64_t x = (uint64_t)p;
    do {
        for (int r = 0; r < 4; ++r) {
            x = (x + k[r]) & mask;
            x ^= x >> sh;
            x = (x * 0x9E3779B97F4A7C15ULL) & mask;
        }
    } while (x >= (uint64_t)m);
    return (int64_t)x;
}

/* the draw of step t over m drawable rows: R8 (sampling 0) or R8b (1) */
int64_t or_draw_index(uint64_t seed, int64_t t, int64_t m, int32_t sampling)
{
    return sampling == 1 ? or_perm_index(seed, t, m) : or_sample_index(seed, t, m);
}

/* --------------------------------------------------------------- schedule */
/* R1 ("The Gaussian decay was used to smooth the learning rate and
 * neighborhood radius"): tau = t/T, f = exp(-k tau^2);
 * alpha_t = alpha0 f, sigma_t = max(sigma_min, sigma0 f).
 * Alternatives (kind 1 linear, kind 2 exponential) end at the same e^-k.
 * R5: cutoff radius^2 r2 = 2 sigma_t^2 ln(1/eps); eps = 0 means no cutoff. */
void or_schedule(int kind, double k, int64_t t, int64_t T, double alpha0,
                 double sigma0, double sigma_min, double eps,
                 double *alpha, double *sigma, double *r2)
{
    double tau = (double)t / (double)T;
    double f;
    if (kind == 0)      f = exp(-k * tau * tau);
    else if (kind == 1) f = 1.0 - (1.0 - exp(-k)) * tau;
    else                f = exp(-k * tau);
    double s = sigma0 * f;
    if (s < sigma_min) s = sigma_min;
    *alpha = alpha0 * f;
    *sigma = s;
    *r2 = (eps > 0.0) ? 2.0 * s * s * log(1.0 / eps) : INFINITY;
}

/* ---------------------------------------------------------------- lattice */
/* P:166 "hexagonal coordinates were calculate[d] before computing the
 * distances"; S:164 hex_position(i,j) = (j + 0.5 (i mod 2), i sqrt(3)/2),
 * u = i*cols + j.  Squared lattice distance, exact: the x
 * offset is a multiple of 1/2 and (dy)^2 = 3/4 (di)^2, so g2 is a multiple
 * of 1/4 and exactly representable.  topo 0 = rectangular (BJ:7),
 * topo 1 = hexagonal. */
double or_lattice_g2(int32_t rows, int32_t cols, int32_t topo, int64_t u, int64_t v)
{
    (void)rows;
    int64_t iu = u / cols, ju = u % cols;
    int64_t iv = v / cols, jv = v % cols;
    double di = (double)(iu - iv);
    if (topo == 0) {
        double dj = (double)(ju - jv);
        return di * di + dj * dj;
    }
    double xu = (double)ju + 0.5 * (double)(iu % 2);
    double xv = (double)jv + 0.5 * (double)(iv % 2);
    double dx = xu - xv;
    return dx * dx + 0.75 * di * di;
}

/* -------------------------------------------------------------- distance */
/* P:106 "The weight vector which is most similar to the input vector, is
 * determined as the winning neuron"; Euclidean distance.
 * R10: difference formed in fp64 from the fp32 operands, summed in fp64,
 * sequentially over k; D_u = RN_fp32(sum). */
double or_dist2_f64(const float *w, const float *x, int64_t d)
{
    double acc = 0.0;
    for (int64_t k = 0; k < d; ++k) {
        double delta = (double)x[k] - (double)w[k];
        acc += delta * delta;
    }
    return acc;
}

/* R9: BMU = lexicographic minimum of (D_u, u): equal fp32 distances go to
 * the lowest flat index.  Returns c; *Dc = D_c (fp32);
 * *margin = (acc_2nd - acc_1st)/max(acc_1st,1e-30) in fp64 (diagnostic). */
int64_t or_bmu(const float *W, int64_t N, int64_t d, const float *x,
               float *Dc, double *margin)
{
    double *acc = (double *)malloc(sizeof(double) * (size_t)N);
#pragma omp parallel for schedule(static) if (N * d > 200000)
    for (int64_t u = 0; u < N; ++u)
        acc[u] = or_dist2_f64(W + u * d, x, d);
    int64_t c = 0;
    float best = (float)acc[0];
    for (int64_t u = 1; u < N; ++u) {
        float D = (float)acc[u];
        if (D < best) { best = D; c = u; }
    }
    if (margin) {
        double a1 = acc[c], a2 = INFINITY;
        for (int64_t u = 0; u < N; ++u)
            if (u != c && acc[u] < a2) a2 = acc[u];
        *margin = (N > 1) ? (a2 - a1) / (a1 > 1e-30 ? a1 : 1e-30) : INFINITY;
    }
    if (Dc) *Dc = best;
    free(acc);
    return c;
}

/* ----------------------------------------------------------------- update */
/* Eq. 1: w_u(t+1) = w_u(t) + h_cu(t) [x(t) - w_u(t)].
 * R4 ("h represents a smoothing kernel like Gaussian"):
 *   h_u = RN_fp32(alpha_t exp(-g2(u,c) / (2 sigma_t^2))).
 * R5: only u with g2 <= r2 adapt ("The neurons in the selected
 * neighborhood then adapt").  R11: per element
 *   w <- fmaf(h, RN_fp32(x - w), w). */
void or_update(float *W, int32_t rows, int32_t cols, int32_t topo, int64_t d,
               const float *x, int64_t c, double alpha, double sigma, double r2)
{
    int64_t N = (int64_t)rows * cols;
#pragma omp parallel for schedule(static) if (N * d > 200000)
    for (int64_t u = 0; u < N; ++u) {
        double g2 = or_lattice_g2(rows, cols, topo, u, c);
        if (!(g2 <= r2)) continue;
        float h = (float)(alpha * exp(-g2 / (2.0 * sigma * sigma)));
        float *w = W + u * d;
        for (int64_t k = 0; k < d; ++k) {
            float diff = x[k] - w[k];
            w[k] = fmaf(h, diff, w[k]);
        }
    }
}

/* ----------------------------------------------------------- online train */
/* The standard (online) SOM, one sample per iteration: compete, cooperate,
 * adapt.  T = epochs * n (R7).  Steps
 * t in [t_begin, t_end) are run; bmu_log[t - t_begin] = c_t (nullable);
 * margin_log likewise (nullable).  Returns 0, or -1 on bad arguments. */
/* Zero rows ("All-zero document rows after filtering are retained
 * but excluded from training sample draws"): the indices of
 * the rows holding at least one non-zero value, ascending, into idx
 * (nullable); returns their count. */
int64_t or_nonzero_rows(const float *X, int64_t n, int64_t d, int64_t *idx)
{
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        int nz = 0;
        for (int64_t k = 0; k < d && !nz; ++k) nz = X[i * d + k] != 0.0f;
        if (nz) { if (idx) idx[m] = i; ++m; }
    }
    return m;
}

/* The same for CSR rows: a row is zero when it stores no non-zero value
 * (explicit zeros, e.g. idf-0 terms of R28, do not count). */
int64_t or_nonzero_rows_csr(const int64_t *rowptr, const float *val, int64_t n, int64_t *idx)
{
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        int nz = 0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1] && !nz; ++p) nz = val[p] != 0.0f;
        if (nz) { if (idx) idx[m] = i; ++m; }
    }
    return m;
}

int or_train_online(float *W, int32_t rows, int32_t cols, int32_t topo, int64_t d,
                    const float *X, int64_t n, int32_t epochs,
                    double alpha0, double sigma0, int32_t decay_kind, double k,
                    double sigma_min, double eps, int32_t sampling, uint64_t seed,
                    int64_t t_begin, int64_t t_end,
                    int32_t *bmu_log, double *margin_log)
{
    int64_t T = (int64_t)epochs * n;
    if (t_end < 0) t_end = T;
    if (t_begin < 0 || t_begin > t_end || t_end > T || sampling < 0 || sampling > 1) return -1;
    if (t_end == t_begin) return 0;
    int64_t N = (int64_t)rows * cols;
    /* R8 + S:218: draws are uniform over the non-zero rows only (the j-th
     * non-zero row for draw j); T = epochs * n stays the step count (R7).
     * Without zero rows this is the plain sampler over [0, n). */
    int64_t *nzr = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!nzr) return -1;
    int64_t m = or_nonzero_rows(X, n, d, nzr);
    if (m == 0) { free(nzr); return -2; }   /* EmptyData */
    for (int64_t t = t_begin; t < t_end; ++t) {
        int64_t i = nzr[or_draw_index(seed, t, m, sampling)];
        const float *x = X + i * d;
        double margin;
        int64_t c = or_bmu(W, N, d, x, NULL, &margin);
        double alpha, sigma, r2;
        or_schedule(decay_kind, k, t, T, alpha0, sigma0, sigma_min, eps,
                    &alpha, &sigma, &r2);
        or_update(W, rows, cols, topo, d, x, c, alpha, sigma, r2);
        if (bmu_log) bmu_log[t - t_begin] = (int32_t)c;
        if (margin_log) margin_log[t - t_begin] = margin;
    }
    free(nzr);
    return 0;
}

/* The same online SOM on CSR rows (the sparse TF-IDF DTM of P:148-154):
 * x_t is densified into a zeroed d-vector and the step is or_bmu +
 * or_update exactly as above.  Lets the oracle follow corpora whose dense
 * copy would not fit (c4: 200k x 20k). */
int or_train_online_csr(float *W, int32_t rows, int32_t cols, int32_t topo, int64_t d,
                        const int64_t *rowptr, const int32_t *col, const float *val,
                        int64_t n, int32_t epochs, double alpha0, double sigma0,
                        int32_t decay_kind, double k, double sigma_min, double eps,
                        int32_t sampling, uint64_t seed, int64_t t_begin, int64_t t_end, int32_t *bmu_log)
{
    int64_t T = (int64_t)epochs * n;
    if (t_end < 0) t_end = T;
    if (t_begin < 0 || t_begin > t_end || t_end > T || sampling < 0 || sampling > 1) return -1;
    if (t_end == t_begin) return 0;
    int64_t N = (int64_t)rows * cols;
    int64_t *nzr = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    float *x = (float *)calloc((size_t)d, sizeof(float));
    if (!nzr || !x) { free(nzr); free(x); return -1; }
    int64_t m = or_nonzero_rows_csr(rowptr, val, n, nzr);
    if (m == 0) { free(nzr); free(x); return -2; }
    for (int64_t t = t_begin; t < t_end; ++t) {
        int64_t i = nzr[or_draw_index(seed, t, m, sampling)];
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) x[col[p]] = val[p];
        int64_t c = or_bmu(W, N, d, x, NULL, NULL);
        double alpha, sigma, r2;
        or_schedule(decay_kind, k, t, T, alpha0, sigma0, sigma_min, eps, &alpha, &sigma, &r2);
        or_update(W, rows, cols, topo, d, x, c, alpha, sigma, r2);
        if (bmu_log) bmu_log[t - t_begin] = (int32_t)c;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) x[col[p]] = 0.0f;
    }
    free(nzr);
    free(x);
    return 0;
}

/* ----------------------------------------------------------------- map */
/* P:248 "we assigned each document vector to the best matching vector on
 * the trained map".  Per document: fp64 distances to all units, rounded to
 * fp32; bmu1 = min (D,u), bmu2 = min (D,u) over u != bmu1 (R9, R15);
 * d1 = D_bmu1.  m12 = (acc2-acc1)/acc1, m23 = (acc3-acc2)/acc2 in fp64
 * (R19 near-tie diagnostics; nullable). */
void or_map(const float *W, int64_t N, int64_t d, const float *X, int64_t n,
            int32_t *bmu1, int32_t *bmu2, float *d1, double *m12, double *m23)
{
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < n; ++i) {
        const float *x = X + i * d;
        int64_t b1 = -1, b2 = -1, b3 = -1;
        float D1 = INFINITY, D2 = INFINITY, D3 = INFINITY;
        double a1 = INFINITY, a2 = INFINITY, a3 = INFINITY;
        for (int64_t u = 0; u < N; ++u) {
            double acc = or_dist2_f64(W + u * d, x, d);
            float D = (float)acc;
            /* strict < keeps the lowest index among equal D (u ascends) */
            if (D < D1) {
                b3 = b2; D3 = D2; a3 = a2;
                b2 = b1; D2 = D1; a2 = a1;
                b1 = u;  D1 = D;  a1 = acc;
            } else if (D < D2) {
                b3 = b2; D3 = D2; a3 = a2;
                b2 = u;  D2 = D;  a2 = acc;
            } else if (D < D3) {
                b3 = u;  D3 = D;  a3 = acc;
            }
        }
        (void)b3; (void)D3;
        if (bmu1) bmu1[i] = (int32_t)b1;
        if (bmu2) bmu2[i] = (int32_t)b2;   /* -1 when N == 1 */
        if (d1) d1[i] = D1;
        if (m12) m12[i] = (N > 1) ? (a2 - a1) / (a1 > 1e-30 ? a1 : 1e-30) : INFINITY;
        if (m23) m23[i] = (N > 2) ? (a3 - a2) / (a2 > 1e-30 ? a2 : 1e-30) : INFINITY;
    }
}

/* Sparse identity for one CSR document (BASELINE.md oracle plan, path 2):
 *   sum_k (x_k - w_k)^2 = sum_{k in nz(x)} [(x_k - w_k)^2 - w_k^2] + |w|^2,
 * exact in real arithmetic, evaluated in fp64 with |w|^2 precomputed in
 * fp64 (wsq).  Used only to make large-n samples of the mapping oracle
 * affordable; tests check it against or_map on dense rows. */
void or_map_csr(const float *W, const double *wsq, int64_t N, int64_t d,
                const int64_t *rowptr, const int32_t *col, const float *val,
                int64_t n, int32_t *bmu1, int32_t *bmu2, float *d1,
                double *m12, double *m23)
{
    (void)d;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < n; ++i) {
        int64_t b1 = -1, b2 = -1;
        float D1 = INFINITY, D2 = INFINITY, D3 = INFINITY;
        double a1 = INFINITY, a2 = INFINITY, a3 = INFINITY;
        for (int64_t u = 0; u < N; ++u) {
            const float *w = W + u * d;
            double acc = 0.0;
            for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
                double wk = (double)w[col[p]];
                double delta = (double)val[p] - wk;
                acc += delta * delta - wk * wk;
            }
            acc += wsq[u];
            if (acc < 0.0) acc = 0.0;
            float D = (float)acc;
            if (D < D1) {
                D3 = D2; a3 = a2;
                b2 = b1; D2 = D1; a2 = a1;
                b1 = u;  D1 = D;  a1 = acc;
            } else if (D < D2) {
                D3 = D2; a3 = a2;
                b2 = u;  D2 = D;  a2 = acc;
            } else if (D < D3) {
                D3 = D; a3 = acc;
            }
        }
        if (bmu1) bmu1[i] = (int32_t)b1;
        if (bmu2) bmu2[i] = (int32_t)b2;
        if (d1) d1[i] = D1;
        if (m12) m12[i] = (N > 1) ? (a2 - a1) / (a1 > 1e-30 ? a1 : 1e-30) : INFINITY;
        if (m23) m23[i] = (N > 2) ? (a3 - a2) / (a2 > 1e-30 ? a2 : 1e-30) : INFINITY;
    }
}

/* ------------------------------------------------------------ batch SOM */
/* Batch SOM (the variant of [25], [26], and
 * "most of the recent proposals have focused on the batch version of SOM",
 * P:158).  The paper does not state it; reading R27 takes Kohonen's batch
 * map: per epoch e in [0, E), with the current W,
 *   c_i  = BMU of x_i (R9, R10, every document),
 *   h_iu = exp(-g2(c_i, u) / (2 sigma_e^2)) if g2 <= r2_e else 0   (R4, R5
 *          without the learning rate: the batch map has none),
 *   W_u  <- RN_fp32( sum_i h_iu x_i / sum_i h_iu )   if sum_i h_iu > 0,
 *          else W_u unchanged,
 * with sigma_e, r2_e from the decay schedule at tau = e/E (R1-R3, R5).
 * Sums run over documents in index order in fp64, straight from the
 * definition (no per-BMU regrouping).  bmu_last (nullable, n) receives the
 * BMUs of the final epoch.  Returns 0, or -1 on bad arguments. */
int or_train_batch(float *W, int32_t rows, int32_t cols, int32_t topo, int64_t d,
                   const float *X, int64_t n, int32_t epochs, double sigma0,
                   int32_t decay_kind, double k, double sigma_min, double eps,
                   int32_t *bmu_last)
{
    if (n < 1 || epochs < 0) return -1;
    int64_t N = (int64_t)rows * cols;
    int64_t *c = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    float *Wn = (float *)malloc(sizeof(float) * (size_t)(N * d));
    if (!c || !Wn) { free(c); free(Wn); return -1; }
    for (int32_t e = 0; e < epochs; ++e) {
        double alpha, sigma, r2;
        or_schedule(decay_kind, k, e, epochs, 1.0, sigma0, sigma_min, eps, &alpha, &sigma, &r2);
        (void)alpha;
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t i = 0; i < n; ++i) c[i] = or_bmu(W, N, d, X + i * d, NULL, NULL);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t u = 0; u < N; ++u) {
            double den = 0.0;
            double *num = (double *)calloc((size_t)d, sizeof(double));
            for (int64_t i = 0; i < n; ++i) {
                double g2 = or_lattice_g2(rows, cols, topo, u, c[i]);
                if (!(g2 <= r2)) continue;
                double h = exp(-g2 / (2.0 * sigma * sigma));
                den += h;
                const float *x = X + i * d;
                for (int64_t kk = 0; kk < d; ++kk) num[kk] += h * (double)x[kk];
            }
            for (int64_t kk = 0; kk < d; ++kk)
                Wn[u * d + kk] = (den > 0.0) ? (float)(num[kk] / den) : W[u * d + kk];
            free(num);
        }
        memcpy(W, Wn, sizeof(float) * (size_t)(N * d));
    }
    if (bmu_last) {
        for (int64_t i = 0; i < n; ++i) bmu_last[i] = (int32_t)or_bmu(W, N, d, X + i * d, NULL, NULL);
    }
    free(c);
    free(Wn);
    return 0;
}

/* fp64 squared norms of the prototypes (input to or_map_csr). */
void or_row_sqnorm(const float *W, int64_t N, int64_t d, double *wsq)
{
    for (int64_t u = 0; u < N; ++u) {
        double acc = 0.0;
        for (int64_t k = 0; k < d; ++k) {
            double wk = (double)W[u * d + k];
            acc += wk * wk;
        }
        wsq[u] = acc;
    }
}

/* ------------------------------------------------------------ QE and TE */
/* R14 (Table 2): quantization error =
 * mean Euclidean (not squared) distance of each row to its BMU. */
double or_qerror_from_d1(const float *d1, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += sqrt((double)d1[i]);
    return s / (double)n;
}

/* S:227 "mean over nonzero rows": keep[i] != 0 marks the rows that
 * count; NAN when none does (EmptyData). */
double or_qerror_masked(const float *d1, const uint8_t *keep, int64_t n)
{
    double s = 0.0;
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!keep[i]) continue;
        s += sqrt((double)d1[i]);
        ++m;
    }
    return m ? s / (double)m : NAN;
}

/* R13, R15 (BJ:5; not in the paper): topographic error = fraction of rows
 * whose first and second BMUs are not lattice-adjacent (g2 != 1).
 * A 1-unit map has no second BMU: TE := 0 (R23). */
double or_topographic_error_from_bmus(int32_t rows, int32_t cols, int32_t topo,
                                      const int32_t *bmu1, const int32_t *bmu2,
                                      int64_t n)
{
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (bmu2[i] < 0) continue;
        if (or_lattice_g2(rows, cols, topo, bmu1[i], bmu2[i]) != 1.0) ++bad;
    }
    return (double)bad / (double)n;
}

/* TE over the rows keep[i] != 0 only (zero rows are scored like QE). */
double or_topographic_error_masked(int32_t rows, int32_t cols, int32_t topo,
                                   const int32_t *bmu1, const int32_t *bmu2,
                                   const uint8_t *keep, int64_t n)
{
    int64_t bad = 0, m = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!keep[i]) continue;
        ++m;
        if (bmu2[i] < 0) continue;
        if (or_lattice_g2(rows, cols, topo, bmu1[i], bmu2[i]) != 1.0) ++bad;
    }
    return m ? (double)bad / (double)m : NAN;
}

/* -------------------------------------------------------------- U-matrix */
/* R16 (BJ:5; S:415 lists it as a viz non-goal there): per unit, the mean
 * Euclidean distance between its prototype and the prototypes of its
 * lattice-adjacent units (g2 == 1); 0 for a unit with no neighbour (R23).
 * Distances in fp64, result rounded to fp32. */
void or_umatrix(const float *W, int32_t rows, int32_t cols, int32_t topo,
                int64_t d, float *U)
{
    int64_t N = (int64_t)rows * cols;
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < N; ++u) {
        double sum = 0.0;
        int64_t cnt = 0;
        for (int64_t v = 0; v < N; ++v) {
            if (or_lattice_g2(rows, cols, topo, u, v) != 1.0) continue;
            sum += sqrt(or_dist2_f64(W + v * d, W + u * d, d));
            ++cnt;
        }
        U[u] = cnt ? (float)(sum / (double)cnt) : 0.0f;
    }
}

/* ------------------------------------------------------------ TF-IDF */
/* Eq. 2 and the row normalisation of P:174, reading R28:
 *   df_t   = #{documents d : tf(d,t) > 0},
 *   idf_t  = ln(n / df_t)                      (natural log),
 *   w_dt   = tf(d,t) idf_t / ||(tf(d,.) idf)||_2,
 * products and the norm in fp64 (sum over the row's entries in order),
 * one rounding to fp32.  The CSR pattern is kept (an entry whose idf is 0
 * stays as an explicit 0); a row whose norm is 0 stays all-zero and is
 * counted in *zero_rows.  counts: raw term frequencies. */
void or_tfidf_csr(const int64_t *rowptr, const int32_t *col, const float *counts,
                  int64_t n, int64_t d, float *out, int64_t *zero_rows)
{
    int64_t *df = (int64_t *)calloc((size_t)d, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p)
            if (counts[p] > 0.0f) df[col[p]] += 1;
    int64_t zr = 0;
    for (int64_t i = 0; i < n; ++i) {
        double ss = 0.0;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            int64_t t = col[p];
            double idf = df[t] > 0 ? log((double)n / (double)df[t]) : 0.0;
            double v = (double)counts[p] * idf;
            ss += v * v;
        }
        double nrm = sqrt(ss);
        if (nrm == 0.0) ++zr;
        for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            int64_t t = col[p];
            double idf = df[t] > 0 ? log((double)n / (double)df[t]) : 0.0;
            double v = (double)counts[p] * idf;
            out[p] = (nrm > 0.0) ? (float)(v / nrm) : 0.0f;
        }
    }
    if (zero_rows) *zero_rows = zr;
    free(df);
}

/* threads the OpenMP regions above will use (for cpu_baseline reporting) */
int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int nt)
{
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}
