// som_train_api.cu — host runtime of libsom, part 2: online training
// (som_train_online / _csr): argument checks, kernel choice and launch
// geometry, L2 residency, launch and error reporting.

#include "som_host.h"

using namespace som;
using namespace som::host;

namespace {

// shared argument checks of som_train_online / som_train_online_csr; on OK
// *sd holds the schedule and [*t_begin, *t_end) the (resolved) step range
som_status check_train(som_ctx* h, int64_t n, int32_t epochs, double alpha0, double sigma0, const som_schedule* s,
                       som_schedule* sd, int64_t* t_begin, int64_t* t_end) {
    som_schedule_default(sd);
    if (s) *sd = *s;
    if (n < 1) return fail(SOM_EEMPTY, "n = 0: no data to train on");
    if (epochs < 0) return fail(SOM_EINVAL, "epochs must be >= 0");
    if (!(alpha0 >= 0.0 && alpha0 <= 1.0)) return fail(SOM_EINVAL, "alpha0 must be in [0, 1]");
    if (!(sigma0 > 0.0) || !std::isfinite(sigma0)) return fail(SOM_EINVAL, "sigma0 must be > 0");
    if (sd->kind < 0 || sd->kind > 2) return fail(SOM_EINVAL, "unknown decay kind");
    if (sd->sampling < 0 || sd->sampling > 1) return fail(SOM_EINVAL, "unknown sampling mode");
    if (!(sd->k > 0.0) || !std::isfinite(sd->k)) return fail(SOM_EINVAL, "decay constant k must be > 0");
    if (!(sd->sigma_min > 0.0)) return fail(SOM_EINVAL, "sigma_min must be > 0");
    if (!(sd->cutoff >= 0.0 && sd->cutoff < 1.0)) return fail(SOM_EINVAL, "cutoff must be in [0, 1)");
    const int64_t T = (int64_t)epochs * n;
    if (*t_end == -1) *t_end = T;
    if (*t_begin < 0 || *t_end < *t_begin || *t_end > T)
        return fail(SOM_EINVAL, "bad t-range [%lld, %lld) for T = %lld", (long long)*t_begin, (long long)*t_end,
                    (long long)T);
    h->last_ms = 0; h->last_units = 0; h->last_launches = 0;
    return SOM_OK;
}

// Unit dealing for the CSR training kernels.  With cyclic dealing (b + s*G)
// the units of one CTA lie on a few long lattice lines, so the disk of units
// a pending update touches gives some CTAs many rows and others none, and the
// step waits for the fullest CTA.  Here unit (i, j) goes to class
// (alpha*i + j) mod G with alpha chosen so that every class is a near-square
// sub-lattice (its shortest vector is maximal), then to the first class with
// room (capacity ceil(NL/G), linear probing): any disk then holds about the
// same number of rows of every CTA, and the all-dense step keeps its balance.
void build_unit_tab(int rows, int cols, int topo, int rank, int world, int NL, int G, std::vector<int>& out) {
    const int S = (NL + G - 1) / G;
    int best_alpha = cols % G;
    double best_len = -1.0;
    for (int al = 1; al < G; ++al) {
        double mn = 1e300;
        for (int di = 0; di < rows && di <= 64; ++di) {
            const int dj0 = (int)((((long long)-al * di) % G + G) % G);
            for (int dj : {dj0, dj0 - G}) {
                if (di == 0 && dj == 0) continue;
                if (dj >= cols || -dj >= cols) continue;   // no such pair of units
                const double len = topo == 0 ? (double)di * di + (double)dj * dj
                                             : (double)dj * dj + 0.75 * (double)di * di;
                mn = std::min(mn, len);
            }
        }
        if (mn > best_len) { best_len = mn; best_alpha = al; }
    }
    out.assign((size_t)G * S + G, -1);
    int* cnt = out.data() + (size_t)G * S;
    for (int b = 0; b < G; ++b) cnt[b] = 0;
    for (int l = 0; l < NL; ++l) {
        const long long u = (long long)rank + (long long)world * l;
        const long long i = u / cols, j = u % cols;
        int k = (int)(((long long)best_alpha * i + j) % G);
        while (cnt[k] >= S) k = (k + 1) % G;
        out[(size_t)k * S + cnt[k]++] = l;
    }
}

// Fraction of the units inside the cutoff disk at step t, averaged over 64
// sampled winner positions (non-increasing in t): the hand-over criterion
// of the two-kernel schedules (kernels 11 and 12).
double mean_cover(const som_ctx* h, const som_schedule& sd, int64_t T, double sigma0, double ln_inv_eps, int64_t t) {
    double f;
    fill_decay(&f, t, t + 1, T, sd.kind, sd.k);
    const double sigma = std::max(sd.sigma_min, sigma0 * f);
    const double r2 = 2.0 * sigma * sigma * ln_inv_eps;
    const int Nm = h->rows * h->cols;
    const int stride = std::max(1, Nm / 64);
    int64_t cnt = 0, pos = 0;
    for (int c = stride / 2; c < Nm; c += stride, ++pos) {
        const int ic = c / h->cols, jc = c - ic * h->cols;
        for (int i = 0; i < h->rows; ++i) {
            const double di = (double)(i - ic);
            for (int j = 0; j < h->cols; ++j) {
                double g2;
                if (h->topo == 0) {
                    const double dj = (double)(j - jc);
                    g2 = di * di + dj * dj;
                } else {
                    const double dx2 = (double)(2 * (j - jc) + ((i & 1) - (ic & 1)));
                    g2 = 0.25 * dx2 * dx2 + 0.75 * di * di;
                }
                cnt += g2 <= r2;
            }
        }
    }
    return (double)cnt / ((double)pos * Nm);
}

// first t in [lo, hi) whose mean coverage is below thr (hi if none)
int64_t first_below(const som_ctx* h, const som_schedule& sd, int64_t T, double sigma0, double ln_inv_eps, double thr,
                    int64_t lo, int64_t hi) {
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (mean_cover(h, sd, T, sigma0, ln_inv_eps, mid) >= thr) lo = mid + 1; else hi = mid;
    }
    return lo;
}

som_status train_impl(som_ctx* h, const void* Xd, const CsrIn* csr, int64_t n, int32_t epochs, double alpha0,
                      double sigma0, const som_schedule& sd, uint64_t seed, int64_t t_begin, int64_t t_end,
                      int32_t* bmu_log) {
    const int64_t T = (int64_t)epochs * n;
    invalidate_w_caches(h);
    som_status st = SOM_OK;
    if ((st = ensure_decay_table(h, T, sd.kind, sd.k, t_begin, t_end))) return st;

    // zero rows are never drawn: the draws go to the list of
    // non-zero rows when some row is zero (R8 over that list)
    int64_t n_draw = 0;
    const int64_t* rowmap = nullptr;
    if ((st = scan_rows(h, (const float*)Xd, csr, n, &n_draw, &rowmap))) return st;
    if (n_draw == 0) return fail(SOM_EEMPTY, "every row is zero: nothing to draw (S:219)");

    TrainArgs a{};
    a.W = h->W; a.X = (const float*)Xd; a.n = n; a.dim = h->dim; a.dimp = (h->dim + 3) & ~3;
    a.rowmap = rowmap; a.n_draw = n_draw; a.sampling = sd.sampling;
    a.rows = h->rows; a.cols = h->cols; a.topo = h->topo; a.N = h->NL;
    a.rank = h->rank; a.world = h->world;
    for (int p = 0; p < kMaxRanks; ++p) a.mail[p] = h->peer_mail[p];
    if (h->xchg_mode == SOM_XCHG_NCCL) {
        // step-at-a-time path, winner exchanged by ncclAllReduce (som_comm.cu)
        a.t0 = t_begin; a.t1 = t_end; a.seed = seed;
        a.f_tab = (const double*)h->ftab.p;
        a.alpha0 = alpha0; a.sigma0 = sigma0; a.sigma_min = sd.sigma_min;
        a.cutoff_on = sd.cutoff > 0.0;
        a.ln_inv_eps = sd.cutoff > 0.0 ? std::log(1.0 / sd.cutoff) : 0.0;
        a.G = h->NL;
        if (csr) {   // the step kernel reads dense rows
            CK(h->dense.ensure(sizeof(float) * (size_t)n * h->dim, h->stream));
            CK(launch_densify(csr->rowptr, csr->col, csr->val, 0, n, h->dim, (float*)h->dense.p, h->stream));
            a.X = (const float*)h->dense.p;
        }
        const int64_t steps = t_end - t_begin;
        const bool log_dev = bmu_log && is_device_ptr(bmu_log);
        if (bmu_log && !log_dev) CK(h->log.ensure(sizeof(int32_t) * (size_t)steps, h->stream));
        a.bmu_log = bmu_log ? (log_dev ? bmu_log : (int32_t*)h->log.p) : nullptr;
        int launches = 0;
        CK(cudaEventRecord(h->ev0, h->stream));
        if ((st = train_nccl_steps(h, a, &launches))) return st;
        CK(cudaEventRecord(h->ev1, h->stream));
        if (bmu_log && !log_dev)
            CK(cudaMemcpyAsync(bmu_log, h->log.p, sizeof(int32_t) * (size_t)steps, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        h->last_ms = ms; h->last_units = steps; h->last_launches = launches;
        h->last_grid = a.G; h->last_kernel = 8;
        return SOM_OK;
    }
    if (h->world > 1) {
        for (int p = 0; p < h->world; ++p)
            if (!h->peer_mail[p]) return fail(SOM_ESTATE, "neuron sharding: peer mailboxes not set (som_comm_set_peers_*)");
    }
    a.x_vec4 = (h->dim % 4 == 0) && (csr || (uintptr_t)Xd % 16 == 0);   // densified CSR is aligned
    // launch geometry.  Register-resident kernel when a CTA's share of W fits
    // the register file: G minimises (all-gather latency + fp64 distance
    // time), both measured on B200 (profiles/probe_*_r01.json).  Otherwise
    // one persistent CTA per SM with W in shared or global memory.
    // short prototypes (d <= 128): the lane-group kernel (train_small.cu).
    // G minimises (all-gather latency + per-CTA rounds of work), with the
    // L2 traffic of the streamed variant when the map exceeds 4 rounds.
    bool use_small = false;
    if ((h->train_mode == SOM_TRAIN_AUTO || h->train_mode == SOM_TRAIN_SHORT_ROWS) && a.x_vec4 &&
        train_small_supported(h->dim)) {
        auto xchg_us = [](int G) { return G <= 32 ? 0.65 : G <= 64 ? 0.70 : G <= 128 ? 0.85 : 1.65; };
        const int gmax = std::min(h->NL, h->sm_count);
        double best = 1e30;
        int bestG = 0;
        for (int G : {8, 16, 32, 64, 128, gmax}) {
            if (h->train_grid > 0) G = std::min(h->train_grid, gmax);
            if (G < 1 || G > gmax) continue;
            const int R = small_rounds((h->NL + G - 1) / G, h->dim);
            double est = xchg_us(G) + 0.35 * R;   // ~0.35 us per round (tools/sweep_small.py, d = 64)
            // streamed: read + ~60 % written per step at ~12 TB/s of L2 over 148 SMs, pro rata G
            if (R > 4) est += 2.6 * 4.0 * (double)h->NL * h->dim / (12.0e6 * G / 148.0);
            if (est < best) { best = est; bestG = G; }
        }
        use_small = bestG > 0;
        a.G = bestG;
    }
    if (h->train_mode == SOM_TRAIN_SHORT_ROWS && !use_small)
        return fail(SOM_EUNSUPPORTED, "short-row kernel needs d <= 128 and d %% 4 == 0");
    bool use_reg = false;
    if (!use_small && (h->train_mode == SOM_TRAIN_AUTO || h->train_mode == SOM_TRAIN_W_REGISTERS) && a.x_vec4) {
        // all-gather latency by grid size (profiles/probe_xchg_r01.json) and
        // per-CTA F2F-bound distance time: (S + 1) * d conversions at 16/clk
        // (power-of-two grids measured fastest: 16-64 ~0.6-0.7 us, 128 ~0.8 us,
        // 48/96/100/112/134/148 all slower; tools/sweep_grid.py on c2)
        auto xchg_us = [](int G) { return G <= 32 ? 0.65 : G <= 64 ? 0.70 : G <= 128 ? 0.85 : 1.65; };
        double best = 1e30;
        int bestG = 0;
        const int gmax = std::min(h->NL, h->sm_count);
        std::vector<int> cands = {16, 32, 64, 128};
        if (gmax <= 32) cands.push_back(gmax);
        for (int G : cands) {
            if (h->train_grid > 0) G = std::min(h->train_grid, gmax);
            if (G < 1 || G > gmax) continue;
            const int S = (h->NL + G - 1) / G;
            if (!train_reg_supported(S, h->dim)) continue;
            const double est = xchg_us(G) + (double)(S + 1) * h->dim / (16.0 * 1965.0);
            if (est < best) { best = est; bestG = G; }
        }
        if (bestG > 0) { use_reg = true; a.G = bestG; }
    }
    if (h->train_mode == SOM_TRAIN_W_REGISTERS && !use_reg)
        return fail(SOM_EUNSUPPORTED, "map share per CTA does not fit registers (or d %% 4 != 0)");
    if (!use_reg && !use_small) {
        a.G = std::min(h->NL, h->sm_count);
        if (h->train_grid > 0) a.G = std::min(a.G, h->train_grid);
    }
    a.S = (h->NL + a.G - 1) / a.G;
    a.t0 = t_begin; a.t1 = t_end; a.seed = seed;
    a.f_tab = (const double*)h->ftab.p;
    a.alpha0 = alpha0; a.sigma0 = sigma0; a.sigma_min = sd.sigma_min;
    a.cutoff_on = sd.cutoff > 0.0;
    a.ln_inv_eps = sd.cutoff > 0.0 ? std::log(1.0 / sd.cutoff) : 0.0;
    a.trace = h->trace;
    a.trace_steps = h->trace ? h->trace_steps : 0;
    a.trace_clk = 0;
    if (const char* e = std::getenv("SOM_TRACE_CLOCK")) a.trace_clk = std::atoi(e) != 0;
    size_t smem = train_smem_bytes(a.S, a.dimp, 1);
    a.w_smem = smem <= (size_t)h->max_smem_optin;
    if (h->train_mode == SOM_TRAIN_W_SHARED && !a.w_smem)
        return fail(SOM_EUNSUPPORTED, "W slice (%zu B/CTA) does not fit shared memory", smem);
    if (h->train_mode == SOM_TRAIN_W_GLOBAL) a.w_smem = 0;
    if (!a.w_smem) smem = train_smem_bytes(a.S, a.dimp, 0);
    // maps that do not fit on chip stream from global memory with the
    // pipelined kernel (train_glb.cu) when its layout applies
    const bool use_glb = !use_small && !use_reg && !a.w_smem && a.x_vec4 && train_glb_supported(a.S, h->dim);
    if (use_reg) smem = sizeof(float) * (3 * (size_t)a.dimp + (size_t)a.rows * (a.topo == 0 ? a.cols : 2 * a.cols));
    if (use_glb) smem = sizeof(float) * 2 * (size_t)a.dimp;
    if (use_small) {
        a.w_smem = 0;
        smem = sizeof(float) * 3 * (size_t)a.dimp +
               sizeof(double) * ((size_t)a.dimp + a.rows + (a.topo == 0 ? a.cols : 2 * a.cols));
    }
    // Dense TF-IDF rows where W streams from global memory: put the rows in
    // CSR form on the device once per call (count, scan, fill) and take the
    // sparse-distance kernel when they are sparse (<= 1.5 % of the terms
    // set; SOM_TRAIN_DENSE_CSR=0 keeps the dense kernels).  Same results: the
    // CSR kernels follow the same contract (R10 via R25) and are
    // parity-tested against the dense oracle.
    CsrIn auto_csr{};
    bool dense_csr = true;
    if (const char* e = std::getenv("SOM_TRAIN_DENSE_CSR")) dense_csr = std::atoi(e) != 0;
    // kernel 10 (train_tier.cu) for CSR rows where W streams from global
    // memory in AUTO mode (SOM_TRAIN_TIER=0: kernel 4 throughout)
    bool tier_env = true;
    if (const char* e = std::getenv("SOM_TRAIN_TIER")) tier_env = std::atoi(e) != 0;
    tier_env = tier_env && h->train_mode == SOM_TRAIN_AUTO && !use_small && !use_reg && !a.w_smem;
    if (!csr && dense_csr && !use_small && !use_reg && !a.w_smem && a.x_vec4 &&
        h->train_mode == SOM_TRAIN_AUTO && h->xchg_mode != SOM_XCHG_NCCL) {
        const size_t tb = dense_csr_temp_bytes(n);
        CK(h->tcsr.ensure(sizeof(int64_t) * 2 * ((size_t)n + 1) + tb + 256, h->stream));
        int64_t* cnt = (int64_t*)h->tcsr.p;
        int64_t* rp = cnt + n + 1;
        void* temp = (void*)(((uintptr_t)(rp + n + 1) + 255) & ~(uintptr_t)255);
        CK(launch_dense_rowptr((const float*)Xd, n, h->dim, cnt, rp, temp, tb, h->stream));
        int64_t nnz = 0;
        CK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if ((double)nnz <= 0.015 * (double)n * h->dim) {
            CK(h->tcsr2.ensure((sizeof(int32_t) + sizeof(float)) * (size_t)std::max<int64_t>(nnz, 1) + 256, h->stream));
            int32_t* col = (int32_t*)h->tcsr2.p;
            float* val = (float*)(((uintptr_t)(col + nnz) + 255) & ~(uintptr_t)255);
            CK(launch_dense_fill((const float*)Xd, n, h->dim, rp, col, val, h->stream));
            CK(h->red.ensure(64, h->stream));
            CK(launch_csr_check(rp, col, n, h->dim, (int*)h->red.p, h->stream));
            int res[2] = {0, 0};
            CK(cudaMemcpyAsync(res, h->red.p, sizeof(res), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            auto_csr = CsrIn{rp, col, val, res[1], nnz};
            if (train_csr_supported(a.S, h->dim, res[1], h->max_smem_optin) ||
                (tier_env && train_tier_supported(a.S, h->dim, res[1], h->max_smem_optin)))
                csr = &auto_csr;
        }
    }
    // CSR input: the sparse-distance kernel where W streams from global
    // memory; on-chip maps (latency-bound, no gain) and layouts it does not
    // cover train on the densified rows
    bool use_csr = false, use_tier = false;
    if (csr) {
        use_tier = tier_env && train_tier_supported(a.S, h->dim, csr->maxnnz, h->max_smem_optin);
        use_csr = use_tier ||
                  (!use_small && !use_reg && !a.w_smem && train_csr_supported(a.S, h->dim, csr->maxnnz, h->max_smem_optin));
        if (use_csr) {
            a.rowptr = csr->rowptr; a.col = csr->col; a.val = csr->val;
            a.nz_cap = csr_nz_cap(csr->maxnnz);
            // upper bound of the lattice g2 between any two units (exact for
            // rect; hex bound takes the half-column offset at the full row span)
            const double dr = h->rows - 1, dc = h->cols - 1;
            a.g2max = h->topo == 0 ? dr * dr + dc * dc : 0.25 * (2 * dc + 1) * (2 * dc + 1) + 0.75 * dr * dr;
            if (h->utab_G != a.G || h->utab_NL != h->NL || h->utab_rank != h->rank || h->utab_world != h->world) {
                std::vector<int> tab;
                build_unit_tab(h->rows, h->cols, h->topo, h->rank, h->world, h->NL, a.G, tab);
                CK(h->utab.ensure(sizeof(int) * tab.size(), h->stream));
                CK(cudaMemcpyAsync(h->utab.p, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, h->stream));
                CK(cudaStreamSynchronize(h->stream));
                h->utab_G = a.G; h->utab_NL = h->NL; h->utab_rank = h->rank; h->utab_world = h->world;
            }
            a.utab = (const int*)h->utab.p;
            a.ucnt = a.utab + (size_t)a.G * a.S;
            smem = sizeof(float) * 2 * (size_t)a.dimp + 24 * (size_t)a.nz_cap;
            if (use_tier) { a.w_smem = 0; smem = 0; }   // kernel 10 sizes its own shared memory
        } else {
            CK(h->dense.ensure(sizeof(float) * (size_t)n * h->dim, h->stream));
            CK(launch_densify(csr->rowptr, csr->col, csr->val, 0, n, h->dim, (float*)h->dense.p, h->stream));
            a.X = (const float*)h->dense.p;
        }
    }
    if (smem > (size_t)h->max_smem_optin)
        return fail(SOM_EUNSUPPORTED, "dim %d too large for the x staging ring (%zu B smem)", h->dim, smem);

    // exchange slots: two parities of G slots, each parity on its own 256-byte
    // lines (a line shared by step t's and step t+1's slots would be written
    // by fast CTAs while slow ones still poll it)
    a.xstride = (a.G + 31) & ~31;
    // exchange variant (som_internal.h), measured on B200 (tools/xchg_ab.py,
    // bit-identical results): the tagged all-gather alone is fastest for
    // small grids (c1, G = 32: 2.27 vs 2.46 us/step); from ~100 CTAs on, the
    // all-gather read once a relaxed arrival counter is complete wins (c2,
    // G = 128: 3.24 vs 3.27; c3, G = 148: 23.0 vs 24.0 us/step early in the
    // schedule, 5.9 vs 7.5 late), the L2 no longer serving G full scans per
    // poll round
    a.xchg_atomic = a.G >= 96 ? 2 : 0;
    if (const char* e = std::getenv("SOM_XCHG_ATOMIC")) a.xchg_atomic = std::max(0, std::min(2, std::atoi(e)));
    a.poll_ns = 0;
    if (const char* e = std::getenv("SOM_POLL_NS")) a.poll_ns = std::max(0, std::atoi(e));
    // exchange wait bound: 60 s of %globaltimer (SOM_SPIN_TIMEOUT_MS), then
    // the abort flag and SOM_ECUDA instead of a hang
    a.spin_ns = 60000ull * 1000000ull;
    if (const char* e = std::getenv("SOM_SPIN_TIMEOUT_MS")) a.spin_ns = (unsigned long long)std::max(1, std::atoi(e)) * 1000000ull;
    // (kernel 6: a second word per CTA, [2][2][xstride]); then the abort flag
    // and the fallback counter
    const size_t xwords = 4 * (size_t)a.xstride;
    CK(h->xchg.ensure(sizeof(unsigned long long) * xwords + 64, h->stream));
    a.xchg = (unsigned long long*)h->xchg.p;
    a.abort_flag = (unsigned*)((char*)h->xchg.p + sizeof(unsigned long long) * xwords);
    a.spec_fallbacks = (unsigned long long*)((char*)h->xchg.p + sizeof(unsigned long long) * xwords + 8);
    CK(cudaMemsetAsync(h->xchg.p, 0, sizeof(unsigned long long) * xwords + 64, h->stream));
    // kernel 6 (train_spec.cu, R32): SOM_TRAIN_SPEC=1 for the whole range;
    // =2 (no forced mode or grid, one GPU): kernel 6 on a balanced grid for
    // the steps whose neighbourhood still covers >= 70 % of the map, then
    // kernel 2 (tools/spec_windows.py); unset / 0: kernel 2.  Both give
    // identical results and the t-range split is exact; the speed relative
    // to kernel 2 varies by box (-4 % .. +3 % at c2), so not the default.
    bool use_spec = false;
    const char* spec_env = std::getenv("SOM_TRAIN_SPEC");
    const int spec_mode = spec_env ? std::atoi(spec_env) : 0;
    if (use_reg && spec_mode == 1 && train_spec_supported(a.S, h->dim, a.G, h->world)) use_spec = true;
    // kernel 10 while the neighbourhood covers most of the lattice (its
    // on-chip rows save the most when most units are updated), then kernel 4
    // (few updated units: kernel 4's step is shorter); an exact t-range
    // split, both kernels give identical results.  The hand-over is the
    // first step whose cutoff disk holds, on average over winner positions
    // (64 sampled units), less than SOM_TIER_COVER (default 0.4) of the
    // units: c3 per 20,000-step segment (tools/prof_tier.py, B200) kernel 10
    // is faster down to ~0.4 mean coverage (t ~ 300k: 15.0 vs 15.1 us/step),
    // kernel 4 after (13.1 vs 12.9).  SOM_TIER_HANDOVER=0: kernel 10 throughout.
    int64_t t_tier = t_end;
    if (use_tier && a.cutoff_on) {
        bool handover = true;
        if (const char* e = std::getenv("SOM_TIER_HANDOVER")) handover = std::atoi(e) != 0;
        double thr = 0.4;
        if (const char* e = std::getenv("SOM_TIER_COVER")) thr = std::atof(e);
        if (handover) t_tier = first_below(h, sd, T, sigma0, a.ln_inv_eps, thr, t_begin, t_end);
    }
    // kernel 3 then kernel 4 (kernel 12): CSR rows too long for kernel 4's
    // TMA row ring (> 6 float4 per thread: c4, d = 20,000) run the dense
    // pipelined kernel while most units update every step (it streams all
    // of W once per step at ~94 % of HBM, kernel 4's register ring reaches
    // ~71 % on the same full-coverage steps), then kernel 4 (sparse
    // distances: only the updated rows move).  Exact t-range split; needs
    // the dense rows (the caller's, or densified when the device has room).
    // SOM_DENSE_COVER: mean-coverage threshold of the hand-over (default
    // 0.6; 0 = kernel 4 throughout).
    int64_t t_dense = t_begin;
    const float* xdense = nullptr;
    if (use_csr && !use_tier && a.cutoff_on && h->world == 1 && h->train_mode == SOM_TRAIN_AUTO &&
        ((a.dimp / 4) + kTrainThreads - 1) / kTrainThreads > 6 && train_glb_supported(a.S, h->dim)) {
        double thr = 0.6;
        if (const char* e = std::getenv("SOM_DENSE_COVER")) thr = std::atof(e);
        if (thr > 0.0) t_dense = first_below(h, sd, T, sigma0, a.ln_inv_eps, thr, t_begin, t_end);
        if (t_dense > t_begin) {
            if (Xd) {
                xdense = (const float*)Xd;
            } else {
                size_t fr = 0, tot = 0;
                const size_t need = sizeof(float) * (size_t)n * h->dim;
                if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && (h->dense.cap >= need || need + ((size_t)1 << 30) <= fr)) {
                    CK(h->dense.ensure(need, h->stream));
                    CK(launch_densify(csr->rowptr, csr->col, csr->val, 0, n, h->dim, (float*)h->dense.p, h->stream));
                    xdense = (const float*)h->dense.p;
                }
            }
            if (!xdense) t_dense = t_begin;
        }
    }
    int64_t t_split = t_begin;   // hybrid: kernel 6 on [t_split), kernel 2 after
    int G6 = 0;
    if (use_reg && spec_mode == 2 && h->train_mode == SOM_TRAIN_AUTO && h->train_grid == 0 && h->world == 1 &&
        (int64_t)a.S * h->dim >= 8192) {
        const int g6 = (h->NL + a.S - 1) / a.S;
        if (train_spec_supported(a.S, h->dim, g6, 1)) {
            // units inside the cutoff around the map centre at step t (non-increasing in t)
            const int ic = h->rows / 2, jc = h->cols / 2;
            double cover = 0.7;   // SOM_SPEC_COVER: coverage threshold of the hand-over
            if (const char* e = std::getenv("SOM_SPEC_COVER")) cover = std::atof(e);
            auto covered = [&](int64_t t) {
                double f;
                fill_decay(&f, t, t + 1, T, sd.kind, sd.k);
                double sigma = std::max(sd.sigma_min, sigma0 * f);
                const double r2 = sd.cutoff > 0.0 ? 2.0 * sigma * sigma * std::log(1.0 / sd.cutoff) : INFINITY;
                int64_t cnt = 0;
                for (int i = 0; i < h->rows; ++i)
                    for (int j = 0; j < h->cols; ++j) {
                        const double di = i - ic;
                        double g2;
                        if (h->topo == 0) { const double dj = j - jc; g2 = di * di + dj * dj; }
                        else { const double dx = 2.0 * (j - jc) + ((i & 1) - (ic & 1)); g2 = 0.25 * dx * dx + 0.75 * di * di; }
                        cnt += g2 <= r2;
                    }
                return cnt >= (int64_t)std::ceil(cover * h->NL);
            };
            int64_t lo = t_begin, hi = t_end;   // first t in [lo, hi) not covered
            while (lo < hi) {
                const int64_t mid = lo + (hi - lo) / 2;
                if (covered(mid)) lo = mid + 1; else hi = mid;
            }
            t_split = lo;
            if (t_split > t_begin) G6 = g6;
        }
    }

    const int64_t steps = t_end - t_begin;
    bool log_dev = bmu_log && is_device_ptr(bmu_log);
    if (bmu_log && !log_dev) CK(h->log.ensure(sizeof(int32_t) * (size_t)steps, h->stream));
    a.bmu_log = bmu_log ? (log_dev ? bmu_log : (int32_t*)h->log.p) : nullptr;

    // W streamed from global memory every step: keep it resident in L2 with a
    // persisting access-policy window (random X rows stream past it), undone
    // after the launch so the caller's stream is left as it was.
    // The caller's persisting-L2 limit and the stream's window are saved and
    // restored afterwards; the persisting lines are demoted only if no
    // persisting set-aside existed before the call (nobody else uses it).
    bool l2_window = false;
    size_t prev_persist = 0;
    cudaStreamAttrValue prev_win{};
    const char* nowin = std::getenv("SOM_NO_L2_WINDOW");
    if (!(nowin && std::atoi(nowin)) && !use_reg && !a.w_smem && (!use_small || small_rounds(a.S, h->dim) > 4)) {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
        const size_t wbytes = sizeof(float) * (size_t)h->NL * h->dim;
        int l2_bytes = 0;
        cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, h->device);
        // only for maps that fit the L2: for a map several times the L2 (c4 on
        // one GPU, 800 MB) the persisting lines of the window crowd out the
        // streamed rest of W and the row writes (measured 664 -> 263 us/step
        // without it)
        if (max_persist > 0 && max_window > 0 && wbytes <= (size_t)l2_bytes) {
            const size_t win = std::min(wbytes, (size_t)max_window);
            const size_t keep = std::min(win, (size_t)max_persist);
            const bool saved = cudaDeviceGetLimit(&prev_persist, cudaLimitPersistingL2CacheSize) == cudaSuccess &&
                               cudaStreamGetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &prev_win) ==
                                   cudaSuccess;
            if (saved && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::max(keep, prev_persist)) == cudaSuccess) {
                cudaStreamAttrValue at{};
                at.accessPolicyWindow.base_ptr = h->W;
                at.accessPolicyWindow.num_bytes = win;
                at.accessPolicyWindow.hitRatio = (float)((double)keep / (double)win);
                at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                l2_window = cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &at) == cudaSuccess;
            }
            cudaGetLastError();
        }
    }
    CK(cudaEventRecord(h->ev0, h->stream));
    int launches = 1;
    if (use_small) CK(launch_train_small(a, h->stream));
    else if (use_spec) CK(launch_train_spec(a, h->stream));
    else if (G6 > 0) {
        TrainArgs a6 = a;
        a6.G = G6;
        a6.S = (h->NL + G6 - 1) / G6;
        a6.xstride = (G6 + 31) & ~31;
        a6.t1 = t_split;
        CK(launch_train_spec(a6, h->stream));
        if (t_split < t_end) {
            // fresh exchange slots (the abort flag and the fallback counter stay)
            CK(cudaMemsetAsync(h->xchg.p, 0, sizeof(unsigned long long) * xwords, h->stream));
            TrainArgs a2 = a;
            a2.t0 = t_split;
            a2.f_tab = a.f_tab + (t_split - t_begin);
            if (a2.bmu_log) a2.bmu_log = a.bmu_log + (t_split - t_begin);
            a2.trace = nullptr;
            a2.trace_steps = 0;
            CK(launch_train_reg(a2, h->stream));
            launches = 2;
        }
    }
    else if (use_reg) CK(launch_train_reg(a, h->stream));
    else if (use_tier) {
        if (t_tier > t_begin) {
            TrainArgs a10 = a;
            a10.t1 = t_tier;
            CK(launch_train_tier(a10, h->max_smem_optin, h->stream));
        }
        if (t_tier < t_end) {
            // kernel 4 from the first step whose radius no longer covers the
            // lattice (fresh exchange slots; the abort flag stays)
            if (t_tier > t_begin) CK(cudaMemsetAsync(h->xchg.p, 0, sizeof(unsigned long long) * xwords, h->stream));
            TrainArgs a4 = a;
            a4.t0 = t_tier;
            a4.f_tab = a.f_tab + (t_tier - t_begin);
            if (a4.bmu_log) a4.bmu_log = a.bmu_log + (t_tier - t_begin);
            if (t_tier > t_begin) { a4.trace = nullptr; a4.trace_steps = 0; }
            CK(launch_train_csr(a4, h->stream));
            if (t_tier > t_begin) launches = 2;
        }
    }
    else if (use_csr) {
        if (t_dense > t_begin) {
            TrainArgs a3 = a;
            a3.X = xdense;
            a3.x_vec4 = 1;
            a3.t1 = t_dense;
            CK(launch_train_glb(a3, h->stream));
            if (t_dense < t_end) {
                // kernel 4 from the hand-over step (fresh exchange slots; the abort flag stays)
                CK(cudaMemsetAsync(h->xchg.p, 0, sizeof(unsigned long long) * xwords, h->stream));
                TrainArgs a4 = a;
                a4.t0 = t_dense;
                a4.f_tab = a.f_tab + (t_dense - t_begin);
                if (a4.bmu_log) a4.bmu_log = a.bmu_log + (t_dense - t_begin);
                a4.trace = nullptr;
                a4.trace_steps = 0;
                CK(launch_train_csr(a4, h->stream));
                launches = 2;
            }
        } else {
            CK(launch_train_csr(a, h->stream));
        }
    }
    else if (use_glb) CK(launch_train_glb(a, h->stream));
    else CK(launch_train(a, smem, h->stream));
    CK(cudaEventRecord(h->ev1, h->stream));
    if (l2_window) {   // later launches on the stream get the caller's window back
        cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &prev_win);
        cudaGetLastError();
    }
    h->last_grid = a.G;
    h->last_kernel = use_small ? 5 : use_spec ? 6 : G6 > 0 ? (t_split < t_end ? 7 : 6) : use_reg ? 2 : use_tier ? (t_tier >= t_end ? 10 : t_tier > t_begin ? 11 : 4) : use_csr ? (t_dense >= t_end ? 3 : t_dense > t_begin ? 12 : 4) : use_glb ? 3 : (a.w_smem ? 1 : 0);
    if (bmu_log && !log_dev)
        CK(cudaMemcpyAsync(bmu_log, h->log.p, sizeof(int32_t) * (size_t)steps, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (l2_window) {   // the kernel is done: demote its persisting lines, restore the set-aside
        if (prev_persist == 0) cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_persist);
        cudaGetLastError();
    }
    unsigned abort_flag = 0;
    CK(cudaMemcpyAsync(&abort_flag, a.abort_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->last_spec_fallbacks = 0;
    if (use_spec || G6 > 0) {
        unsigned long long fb = 0;
        CK(cudaMemcpyAsync(&fb, a.spec_fallbacks, sizeof(fb), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->last_spec_fallbacks = (int64_t)fb;
    }
    if (abort_flag) {
        h->poisoned = true;
        return fail(SOM_ECUDA, "training exchange timed out (a CTA or rank stopped publishing its BMU candidate)");
    }
    // neuron sharding: clear the own mailbox so the next call's tags cannot
    // match stale entries (callers barrier between sharded calls)
    if (h->world > 1) {
        CK(cudaMemsetAsync(h->mail, 0, sizeof(unsigned long long) * 2 * (size_t)h->world, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms; h->last_units = steps; h->last_launches = launches;
    return SOM_OK;
}

}  // namespace

extern "C" {

som_status som_train_online(som_ctx* h, const float* X, int64_t n, int32_t epochs, double alpha0, double sigma0,
                            const som_schedule* s, uint64_t seed, int64_t t_begin, int64_t t_end, int32_t* bmu_log) {
    CHECK_HANDLE(h);
    if (!X) return fail(SOM_EINVAL, "null X");
    som_schedule sd;
    som_status st = check_train(h, n, epochs, alpha0, sigma0, s, &sd, &t_begin, &t_end);
    if (st) return st;
    if (t_end == t_begin) return SOM_OK;   // epochs = 0 or empty range: weights unchanged
    const void* Xd = nullptr;
    if ((st = stage_in(h, h->xin, X, sizeof(float) * (size_t)n * h->dim, &Xd))) return st;
    return train_impl(h, Xd, nullptr, n, epochs, alpha0, sigma0, sd, seed, t_begin, t_end, bmu_log);
}

som_status som_train_online_csr(som_ctx* h, const int64_t* rowptr, const int32_t* col, const float* val, int64_t n,
                                int32_t epochs, double alpha0, double sigma0, const som_schedule* s, uint64_t seed,
                                int64_t t_begin, int64_t t_end, int32_t* bmu_log) {
    CHECK_HANDLE(h);
    som_schedule sd;
    som_status st = check_train(h, n, epochs, alpha0, sigma0, s, &sd, &t_begin, &t_end);
    if (st) return st;
    CsrIn csr{};
    if ((st = stage_csr(h, rowptr, col, val, n, &csr))) return st;
    if (t_end == t_begin) return SOM_OK;
    return train_impl(h, nullptr, &csr, n, epochs, alpha0, sigma0, sd, seed, t_begin, t_end, bmu_log);
}

}  // extern "C"
