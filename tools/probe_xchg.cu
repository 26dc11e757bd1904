// probe_xchg.cu — per-step argmin exchange protocols for the persistent
// training kernel: latency per step vs grid size and protocol.  Dev tooling.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long umin(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

// P0: all-gather of tagged slots; stride = slot stride in u64 (1 = packed, 16 = one line each)
__global__ void p_gather(unsigned long long* slots, int steps, int stride, unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < 32) {
            unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* s = slots + (size_t)(t & 1) * G * stride;
            if (lane == 0) st_relaxed_u64(s + (size_t)b * stride, ((unsigned long long)((b * 7 + t) % 1000) << 8) | tag);
            for (;;) {
                unsigned long long m = ~0ull;
                bool ok = true;
                for (int j = lane; j < G; j += 32) {
                    unsigned long long v = ld_relaxed_u64(s + (size_t)j * stride);
                    ok &= (v & 0xFF) == tag;
                    m = umin(m, v);
                }
                if (__all_sync(0xffffffffu, ok)) { acc += m; break; }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

// P0r: R replicas of the tagged slot array; CTA b writes its key into every
// replica (lanes over replicas) and polls replica b % R.  R = G is a private
// mailbox per CTA.  Replica r lives at slots + r * 2 * G * stride_r.
__global__ void p_gather_rep(unsigned long long* slots, int steps, int R, unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31;
    const size_t rep_stride = ((size_t)2 * G + 31) & ~(size_t)31;   // 256 B aligned replicas
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < 32) {
            const unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            const unsigned long long key = ((unsigned long long)((b * 7 + t) % 1000) << 8) | tag;
            for (int r = lane; r < R; r += 32) st_relaxed_u64(slots + r * rep_stride + (size_t)(t & 1) * G + b, key);
            const unsigned long long* s = slots + (size_t)(b % R) * rep_stride + (size_t)(t & 1) * G;
            for (;;) {
                unsigned long long m = ~0ull;
                bool ok = true;
                for (int j = lane; j < G; j += 32) {
                    unsigned long long v = ld_relaxed_u64(s + j);
                    ok &= (v & 0xFF) == tag;
                    m = umin(m, v);
                }
                if (__all_sync(0xffffffffu, ok)) { acc += m; break; }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

// P0b: reducer + broadcast: all CTAs publish; CTA 0 polls the G slots, writes
// one tagged result word; the others poll only that word.  `sleep_ns` adds
// a nanosleep backoff between polls of the all-gather variant when > 0.
__global__ void p_reduce_bcast(unsigned long long* slots, unsigned long long* result, int steps,
                               unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < 32) {
            const unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* s = slots + (size_t)(t & 1) * G;
            if (lane == 0) st_relaxed_u64(s + b, ((unsigned long long)((b * 7 + t) % 1000) << 8) | tag);
            if (b == 0) {
                unsigned long long m;
                for (;;) {
                    unsigned long long mm = ~0ull;
                    bool ok = true;
                    for (int j = lane; j < G; j += 32) {
                        unsigned long long v = ld_relaxed_u64(s + j);
                        ok &= (v & 0xFF) == tag;
                        mm = umin(mm, v);
                    }
                    if (__all_sync(0xffffffffu, ok)) {
                        for (int o = 16; o; o >>= 1) mm = umin(mm, __shfl_xor_sync(0xffffffffu, mm, o));
                        m = mm;
                        break;
                    }
                }
                if (lane == 0) st_relaxed_u64(result + (t & 1), m);
                acc += m;
            } else {
                for (;;) {
                    unsigned long long v = ld_relaxed_u64(result + (t & 1));
                    if ((v & 0xFF) == tag) { acc += v; break; }
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

__global__ void p_gather_sleep(unsigned long long* slots, int steps, int sleep_ns, unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < 32) {
            unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* s = slots + (size_t)(t & 1) * G;
            if (lane == 0) st_relaxed_u64(s + b, ((unsigned long long)((b * 7 + t) % 1000) << 8) | tag);
            for (;;) {
                unsigned long long m = ~0ull;
                bool ok = true;
                for (int j = lane; j < G; j += 32) {
                    unsigned long long v = ld_relaxed_u64(s + j);
                    ok &= (v & 0xFF) == tag;
                    m = umin(m, v);
                }
                if (__all_sync(0xffffffffu, ok)) { acc += m; break; }
                __nanosleep(sleep_ns);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

// P1: atomicMin into slot[t%3] + release-add arrival counter; poll counter (acquire), read slot
__global__ void p_atomic(unsigned long long* slot3, unsigned* cnt3, int steps, unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x == 0) {
            const int i = t % 3;
            atomicMin(slot3 + i, (unsigned long long)((b * 7 + t) % 1000) << 8);
            red_release_add(cnt3 + i, 1u);
            const unsigned target = (unsigned)G * (unsigned)(t / 3 + 1);
            while (ld_acquire_u32(cnt3 + i) < target) {}
            acc += ld_relaxed_u64(slot3 + i);
            // reset the slot two steps ahead (everyone is past step t-1's read of it)
            if (b == 0) st_relaxed_u64(slot3 + (t + 2) % 3, ~0ull);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

// P2: cluster of C CTAs reduces through DSMEM, one leader per cluster joins a
// gather among G/C leaders, then writes the result into every member's smem.
template <int C>
__global__ void p_cluster(unsigned long long* slots, int steps, unsigned long long* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ unsigned long long box[C];
    __shared__ unsigned long long res;
    const int rank = cl.block_rank();
    const int L = gridDim.x / C, leader = blockIdx.x / C;
    const int lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x == 0) {
            unsigned long long* lbox = cl.map_shared_rank(box, 0);
            lbox[rank] = ((unsigned long long)((blockIdx.x * 7 + t) % 1000) << 8);
        }
        cl.sync();
        if (rank == 0 && threadIdx.x < 32) {
            unsigned long long m = ~0ull;
            for (int j = lane; j < C; j += 32) m = umin(m, box[j]);
            for (int o = 16; o; o >>= 1) m = umin(m, __shfl_xor_sync(0xffffffffu, m, o));
            unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* s = slots + (size_t)(t & 1) * L;
            if (lane == 0) st_relaxed_u64(s + leader, (m & ~0xFFull) | tag);
            for (;;) {
                unsigned long long mm = ~0ull;
                bool ok = true;
                for (int j = lane; j < L; j += 32) {
                    unsigned long long v = ld_relaxed_u64(s + j);
                    ok &= (v & 0xFF) == tag;
                    mm = umin(mm, v);
                }
                if (__all_sync(0xffffffffu, ok)) {
                    for (int o = 16; o; o >>= 1) mm = umin(mm, __shfl_xor_sync(0xffffffffu, mm, o));
                    if (lane < C) *cl.map_shared_rank(&res, lane) = mm;
                    break;
                }
            }
        }
        cl.sync();
        acc += res;
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

// P3: plain cooperative-groups grid.sync() per step (reference point)
__global__ void p_gridsync(int steps, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) { g.sync(); acc += t; }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

int main() {
    unsigned long long *slots, *out;
    unsigned* cnt;
    CK(cudaMalloc(&slots, 2 * 148 * 16 * 8));
    CK(cudaMalloc(&cnt, 64));
    CK(cudaMalloc(&out, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int steps = 20000;
    float ms;
    printf("{\n");
    auto timeit = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms * 1e3 / steps;
    };
    if (getenv("PROBE_QUICK")) {
        for (int G : {148, 128, 64, 32}) {
            float us = timeit([&] {
                CK(cudaMemset(slots, 0, 2 * 148 * 16 * 8));
                int st = steps, sd = 1;
                void* a[] = {&slots, &st, &sd, &out};
                CK(cudaLaunchCooperativeKernel((void*)p_gather, G, 512, a, 0, 0));
            });
            printf("  \"gather_G%d\": %.3f,\n", G, us);
            unsigned long long* res = slots + 2 * 148 * 8;
            us = timeit([&] {
                CK(cudaMemset(slots, 0, 2 * 148 * 16 * 8));
                int st = steps;
                void* a[] = {&slots, &res, &st, &out};
                CK(cudaLaunchCooperativeKernel((void*)p_reduce_bcast, G, 512, a, 0, 0));
            });
            printf("  \"reduce_bcast_G%d\": %.3f,\n", G, us);
            for (int sl : {20, 50, 100}) {
                us = timeit([&] {
                    CK(cudaMemset(slots, 0, 2 * 148 * 16 * 8));
                    int st = steps, s2 = sl;
                    void* a[] = {&slots, &st, &s2, &out};
                    CK(cudaLaunchCooperativeKernel((void*)p_gather_sleep, G, 512, a, 0, 0));
                });
                printf("  \"gather_sleep%d_G%d\": %.3f,\n", sl, G, us);
            }
        }
        printf("  \"steps\": %d\n}\n", steps);
        return 0;
    }
    for (int stride : {1, 16}) {
        for (int G : {148, 128, 96, 74, 64, 48, 32, 16}) {
            float us = timeit([&] {
                CK(cudaMemset(slots, 0, 2 * 148 * 16 * 8));
                int st = steps, sd = stride;
                void* a[] = {&slots, &st, &sd, &out};
                CK(cudaLaunchCooperativeKernel((void*)p_gather, G, 512, a, 0, 0));
            });
            printf("  \"gather_stride%d_G%d\": %.3f,\n", stride, G, us);
        }
    }
    {
        unsigned long long* rep;
        const size_t rep_bytes = (size_t)148 * 320 * 8;
        CK(cudaMalloc(&rep, rep_bytes));
        for (int G : {148, 128, 64, 32}) {
            for (int R : {1, 2, 4, 8, 16, 32, 64, 148}) {
                if (R > G) continue;
                float us = timeit([&] {
                    CK(cudaMemset(rep, 0, rep_bytes));
                    int st = steps, r = R;
                    void* a[] = {&rep, &st, &r, &out};
                    CK(cudaLaunchCooperativeKernel((void*)p_gather_rep, G, 512, a, 0, 0));
                });
                printf("  \"rep%d_G%d\": %.3f,\n", R, G, us);
            }
        }
    }
    for (int G : {148, 74, 32}) {
        float us = timeit([&] {
            unsigned long long init[3] = {~0ull, ~0ull, ~0ull};
            CK(cudaMemcpy(slots, init, 24, cudaMemcpyHostToDevice));
            CK(cudaMemset(cnt, 0, 64));
            int st = steps;
            void* a[] = {&slots, &cnt, &st, &out};
            CK(cudaLaunchCooperativeKernel((void*)p_atomic, G, 512, a, 0, 0));
        });
        printf("  \"atomic_G%d\": %.3f,\n", G, us);
    }
    {
        auto run_cluster = [&](auto kern, int C, int G) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(512);
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeCooperative;
            at[1].val.cooperative = 1;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            if (C > 8) CK(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            return timeit([&] {
                CK(cudaMemset(slots, 0, 2 * 148 * 16 * 8));
                int st = steps;
                CK(cudaLaunchKernelEx(&cfg, kern, slots, st, out));
            });
        };
        printf("  \"cluster2_G148\": %.3f,\n", run_cluster(p_cluster<2>, 2, 148));
        printf("  \"cluster4_G128\": %.3f,\n", run_cluster(p_cluster<4>, 4, 128));
        printf("  \"cluster8_G144\": %.3f,\n", run_cluster(p_cluster<8>, 8, 144));
        printf("  \"cluster8_G64\": %.3f,\n", run_cluster(p_cluster<8>, 8, 64));
        printf("  \"cluster16_G16\": %.3f,\n", run_cluster(p_cluster<16>, 16, 16));
        printf("  \"cluster16_G32\": %.3f,\n", run_cluster(p_cluster<16>, 16, 32));
        printf("  \"cluster16_G128\": %.3f,\n", run_cluster(p_cluster<16>, 16, 128));
    }
    for (int G : {148, 32}) {
        float us = timeit([&] {
            int st = steps;
            void* a[] = {&st, &out};
            CK(cudaLaunchCooperativeKernel((void*)p_gridsync, G, 512, a, 0, 0));
        });
        printf("  \"gridsync_G%d\": %.3f,\n", G, us);
    }
    printf("  \"steps\": %d\n}\n", steps);
    return 0;
}
