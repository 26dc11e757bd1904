// probes.cu — B200 microbenchmarks for the roofline denominators SURVEY §7.1
// step 0 asks for: FP64 DFMA rate, fp32->fp64 conversion rate, the
// publish/poll exchange latency of the training kernel's per-step argmin,
// L2 read+write bandwidth vs footprint.  Dev tooling, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probes tools/probes.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void dfma_kernel(double* out, int iters, double s) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 0.5);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.678) out[0] = t;
}

// one F2F.F64.F32 + one DADD per element-step (the distance loop's mix minus the DFMA)
__global__ void f2f_kernel(double* out, int iters) {
    float f[8];
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x + i; a[i] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] += (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.678) out[0] = t;
}

// the training kernel's inner element: x, w fp32 -> d = (double)x - (double)w; acc = fma(d, d, acc)
__global__ void dist_kernel(double* out, int iters) {
    float x[8], w[8];
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; w[i] = i * 0.5f; a[i] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d = (double)x[i] - (double)w[i];
            a[i] = fma(d, d, a[i]);
            x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);
        }
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.678) out[0] = t;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// publish/poll all-gather of one u64 per CTA per step (the training exchange), no work
__global__ void xchg_kernel(unsigned long long* slots, int steps, unsigned long long* out) {
    const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int t = 0; t < steps; ++t) {
        if (threadIdx.x < 32) {
            unsigned long long tag = 0x80ull | (unsigned long long)(t & 0x7F);
            unsigned long long* s = slots + (size_t)(t & 1) * G;
            if (lane == 0) st_relaxed_u64(s + b, ((unsigned long long)(b * 7 + t) << 8) | tag);
            for (;;) {
                unsigned long long m = ~0ull;
                bool ok = true;
                for (int j = lane; j < G; j += 32) {
                    unsigned long long v = ld_relaxed_u64(s + j);
                    ok &= (v & 0xFF) == tag;
                    m = v < m ? v : m;
                }
                if (__all_sync(0xffffffffu, ok)) { acc += m; break; }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc == 42) out[0] = acc;
}

__global__ void l2rw_kernel(float4* buf, size_t n4, int reps) {
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(buf + i);
            v.x += 1.0f;
            __stcg(buf + i, v);
        }
    }
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk_khz;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    double* dout;
    CK(cudaMalloc(&dout, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms;
    printf("{\n  \"sms\": %d,\n", sms);

    {   // DFMA
        int blocks = sms * 8, threads = 256, iters = 20000;
        dfma_kernel<<<blocks, threads>>>(dout, 100, 1.0000001);
        CK(cudaEventRecord(e0));
        dfma_kernel<<<blocks, threads>>>(dout, iters, 1.0000001);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double fmas = (double)blocks * threads * iters * 8;
        printf("  \"dfma_tflops\": %.3f,\n  \"dfma_per_clk_per_sm_at_max\": %.2f,\n", 2 * fmas / (ms * 1e-3) / 1e12,
               fmas / (ms * 1e-3) / (sms * clk_khz * 1e3));
    }
    {   // F2F + DADD
        int blocks = sms * 8, threads = 256, iters = 20000;
        f2f_kernel<<<blocks, threads>>>(dout, 100);
        CK(cudaEventRecord(e0));
        f2f_kernel<<<blocks, threads>>>(dout, iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double el = (double)blocks * threads * iters * 8;
        printf("  \"f2f_plus_dadd_G_per_s\": %.1f,\n", el / (ms * 1e-3) / 1e9);
    }
    {   // distance element
        int blocks = sms * 8, threads = 256, iters = 20000;
        dist_kernel<<<blocks, threads>>>(dout, 100);
        CK(cudaEventRecord(e0));
        dist_kernel<<<blocks, threads>>>(dout, iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double el = (double)blocks * threads * iters * 8;
        printf("  \"dist_elements_G_per_s\": %.1f,\n  \"dist_elements_per_clk_per_sm_at_max\": %.2f,\n",
               el / (ms * 1e-3) / 1e9, el / (ms * 1e-3) / (sms * clk_khz * 1e3));
    }
    {   // exchange latency
        unsigned long long* slots;
        CK(cudaMalloc(&slots, 2 * 1024 * sizeof(unsigned long long)));
        for (int G : {sms, 74, 32, 8}) {
            CK(cudaMemset(slots, 0, 2 * 1024 * sizeof(unsigned long long)));
            int steps = 20000;
            void* args[] = {&slots, &steps, &dout};
            CK(cudaLaunchCooperativeKernel((void*)xchg_kernel, G, 512, args, 0, 0));
            CK(cudaDeviceSynchronize());
            CK(cudaMemset(slots, 0, 2 * 1024 * sizeof(unsigned long long)));
            CK(cudaEventRecord(e0));
            CK(cudaLaunchCooperativeKernel((void*)xchg_kernel, G, 512, args, 0, 0));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("  \"xchg_us_per_step_G%d\": %.3f,\n", G, ms * 1e3 / steps);
        }
    }
    {   // L2 read+write bandwidth vs footprint
        size_t maxb = (size_t)512 << 20;
        float4* buf;
        CK(cudaMalloc(&buf, maxb));
        CK(cudaMemset(buf, 0, maxb));
        printf("  \"l2_rw_GBps\": {");
        bool first = true;
        for (size_t mb : {8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 512}) {
            size_t n4 = (mb << 20) / 16;
            int reps = (int)std::max<size_t>(2, (size_t)4096 / mb);
            l2rw_kernel<<<sms * 4, 512>>>(buf, n4, 2);
            CK(cudaEventRecord(e0));
            l2rw_kernel<<<sms * 4, 512>>>(buf, n4, reps);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            double gbps = 2.0 * (mb << 20) * reps / (ms * 1e-3) / 1e9;
            printf("%s\"%zu\": %.0f", first ? "" : ", ", mb, gbps);
            first = false;
        }
        printf("},\n");
    }
    printf("  \"clock_rate_max_mhz\": %.0f\n}\n", clk_khz / 1e3);
    return 0;
}
