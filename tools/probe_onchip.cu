// probe_onchip.cu — measurement probes for the on-chip training kernel
// design (not product code):
//  1. TMEM read-modify-write throughput per SM: every warp of a 512-thread
//     CTA loads 20 columns of its lane quarter (tcgen05.ld 32x32b x16 + x4),
//     adds, stores back (tcgen05.st), rows after rows.
//  2. shared-memory read-modify-write throughput in the same element layout.
//  3. fp32 -> fp64 widening rate on the integer pipe (the exact bit
//     construction for +0 / positive normals) vs F2F.F64.F32, with a DFMA
//     consuming each value (the norm accumulation of the training pass).
// Output: one JSON object (elements or bytes per clock per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void ld4(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                    "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void st4(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}

// rows x (128 lanes x 80 columns) of fp32 in TMEM, iters passes of RMW over all rows
__global__ void __launch_bounds__(512, 1) tmem_rmw(int rows, int iters, float add, long long* clk, float* sink) {
    __shared__ uint32_t base_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&base_s)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = base_s;
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t colg = 20 * (warp >> 2);
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int r = 0; r < rows; ++r) {
            const uint32_t a = base + lane_off + (uint32_t)(80 * r) + colg;
            uint32_t v[20];
            ld16(a, v);
            ld4(a + 16, v + 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 20; ++i) {
                float f = __uint_as_float(v[i]) + add;
                acc += f;
                v[i] = __float_as_uint(f);
            }
            st16(a, v);
            st4(a + 16, v + 16);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512) : "memory");
}

// the same RMW on shared memory rows (float4 per thread per j: the register chunking)
__global__ void __launch_bounds__(512, 1) smem_rmw(int rows, int iters, float add, long long* clk, float* sink) {
    extern __shared__ float4 sm4[];
    const int d4 = 2500;   // 10,000 floats per row
    for (int i = threadIdx.x; i < rows * d4; i += 512) sm4[i] = make_float4(0, 0, 0, 0);
    __syncthreads();
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int r = 0; r < rows; ++r) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int c = threadIdx.x + 512 * j;
                if (c < d4) {
                    float4 v = sm4[r * d4 + c];
                    v.x += add; v.y += add; v.z += add; v.w += add;
                    acc += v.x;
                    sm4[r * d4 + c] = v;
                }
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
}

// fp32 -> fp64 widening + DFMA: mode 0 = F2F (cvt.f64.f32), 1 = integer
// construction (+0 / positive normals), 2 = half and half
__global__ void __launch_bounds__(512, 1) widen(const float* __restrict__ src, int n, int iters, int mode,
                                                long long* clk, double* sink) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = src[(threadIdx.x * 16 + i) % n];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            double w;
            const bool use_int = mode == 1 || (mode == 2 && (i & 1));
            if (use_int) {
                const uint32_t b = __float_as_uint(v[i]);
                const uint32_t hi = (b >> 3) + (896u << 20);
                const uint32_t lo = b << 29;
                w = (b & 0x7F800000u) ? __hiloint2double((int)hi, (int)lo) : 0.0;
            } else {
                w = (double)v[i];
            }
            if (i & 2) { if (i & 1) a3 = fma(w, w, a3); else a2 = fma(w, w, a2); }
            else { if (i & 1) a1 = fma(w, w, a1); else a0 = fma(w, w, a0); }
            v[i] = __uint_as_float(__float_as_uint(v[i]) ^ (it & 1));   // keep the loop honest
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = a0 + a1 + a2 + a3;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long long* clk;
    float* sink;
    double* dsink;
    float* src;
    CK(cudaMalloc(&clk, sizeof(long long) * sms));
    CK(cudaMalloc(&sink, sizeof(float) * sms * 512));
    CK(cudaMalloc(&dsink, sizeof(double) * sms * 512));
    CK(cudaMalloc(&src, sizeof(float) * 8192));
    {
        float h[8192];
        for (int i = 0; i < 8192; ++i) h[i] = 0.001f * (1 + (i % 977));
        CK(cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice));
    }
    long long hc[256];
    auto median_clk = [&](int n) -> double {
        if (cudaMemcpy(hc, clk, sizeof(long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1.0;
        long long s = 0;
        for (int i = 0; i < n; ++i) s += hc[i];
        return (double)s / n;
    };
    printf("{");
    // 1. TMEM RMW: 6 rows x 10,240 fp32, 200 passes, one CTA per SM
    const int rows = 6, iters = 200;
    tmem_rmw<<<sms, 512>>>(rows, iters, 1.0f, clk, sink);
    CK(cudaDeviceSynchronize());
    tmem_rmw<<<sms, 512>>>(rows, iters, 1.0f, clk, sink);
    CK(cudaDeviceSynchronize());
    double c = median_clk(sms);
    double bytes = 2.0 * rows * iters * 128 * 80 * 4;   // read + write
    printf("\"tmem_rmw_bytes_per_clk_per_sm\": %.2f, \"tmem_rmw_elems_per_clk_per_sm\": %.2f, ", bytes / c, bytes / 8 / c);
    // 2. SMEM RMW: 5 rows x 10,000 fp32 (200 KB)
    CK(cudaFuncSetAttribute(smem_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 40000));
    smem_rmw<<<sms, 512, 5 * 40000>>>(5, iters, 1.0f, clk, sink);
    CK(cudaDeviceSynchronize());
    smem_rmw<<<sms, 512, 5 * 40000>>>(5, iters, 1.0f, clk, sink);
    CK(cudaDeviceSynchronize());
    c = median_clk(sms);
    bytes = 2.0 * 5 * iters * 40000;
    printf("\"smem_rmw_bytes_per_clk_per_sm\": %.2f, \"smem_rmw_elems_per_clk_per_sm\": %.2f, ", bytes / c, bytes / 8 / c);
    // 3. widening + DFMA
    const char* names[3] = {"f2f", "int", "split"};
    for (int mode = 0; mode < 3; ++mode) {
        widen<<<sms, 512>>>(src, 8192, 2000, mode, clk, dsink);
        CK(cudaDeviceSynchronize());
        widen<<<sms, 512>>>(src, 8192, 2000, mode, clk, dsink);
        CK(cudaDeviceSynchronize());
        c = median_clk(sms);
        const double el = 512.0 * 16 * 2000;
        printf("\"widen_dfma_%s_per_clk_per_sm\": %.2f%s", names[mode], el / c, mode < 2 ? ", " : "");
    }
    printf("}\n");
    return 0;
}
