// probe_tmem_align.cu — correctness probe of tcgen05.ld/st (32x32b) at
// unaligned column offsets: every warp of a 4-warp CTA stores a pattern
// (lane, column) with .x4/.x8/.x16 at base offsets 0..47, reads it back with
// a different shape split, and counts mismatches.  Also checks store-A /
// load-B / store-B / load-A sequences without intermediate waits.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ptm tools/probe_tmem_align.cu && /tmp/ptm
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void st4(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]) : "memory");
}
__device__ __forceinline__ void st8(uint32_t ta, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
__device__ __forceinline__ void ld1(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(ta));
}
__device__ __forceinline__ void ld4(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]),
                 "=r"(r[3]) : "r"(ta));
}
__device__ __forceinline__ void ld16(uint32_t ta, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void probe(int* bad) {
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = s_tmem + ((uint32_t)(32 * warp) << 16);
    int nbad = 0;
    // 1) stores of 8 columns at every offset 0..47 (x4 pairs and x8), read back 16 + 4 + ... via x1
    for (int off = 0; off < 48; ++off) {
        for (int mode = 0; mode < 2; ++mode) {
            uint32_t r[8];
            for (int i = 0; i < 8; ++i) r[i] = (uint32_t)(mode * 1000000 + off * 10000 + lane * 100 + i);
            if (mode == 0) st8(base + off, r); else { st4(base + off, r); st4(base + off + 4, r + 4); }
            wait_st();
            uint32_t q[8];
            for (int i = 0; i < 8; ++i) ld1(base + off + i, q + i);
            wait_ld();
            for (int i = 0; i < 8; ++i) nbad += q[i] != r[i];
        }
    }
    // 2) x16 load at unaligned offsets of a column ramp written with x1-equivalent x4 stores
    for (int c = 0; c < 128; c += 4) {
        uint32_t r[4];
        for (int i = 0; i < 4; ++i) r[i] = (uint32_t)(lane * 1000 + c + i);
        st4(base + 256 + c, r);
    }
    wait_st();
    for (int off = 0; off < 100; ++off) {
        uint32_t q[16];
        ld16(base + 256 + off, q);
        wait_ld();
        for (int i = 0; i < 16; ++i) nbad += q[i] != (uint32_t)(lane * 1000 + off + i);
    }
    // 3) st A; ld B; st B; ld A (no wait between st A and ld B)
    for (int it = 0; it < 64; ++it) {
        uint32_t a[8], b[8], q[8];
        for (int i = 0; i < 8; ++i) { a[i] = 7 * it + i + lane; b[i] = 13 * it + i + 3 * lane; }
        const uint32_t A = base + 28 * (it % 5), B = base + 200 + 28 * (it % 7);
        st8(A, a);
        ld4(B, q); ld4(B + 4, q + 4);
        wait_ld();
        st8(B, b);
        wait_st();
        ld4(A, q); ld4(A + 4, q + 4);
        wait_ld();
        for (int i = 0; i < 8; ++i) nbad += q[i] != a[i];
        ld4(B, q); ld4(B + 4, q + 4);
        wait_ld();
        for (int i = 0; i < 8; ++i) nbad += q[i] != b[i];
    }
    atomicAdd(bad, nbad);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaMemset(d, 0, 4);
    probe<<<148, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("{\"tmem_align_probe\": {\"cuda\": \"%s\", \"mismatches\": %d}}\n", cudaGetErrorString(e), h);
    return 0;
}
