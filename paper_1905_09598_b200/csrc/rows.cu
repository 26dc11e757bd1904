// rows.cu — zero-row detection and the list of drawable rows ("All-zero
// document rows after filtering are retained but excluded from training
// sample draws").  A row is zero when it stores no
// non-zero value (explicit zeros of a CSR row, e.g. the idf-0 entries of
// R28, do not count).  Training draws i_t over the non-zero rows only
// (train_row() in som_internal.h); QE / TE score the non-zero rows only.
#include <algorithm>

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "som_internal.h"

namespace som {

namespace {

// one warp per row: flag = row holds a value != 0
__global__ void row_flags_dense_kernel(const float* X, int64_t n, int dim, uint8_t* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool vec = (dim & 3) == 0 && ((uintptr_t)X & 15) == 0;
    for (int64_t r = w0; r < n; r += nw) {
        const float* row = X + r * (int64_t)dim;
        bool nz = false;
        if (vec) {
            const float4* r4 = reinterpret_cast<const float4*>(row);
            for (int k = lane; k < (dim >> 2) && !nz; k += 32) {
                const float4 v = __ldcs(r4 + k);
                nz = v.x != 0.0f || v.y != 0.0f || v.z != 0.0f || v.w != 0.0f;
            }
        } else {
            for (int k = lane; k < dim && !nz; k += 32) nz = row[k] != 0.0f;
        }
        nz = __any_sync(0xffffffffu, nz);
        if (lane == 0) flags[r] = nz ? 1 : 0;
    }
}

__global__ void row_flags_csr_kernel(const int64_t* rowptr, const float* val, int64_t n, uint8_t* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw) {
        bool nz = false;
        for (int64_t p = rowptr[r] + lane; p < rowptr[r + 1] && !nz; p += 32) nz = val[p] != 0.0f;
        nz = __any_sync(0xffffffffu, nz);
        if (lane == 0) flags[r] = nz ? 1 : 0;
    }
}

unsigned flag_blocks(int64_t n) {
    const int64_t warps = std::max<int64_t>(1, std::min<int64_t>(n, 148 * 64));
    return (unsigned)((warps * 32 + 255) / 256);
}

}  // namespace

cudaError_t launch_row_flags_dense(const float* X, int64_t n, int dim, uint8_t* flags, cudaStream_t st) {
    row_flags_dense_kernel<<<flag_blocks(n), 256, 0, st>>>(X, n, dim, flags);
    return cudaGetLastError();
}

cudaError_t launch_row_flags_csr(const int64_t* rowptr, const float* val, int64_t n, uint8_t* flags,
                                 cudaStream_t st) {
    row_flags_csr_kernel<<<flag_blocks(n), 256, 0, st>>>(rowptr, val, n, flags);
    return cudaGetLastError();
}

// scratch bytes of select_rows for n rows
size_t select_rows_temp_bytes(int64_t n) {
    size_t tb = 0;
    cub::CountingInputIterator<int64_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, tb, it, (const uint8_t*)nullptr, (int64_t*)nullptr, (int64_t*)nullptr, n);
    return tb;
}

// idx[0 .. *count) = ascending indices i with flags[i] != 0 (stable).
cudaError_t launch_select_rows(const uint8_t* flags, int64_t n, int64_t* idx, int64_t* count, void* temp,
                               size_t temp_bytes, cudaStream_t st) {
    cub::CountingInputIterator<int64_t> it(0);
    return cub::DeviceSelect::Flagged(temp, temp_bytes, it, flags, idx, count, n, st);
}

}  // namespace som
