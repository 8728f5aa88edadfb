// dist_kernels.cu -- create-time checks of the distributed SpMV plan
// (dist.cpp): one pass over a part's local CSR that records the widest
// |column - row| and the number of columns outside [0, n), so a matrix whose
// band is wider than the plan's halo fails with ValidationError instead of
// reading outside the x window.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

// out[0] = max |col - (row0 + i)|, out[1] = #columns outside [0, n),
// out[2] = #rows whose row_ptr decreases.
__global__ void __launch_bounds__(256) band_check_kernel(uint64_t rows, const int* __restrict__ rp,
                                                         const int* __restrict__ col, int64_t row0, int64_t n,
                                                         unsigned long long* __restrict__ out) {
    unsigned long long wid = 0, bad = 0, dec = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
        const int s = __ldg(rp + i), e = __ldg(rp + i + 1);
        if (e < s) ++dec;
        const int64_t r = row0 + (int64_t)i;
        for (int k = s; k < e; ++k) {
            const int64_t c = __ldg(col + k);
            if (c < 0 || c >= n) ++bad;
            const unsigned long long d = (unsigned long long)(c > r ? c - r : r - c);
            wid = d > wid ? d : wid;
        }
    }
    for (int o = 16; o; o >>= 1) {
        wid = max(wid, __shfl_xor_sync(0xffffffffu, wid, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        dec += __shfl_xor_sync(0xffffffffu, dec, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, wid);
        if (bad) atomicAdd(out + 1, bad);
        if (dec) atomicAdd(out + 2, dec);
    }
}

}  // namespace

cudaError_t launch_band_check(uint64_t rows, const int* rp, const int* col, int64_t row0, int64_t n,
                              unsigned long long* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), s);
    if (e != cudaSuccess || rows == 0) return e;
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > (uint64_t)kNumSMs * 8) blocks = (uint64_t)kNumSMs * 8;
    band_check_kernel<<<(unsigned)blocks, 256, 0, s>>>(rows, rp, col, row0, n, out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
