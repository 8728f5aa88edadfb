// Minimal TMA 2D load test: isolates descriptor / mbarrier / TMA issues.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ int g_cx, g_cy;

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, double* out, int bx, int by) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(&bar)), "r"(bx * by * 8) : "memory");
        const void* desc = MODE == 0 ? (const void*)&tm : (const void*)gtm;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            ::"r"(sptr(smem)), "l"(desc), "r"(sptr(&bar)), "r"(g_cx), "r"(g_cy) : "memory");
    }
    asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}"
                 ::"r"(sptr(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = smem[i];
}

int main(int argc, char** argv) {
    int nx = argc > 6 ? atoi(argv[6]) : 128, ny = argc > 7 ? atoi(argv[7]) : 64; int bx = atoi(argv[1]), by = atoi(argv[2]); int prom = atoi(argv[3]); int cx = atoi(argv[4]), cy = atoi(argv[5]);
    double *u, *out; cudaMalloc(&u, nx * ny * 8); cudaMalloc(&out, bx * by * 8);
    static double h[1 << 22]; cudaMemcpyToSymbol(g_cx, &cx, 4); cudaMemcpyToSymbol(g_cy, &cy, 4); for (int i = 0; i < nx * ny; ++i) h[i] = i;
    cudaMemcpy(u, h, (size_t)nx * ny * 8, cudaMemcpyHostToDevice);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap m;
    cuuint64_t gdim[2] = {(cuuint64_t)nx, (cuuint64_t)ny}; cuuint64_t gs[1] = {(cuuint64_t)nx * 8}; cuuint32_t box[2] = {bx, by}; cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, u, gdim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode r=%d q=%d\n", (int)r, (int)q);
    CUtensorMap* gm; cudaMalloc(&gm, sizeof m); cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(out, 0xff, bx * by * 8);
        if (mode == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384); k<0><<<1, 128, 16384>>>(m, gm, out, bx, by); }
        else { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384); k<1><<<1, 128, 16384>>>(m, gm, out, bx, by); }
        cudaError_t e = cudaDeviceSynchronize();
        static double o[256*256]; cudaMemcpy(o, out, bx*by*8, cudaMemcpyDeviceToHost);
        printf("nx %d ny %d box %dx%d prom %d c=(%d,%d) mode %d: %s out[0]=%g out[bx+1]=%g\n", nx, ny, bx, by, prom, cx, cy, mode, cudaGetErrorString(e), o[0], o[bx+1]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
