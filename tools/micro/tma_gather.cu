// tma_gather.cu -- is a TMA tile::gather4 stream a faster way to gather
// random FP64 values from an L2-resident vector than per-lane LDG?
// (SpMV x gathers are bound by ~1 L1 request per SM per cycle.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather tma_gather.cu -lcuda
//   ./tma_gather
//
// x (n doubles, 32 MB) is viewed as a 2D tensor of n/2 rows x 2 columns
// (16-byte rows).  Each lane gathers 4 rows per gather4 into its 64-byte
// shared slot; a warp's 32 gathers complete on one mbarrier per stage.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Baseline: per-lane 8-byte gathers, 16 in flight per lane.  MODE 0
// ld.global.nc.L1::no_allocate, 1 __ldg (L1 allocate), 2 ld.global.nc.L2::cache_hint evict_last (the SpMV path).
template <int MODE>
__global__ void __launch_bounds__(256) ldg_gather(const double* __restrict__ x, const int* __restrict__ idx, int per_thread,
                                                  double* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int T = gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int i = 0; i < per_thread; i += 16) {
        int c[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] = __ldg(idx + (size_t)(i + k) * T + t);
        double v[16];
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MODE == 0)
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[k]) : "l"(x + c[k]));
            else if (MODE == 1)
                v[k] = __ldg(x + c[k]);
            else
                asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(x + c[k]), "l"(pol));
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += v[k];
    }
    if (acc == 123.456) out[0] = acc;
}

// gather4: lane issues one gather4 (4 random x elements) per stage.
template <int S>
__global__ void __launch_bounds__(256) tma_gather4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                   int per_thread, double* out) {
    extern __shared__ __align__(128) double dyn[];
    double(*slot)[256][16] = reinterpret_cast<double(*)[256][16]>(dyn);  // [stage][thread][4 rows x 2], 128-byte slots (TMA destination alignment)
    __shared__ __align__(8) uint64_t bar[S][8];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int T = gridDim.x * blockDim.x;
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(&bar[s][w])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int groups = per_thread / 4;
    auto issue = [&](int g) {
        const int s = g % S;
        int c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = __ldg(idx + (size_t)(4 * g + k) * T + t);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(&bar[s][w])), "r"(32 * 64)
                         : "memory");
        __syncwarp();
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(sptr(&slot[s][tid][0])),
            "l"(&tm), "r"(0), "r"(c[0] >> 1), "r"(c[1] >> 1), "r"(c[2] >> 1), "r"(c[3] >> 1), "r"(sptr(&bar[s][w]))
            : "memory");
    };
    for (int g = 0; g < S && g < groups; ++g) issue(g);
    double acc = 0.0;
    for (int g = 0; g < groups; ++g) {
        const int s = g % S;
        const uint32_t par = (uint32_t)((g / S) & 1);
        asm volatile(
            "{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
                sptr(&bar[s][w])),
            "r"(par)
            : "memory");
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int c = __ldg(idx + (size_t)(4 * g + k) * T + t);
            acc += slot[s][tid][2 * k + (c & 1)];
        }
        __syncwarp();
        if (g + S < groups) issue(g + S);
    }
    if (acc == 123.456) out[0] = acc;
    if (blockIdx.x == 0 && tid == 0) out[1] = acc;
    if (t < 64) out[2 + t] = acc;
}

int main() {
    const size_t n = 1u << 22;  // 32 MB
    std::vector<double> hx(n);
    for (size_t i = 0; i < n; ++i) hx[i] = (double)(i % 1000) * 0.001 + 1.0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int blocks = sms * 8, threads = 256, T = blocks * threads, per_thread = 256;
    std::vector<int> hi((size_t)T * per_thread);
    uint64_t z = 12345;
    for (auto& v : hi) {
        z = z * 6364136223846793005ull + 1442695040888963407ull;
        v = (int)((z >> 33) % n);
    }
    double *x, *out;
    int* idx;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&out, 128 * 8));
    CK(cudaMalloc(&idx, hi.size() * 4));
    CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {2, n / 2};
    cuuint64_t gstr[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box{2,1}: %d\n", (int)r);

    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gathers = (double)T * per_thread;
    auto run_ldg = [&](auto kern, const char* name) {
        for (int rep = 0; rep < 2; ++rep) {
            kern<<<blocks, threads>>>(x, idx, per_thread, out);
            CK(cudaEventRecord(a));
            kern<<<blocks, threads>>>(x, idx, per_thread, out);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s: %.3f ms  %.1f G gathers/s  %.3f per SM per cycle@1.9GHz\n", name, ms, gathers / ms / 1e6,
                   gathers / ms / 1e6 / sms / 1.9);
        }
    };
    run_ldg(ldg_gather<0>, "ldg no_allocate ");
    run_ldg(ldg_gather<1>, "ldg __ldg       ");
    run_ldg(ldg_gather<2>, "ldg L2 evict_last");
    CK(cudaFuncSetAttribute(tma_gather4<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 256 * 128));
    CK(cudaFuncSetAttribute(tma_gather4<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 256 * 128));
    // correctness of gather4 (sum of a thread's values vs host)
    tma_gather4<4><<<blocks, threads, 4 * 256 * 128>>>(tm, idx, per_thread, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> ho(66);
    CK(cudaMemcpy(ho.data(), out, 66 * 8, cudaMemcpyDeviceToHost));
    double ref = 0.0;
    for (int g = 0; g < per_thread; ++g) ref += hx[hi[(size_t)g * T + 0]];
    printf("gather4 check: got %.6f want %.6f\n", ho[2], ref);
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(a));
        tma_gather4<4><<<blocks, threads, 4 * 256 * 128>>>(tm, idx, per_thread, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("gather4 S4: %.3f ms  %.1f G gathers/s  %.3f per SM per cycle@1.9GHz\n", ms, gathers / ms / 1e6,
               gathers / ms / 1e6 / sms / 1.9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        tma_gather4<2><<<blocks, threads, 2 * 256 * 128>>>(tm, idx, per_thread, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("gather4 S2: %.3f ms  %.1f G gathers/s  %.3f per SM per cycle@1.9GHz\n", ms, gathers / ms / 1e6,
               gathers / ms / 1e6 / sms / 1.9);
    }
    return 0;
}
