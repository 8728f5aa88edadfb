// common.cuh -- device helpers shared by the sm_100a kernels.
//
// Memory-access primitives are inline PTX so the exact instruction is
// explicit: 256-bit LDG/STG (ld/st.global.v4.f64 -> LDG.E.ENL2.256, sm_100a
// only), L1::no_allocate for streamed data, and L2 cache_hint policies
// (evict_first for data touched once, evict_last for the SpMV x vector that
// every row gathers from).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rlb {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// ---------------------------------------------------------------------------
// Counter-based RNG: splitmix64 finaliser keyed by (key, index).  Restated
// independently in oracle/oracle.c; tests check the bits agree.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t fmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix(uint64_t key, uint64_t idx) {
    return fmix(key + (idx + 1ull) * 0x9E3779B97F4A7C15ull);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix(fmix(seed ^ 0x243F6A8885A308D3ull), stream);
}
__host__ __device__ __forceinline__ double u01(uint64_t h) {
    return (double)(h >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// L2 cache policies
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---------------------------------------------------------------------------
// Loads.  Non-volatile asm: the compiler may schedule them freely (inputs are
// read-only for the kernel's lifetime -- required by .nc).
// ---------------------------------------------------------------------------
struct d4 {
    double x, y, z, w;
};

__device__ __forceinline__ d4 ld4_stream(const double* p, uint64_t pol) {
    d4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ d4 ld4_cached(const double* p) {
    d4 v;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream_i32(const int* p, uint64_t pol) {
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_policy(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_cached(const double* p) {
    double v;
    asm("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------
// Stores (volatile + memory clobber: ordered, never elided).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st4_stream(double* p, d4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;"
                 :
                 : "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st4(double* p, d4 v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                 :
                 : "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;"
                 :
                 : "l"(p), "d"(v), "l"(pol)
                 : "memory");
}

// ---------------------------------------------------------------------------
// FP64 tensor core: mma.sync m8n8k4 (lowers to DMMA.8x8x4 on sm_100a).
//   A 8x4 row-major: lane holds A[lane/4][lane%4]
//   B 4x8 col-major: lane holds B[lane%4][lane/4]
//   C/D 8x8:         lane holds D[lane/4][2*(lane%4) + {0,1}]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b,
                                            double c0, double c1) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
        : "=d"(d0), "=d"(d1)
        : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__host__ __device__ __forceinline__ bool aligned32(const void* p) {
    return (reinterpret_cast<uintptr_t>(p) & 31u) == 0;
}

}  // namespace rlb
