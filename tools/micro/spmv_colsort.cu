// spmv_colsort.cu -- can a column-sorted, large-row-block SpMV layout beat
// the CSR kernel's L1-request roof on the BASELINE band matrix?
//
// Layout (per block of R rows): the block's nonzeros sorted by column, stored
// as val f64 + meta u32 = (col - block_col_lo) << RB | (row - r0).  A warp
// instruction's 32 consecutive entries then span ~34-70 columns (a few L1
// lines) instead of 32 random lines; the products go into y[R] in shared
// memory with atomicAdd (FP64 shared atomics are a CAS loop on sm_100a).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o spmv_colsort spmv_colsort.cu \
//        -I../../include -L../../paper_2502_16851_b200 -lrooflens_b200 -Xlinker -rpath=$PWD/../../paper_2502_16851_b200
//   ./spmv_colsort
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "rooflens_b200.h"

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned ld_stream_u(const unsigned* p) {
    unsigned v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// 64-bit fixed point (scale 2^52) accumulated with two native 32-bit shared
// atomics: the low word's return value gives the carry into the high word.
__device__ __forceinline__ void fx_add(double* ys, int R, unsigned row, double p) {
    const long long q = __double2ll_rn(p * 0x1p52);
    unsigned* lo = reinterpret_cast<unsigned*>(ys);
    int* hi = reinterpret_cast<int*>(ys) + R;
    const unsigned ql = (unsigned)q;
    const unsigned old = atomicAdd(lo + row, ql);
    const int carry = (old + ql) < old;
    atomicAdd(hi + row, (int)(q >> 32) + carry);
}

__device__ __forceinline__ void add96(unsigned* __restrict__ w, double p, double f) {
    const double P = p * f;
    const long long h = __double2ll_rn(P * 0x1p-32);
    const long long l = __double2ll_rn(fma(-(double)h, 0x1p32, P));
    const unsigned long long U = (unsigned long long)(h + (l >> 63));
    const unsigned a0 = (unsigned)l, a1 = (unsigned)U, a2 = (unsigned)(U >> 32);
    const unsigned o0 = atomicAdd(w, a0);
    const unsigned c0 = (o0 + a0) < o0 ? 1u : 0u;
    const unsigned b1 = a1 + c0;
    const unsigned c1a = (b1 < a1) ? 1u : 0u;
    const unsigned o1 = atomicAdd(w + 1, b1);
    const unsigned c1b = (o1 + b1) < o1 ? 1u : 0u;
    atomicAdd(w + 2, a2 + c1a + c1b);
}
// 64-bit variant with the row's two words interleaved
__device__ __forceinline__ void add64i(unsigned* __restrict__ w, double p) {
    const long long q = __double2ll_rn(p * 0x1p52);
    const unsigned ql = (unsigned)q;
    const unsigned old = atomicAdd(w, ql);
    const int carry = (old + ql) < old;
    atomicAdd(w + 1, (unsigned)(q >> 32) + carry);
}

// MODE 0: atomicAdd into smem y;  1: plain (racy) RMW -- timing bound only;
// 2: loads + gathers, no y update (data movement);  3: shared f64 add emulated
// through two u32 atomics? (not used)
template <int MODE, int U>
__global__ void __launch_bounds__(1024, 2) colsort_spmv(int nblocks, int R, int RB, const uint64_t* __restrict__ boff,
                                                         const int* __restrict__ bcol, const int* __restrict__ brow,
                                                         const double* __restrict__ val,
                                                         const unsigned* __restrict__ meta,
                                                         const double* __restrict__ x, double* __restrict__ y,
                                                         int m) {
    extern __shared__ double ys[];
    const unsigned rmask = (1u << RB) - 1;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < R; i += blockDim.x) ys[i] = 0.0;
        __syncthreads();
        const uint64_t e0 = boff[b], e1 = boff[b + 1];
        const double* xb = x + bcol[b];
        uint64_t e = e0 + threadIdx.x;
        const unsigned step = blockDim.x;
        for (; e + (U - 1) * step < e1; e += U * step) {
            double v[U];
            unsigned mt[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = ld_stream(val + e + u * step);
                mt[u] = ld_stream_u(meta + e + u * step);
            }
            double xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = __ldg(xb + (mt[u] >> RB));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double p = v[u] * xv[u];
                if (MODE == 0) atomicAdd(&ys[mt[u] & rmask], p);
                else if (MODE == 1) ys[mt[u] & rmask] += p;
                else if (MODE == 3) fx_add(ys, R, mt[u] & rmask, p);
                else if (MODE == 4) add96(reinterpret_cast<unsigned*>(ys) + 3 * (mt[u] & rmask), p, 0x1p60);
                else if (MODE == 5) add64i(reinterpret_cast<unsigned*>(ys) + 2 * (mt[u] & rmask), p);
                else if (p == 1.2345) ys[0] = p;
            }
        }
        for (; e < e1; e += step) {
            const double v = val[e];
            const unsigned mt = meta[e];
            const double p = v * __ldg(xb + (mt >> RB));
            if (MODE == 0) atomicAdd(&ys[mt & rmask], p);
            else if (MODE == 1) ys[mt & rmask] += p;
            else if (MODE == 3) fx_add(ys, R, mt & rmask, p);
            else if (MODE == 4) add96(reinterpret_cast<unsigned*>(ys) + 3 * (mt & rmask), p, 0x1p60);
            else if (MODE == 5) add64i(reinterpret_cast<unsigned*>(ys) + 2 * (mt & rmask), p);
            else if (p == 1.2345) ys[0] = p;
        }
        __syncthreads();
        const int r0 = brow[b];
        const int rn = min(R, m - r0);
        if (MODE == 4) {
            const unsigned* w = reinterpret_cast<const unsigned*>(ys);
            for (int i = threadIdx.x; i < rn; i += blockDim.x) {
                long long v = ((long long)w[3 * i + 1] << 32) | w[3 * i];
                y[r0 + i] = (double)v * 0x1p-60 + (double)(int)w[3 * i + 2] * 0x1p4;
            }
        } else if (MODE == 5) {
            const unsigned* w = reinterpret_cast<const unsigned*>(ys);
            for (int i = threadIdx.x; i < rn; i += blockDim.x)
                y[r0 + i] = (double)(((long long)w[2 * i + 1] << 32) | w[2 * i]) * 0x1p-52;
        } else if (MODE == 3) {
            const unsigned* lo = reinterpret_cast<const unsigned*>(ys);
            const int* hi = reinterpret_cast<const int*>(ys) + R;
            for (int i = threadIdx.x; i < rn; i += blockDim.x)
                y[r0 + i] = (double)(((long long)hi[i] << 32) | lo[i]) * 0x1p-52;
        } else
        for (int i = threadIdx.x; i < rn; i += blockDim.x) y[r0 + i] = ys[i];
        __syncthreads();
    }
}

// Reorder entries inside each window of PW column-sorted entries so that each
// aligned group of 16 (one half-warp of 64-bit shared accesses) has distinct
// row % 16 (distinct 8-byte bank pairs) where the window allows: greedy, the
// class with the most entries left goes first.
static void bank_order(std::vector<std::pair<uint64_t, double>>& t, int PW, unsigned rmask) {
    std::vector<std::pair<uint64_t, double>> out;
    out.reserve(t.size());
    std::vector<std::vector<std::pair<uint64_t, double>>> cls(16);
    for (size_t w0 = 0; w0 < t.size(); w0 += PW) {
        const size_t w1 = std::min(t.size(), w0 + PW);
        for (auto& c : cls) c.clear();
        for (size_t i = w0; i < w1; ++i) cls[(t[i].first & rmask) & 15].push_back(t[i]);
        size_t left = w1 - w0;
        while (left) {
            // one group of up to 16: take one from each class, largest first
            int order[16];
            for (int c = 0; c < 16; ++c) order[c] = c;
            std::sort(order, order + 16, [&](int a, int b) { return cls[a].size() > cls[b].size(); });
            int taken = 0;
            for (int oi = 0; oi < 16 && left; ++oi) {
                auto& c = cls[order[oi]];
                if (c.empty()) continue;
                out.push_back(c.back());
                c.pop_back();
                --left;
                ++taken;
            }
            // fill the rest of the group of 16 from the largest classes (conflicts)
            while (taken < 16 && left) {
                int big = 0;
                for (int c = 1; c < 16; ++c) if (cls[c].size() > cls[big].size()) big = c;
                out.push_back(cls[big].back());
                cls[big].pop_back();
                --left;
                ++taken;
            }
        }
    }
    t.swap(out);
}

template <int MODE, int U>
__global__ void __launch_bounds__(1024, 1) colsort_spmv1(int nblocks, int R, int RB, const uint64_t* __restrict__ boff,
                                                          const int* __restrict__ bcol, const int* __restrict__ brow,
                                                          const double* __restrict__ val,
                                                          const unsigned* __restrict__ meta,
                                                          const double* __restrict__ x, double* __restrict__ y, int m) {
    extern __shared__ double ys[];
    const unsigned rmask = (1u << RB) - 1;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
        for (int i = threadIdx.x; i < R; i += blockDim.x) ys[i] = 0.0;
        __syncthreads();
        const uint64_t e0 = boff[b], e1 = boff[b + 1];
        const double* xb = x + bcol[b];
        uint64_t e = e0 + threadIdx.x;
        const unsigned step = blockDim.x;
        for (; e + (U - 1) * step < e1; e += U * step) {
            double v[U];
            unsigned mt[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = ld_stream(val + e + u * step);
                mt[u] = ld_stream_u(meta + e + u * step);
            }
            double xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = __ldg(xb + (mt[u] >> RB));
#pragma unroll
            for (int u = 0; u < U; ++u) atomicAdd(&ys[mt[u] & rmask], v[u] * xv[u]);
        }
        for (; e < e1; e += step) atomicAdd(&ys[meta[e] & rmask], val[e] * __ldg(xb + (meta[e] >> RB)));
        __syncthreads();
        const int r0 = brow[b];
        const int rn = min(R, m - r0);
        for (int i = threadIdx.x; i < rn; i += blockDim.x) y[r0 + i] = ys[i];
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    const int m = 1 << 22, k = 16, hb = 65536;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    // CSR band matrix (16 distinct sorted columns per row in [i-hb, i+hb])
    std::vector<int> rp(m + 1), col((size_t)m * k);
    std::vector<double> val((size_t)m * k), x(m);
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    for (int i = 0; i < m; ++i) {
        rp[i] = i * k;
        const long lo = std::max<long>(0, i - hb), hi = std::min<long>(m - 1, i + hb);
        int* c = &col[(size_t)i * k];
        int n = 0;
        while (n < k) {
            const int cand = (int)(lo + (long)(rng() % (uint64_t)(hi - lo + 1)));
            bool dup = false;
            for (int j = 0; j < n; ++j) dup |= c[j] == cand;
            if (!dup) c[n++] = cand;
        }
        std::sort(c, c + k);
        for (int j = 0; j < k; ++j) val[(size_t)i * k + j] = U(rng);
    }
    rp[m] = m * k;
    for (auto& v : x) v = U(rng);
    // reference y (serial CSR)
    std::vector<double> yref(m);
    for (int i = 0; i < m; ++i) {
        double a = 0;
        for (int j = rp[i]; j < rp[i + 1]; ++j) a += val[j] * x[col[j]];
        yref[i] = a;
    }
    int *d_rp, *d_col;
    double *d_val, *d_x, *d_y;
    CK(cudaMalloc(&d_rp, (m + 1) * 4));
    CK(cudaMalloc(&d_col, (size_t)m * k * 4));
    CK(cudaMalloc(&d_val, (size_t)m * k * 8));
    CK(cudaMalloc(&d_x, (size_t)m * 8));
    CK(cudaMalloc(&d_y, (size_t)m * 8));
    CK(cudaMemcpy(d_rp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_col, col.data(), (size_t)m * k * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_val, val.data(), (size_t)m * k * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_x, x.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double model_bytes = 889192452.0;
    auto check = [&](const char* name) {
        std::vector<double> yg(m);
        CK(cudaMemcpy(yg.data(), d_y, (size_t)m * 8, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (int i = 0; i < m; ++i) num += (yg[i] - yref[i]) * (yg[i] - yref[i]), den += yref[i] * yref[i];
        printf("  %s rel err %.3e\n", name, std::sqrt(num / den));
    };
    // CSR kernel of the library
    {
        rl_kchar kc;
        for (int it = 0; it < 3; ++it)
            rl_spmv_csr(RL_CUDA_CORE, RL_FP64, m, m, (uint64_t)m * k, d_rp, d_col, d_val, d_x, d_y, nullptr, &kc);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int it = 0; it < 20; ++it)
            rl_spmv_csr(RL_CUDA_CORE, RL_FP64, m, m, (uint64_t)m * k, d_rp, d_col, d_val, d_x, d_y, nullptr, &kc);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("CSR (rl_spmv_csr): %.4f ms  %.1f GB/s\n", ms / 20, model_bytes / (ms / 20 * 1e-3) / 1e9);
        check("csr");
    }
    for (int cfg = 0; cfg < 2; ++cfg) {
        const int waves = 2;
        const int PW = (int[]){64, 128}[cfg];
        // R = rows per block so that nblocks = waves * 2 * sms exactly covers m
        const int nb_target = waves * 2 * sms;
        const int R = (m + nb_target - 1) / nb_target;
        int RB = 0;
        while ((1 << RB) < R) ++RB;
        const int nblocks = (m + R - 1) / R;
        std::vector<uint64_t> boff(nblocks + 1);
        std::vector<int> bcol(nblocks), brow(nblocks);
        std::vector<double> sval((size_t)m * k);
        std::vector<unsigned> smeta((size_t)m * k);
        bool ok = true;
        std::vector<std::pair<uint64_t, double>> tmp;
        for (int b = 0; b < nblocks; ++b) {
            const int r0 = b * R, r1 = std::min(m, r0 + R);
            boff[b] = rp[r0];
            brow[b] = r0;
            int clo = m, chi = 0;
            for (int j = rp[r0]; j < rp[r1]; ++j) clo = std::min(clo, col[j]), chi = std::max(chi, col[j]);
            bcol[b] = clo;
            if ((uint64_t)(chi - clo) >= (1ull << (32 - RB))) ok = false;
            tmp.clear();
            for (int r = r0; r < r1; ++r)
                for (int j = rp[r]; j < rp[r + 1]; ++j)
                    tmp.push_back({((uint64_t)(col[j] - clo) << RB) | (uint64_t)(r - r0), val[j]});
            std::sort(tmp.begin(), tmp.end(), [](auto& a, auto& b) { return a.first < b.first; });
            if (PW) bank_order(tmp, PW, (1u << RB) - 1);
            for (size_t t = 0; t < tmp.size(); ++t) {
                smeta[boff[b] + t] = (unsigned)tmp[t].first;
                sval[boff[b] + t] = tmp[t].second;
            }
        }
        boff[nblocks] = rp[m];
        if (!ok) {
            printf("R=%d: span does not fit\n", R);
            continue;
        }
        uint64_t* d_boff;
        int *d_bcol, *d_brow;
        double* d_sval;
        unsigned* d_meta;
        CK(cudaMalloc(&d_boff, (nblocks + 1) * 8));
        CK(cudaMalloc(&d_bcol, nblocks * 4));
        CK(cudaMalloc(&d_brow, nblocks * 4));
        CK(cudaMalloc(&d_sval, (size_t)m * k * 8));
        CK(cudaMalloc(&d_meta, (size_t)m * k * 4));
        CK(cudaMemcpy(d_boff, boff.data(), (nblocks + 1) * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_bcol, bcol.data(), nblocks * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_brow, brow.data(), nblocks * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_sval, sval.data(), (size_t)m * k * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_meta, smeta.data(), (size_t)m * k * 4, cudaMemcpyHostToDevice));
        const size_t smem = (size_t)R * 12 + 16;
        auto run = [&](auto kern, const char* name, int threads, int grid) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int it = 0; it < 3; ++it)
                kern<<<grid, threads, smem>>>(nblocks, R, RB, d_boff, d_bcol, d_brow, d_sval, d_meta, d_x, d_y, m);
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            for (int it = 0; it < 20; ++it)
                kern<<<grid, threads, smem>>>(nblocks, R, RB, d_boff, d_bcol, d_brow, d_sval, d_meta, d_x, d_y, m);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("R=%d PW=%d (%d blocks, grid %d x %d) %s: %.4f ms  %.1f GB/s\n", R, PW, nblocks, grid, threads, name,
                   ms / 20, model_bytes / (ms / 20 * 1e-3) / 1e9);
        };
        run(colsort_spmv<0, 3>, "atomic U3", 1024, 2 * sms);
        run(colsort_spmv<3, 4>, "fixed-point u32x2 U4", 1024, 2 * sms);
        check("fixed");
        run(colsort_spmv<5, 4>, "fixed-point 64 interleaved U4", 1024, 2 * sms);
        check("fixed64i");
        run(colsort_spmv<5, 2>, "fixed-point 64 interleaved U2", 1024, 2 * sms);
        run(colsort_spmv<4, 2>, "fixed-point 96 U2", 1024, 2 * sms);
        check("fixed96");
        run(colsort_spmv<4, 3>, "fixed-point 96 U3", 1024, 2 * sms);
        run(colsort_spmv<4, 4>, "fixed-point 96 U4", 1024, 2 * sms);
        CK(cudaFree(d_boff));
        CK(cudaFree(d_bcol));
        CK(cudaFree(d_brow));
        CK(cudaFree(d_sval));
        CK(cudaFree(d_meta));
    }
    return 0;
}
