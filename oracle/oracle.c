/*
 * oracle.c -- CPU restatement of the three memory-bound kernels of
 * arXiv 2502.16851 ("Can Tensor Cores Benefit Memory-Bound Kernels? (No!)").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker (or the timed CPU baseline).  The product path
 * (paper_2502_16851_b200/) never links, loads or calls it.
 *
 * Parity status: the reference (/root/reference) contains NO executing
 * kernel, no golden vectors and no fixtures for the kernel *results*; it only
 * ships the analytic W/Q models (proj/src/kernels.cpp).  Kernel-result parity
 * is therefore "parity unpinned" by the reference: this file restates the
 * paper's equations directly and is cross-checked in tests/ against
 * independent numpy / scipy.sparse restatements.  The accounting side (W, Q)
 * IS pinned: oracle/_ref is the reference library itself, built from its own
 * sources by oracle/Makefile.
 *
 *   scale        a_i = q * b_i                         PAPER.md:147-151 (Eq. 5)
 *   spmv_csr     y_i = sum_k val[k] * x[col[k]]
 *   stencil      v(p) = sum_s w_s * u(p + s)           PAPER.md:211-215 (Eq. 11)
 *
 * Inputs follow BASELINE.json's configs: counter-based splitmix64 RNG so the
 * device generators (csrc/gen.cu) can reproduce the same bits independently.
 * Built with -ffp-contract=off: every sum below is evaluated exactly in the
 * order written (no FMA contraction), one rounding per operation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Counter-based RNG (splitmix64 finaliser keyed by seed and index).        */
/* ------------------------------------------------------------------------ */

static inline uint64_t fmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

ORC_API uint64_t orc_mix(uint64_t key, uint64_t idx) {
    return fmix(key + (idx + 1ull) * 0x9E3779B97F4A7C15ull);
}

/* Stream keys: 1 = STREAM b, 2 = CSR columns, 3 = CSR values, 4 = x,
 * 5 = stencil initial field. */
ORC_API uint64_t orc_key(uint64_t seed, uint64_t stream) {
    return orc_mix(fmix(seed ^ 0x243F6A8885A308D3ull), stream);
}

static inline double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* kind 0: U[0,1);  kind 1: U[-1,1) = 2u - 1 (exact in binary64). */
ORC_API void orc_fill_uniform(double* out, uint64_t n, uint64_t seed, uint64_t stream,
                              uint64_t idx0, int kind) {
    const uint64_t key = orc_key(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const double u = u01(orc_mix(key, idx0 + (uint64_t)i));
        out[i] = kind ? 2.0 * u - 1.0 : u;
    }
}

/* ------------------------------------------------------------------------ */
/* STREAM SCALE  (reference model kernels.cpp:74-86)      */
/* ------------------------------------------------------------------------ */

ORC_API void orc_scale(double* a, const double* b, double q, uint64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) a[i] = q * b[i];
}

/* Dense GEMV y = A x, row-major (model kernels.cpp:88-101). */
ORC_API void orc_gemv(uint64_t m, uint64_t n, const double* A, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)m; ++i) {
        double acc = 0.0;
        for (uint64_t k = 0; k < n; ++k) acc = acc + A[(uint64_t)i * n + k] * x[k];
        y[i] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* Banded CSR generator (BASELINE.json configs[1]).                         */
/* Row i (global) gets k distinct columns drawn uniformly from              */
/* [max(0,i-hb), min(n-1,i+hb)], sorted ascending.  Requires the band width */
/* to hold k columns for every row.  Values keyed by the global nnz index   */
/* i*k + j so a row-partitioned matrix equals the corresponding rows of the */
/* global matrix.                                                           */
/* ------------------------------------------------------------------------ */

ORC_API int orc_gen_band_csr(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k,
                             uint64_t hb, uint64_t seed, int32_t* rp, int32_t* col,
                             double* val) {
    if (k == 0 || k > 64 || n < k || hb + 1 < k) return 1;
    const uint64_t kc = orc_key(seed, 2), kv = orc_key(seed, 3);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)m_local; ++r) {
        const uint64_t i = row0 + (uint64_t)r;
        const uint64_t lo = i > hb ? i - hb : 0;
        const uint64_t hi = (i + hb < n - 1) ? i + hb : n - 1;
        const uint64_t width = hi - lo + 1;
        int32_t c[64];
        uint32_t cnt = 0;
        const uint64_t rowkey = orc_mix(kc, i);
        for (uint64_t t = 0; cnt < k; ++t) {
            const uint64_t h = orc_mix(rowkey, t);
            const uint64_t cand = lo + (((h >> 32) * width) >> 32);
            int dup = 0;
            for (uint32_t j = 0; j < cnt; ++j) dup |= (c[j] == (int32_t)cand);
            if (!dup) c[cnt++] = (int32_t)cand;
        }
        for (uint32_t a = 1; a < k; ++a) { /* insertion sort */
            int32_t v = c[a];
            int32_t b = (int32_t)a - 1;
            while (b >= 0 && c[b] > v) { c[b + 1] = c[b]; --b; }
            c[b + 1] = v;
        }
        for (uint32_t j = 0; j < k; ++j) {
            col[(uint64_t)r * k + j] = c[j];
            val[(uint64_t)r * k + j] = 2.0 * u01(orc_mix(kv, i * k + j)) - 1.0;
        }
    }
    for (uint64_t r = 0; r <= m_local; ++r) rp[r] = (int32_t)(r * k);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* CSR SpMV  (CSR traffic 182-190; reference model        */
/* kernels.cpp:123-135).  Row sums in storage order, starting from +0.0.    */
/* col_base: x is indexed as x[col[k] - col_base] (row-partitioned halos).  */
/* ------------------------------------------------------------------------ */

ORC_API void orc_spmv_csr(uint64_t m, const int32_t* rp, const int32_t* col,
                          const double* val, const double* x, int64_t col_base,
                          double* y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)m; ++i) {
        double acc = 0.0;
        for (int32_t k = rp[i]; k < rp[i + 1]; ++k)
            acc = acc + val[k] * x[(int64_t)col[k] - col_base];
        y[i] = acc;
    }
}

/* ------------------------------------------------------------------------ */
/* Jacobi stencils  (Eq. 11; presets kernels.cpp:54-68).   */
/*                                                                          */
/* Grid layout: x fastest; 2D arrays are ny rows of nx, 3D nz planes of     */
/* ny*nx.  The outer ring of width `radius` is a Dirichlet boundary: never  */
/* written.  Each step writes every interior point of v from u, then the    */
/* roles swap; after `steps` steps the result is in u if steps is even,     */
/* else in v.  Offsets are summed in the canonical order below, starting    */
/* from +0.0 with one rounding per multiply and per add.                    */
/* ------------------------------------------------------------------------ */

typedef struct { int dz, dy, dx; } off3;

static const off3 OFF_2D5[5] = {{0, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
static const off3 OFF_3D7[7] = {{0, 0, 0},  {-1, 0, 0}, {1, 0, 0}, {0, -1, 0},
                                {0, 1, 0},  {0, 0, -1}, {0, 0, 1}};

static int preset_info(const char* name, int* dim, int* npts, int* radius) {
    if (!strcmp(name, "2d5pt")) { *dim = 2; *npts = 5; *radius = 1; return 0; }
    if (!strcmp(name, "2d9pt")) { *dim = 2; *npts = 9; *radius = 1; return 0; }
    if (!strcmp(name, "2d13pt")) { *dim = 2; *npts = 13; *radius = 3; return 0; }
    if (!strcmp(name, "2d49pt")) { *dim = 2; *npts = 49; *radius = 3; return 0; }
    if (!strcmp(name, "3d7pt")) { *dim = 3; *npts = 7; *radius = 1; return 0; }
    if (!strcmp(name, "3d27pt")) { *dim = 3; *npts = 27; *radius = 1; return 0; }
    return 1;
}

/* Canonical offsets for every preset (count returned). */
static int preset_offsets(const char* name, off3* o) {
    int n = 0;
    if (!strcmp(name, "2d5pt")) { memcpy(o, OFF_2D5, sizeof OFF_2D5); return 5; }
    if (!strcmp(name, "3d7pt")) { memcpy(o, OFF_3D7, sizeof OFF_3D7); return 7; }
    if (!strcmp(name, "2d9pt") || !strcmp(name, "2d49pt")) {
        const int r = name[2] == '9' ? 1 : 3;
        for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx) o[n++] = (off3){0, dy, dx};
        return n;
    }
    if (!strcmp(name, "2d13pt")) {
        o[n++] = (off3){0, 0, 0};
        for (int d = 1; d <= 3; ++d) {
            o[n++] = (off3){0, -d, 0}; o[n++] = (off3){0, d, 0};
            o[n++] = (off3){0, 0, -d}; o[n++] = (off3){0, 0, d};
        }
        return n;
    }
    if (!strcmp(name, "3d27pt")) {
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) o[n++] = (off3){dz, dy, dx};
        return n;
    }
    return 0;
}

ORC_API int orc_preset_points(const char* name) {
    int d, p, r;
    return preset_info(name, &d, &p, &r) ? -1 : p;
}

ORC_API int orc_preset_offsets(const char* name, int32_t* dz_dy_dx) {
    off3 o[64];
    const int n = preset_offsets(name, o);
    for (int s = 0; s < n; ++s) {
        dz_dy_dx[3 * s] = o[s].dz; dz_dy_dx[3 * s + 1] = o[s].dy; dz_dy_dx[3 * s + 2] = o[s].dx;
    }
    return n;
}

/* BASELINE.json weights: 2d5pt c0=0.5 c1=0.125; 3d7pt c0=0.4 c1=0.1;
 * 3d27pt raw = 1/(1+|dx|+|dy|+|dz|), S = sum(raw) = 10, w = raw / S.
 * The other presets use the same normalised 1/(1+manhattan) rule. */
ORC_API int orc_default_weights(const char* name, double* w) {
    if (!strcmp(name, "2d5pt")) {
        w[0] = 0.5; for (int s = 1; s < 5; ++s) w[s] = 0.125; return 5;
    }
    if (!strcmp(name, "3d7pt")) {
        w[0] = 0.4; for (int s = 1; s < 7; ++s) w[s] = 0.1; return 7;
    }
    off3 o[64];
    const int n = preset_offsets(name, o);
    if (n == 0) return -1;
    double raw[64], S = 0.0;
    for (int s = 0; s < n; ++s) {
        raw[s] = 1.0 / (double)(1 + abs(o[s].dx) + abs(o[s].dy) + abs(o[s].dz));
        S = S + raw[s];
    }
    for (int s = 0; s < n; ++s) w[s] = raw[s] / S;
    return n;
}

/* Interior U[0,1) keyed by the global linear index, boundary ring 0.
 * Global grid nx * ny (* nz for dim 3); u holds outer indices [o0, o1)
 * (rows in 2D, planes in 3D). */
ORC_API void orc_stencil_init(double* u, uint64_t nx, uint64_t ny, uint64_t nz, int dim,
                              uint64_t o0, uint64_t o1, int radius, uint64_t seed) {
    const uint64_t key = orc_key(seed, 5);
    const uint64_t per_outer = dim == 2 ? nx : nx * ny;
    const uint64_t r = (uint64_t)radius;
#pragma omp parallel for schedule(static)
    for (int64_t oo = 0; oo < (int64_t)(o1 - o0); ++oo) {
        const uint64_t o = o0 + (uint64_t)oo;
        for (uint64_t in = 0; in < per_outer; ++in) {
            const uint64_t x = in % nx;
            const uint64_t y = dim == 2 ? o : in / nx;
            const int zin = dim == 2 || (o >= r && o + r < nz);
            const int yin = y >= r && y + r < ny;
            const int xin = x >= r && x + r < nx;
            u[(uint64_t)oo * per_outer + in] =
                (zin && yin && xin) ? u01(orc_mix(key, o * per_outer + in)) : 0.0;
        }
    }
}

/* Outer range [olo, ohi) (rows in 2D, planes in 3D) is clipped to the
 * interior; the full-grid sweep passes [0, n_outer). */
static void sweep_generic(int n_off, const off3* o, const double* w, uint64_t nx,
                          uint64_t ny, uint64_t nz, int r, int is2d, const double* u,
                          double* v, uint64_t olo, uint64_t ohi) {
    const int64_t sx = 1, sy = (int64_t)nx, sz = (int64_t)(nx * ny);
    int64_t d[64];
    for (int s = 0; s < n_off; ++s) d[s] = o[s].dz * sz + o[s].dy * sy + o[s].dx * sx;
    const uint64_t n_outer = is2d ? ny : nz;
    const uint64_t lo = olo > (uint64_t)r ? olo : (uint64_t)r;
    const uint64_t hi = ohi < n_outer - r ? ohi : n_outer - r;
    const uint64_t zlo = is2d ? 0 : lo, zhi = is2d ? 1 : hi;
    const uint64_t ylo = is2d ? lo : (uint64_t)r, yhi = is2d ? hi : ny - r;
    if (lo >= hi) return;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = (int64_t)zlo; z < (int64_t)zhi; ++z)
        for (int64_t y = (int64_t)ylo; y < (int64_t)yhi; ++y) {
            const int64_t base = z * sz + y * sy;
            for (int64_t x = r; x < (int64_t)(nx - r); ++x) {
                const int64_t p = base + x;
                double acc = 0.0;
                for (int s = 0; s < n_off; ++s) acc = acc + w[s] * u[p + d[s]];
                v[p] = acc;
            }
        }
}

/* Specialised sweeps for the three BASELINE presets: identical summation
 * order to sweep_generic, written out so the compiler vectorises along x
 * (this is also the timed CPU baseline, so it should not be sandbagged). */
static void sweep_2d5(const double* w, uint64_t nx, uint64_t ny, const double* u, double* v) {
    const int64_t X = (int64_t)nx;
    const double w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
#pragma omp parallel for schedule(static)
    for (int64_t y = 1; y < (int64_t)ny - 1; ++y) {
        const double* c = u + y * X;
        const double* n = c - X;
        const double* s = c + X;
        double* o = v + y * X;
        for (int64_t x = 1; x < X - 1; ++x) {
            double acc = 0.0;
            acc = acc + w0 * c[x];
            acc = acc + w1 * n[x];
            acc = acc + w2 * s[x];
            acc = acc + w3 * c[x - 1];
            acc = acc + w4 * c[x + 1];
            o[x] = acc;
        }
    }
}

static void sweep_3d7(const double* w, uint64_t nx, uint64_t ny, uint64_t nz, const double* u,
                      double* v) {
    const int64_t X = (int64_t)nx, P = (int64_t)(nx * ny);
    const double w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4], w5 = w[5], w6 = w[6];
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 1; z < (int64_t)nz - 1; ++z)
        for (int64_t y = 1; y < (int64_t)ny - 1; ++y) {
            const double* c = u + z * P + y * X;
            double* o = v + z * P + y * X;
            for (int64_t x = 1; x < X - 1; ++x) {
                double acc = 0.0;
                acc = acc + w0 * c[x];
                acc = acc + w1 * c[x - P];
                acc = acc + w2 * c[x + P];
                acc = acc + w3 * c[x - X];
                acc = acc + w4 * c[x + X];
                acc = acc + w5 * c[x - 1];
                acc = acc + w6 * c[x + 1];
                o[x] = acc;
            }
        }
}

static void sweep_3d27(const double* w, uint64_t nx, uint64_t ny, uint64_t nz, const double* u,
                       double* v) {
    const int64_t X = (int64_t)nx, P = (int64_t)(nx * ny);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t z = 1; z < (int64_t)nz - 1; ++z)
        for (int64_t y = 1; y < (int64_t)ny - 1; ++y) {
            const double* c = u + z * P + y * X;
            double* o = v + z * P + y * X;
            for (int64_t x = 1; x < X - 1; ++x) {
                double acc = 0.0;
                int s = 0;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx, ++s)
                            acc = acc + w[s] * c[x + dz * P + dy * X + dx];
                o[x] = acc;
            }
        }
}

/* dims = {nx, ny, nz}; nz = 1 (or 0) for 2D presets.  weights NULL selects
 * the BASELINE defaults.  Returns 0 on success, nonzero on bad arguments. */
ORC_API int orc_stencil(const char* preset, const uint64_t* dims, const double* weights,
                        uint64_t steps, double* u, double* v) {
    int dim, npts, r;
    if (preset_info(preset, &dim, &npts, &r)) return 1;
    const uint64_t nx = dims[0], ny = dims[1], nz = dim == 3 ? dims[2] : 1;
    if (nx < (uint64_t)(2 * r + 1) || ny < (uint64_t)(2 * r + 1) ||
        (dim == 3 && nz < (uint64_t)(2 * r + 1)))
        return 2;
    double w[64];
    if (weights) memcpy(w, weights, sizeof(double) * (size_t)npts);
    else orc_default_weights(preset, w);
    off3 o[64];
    const int n_off = preset_offsets(preset, o);
    for (uint64_t t = 0; t < steps; ++t) {
        const double* src = (t & 1) ? v : u;
        double* dst = (t & 1) ? u : v;
        if (!strcmp(preset, "2d5pt")) sweep_2d5(w, nx, ny, src, dst);
        else if (!strcmp(preset, "3d7pt")) sweep_3d7(w, nx, ny, nz, src, dst);
        else if (!strcmp(preset, "3d27pt")) sweep_3d27(w, nx, ny, nz, src, dst);
        else sweep_generic(n_off, o, w, nx, ny, nz, r, dim == 2, src, dst, 0, dim == 2 ? ny : nz);
    }
    return 0;
}

/* One sweep v = S(u) over outer indices [o0, o1) (clipped to the interior):
 * the slab building block the distributed tests check against. */
ORC_API int orc_stencil_sweep(const char* preset, const uint64_t* dims, const double* weights,
                              uint64_t o0, uint64_t o1, const double* u, double* v) {
    int dim, npts, r;
    if (preset_info(preset, &dim, &npts, &r)) return 1;
    const uint64_t nx = dims[0], ny = dims[1], nz = dim == 3 ? dims[2] : 1;
    double w[64];
    if (weights) memcpy(w, weights, sizeof(double) * (size_t)npts);
    else orc_default_weights(preset, w);
    off3 o[64];
    const int n_off = preset_offsets(preset, o);
    sweep_generic(n_off, o, w, nx, ny, nz, r, dim == 2, u, v, o0, o1);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Checkers.                                                                 */
/* ------------------------------------------------------------------------ */

/* ||a - b||_2 / ||b||_2 (||a - b||_2 if b == 0), accumulated in long double. */
ORC_API double orc_rel_err(const double* a, const double* b, uint64_t n) {
    long double num = 0.0L, den = 0.0L;
#pragma omp parallel for reduction(+ : num, den) schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const long double d = (long double)a[i] - (long double)b[i];
        num += d * d;
        den += (long double)b[i] * (long double)b[i];
    }
    return den > 0.0L ? (double)sqrtl(num / den) : (double)sqrtl(num);
}

/* Number of positions whose 64-bit patterns differ (bit-exact check). */
ORC_API uint64_t orc_bit_mismatches(const double* a, const double* b, uint64_t n) {
    uint64_t bad = 0;
#pragma omp parallel for reduction(+ : bad) schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) bad += memcmp(&a[i], &b[i], 8) != 0;
    return bad;
}

ORC_API int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
