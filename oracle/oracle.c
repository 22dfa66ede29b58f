/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline "port").
 * Never linked into, called by, or shipped with the product library; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Plain-C restatement of the reference CPU stencil sweep and its synthetic
 * inputs (/root/reference/proj/core/src/stencil.cpp):
 *   or_random_grid   stencil.cpp:361-369  mt19937_64(seed), (x & 0xff) / 256
 *   or_preset        stencil.cpp:90-159   Table-2 shapes, dyadic weights,
 *                                         points sorted lexicographically
 *   or_direct_apply  stencil.cpp:231-270  valid region (N - k + 1 per axis per
 *                                         step), fp64, lexicographic point order
 *   or_direct_apply_mt   the same sweep with its output rows split over host
 *                        threads (every output is computed exactly as in the
 *                        serial sweep: bitwise identical), plus the round16
 *                        semantics of the device path as an option: each step
 *                        rounds its inputs to binary16 (RNE; fp16.hpp:13-59,
 *                        emulator.cpp:100-117), sums in fp64 and stores fp32
 * Pinned against the reference itself: tests/golden/direct_apply.npz is written
 * by oracle/make_golden.py from oracle/_ref/libstensor_ref.so (the unmodified
 * reference sources) and tests/test_oracle.py checks this file bit-for-bit.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ mt19937_64 */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void or_random_grid(int ndims, const uint64_t* dims, uint64_t seed, double* out) {
    uint64_t n = 1;
    for (int a = 0; a < ndims; ++a) n *= dims[a];
    mt64 g;
    mt64_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = (double)(mt64_next(&g) & 0xffu) / 256.0;
}

/* float variant for device uploads (values are exact in fp32) */
void or_random_grid_f32(int ndims, const uint64_t* dims, uint64_t seed, float* out) {
    uint64_t n = 1;
    for (int a = 0; a < ndims; ++a) n *= dims[a];
    mt64 g;
    mt64_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)(mt64_next(&g) & 0xffu) / 256.0f;
}

/* ---------------------------------------------------------------- presets */
static int cmp_off(const int* a, const int* b) {
    for (int i = 0; i < 3; ++i)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

static void sort_points(int n, int* offs, double* w) {
    for (int i = 1; i < n; ++i) /* insertion sort: n <= 49 */
        for (int j = i; j > 0 && cmp_off(offs + 3 * j, offs + 3 * (j - 1)) < 0; --j) {
            for (int c = 0; c < 3; ++c) {
                const int t = offs[3 * j + c];
                offs[3 * j + c] = offs[3 * (j - 1) + c];
                offs[3 * (j - 1) + c] = t;
            }
            const double tw = w[j];
            w[j] = w[j - 1];
            w[j - 1] = tw;
        }
}

/* Returns the point count (<= 49), or -1 for an unknown name. offs: 3 ints per point. */
int or_preset(const char* name, int* dims, int* k, int* offs, double* w) {
    int d, kk, star;
    double centre, other;
    if (!strcmp(name, "Heat-1D")) { d = 1; kk = 3; star = 1; centre = 0.5; other = 0.25; }
    else if (!strcmp(name, "1D5P")) { d = 1; kk = 5; star = 1; centre = 0.375; other = 0; }
    else if (!strcmp(name, "Heat-2D")) { d = 2; kk = 3; star = 1; centre = 0.5; other = 0.125; }
    else if (!strcmp(name, "Box-2D9P")) { d = 2; kk = 3; star = 0; centre = 0.5; other = 0.0625; }
    else if (!strcmp(name, "Star-2D13P")) { d = 2; kk = 7; star = 1; centre = 0.25; other = 0.0625; }
    else if (!strcmp(name, "Box-2D49P")) { d = 2; kk = 7; star = 0; centre = 0.25; other = 0.015625; }
    else if (!strcmp(name, "Heat-3D")) { d = 3; kk = 3; star = 1; centre = 0.25; other = 0.125; }
    else if (!strcmp(name, "Box-3D27P")) { d = 3; kk = 3; star = 0; centre = 0.1875; other = 0.03125; }
    else return -1;
    const int r = (kk - 1) / 2;
    int n = 0;
    if (star) {
        memset(offs, 0, 3 * sizeof(int));
        w[n++] = centre;
        for (int a = 0; a < d; ++a)
            for (int o = 1; o <= r; ++o)
                for (int s = -1; s <= 1; s += 2) {
                    memset(offs + 3 * n, 0, 3 * sizeof(int));
                    offs[3 * n + a] = s * o;
                    /* 1D5P carries distance-dependent weights (stencil.cpp:141-147) */
                    w[n++] = strcmp(name, "1D5P") ? other : (o == 1 ? 0.25 : 0.0625);
                }
    } else {
        int cells = 1;
        for (int a = 0; a < d; ++a) cells *= kk;
        for (int c = 0; c < cells; ++c) {
            int rem = c, z = 1;
            memset(offs + 3 * n, 0, 3 * sizeof(int));
            for (int a = d - 1; a >= 0; --a) {
                offs[3 * n + a] = rem % kk - r;
                rem /= kk;
                if (offs[3 * n + a] != 0) z = 0;
            }
            w[n++] = z ? centre : other;
        }
    }
    sort_points(n, offs, w);
    *dims = d;
    *k = kk;
    return n;
}

/* -------------------------------------------------------------- the sweep */
/* One valid-region step: out extents = in extents - (k - 1). */
static void sweep_once(int ndims, const uint64_t* in_dims, int k, int npts, const int* offs,
                       const double* w, const double* in, double* out) {
    const int r = (k - 1) / 2;
    uint64_t od[3] = {1, 1, 1}, id[3] = {1, 1, 1};
    /* right-align into (z, y, x) */
    for (int a = 0; a < ndims; ++a) {
        id[3 - ndims + a] = in_dims[a];
        od[3 - ndims + a] = in_dims[a] - (uint64_t)k + 1;
    }
    /* per-point flat offsets relative to the window origin (z0, y0, x0) */
    int64_t rel[64];
    for (int p = 0; p < npts; ++p) {
        int o[3] = {0, 0, 0};
        for (int a = 0; a < ndims; ++a) o[3 - ndims + a] = offs[3 * p + a] + r;
        rel[p] = ((int64_t)o[0] * (int64_t)id[1] + o[1]) * (int64_t)id[2] + o[2];
    }
    for (uint64_t z = 0; z < od[0]; ++z)
        for (uint64_t y = 0; y < od[1]; ++y) {
            const double* src = in + (z * id[1] + y) * id[2];
            double* dst = out + (z * od[1] + y) * od[2];
            for (uint64_t x = 0; x < od[2]; ++x) {
                double acc = 0.0;
                for (int p = 0; p < npts; ++p) acc += w[p] * src[x + (uint64_t)rel[p]];
                dst[x] = acc;
            }
        }
}

/* T valid-region steps; out must hold prod(dims - T(k-1)) doubles. 0 = ok. */
int or_direct_apply(int ndims, const uint64_t* dims, int k, int npts, const int* offs,
                    const double* w, const double* in, uint64_t steps, double* out) {
    if (steps == 0 || ndims < 1 || ndims > 3 || npts < 1 || npts > 64) return 1;
    uint64_t cur[3], n = 1;
    for (int a = 0; a < ndims; ++a) {
        if (dims[a] < (uint64_t)k + (steps - 1) * (uint64_t)(k - 1)) return 2;
        cur[a] = dims[a];
        n *= dims[a];
    }
    double* a = (double*)malloc(n * sizeof(double));
    double* b = (double*)malloc(n * sizeof(double));
    if (!a || !b) {
        free(a);
        free(b);
        return 3;
    }
    memcpy(a, in, n * sizeof(double));
    for (uint64_t s = 0; s < steps; ++s) {
        sweep_once(ndims, cur, k, npts, offs, w, a, b);
        for (int d = 0; d < ndims; ++d) cur[d] -= (uint64_t)k - 1;
        double* t = a;
        a = b;
        b = t;
    }
    uint64_t m = 1;
    for (int d = 0; d < ndims; ++d) m *= cur[d];
    memcpy(out, a, m * sizeof(double));
    free(a);
    free(b);
    return 0;
}

/* ------------------------------------------------- threaded / round16 sweep */
/* binary16 RNE of a value exactly representable in fp32 (the device rounds its
 * fp32 grid values with __floats2half2_rn), widened back. Bit arithmetic rather
 * than _Float16 casts (software conversions without F16C: 10x slower). */
static double round16(double x) {
    float f = (float)x;
    uint32_t u;
    memcpy(&u, &f, 4);
    const uint32_t e = (u >> 23) & 0xffu;
    if (e == 0xffu) return x;                   /* inf / nan */
    if (e >= 113u) {                            /* binary16 normal range: keep 10 bits */
        u += 0x0fffu + ((u >> 13) & 1u);        /* round half to even (carries into e) */
        u &= ~0x1fffu;
        if (((u >> 23) & 0xffu) > 142u) u = (u & 0x80000000u) | 0x7f800000u; /* > 65504: inf */
        memcpy(&f, &u, 4);
        return (double)f;
    }
    /* binary16 subnormals: multiples of 2^-24, ties to even (default rounding mode) */
    return (double)(nearbyintf(f * 16777216.0f) / 16777216.0f);
}

typedef struct {
    const uint64_t* id;
    const uint64_t* od;
    int npts;
    const int64_t* rel;
    const double* w;
    const double* in;
    double* out;
    uint64_t row0, row1; /* output rows (z * od[1] + y) of this worker */
    int store_f32;
} sweep_job;

static void* sweep_rows(void* arg) {
    const sweep_job* j = (const sweep_job*)arg;
    for (uint64_t row = j->row0; row < j->row1; ++row) {
        const uint64_t z = row / j->od[1], y = row % j->od[1];
        const double* src = j->in + (z * j->id[1] + y) * j->id[2];
        double* dst = j->out + row * j->od[2];
        for (uint64_t x = 0; x < j->od[2]; ++x) {
            double acc = 0.0;
            for (int p = 0; p < j->npts; ++p) acc += j->w[p] * src[x + (uint64_t)j->rel[p]];
            dst[x] = j->store_f32 == 2 ? round16((double)(float)acc)
                     : j->store_f32 ? (double)(float)acc : acc;
        }
    }
    return NULL;
}

/* T valid-region steps over `nthreads` host threads. round16 != 0: every step
 * rounds its input values to binary16 first and stores its outputs as fp32 (the
 * operand / storage semantics of the device path, SST_PREC_F16); round16 == 0 is
 * bitwise identical to or_direct_apply. 0 = ok. */
int or_direct_apply_mt(int ndims, const uint64_t* dims, int k, int npts, const int* offs, const double* w,
                       const double* in, uint64_t steps, double* out, int nthreads, int round16_ops) {
    if (steps == 0 || ndims < 1 || ndims > 3 || npts < 1 || npts > 64) return 1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    const int r = (k - 1) / 2;
    uint64_t cur[3] = {1, 1, 1}, n = 1;
    for (int a = 0; a < ndims; ++a) {
        if (dims[a] < (uint64_t)k + (steps - 1) * (uint64_t)(k - 1)) return 2;
        cur[3 - ndims + a] = dims[a];
        n *= dims[a];
    }
    double* a = (double*)malloc(n * sizeof(double));
    double* b = (double*)malloc(n * sizeof(double));
    if (!a || !b) {
        free(a);
        free(b);
        return 3;
    }
    memcpy(a, in, n * sizeof(double));
    pthread_t th[256];
    sweep_job jobs[256];
    for (uint64_t s = 0; s < steps; ++s) {
        uint64_t od[3] = {1, 1, 1}, m = 1;
        for (int d = 3 - ndims; d < 3; ++d) od[d] = cur[d] - (uint64_t)k + 1;
        for (int d = 0; d < 3; ++d) m *= cur[d];
        if (round16_ops && s == 0)  /* later steps' inputs were rounded as they were stored */
            for (uint64_t i = 0; i < m; ++i) a[i] = round16(a[i]);
        int64_t rel[64];
        for (int p = 0; p < npts; ++p) {
            int o[3] = {0, 0, 0};
            for (int d = 0; d < ndims; ++d) o[3 - ndims + d] = offs[3 * p + d] + r;
            rel[p] = ((int64_t)o[0] * (int64_t)cur[1] + o[1]) * (int64_t)cur[2] + o[2];
        }
        const uint64_t rows = od[0] * od[1];
        const int nt = (uint64_t)nthreads < rows ? nthreads : (int)rows;
        for (int t = 0; t < nt; ++t) {
            sweep_job* j = &jobs[t];
            j->id = cur;
            j->od = od;
            j->npts = npts;
            j->rel = rel;
            j->w = w;
            j->in = a;
            j->out = b;
            j->row0 = rows * (uint64_t)t / (uint64_t)nt;
            j->row1 = rows * (uint64_t)(t + 1) / (uint64_t)nt;
            /* round16: store fp32; an input of the next step is stored already rounded */
            j->store_f32 = round16_ops ? (s + 1 < steps ? 2 : 1) : 0;
        }
        int started = 0;
        for (int t = 1; t < nt; ++t)
            if (pthread_create(&th[t], NULL, sweep_rows, &jobs[t]) == 0) {
                ++started;
            } else {
                sweep_rows(&jobs[t]); /* no thread: run it here */
                th[t] = 0;
            }
        sweep_rows(&jobs[0]);
        for (int t = 1; t < nt; ++t)
            if (th[t]) pthread_join(th[t], NULL);
        (void)started;
        for (int d = 3 - ndims; d < 3; ++d) cur[d] -= (uint64_t)k - 1;
        double* t = a;
        a = b;
        b = t;
    }
    uint64_t m = 1;
    for (int d = 0; d < 3; ++d) m *= cur[d];
    memcpy(out, a, m * sizeof(double));
    free(a);
    free(b);
    return 0;
}
