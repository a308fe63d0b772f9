/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 DOT / GEMV / GER
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it, and only as the checker.  The product
 * library (paper_2108_02025_b200/csrc) never links or calls it.
 *
 * A plain-C restatement of the reference's naive oracles, with their floating
 * point semantics pinned explicitly instead of being left to the compiler:
 *
 *   dot_ref   reference kernels.hpp:119-127  acc = alpha0; acc += x_p*y_p, p ascending
 *   gemv_ref  reference kernels.hpp:171-181  acc = c_i; acc += A(i,j)*x_j, j ascending
 *   ger_ref   reference kernels.hpp:264-270  C(i,j) += x_i*y_j, one fused op
 *
 * The reference's accumulation statements are compiled by GCC 13 with
 * `-O3 -march=native -std=gnu++20` (reference proj/CMakeLists.txt:3-22), and
 * what `acc += a*b` means then depends on the code the compiler emits.
 * Measured on the compiled reference (oracle/_ref, tests/test_oracle.py):
 *
 *   dot_ref / gemv_ref  the first V*floor(n/V) terms are multiplied in 16-byte
 *                       vectors and added to the accumulator one by one in
 *                       ascending order (separately rounded mul, then add);
 *                       the n mod V remainder runs as scalar FMA.
 *                       V = 16 / sizeof(T): 4 for fp32, 2 for fp64.
 *   ger_ref             one FMA per element.
 *
 * The functions below take V as an argument (`vec`): vec = 16/sizeof(T)
 * reproduces the compiled reference bit for bit; vec = 0 gives the pure
 * "multiply then add" reading of the source.  This file is compiled with
 * -ffp-contract=off so every multiply/add/fma here means exactly what it says.
 *
 * Also here: the counter-based SplitMix64 input generator shared bit-for-bit
 * with the device generator (paper_2108_02025_b200/csrc/datagen.cu), and
 * extended-precision "truth" used for the non-vacuous accuracy check that
 * SURVEY.md §8(c) recommends next to BASELINE's contract tolerance.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#include "cabl_oracle.h"

/* ------------------------------------------------------------------------ */
/* SplitMix64, counter form.  value(seed, stream, i) is the (i+1)-th output   */
/* of a SplitMix64 sequence whose state starts at key(seed, stream).          */
/* ------------------------------------------------------------------------ */
#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_sm64_key(uint64_t seed, uint64_t stream) {
    return sm_mix(seed + GOLDEN * (stream + 1ULL));
}

uint64_t oracle_sm64(uint64_t key, uint64_t index) {
    return sm_mix(key + GOLDEN * (index + 1ULL));
}

void oracle_gen_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset) {
    const uint64_t key = oracle_sm64_key(seed, stream);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t u = oracle_sm64(key, offset + i);
        /* 24-bit integer * 2^-23 - 1: exact in fp32, lies in [-1, 1) */
        out[i] = (float)(int32_t)(u >> 40) * (1.0f / 8388608.0f) - 1.0f;
    }
}

void oracle_gen_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset) {
    const uint64_t key = oracle_sm64_key(seed, stream);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t u = oracle_sm64(key, offset + i);
        out[i] = (double)(int64_t)(u >> 11) * (1.0 / 4503599627370496.0) - 1.0;
    }
}

/* Box-Muller on counters (2i, 2i+1).  libm and CUDA math differ in the last
 * ulp, so parity tests copy the device-generated normals back instead of
 * regenerating them here; this host version feeds CPU-only timing runs. */
void oracle_gen_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream,
                           uint64_t offset) {
    const uint64_t key = oracle_sm64_key(seed, stream);
    const double two_pi = 6.283185307179586476925286766559;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t a = oracle_sm64(key, 2 * (offset + i));
        const uint64_t b = oracle_sm64(key, 2 * (offset + i) + 1);
        const double u1 = ((double)(int64_t)(a >> 11) + 1.0) * (1.0 / 9007199254740992.0);
        const double u2 = (double)(int64_t)(b >> 11) * (1.0 / 9007199254740992.0);
        out[i] = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    }
}

/* ------------------------------------------------------------------------ */
/* Naive oracles (reference kernels.hpp:119-127, :171-181, :264-270)        */
/* ------------------------------------------------------------------------ */
/* number of leading terms accumulated as separately rounded mul-then-add */
static inline uint64_t muladd_terms(uint64_t n, unsigned vec) {
    return vec == 0 ? n : (n / vec) * vec;
}

float oracle_dot_ref_f32(const float* x, const float* y, uint64_t n, float alpha0,
                         unsigned vec) {
    const uint64_t cut = muladd_terms(n, vec);
    float acc = alpha0;
    for (uint64_t p = 0; p < cut; ++p) {
        const float prod = x[p] * y[p];
        acc = acc + prod;
    }
    for (uint64_t p = cut; p < n; ++p) acc = fmaf(x[p], y[p], acc);
    return acc;
}

double oracle_dot_ref_f64(const double* x, const double* y, uint64_t n, double alpha0,
                          unsigned vec) {
    const uint64_t cut = muladd_terms(n, vec);
    double acc = alpha0;
    for (uint64_t p = 0; p < cut; ++p) {
        const double prod = x[p] * y[p];
        acc = acc + prod;
    }
    for (uint64_t p = cut; p < n; ++p) acc = fma(x[p], y[p], acc);
    return acc;
}

/* layout: 0 = row-major (A(i,j) at j + i*n), 1 = col-major (i + j*m);
 * reference dense.hpp:54-56 */
static inline uint64_t idx(int layout, uint64_t m, uint64_t n, uint64_t i, uint64_t j) {
    return layout == 1 ? i + j * m : j + i * n;
}

void oracle_gemv_ref_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                         float* c, unsigned vec) {
    const uint64_t cut = muladd_terms(n, vec);
    for (uint64_t i = 0; i < m; ++i) {
        float acc = c[i];
        for (uint64_t j = 0; j < cut; ++j) {
            const float prod = A[idx(layout, m, n, i, j)] * x[j];
            acc = acc + prod;
        }
        for (uint64_t j = cut; j < n; ++j) acc = fmaf(A[idx(layout, m, n, i, j)], x[j], acc);
        c[i] = acc;
    }
}

void oracle_gemv_ref_f64(const double* A, int layout, uint64_t m, uint64_t n,
                         const double* x, double* c, unsigned vec) {
    const uint64_t cut = muladd_terms(n, vec);
    for (uint64_t i = 0; i < m; ++i) {
        double acc = c[i];
        for (uint64_t j = 0; j < cut; ++j) {
            const double prod = A[idx(layout, m, n, i, j)] * x[j];
            acc = acc + prod;
        }
        for (uint64_t j = cut; j < n; ++j) acc = fma(A[idx(layout, m, n, i, j)], x[j], acc);
        c[i] = acc;
    }
}

void oracle_ger_ref_f32(const float* x, const float* y, float* C, int layout, uint64_t m,
                        uint64_t n) {
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j) {
            float* cij = &C[idx(layout, m, n, i, j)];
            *cij = fmaf(x[i], y[j], *cij);
        }
}

void oracle_ger_ref_f64(const double* x, const double* y, double* C, int layout, uint64_t m,
                        uint64_t n) {
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j) {
            double* cij = &C[idx(layout, m, n, i, j)];
            *cij = fma(x[i], y[j], *cij);
        }
}

/* ------------------------------------------------------------------------ */
/* Extended-precision truth and the error-bound sums.                        */
/* fp32: products are exact in fp64, summed in 80-bit long double.           */
/* fp64: Dot2 (Ogita-Rump-Oishi) — TwoProd via fma, TwoSum — as accurate as   */
/* computing in twice the working precision.                                 */
/* ------------------------------------------------------------------------ */
void oracle_dot_truth_f32(const float* x, const float* y, uint64_t n, float alpha0,
                          double* truth, double* sumabs) {
    long double s = (long double)alpha0, a = 0.0L;
    for (uint64_t p = 0; p < n; ++p) {
        const double prod = (double)x[p] * (double)y[p];
        s += (long double)prod;
        a += (long double)fabs(prod);
    }
    *truth = (double)s;
    *sumabs = (double)a;
}

static inline void two_sum(double a, double b, double* s, double* e) {
    const double t = a + b;
    const double z = t - a;
    *e = (a - (t - z)) + (b - z);
    *s = t;
}

void oracle_dot_truth_f64(const double* x, const double* y, uint64_t n, double alpha0,
                          double* truth, double* sumabs) {
    double s = alpha0, c = 0.0, a = 0.0;
    for (uint64_t p = 0; p < n; ++p) {
        const double h = x[p] * y[p];
        const double l = fma(x[p], y[p], -h);
        double e;
        two_sum(s, h, &s, &e);
        c += e + l;
        a += fabs(h);
    }
    *truth = s + c;
    *sumabs = a;
}

void oracle_gemv_truth_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                           const float* c0, double* truth, double* rowabs) {
    for (uint64_t i = 0; i < m; ++i) {
        long double s = (long double)c0[i], a = 0.0L;
        for (uint64_t j = 0; j < n; ++j) {
            const double prod = (double)A[idx(layout, m, n, i, j)] * (double)x[j];
            s += (long double)prod;
            a += (long double)fabs(prod);
        }
        truth[i] = (double)s;
        rowabs[i] = (double)a;
    }
}

void oracle_gemv_truth_f64(const double* A, int layout, uint64_t m, uint64_t n,
                           const double* x, const double* c0, double* truth, double* rowabs) {
    for (uint64_t i = 0; i < m; ++i) {
        double s = c0[i], c = 0.0, a = 0.0;
        for (uint64_t j = 0; j < n; ++j) {
            const double av = A[idx(layout, m, n, i, j)];
            const double h = av * x[j];
            const double l = fma(av, x[j], -h);
            double e;
            two_sum(s, h, &s, &e);
            c += e + l;
            a += fabs(h);
        }
        truth[i] = s + c;
        rowabs[i] = a;
    }
}
