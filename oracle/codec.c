/*
 * oracle/codec.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously
 * correct ExMy codec the CUDA path is checked against.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code with paper_2310_07854_b200/csrc.
 *
 * What it computes ("E3M1 as a FP data type of 3-bit exponent,
 * 1-bit mantissa, and 1 sign bit"; "quantizing the tensors from
 * FP32 to the specified data format and dequantizing them back to FP32";
 * PAPER.md:259 the `_rn` FP16 intrinsics), with the readings of DESIGN.md §3
 * (= SURVEY.md §8(c) c1-c8):
 *   bias = 2^(E-1) - 1 (c1); subnormals representable (c2); no inf/NaN codes
 *   for t < 32 (c3); round to nearest, ties to even, ONE rounding from the FP32
 *   value (c4); overflow and +-inf saturate to +-max_finite (c5); NaN -> the
 *   +max_finite code (c6); for E = 8 the largest code is exponent field 254
 *   (c7); -0 keeps its sign (c8); E8M23 is the raw-bit identity.
 *
 * Step by step ("Formula"): a = |x| taken exactly in
 * double; E_a = max(floor(log2 a), 1 - bias) computed with ilogb (never log2);
 * quantum q = 2^(E_a - M); N = nearbyint(a / q) under FE_TONEAREST; v = N q;
 * v = min(v, max_finite); then the sign / exponent / mantissa fields.
 * All of it is exact in double because a has a 24-bit significand and q is a
 * power of two.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <stdlib.h>

static double max_finite(int E, int M) {
    int bias = (1 << (E - 1)) - 1;
    int emax_field = (E == 8) ? 254 : (1 << E) - 1;          /* c3, c7 */
    /* (2 - 2^-M) * 2^(emax_field - bias) */
    return ldexp(2.0 - ldexp(1.0, -M), emax_field - bias);
}

/* Encode an exactly-representable, non-negative value v of the format. */
static uint32_t encode_exact(double v, int E, int M) {
    int bias = (1 << (E - 1)) - 1;
    double min_normal = ldexp(1.0, 1 - bias);
    if (v < min_normal) {                       /* subnormal: exp field 0 */
        double mant = v / ldexp(1.0, 1 - bias - M);
        return (uint32_t)mant;
    }
    int e = ilogb(v);
    uint32_t expf = (uint32_t)(e + bias);
    double mant = v / ldexp(1.0, e - M) - ldexp(1.0, M);
    return (expf << M) | (uint32_t)mant;
}

uint32_t oracle_quantize_code(float x, int E, int M) {
    int t = 1 + E + M;
    if (E == 8 && M == 23) {                    /* identity on all patterns */
        uint32_t u;
        memcpy(&u, &x, 4);
        return u;
    }
    double vmax = max_finite(E, M);
    uint32_t maxcode = encode_exact(vmax, E, M);
    if (isnan(x)) return maxcode;               /* c6: +max_finite */
    uint32_t sign = signbit(x) ? (1u << (t - 1)) : 0u;
    double a = fabs((double)x);
    if (isinf(a)) return sign | maxcode;         /* c5 */
    if (a == 0.0) return sign;                   /* c8 */
    int bias = (1 << (E - 1)) - 1;
    int Ea = ilogb(a);
    if (Ea < 1 - bias) Ea = 1 - bias;
    double q = ldexp(1.0, Ea - M);
    double N = nearbyint(a / q);                 /* ties to even (FE_TONEAREST) */
    double v = N * q;
    if (v > vmax) v = vmax;                      /* c5: saturate */
    return sign | encode_exact(v, E, M);
}

/* Quantise a DOUBLE value with one rounding (the
 * oracle quantises its double-precision FK output "from the double value (a
 * single rounding)").  Same formula as above; E8M23 is treated as a format
 * like any other (RNE to FP32, saturating to +-FLT_MAX), NaN -> +max. */
uint32_t oracle_quantize_code_f64(double x, int E, int M) {
    int t = 1 + E + M;
    double vmax = max_finite(E, M);
    uint32_t maxcode = encode_exact(vmax, E, M);
    if (isnan(x)) return maxcode;
    uint32_t sign = signbit(x) ? (t == 32 ? 0x80000000u : (1u << (t - 1))) : 0u;
    double a = fabs(x);
    if (isinf(a)) return sign | maxcode;
    if (a == 0.0) return sign;
    int bias = (1 << (E - 1)) - 1;
    int Ea = ilogb(a);
    if (Ea < 1 - bias) Ea = 1 - bias;
    double q = ldexp(1.0, Ea - M);
    double N = nearbyint(a / q);   /* a/q is exact: q is a power of two */
    double v = N * q;
    if (v > vmax) v = vmax;
    return sign | encode_exact(v, E, M);
}

void oracle_quantize_f64(const double *x, size_t n, int E, int M, uint32_t *codes) {
    fesetround(FE_TONEAREST);
    for (size_t i = 0; i < n; ++i) codes[i] = oracle_quantize_code_f64(x[i], E, M);
}

float oracle_dequantize_code(uint32_t c, int E, int M) {
    if (E == 8 && M == 23) {
        float f;
        memcpy(&f, &c, 4);
        return f;
    }
    int t = 1 + E + M;
    int bias = (1 << (E - 1)) - 1;
    uint32_t mant = c & ((1u << M) - 1);
    uint32_t expf = (c >> M) & ((1u << E) - 1);
    int neg = (c >> (t - 1)) & 1;
    double v;
    if (E == 8 && expf == 255) {                 /* never produced (c7) */
        v = mant ? NAN : INFINITY;
    } else if (expf == 0) {
        v = ldexp((double)mant, 1 - bias - M);
    } else {
        v = ldexp((double)((1u << M) + mant), (int)expf - bias - M);
    }
    float f = (float)v;                          /* exact: every code fits FP32 */
    return neg ? -f : f;
}

void oracle_quantize(const float *x, size_t n, int E, int M, uint32_t *codes) {
    fesetround(FE_TONEAREST);
    for (size_t i = 0; i < n; ++i) codes[i] = oracle_quantize_code(x[i], E, M);
}

void oracle_dequantize(const uint32_t *codes, size_t n, int E, int M, float *y) {
    for (size_t i = 0; i < n; ++i) y[i] = oracle_dequantize_code(codes[i], E, M);
}

/* ---- multithreaded driver (for the exhaustive 2^32 test and CPU timing) ---- */
typedef struct { const float *x; size_t lo, hi; int E, M; uint32_t *codes;
                 uint32_t base; int from_bits; } job_t;

static void *run_job(void *p) {
    job_t *j = (job_t *)p;
    fesetround(FE_TONEAREST);
    for (size_t i = j->lo; i < j->hi; ++i) {
        float xi;
        if (j->from_bits) { uint32_t u = j->base + (uint32_t)i; memcpy(&xi, &u, 4); }
        else xi = j->x[i];
        j->codes[i] = oracle_quantize_code(xi, j->E, j->M);
    }
    return NULL;
}

static void run_mt(const float *x, size_t n, int E, int M, uint32_t *codes,
                   int nthreads, uint32_t base, int from_bits) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    job_t jobs[256];
    size_t chunk = (n + nthreads - 1) / nthreads;
    for (int k = 0; k < nthreads; ++k) {
        size_t lo = k * chunk, hi = lo + chunk;
        if (lo > n) lo = n;
        if (hi > n) hi = n;
        jobs[k] = (job_t){x, lo, hi, E, M, codes, base, from_bits};
        pthread_create(&th[k], NULL, run_job, &jobs[k]);
    }
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
}

void oracle_quantize_mt(const float *x, size_t n, int E, int M, uint32_t *codes,
                        int nthreads) {
    run_mt(x, n, E, M, codes, nthreads, 0, 0);
}

/* codes[i] = quantize(bits_as_float(base + i)), i < n: enumerates FP32 bit
 * patterns without materialising the inputs (exhaustive test). */
void oracle_quantize_bits_range(uint32_t base, size_t n, int E, int M,
                                uint32_t *codes, int nthreads) {
    run_mt(NULL, n, E, M, codes, nthreads, base, 1);
}
