// common.cuh -- device-side building blocks shared by the libvapr kernels:
// the ExMy codec (a1), the packed-row geometry, and the robot description that
// travels to every kernel as a __grid_constant__ parameter.
//
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/vapr.h"

namespace vapr {

constexpr int kMaxSpheres = VAPR_MAX_SPHERES;
constexpr int kMaxPairs = VAPR_MAX_PAIRS;
constexpr int kMaxCuboids = VAPR_MAX_CUBOIDS_PER_WORLD;
constexpr int kLinks = 9;          // link0..link7, hand
constexpr int kJoints = 7;

// ---------------------------------------------------------------------------
// ExMy format descriptor (readings c1-c9).  All derived constants are
// computed once on the host (make_fmt in api.cu) so the device codec is a
// handful of integer/FP32 ops with no table lookups.
// ---------------------------------------------------------------------------
struct Fmt {
    int32_t E, M, t, pf;
    int32_t sh;            // 23 - M: FP32 mantissa bits dropped
    uint32_t rnd;          // (1 << (sh-1)) - 1: round-half-1 for RNE
    uint32_t off;          // (127 - bias) << M: exponent re-bias in code units
    uint32_t minnorm;      // FP32 bits of 2^(1-bias): smallest normal of the format
    uint32_t magic_bits;   // FP32 bits of 2^(24-bias-M): its ulp is the subnormal quantum
    uint32_t maxcode;      // largest finite magnitude code (exp field 254 for E=8, c7)
    uint32_t mask;         // (1 << t) - 1
    uint32_t magmask;      // (1 << (t-1)) - 1
    float dscale;          // 2^(127 - bias): decode re-bias
    int32_t identity;      // E8M23: raw FP32 bits
};

// FP32 -> code, round to nearest even (single rounding), saturating, NaN ->
// +max, -0 kept (readings c2-c8).  Normal range: integer RNE on the FP32 bit
// pattern (carry into the exponent is the correct binade change).  Format
// subnormal range: x + 2^(24-bias-M) rounds x to the subnormal quantum in the
// FP32 adder (RN-even), exact because no FTZ is used anywhere.
__device__ __forceinline__ uint32_t encode(float x, const Fmt& f) {
    const uint32_t u = __float_as_uint(x);
    if (f.identity) return u;
    const uint32_t s = u & 0x80000000u;
    const uint32_t a = u ^ s;
    const uint32_t r = a + f.rnd + ((a >> f.sh) & 1u);
    const uint32_t cn = (r >> f.sh) - f.off;
    const uint32_t cs = __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(f.magic_bits)))
                        - f.magic_bits;
    uint32_t c = (a < f.minnorm) ? cs : cn;
    c = min(c, f.maxcode);
    c |= s >> (32 - f.t);
    return (a > 0x7f800000u) ? f.maxcode : c;
}

// code -> FP32 (exact).  The magnitude bits placed into an FP32 pattern read as
// (1.m) 2^(e-127) (or the FP32 subnormal m 2^-149 ...); one multiply by the
// power of two 2^(127-bias) re-biases both normals and subnormals exactly.
__device__ __forceinline__ float decode(uint32_t c, const Fmt& f) {
    if (f.identity) return __uint_as_float(c);
    const uint32_t s = (c << (32 - f.t)) & 0x80000000u;
    const float v = __fmul_rn(__uint_as_float((c & f.magmask) << f.sh), f.dscale);
    return __uint_as_float(__float_as_uint(v) | s);
}

__device__ __forceinline__ uint32_t code_at(uint32_t word, int slot, const Fmt& f) {
    return (f.t == 32) ? word : ((word >> (slot * f.t)) & f.mask);
}

// ---------------------------------------------------------------------------
// Robot description (built by vapr_set_robot).  Passed by value as a
// __grid_constant__ kernel parameter: every lane reads the same entry at the
// same time, which the constant bank serves as a broadcast.
// ---------------------------------------------------------------------------
struct RobotDev {
    int32_t n_spheres;
    int32_t cols;                        // 3 * n_spheres
    float ca[8], sa[8], a[8], d[8];      // modified-DH rows (cos/sin alpha, a, d)
    float hand_c, hand_s;                // RotZ(hand_rz)
    int32_t link_start[kLinks + 1];      // spheres sorted by link
    float sx[kMaxSpheres], sy[kMaxSpheres], sz[kMaxSpheres], sr[kMaxSpheres];
    // self-collision adjacency (CSR): partners of sphere s are
    // adj[adj_off[s] .. adj_off[s+1]), each pair listed from both ends.
    uint16_t adj_off[kMaxSpheres + 1];
    uint8_t adj[2 * kMaxPairs];
};

// 3x4 rigid transform, row-major rotation r[3][3] and translation p[3].
struct Xf {
    float r[9];
    float p[3];
};

__device__ __forceinline__ void xf_identity(Xf& X) {
#pragma unroll
    for (int i = 0; i < 9; ++i) X.r[i] = (i % 4 == 0) ? 1.f : 0.f;
    X.p[0] = X.p[1] = X.p[2] = 0.f;
}

// X <- X . T_i with T_i = RotX(alpha) TransX(a) RotZ(theta) TransZ(d):
//   T = [[ct, -st, 0, a], [ca st, ca ct, -sa, -sa d], [sa st, sa ct, ca, ca d]]
__device__ __forceinline__ void xf_dh(Xf& X, float ca, float sa, float a, float d, float ct,
                                      float st) {
    const float t00 = ct, t01 = -st;
    const float t10 = ca * st, t11 = ca * ct, t12 = -sa, t13 = -sa * d;
    const float t20 = sa * st, t21 = sa * ct, t22 = ca, t23 = ca * d;
    Xf Y;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float x0 = X.r[3 * i + 0], x1 = X.r[3 * i + 1], x2 = X.r[3 * i + 2];
        Y.r[3 * i + 0] = fmaf(x0, t00, fmaf(x1, t10, x2 * t20));
        Y.r[3 * i + 1] = fmaf(x0, t01, fmaf(x1, t11, x2 * t21));
        Y.r[3 * i + 2] = fmaf(x1, t12, x2 * t22);
        Y.p[i] = fmaf(x0, a, fmaf(x1, t13, fmaf(x2, t23, X.p[i])));
    }
    X = Y;
}

// X <- X . RotZ(c, s)
__device__ __forceinline__ void xf_rotz(Xf& X, float c, float s) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float x0 = X.r[3 * i + 0], x1 = X.r[3 * i + 1];
        X.r[3 * i + 0] = fmaf(x0, c, x1 * s);
        X.r[3 * i + 1] = fmaf(x1, c, -x0 * s);
    }
}

__device__ __forceinline__ void xf_apply(const Xf& X, float x, float y, float z, float& ox,
                                         float& oy, float& oz) {
    ox = fmaf(X.r[0], x, fmaf(X.r[1], y, fmaf(X.r[2], z, X.p[0])));
    oy = fmaf(X.r[3], x, fmaf(X.r[4], y, fmaf(X.r[5], z, X.p[1])));
    oz = fmaf(X.r[6], x, fmaf(X.r[7], y, fmaf(X.r[8], z, X.p[2])));
}

// Advance the kinematic chain from frame j-1 to frame j (j = 1..7), using the
// joint angle q.  Full-precision sincosf (no fast-math anywhere in libvapr).
__device__ __forceinline__ void fk_step(Xf& X, const RobotDev& R, int row, float q) {
    float s, c;
    sincosf(q, &s, &c);
    xf_dh(X, R.ca[row], R.sa[row], R.a[row], R.d[row], c, s);
}

// Flange (fixed row 7, theta = 0) followed by the hand rotation.
__device__ __forceinline__ void fk_hand(Xf& X, const RobotDev& R) {
    xf_dh(X, R.ca[7], R.sa[7], R.a[7], R.d[7], 1.f, 0.f);
    xf_rotz(X, R.hand_c, R.hand_s);
}

}  // namespace vapr
