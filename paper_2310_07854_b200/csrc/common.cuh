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
constexpr int kMaxGroupPairs = 128;

// ---------------------------------------------------------------------------
// ExMy format descriptor (readings c1-c9).  All derived constants are
// computed once on the host (make_fmt in api.cu) so the device codec is a
// handful of integer/FP32 ops with no table lookups.
// ---------------------------------------------------------------------------
enum FmtKind : int32_t {
    KIND_GENERIC = 0,   // integer RNE path
    KIND_IDENTITY = 1,  // E8M23: FP32 bits
    KIND_F16 = 2,       // E5M10: cvt.rn.f16x2.f32, |x| >= 65520 / NaN -> generic
    KIND_BF16 = 3,      // E8M7:  cvt.rn.bf16x2.f32, |x| >= bf16max + ulp/2 / NaN -> generic
    KIND_E4M3 = 4,      // cvt.rn.satfinite.e4m3x2.f32, |x| > 464 / NaN -> generic
    KIND_E5M2 = 5,      // cvt.rn.satfinite.e5m2x2.f32, |x| >= 61440 / NaN -> generic
    KIND_E2M1 = 6,      // cvt.rn.satfinite.e2m1x2.f32, NaN -> generic
    KIND_E2M3 = 7,      // cvt.rn.satfinite.e2m3x2.f32, NaN -> generic
    KIND_E3M2 = 8,      // cvt.rn.satfinite.e3m2x2.f32, NaN -> generic
    // IEEE special-value mode (VAPR_FMT_IEEE; reading c41).  Encoding is the
    // generic path for both IEEE formats -- exact IEEE RNE once maxcode is the
    // inf code (overflow clamps to +-inf) and nancode the conversions'
    // canonical NaN 0x7FFF.  IEEE E8M7 is KIND_GENERIC (exponent 255 decodes
    // to inf / NaN by itself); IEEE E5M10 gets this kind, tested only on the
    // decode slow paths, so the all-finite fast paths are unchanged.
    KIND_F16_IEEE = 9
};

struct Fmt {
    int32_t E, M, t, pf;
    int32_t kind;
    int32_t sh;            // 23 - M: FP32 mantissa bits dropped
    uint32_t K;            // rnd - (off << sh) (mod 2^32): fused RNE + re-bias constant
    uint32_t minnorm;      // FP32 bits of 2^(1-bias): smallest normal of the format
    uint32_t magic_bits;   // FP32 bits of 2^(24-bias-M): its ulp is the subnormal quantum
    uint32_t maxcode;      // encode clamp: largest finite magnitude code (exp field 254
                           // for E=8, c7); IEEE mode: the inf code
    uint32_t mask;         // (1 << t) - 1
    uint32_t signbit;      // 1 << (t-1)
    uint32_t keep;         // decode: sign | exponent+mantissa field mask in FP32 position
    uint32_t hw_limit;     // hardware fast path valid while |x| bits < hw_limit
    float dscale;          // 2^(127 - bias): decode re-bias
    uint32_t nancode;      // encode of NaN: maxcode (c8) / 0x7FFF (IEEE)
    uint32_t lsb;          // RNE tie bit mask: 1 when sh > 0; 0 for M = 23 (nothing is
                           // dropped, so nothing rounds: code = a - off exactly)
    // fake_quant (N4): decode(encode(x)) straight on the FP32 bit pattern
    uint32_t fq_rnd;       // (1 << (sh-1)) - 1: the RNE half-ulp constant (0 for sh = 0)
    uint32_t fq_keep;      // ~((1 << sh) - 1): the kept mantissa bits
    uint32_t fq_maxfin;    // FP32 bits of the largest finite value of the format
    uint32_t fq_sat;       // bits of an overflow's result: fq_maxfin (c7) / inf (IEEE)
    uint32_t fq_nan;       // bits of decode(nancode)
};

// FP32 -> code, round to nearest even (single rounding), saturating, NaN ->
// +max, -0 kept (readings c2-c8).  Normal range: integer RNE on the FP32 bit
// pattern (a carry into the exponent is the correct binade change; for M = 23
// nothing is dropped and both the half-ulp constant and the tie bit are 0).  Format
// subnormal range: |x| + 2^(24-bias-M) rounds |x| to the subnormal quantum in
// the FP32 adder (RN-even), exact because no FTZ is used anywhere.
__device__ __forceinline__ uint32_t encode_generic(float x, const Fmt& f) {
    const uint32_t u = __float_as_uint(x);
    const uint32_t a = u & 0x7fffffffu;
    const uint32_t cn = (a + f.K + ((a >> f.sh) & f.lsb)) >> f.sh;
    const uint32_t cs =
        __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(f.magic_bits))) - f.magic_bits;
    uint32_t c = (a < f.minnorm) ? cs : cn;
    c = min(c, f.maxcode) | ((u >> (32 - f.t)) & f.signbit);
    return (a > 0x7f800000u) ? f.nancode : c;
}

__device__ __forceinline__ uint32_t encode(float x, const Fmt& f) {
    return (f.kind == KIND_IDENTITY) ? __float_as_uint(x) : encode_generic(x, f);
}

// code at slot j of a word -> FP32 (exact).  The code is shifted to the top of
// the word, an arithmetic shift moves its exponent into the FP32 exponent
// field (the sign copies land in bits the mask clears), and one multiply by
// the power of two 2^(127-bias) re-biases normals and subnormals alike.
__device__ __forceinline__ float decode_slot(uint32_t w, int j, const Fmt& f) {
    if (f.kind == KIND_IDENTITY) return __uint_as_float(w);
    // (E8M7 exponent 255 lands in the FP32 exponent field as inf / NaN: codes
    // the all-finite reading never produces, IEEE mode's specials; IEEE E5M10
    // exponent-31 codes are fixed up by decode() / taken by the hardware path)
    const uint32_t u = w << (32 - f.t - j * f.t);
    const uint32_t x = uint32_t(int32_t(u) >> (8 - f.E)) & f.keep;
    return (f.E == 8) ? __uint_as_float(x) : __fmul_rn(__uint_as_float(x), f.dscale);
}

__device__ __forceinline__ float decode(uint32_t c, const Fmt& f) { return decode_slot(c, 0, f); }

// decode() for a format that may be IEEE E5M10 (KIND_F16_IEEE): exponent 31 ->
// FP32 inf / NaN, sign and payload kept.  Kept apart so decode() carries no
// fixup in the kernels' common instantiations.
__device__ __forceinline__ float decode_sp(uint32_t c, const Fmt& f) {
    const float v = decode_slot(c, 0, f);
    const uint32_t sp = ((c & 0x8000u) << 16) | 0x7F800000u | ((c & 0x3FFu) << 13);
    return (f.kind == KIND_F16_IEEE && (c & 0x7C00u) == 0x7C00u) ? __uint_as_float(sp) : v;
}

__device__ __forceinline__ uint32_t code_at(uint32_t word, int slot, const Fmt& f) {
    return (f.t == 32) ? word : ((word >> (slot * f.t)) & f.mask);
}

// ---- hardware conversions (sm_100a) -------------------------------------
__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_e4m3x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_e5m2x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_e2m1x2(float lo, float hi) {
    uint16_t r;
    asm("{ .reg .b8 t;\n cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n mov.b16 %0, {t, 0};}"
        : "=h"(r) : "f"(hi), "f"(lo));
    return r & 0xffu;
}
__device__ __forceinline__ uint32_t cvt_e2m3x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t cvt_e3m2x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

// One value -> its code: the hardware conversion where it is bit-identical to
// the reading (|x| below the format's hw_limit, non-NaN), the generic integer
// path elsewhere.  Exact either way, so the choice may be made per value.
__device__ __forceinline__ uint32_t encode1(float x, const Fmt& f) {
    if (f.kind == KIND_IDENTITY) return __float_as_uint(x);
    const uint32_t a = __float_as_uint(x) & 0x7fffffffu;
    if (a < f.hw_limit) {
        switch (f.kind) {
            case KIND_F16: {
                uint16_t h;
                asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(x));
                return h;
            }
            case KIND_BF16: {
                uint16_t h;
                asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(x));
                return h;
            }
            case KIND_E4M3: return cvt_e4m3x2(x, 0.f) & 0xffu;
            case KIND_E5M2: return cvt_e5m2x2(x, 0.f) & 0xffu;
            case KIND_E2M1: return cvt_e2m1x2(x, 0.f) & 0xfu;
            case KIND_E2M3: return cvt_e2m3x2(x, 0.f) & 0x3fu;
            case KIND_E3M2: return cvt_e3m2x2(x, 0.f) & 0x3fu;
            default: break;
        }
    }
    return encode_generic(x, f);
}

// Encode PF values x[0..PF) into one packed word (the caller sets values
// beyond the row end to +0).  Formats with a hardware conversion use it unless
// some value of the word needs the reading's special handling (top binade,
// NaN), which the generic path provides; the choice is per word and bit-exact
// either way.  PF is a compile-time constant (see with_pf).
template <int PF>
__device__ __forceinline__ uint32_t encode_word_t(const float* x, const Fmt& f) {
    if (PF == 1 && f.kind == KIND_IDENTITY) return __float_as_uint(x[0]);
    uint32_t amax = 0;
#pragma unroll
    for (int j = 0; j < PF; ++j) amax = max(amax, __float_as_uint(x[j]) & 0x7fffffffu);
#ifdef VAPR_NO_HW_ENCODE
    if (false) {
#else
    if (amax < f.hw_limit) {
#endif
        if constexpr (PF == 2) {
            if (f.kind == KIND_F16) return cvt_f16x2(x[0], x[1]);
            if (f.kind == KIND_BF16) return cvt_bf16x2(x[0], x[1]);
        } else if constexpr (PF == 4) {
            if (f.kind == KIND_E4M3) return cvt_e4m3x2(x[0], x[1]) | (cvt_e4m3x2(x[2], x[3]) << 16);
            if (f.kind == KIND_E5M2) return cvt_e5m2x2(x[0], x[1]) | (cvt_e5m2x2(x[2], x[3]) << 16);
        } else if constexpr (PF == 8) {
            if (f.kind == KIND_E2M1)
                return cvt_e2m1x2(x[0], x[1]) | (cvt_e2m1x2(x[2], x[3]) << 8) |
                       (cvt_e2m1x2(x[4], x[5]) << 16) | (cvt_e2m1x2(x[6], x[7]) << 24);
        } else if constexpr (PF == 5) {
            if (f.kind == KIND_E2M3 || f.kind == KIND_E3M2) {
                uint32_t p0, p1, p2;
                if (f.kind == KIND_E2M3) {
                    p0 = cvt_e2m3x2(x[0], x[1]);
                    p1 = cvt_e2m3x2(x[2], x[3]);
                    p2 = cvt_e2m3x2(x[4], 0.f);
                } else {
                    p0 = cvt_e3m2x2(x[0], x[1]);
                    p1 = cvt_e3m2x2(x[2], x[3]);
                    p2 = cvt_e3m2x2(x[4], 0.f);
                }
                return (p0 & 0x3fu) | ((p0 >> 8) << 6) | ((p1 & 0x3fu) << 12) |
                       ((p1 >> 8) << 18) | ((p2 & 0x3fu) << 24);
            }
        }
    }
    // generic path (the hardware conversions above already map +-0 exactly)
    if (amax == 0u) {               // all +-0: only the signs can be set
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < PF; ++j) w |= ((__float_as_uint(x[j]) >> (32 - f.t)) & f.signbit) << (j * f.t);
        return w;
    }
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < PF; ++j) w |= encode_generic(x[j], f) << (j * f.t);
    return w;
}

// two 8-bit codes (low 16 bits of w) -> two FP32 values via f16x2
__device__ __forceinline__ void cvt2_f8(uint32_t w, float* out, bool e5m2) {
    uint32_t h;
    const uint16_t c = (uint16_t)(w & 0xffffu);
    if (e5m2) asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h) : "h"(c));
    else asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(c));
    asm("{ .reg .f16 a, b;\n mov.b32 {a, b}, %2;\n cvt.f32.f16 %0, a;\n cvt.f32.f16 %1, b;}"
        : "=f"(out[0]), "=f"(out[1]) : "r"(h));
}

template <int PF>
__device__ __forceinline__ void decode_word_t(uint32_t w, float* out, const Fmt& f) {
    if constexpr (PF == 4) {
        // E4M3 / E5M2 through the hardware f8 -> f16 conversion (exact: every
        // value of both formats is an f16 value), except the codes that are
        // finite in this reading but NaN / inf in the hardware encodings:
        // E4M3 S.1111.111 (480), E5M2 exponent field 31
        if (f.kind == KIND_E4M3) {
            if ((((w & 0x7f7f7f7fu) + 0x01010101u) & 0x80808080u) == 0u) {
                cvt2_f8(w, out, false);
                cvt2_f8(w >> 16, out + 2, false);
                return;
            }
        } else if (f.kind == KIND_E5M2) {
            const uint32_t e = w & 0x7c7c7c7cu;
            // a byte's exponent field is 31 iff (e_byte + 0x04) carries into bit 7
            if ((((e + 0x04040404u) & 0x80808080u)) == 0u) {
                cvt2_f8(w, out, true);
                cvt2_f8(w >> 16, out + 2, true);
                return;
            }
        }
    }
    if constexpr (PF == 8) {
        // E2M1 (no special codes) through cvt.rn.f16x2.e2m1x2, one byte = two codes
        if (f.kind == KIND_E2M1) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                uint32_t h;
                const uint16_t c = (uint16_t)((w >> (8 * b)) & 0xffu);
                asm("{ .reg .b8 t;\n cvt.u8.u16 t, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;}" : "=r"(h) : "h"(c));
                asm("{ .reg .f16 a, b;\n mov.b32 {a, b}, %2;\n cvt.f32.f16 %0, a;\n cvt.f32.f16 %1, b;}"
                    : "=f"(out[2 * b]), "=f"(out[2 * b + 1]) : "r"(h));
            }
            return;
        }
    }
    if constexpr (PF == 2) {
        // E5M10: the hardware f16 -> f32 conversion is exact except for the
        // exponent-31 codes, which are finite in this reading (c3; IEEE mode:
        // they are inf / NaN, and the hardware decode takes every code)
        if ((f.kind == KIND_F16 && (w & 0x7C00u) != 0x7C00u && (w & 0x7C000000u) != 0x7C000000u) ||
            f.kind == KIND_F16_IEEE) {
            float lo, hi;
            asm("{ .reg .f16 a, b;\n mov.b32 {a, b}, %2;\n cvt.f32.f16 %0, a;\n cvt.f32.f16 %1, b;}"
                : "=f"(lo), "=f"(hi) : "r"(w));
            out[0] = lo;
            out[1] = hi;
            return;
        }
    }
#pragma unroll
    for (int j = 0; j < PF; ++j) out[j] = decode_slot(w, j, f);
}

// A 16-byte group of 4 words -> 4 PF values.  For E5M10 the exponent-31
// test (the codes the hardware conversion cannot take, c3) is one SWAR test
// for all eight halves: (e + 0x0400) carries into bit 15 of a half iff its
// exponent field e is 0x7C00.
template <int PF>
__device__ __forceinline__ void decode_group_t(const uint4& v, float* out, const Fmt& f) {
    if constexpr (PF == 2) {
        if (f.kind == KIND_F16) {
            const uint32_t t = (((v.x & 0x7C007C00u) + 0x04000400u) | ((v.y & 0x7C007C00u) + 0x04000400u) |
                                ((v.z & 0x7C007C00u) + 0x04000400u) | ((v.w & 0x7C007C00u) + 0x04000400u)) &
                               0x80008000u;
            if (t == 0u) {
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    asm("{ .reg .f16 a, b;\n mov.b32 {a, b}, %2;\n cvt.f32.f16 %0, a;\n cvt.f32.f16 %1, b;}"
                        : "=f"(out[2 * k]), "=f"(out[2 * k + 1]) : "r"(w4[k]));
                return;
            }
        }
    }
    decode_word_t<PF>(v.x, out, f);
    decode_word_t<PF>(v.y, out + PF, f);
    decode_word_t<PF>(v.z, out + 2 * PF, f);
    decode_word_t<PF>(v.w, out + 3 * PF, f);
}

// Run fn(std::integral_constant<int, pf>) for the runtime packing factor
// (one uniform branch), so the per-word loops above unroll at compile time.
template <int V>
struct IC {
    static constexpr int value = V;
};
template <class Fn>
__device__ __forceinline__ void with_pf(int pf, Fn&& fn) {
    switch (pf) {
        case 1: fn(IC<1>{}); break;
        case 2: fn(IC<2>{}); break;
        case 3: fn(IC<3>{}); break;
        case 4: fn(IC<4>{}); break;
        case 5: fn(IC<5>{}); break;
        case 6: fn(IC<6>{}); break;
        default: fn(IC<8>{}); break;
    }
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
    float q_lo[kJoints], q_hi[kJoints];  // joint limits (bound cost, N2)
    int32_t link_start[kLinks + 1];      // spheres sorted by link
    float sx[kMaxSpheres], sy[kMaxSpheres], sz[kMaxSpheres], sr[kMaxSpheres];
    // self-collision adjacency (CSR): partners of sphere s are
    // adj[adj_off[s] .. adj_off[s+1]), each pair listed from both ends, in
    // ascending partner order; the partners on link L are the sub-range
    // adj[adj_link_off[s][L] .. adj_link_off[s][L+1]).
    uint16_t adj_off[kMaxSpheres + 1];
    uint16_t adj_link_off[kMaxSpheres][kLinks + 1];
    // link-pair broadphase: index (0..31) of the link pair (a, b) in the
    // per-pose self mask, -1 when no listed sphere pair joins the two links
    int8_t lp_index[kLinks][kLinks];
    int8_t lp_a[32], lp_b[32];           // links of link pair i (lp_a <= lp_b)
    int32_t n_link_pairs;
    // link bounding spheres: reference sphere of each link and the radius
    // max_s(|o_s - o_ref| + r_s) over its spheres (rigid: the same in any pose)
    int32_t link_ref[kLinks];
    float link_rl[kLinks];
    // canonical pair ids: pairs sorted by (i, j), i < j; adj_pid[jj] is the id
    // of the pair (s, adj[jj]); pair_i / pair_j map an id back to its spheres
    int32_t n_pairs;
    uint16_t adj_pid[2 * kMaxPairs];
    uint8_t pair_i[kMaxPairs], pair_j[kMaxPairs];
    // sub-link groups (each link's spheres split in two contiguous halves),
    // each with a reference sphere and a rigid bounding radius, for the
    // two-level self-collision broadphase: link pair -> group pairs -> pairs.
    int32_t n_groups;
    int32_t grp_ref[2 * kLinks];
    float grp_rl[2 * kLinks];
    uint8_t lp_gp_off[33];               // group pairs of link pair lp: [off[lp], off[lp+1])
    uint8_t gp_a[kMaxGroupPairs], gp_b[kMaxGroupPairs];
    uint16_t gp_off[kMaxGroupPairs + 1]; // pair ids of group pair g: gp_pid[gp_off[g] ..]
    uint16_t gp_pid[kMaxPairs];
    uint8_t adj[2 * kMaxPairs];
};

// Programmatic dependent launch (vapr_cost_grad chains its kernels with it:
// a kernel launched with the programmatic-serialization attribute may start
// while its predecessor drains; pdl_wait() returns once the predecessor grid
// has completed and its writes are visible -- a no-op for a kernel launched
// normally).  pdl_trigger() lets the successor launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

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

// sin and cos of a joint angle: Cody-Waite reduction by pi/2 (three-part
// constant, exact k * P1 for |k| < 2^16) and the classic single-precision
// minimax polynomials on [-pi/4, pi/4] (Cephes sinf / cosf coefficients).
// Max error 1.5 ulp on |x| <= 4 (checked against double sin / cos on 2e5
// points), the accuracy of CUDA's sincosf, without its large-argument
// Payne-Hanek path (whose local-memory frame made FK and BK spill).  Joint
// angles are bounded by the limits (|q| < 3.8 rad); the reduction stays
// accurate to ~1e-7 relative for |x| < 2^10.
__device__ __forceinline__ void sincos_joint(float x, float& s, float& c) {
    const float k = rintf(x * 0.636619772367581343f);
    float r = fmaf(-k, 1.5703125f, x);
    r = fmaf(-k, 4.837512969970703125e-4f, r);
    r = fmaf(-k, 7.54978995489188216e-8f, r);
    const float r2 = r * r;
    const float ps = fmaf(fmaf(-1.9515295891e-4f, r2, 8.3321608736e-3f), r2, -1.6666654611e-1f);
    const float sr = fmaf(ps * r2, r, r);
    const float pc = fmaf(fmaf(2.443315711809948e-5f, r2, -1.388731625493765e-3f), r2,
                          4.166664568298827e-2f);
    const float cr = fmaf(pc * r2, r2, fmaf(-0.5f, r2, 1.f));
    const int q = int(k) & 3;
    const float sa = (q & 1) ? cr : sr, ca = (q & 1) ? sr : cr;
    s = (q & 2) ? -sa : sa;
    c = ((q + 1) & 2) ? -ca : ca;
}

// Advance the kinematic chain from frame j-1 to frame j (j = 1..7), using the
// joint angle q (sincos_joint: ~1 ulp, no fast-math anywhere in libvapr).
__device__ __forceinline__ void fk_step(Xf& X, const RobotDev& R, int row, float q) {
    float s, c;
    sincos_joint(q, s, c);
    xf_dh(X, R.ca[row], R.sa[row], R.a[row], R.d[row], c, s);
}

// Flange (fixed row 7, theta = 0) followed by the hand rotation.
__device__ __forceinline__ void fk_hand(Xf& X, const RobotDev& R) {
    xf_dh(X, R.ca[7], R.sa[7], R.a[7], R.d[7], 1.f, 0.f);
    xf_rotz(X, R.hand_c, R.hand_s);
}

// N2 pose cost of the hand frame X against the goal G (12 floats: R
// row-major, p) -- reading c35: w_pos |p - p_g|^2 + w_rot |R - R_g|_F^2, with
// the force F = 2 w_pos (p - p_g) at p and the torque
// tau = -2 w_rot sum_k r_k x g_k (columns) that carry its gradient to the joints.
__device__ __forceinline__ float ik_pose_cost(const Xf& X, const float* G, float w_pos, float w_rot,
                                              float* F, float* tau) {
    const float dx = X.p[0] - G[9], dy = X.p[1] - G[10], dz = X.p[2] - G[11];
    float rr = 0.f;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const float e = X.r[i] - G[i];
        rr = fmaf(e, e, rr);
    }
    F[0] = 2.f * w_pos * dx;
    F[1] = 2.f * w_pos * dy;
    F[2] = 2.f * w_pos * dz;
    float tx = 0.f, ty = 0.f, tz = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {        // r_k = (r[k], r[3+k], r[6+k]), g_k likewise
        const float ax = X.r[k], ay = X.r[3 + k], az = X.r[6 + k];
        const float bx = G[k], by = G[3 + k], bz = G[6 + k];
        tx += ay * bz - az * by;
        ty += az * bx - ax * bz;
        tz += ax * by - ay * bx;
    }
    tau[0] = -2.f * w_rot * tx;
    tau[1] = -2.f * w_rot * ty;
    tau[2] = -2.f * w_rot * tz;
    return w_pos * fmaf(dx, dx, fmaf(dy, dy, dz * dz)) + w_rot * rr;
}

// N2 joint-bound cost (reading c36) of one joint and its derivative.
__device__ __forceinline__ float ik_bound(float q, float lo, float hi, float w, float& dq) {
    const float a = fmaxf(q - hi, 0.f), b = fmaxf(lo - q, 0.f);
    dq = 2.f * w * (a - b);
    return w * fmaf(a, a, b * b);
}

}  // namespace vapr
