// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients, reading packed
// out_spheres and writing packed closest_pt[_swept] / out_vec.
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// One warp per tile of up to 16 consecutive poses, two lanes per pose (lane =
// half * 16 + pose): kTP = 15 poses for the swept world pass, whose pose lane
// 15 / 31 is the halo pose p0 + 15 and whose tile adds the halo rows p0-1 and
// p0+15 for the swept samples; 16 for the self pass and the discrete world
// pass (warps are independent: no CTA barrier in the tile loop; the robot
// tables are staged once per CTA from a device image).  World and self run as
// two passes, each its own kernel instantiation (PASS 1 / 2):
//  1. stage the packed rows (cp.async, all 16-byte copies in flight) and
//     decode them in place into an FP32 tile (odd row stride: pose-per-lane
//     accesses are conflict-free); track the largest decoded coordinate.
//     The self pass with E5M10 out_spheres (H16) keeps the staged codes as
//     16-bit rows instead and converts each coordinate as it reads it
//     (RowView): half the shared memory, 26 warps per SM;
//  2. broadphase, 16 poses per instruction, the two lanes of a pose splitting
//     its list.  The spheres of a link (or of a
//     half-link group) lie in a ball around a reference sphere whose radius is
//     rigid (computed once on the host) plus the quantisation-error margin.
//     World: per (segment, link, cuboid) -- or per (pose, link, cuboid) for
//     the discrete cost -- a cull bit from the squared distance of the ball
//     centre to the box.  Self: per (pose, link pair) a ball-ball test, then
//     per live link pair its half-link group pairs;
//  3. the sparse work goes through warp work queues (every lane gets an item):
//     live (pose, sphere) world items gather the complete gradient of the
//     sphere (no scatter) and OR its codes into shared packed rows (OR is
//     order-independent); live (pose, group pair) self items test the group
//     balls and then the candidate sphere pairs, marking active pairs in a
//     per-pose bitmask over canonical pair ids; (pose, touched sphere) items
//     gather the self gradient over the active pairs in id order (the
//     sphere's partner mask first, then its pairs evaluated together).  Costs
//     come back to the pose's lane and are summed in a fixed order;
//  4. outputs: dense rows (codes ORed into zero-filled rows) or the N3 sparse
//     form (each pose's owner lane appends its codes in sphere order).
//
// Culling is exact: a term is skipped only when its bound clears the
// activation distance by kSlack = 1e-4 m, orders of magnitude above the FP32
// evaluation error of the distances for workspace-scale coordinates
// (|x| < 100 m), so every skipped term would evaluate to phi <= 0, i.e. to
// exactly 0; surviving terms are accumulated in the same order with and
// without culling, so VAPR_OPT_CULL on and off give bit-identical results
// (tests/test_gpu_parity.py::test_cull_is_exact).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "tap.cuh"

namespace vapr {

namespace {

constexpr float kSlack = 1e-4f;

struct Acc {
    float cost, gx, gy, gz;
};

struct Cub {
    float4 q0, q1, q2, q3;   // R^T (9), t (3), h (3), pad
};

// One sphere-vs-cuboid term: adds cw * w * h(phi) to the cost and
// -gw * w * h'(phi) * grad sdf to the gradient.
__device__ __forceinline__ void world_term(const Cub& b, float cx, float cy, float cz, float A,
                                           float eta, float inv_eta, float half_over_eta,
                                           float w, float cw, float gw, Acc& acc) {
    const float dx = cx - b.q2.y, dy = cy - b.q2.z, dz = cz - b.q2.w;
    const float px = fmaf(b.q0.x, dx, fmaf(b.q0.y, dy, b.q0.z * dz));
    const float py = fmaf(b.q0.w, dx, fmaf(b.q1.x, dy, b.q1.y * dz));
    const float pz = fmaf(b.q1.z, dx, fmaf(b.q1.w, dy, b.q2.x * dz));
    const float ux = fabsf(px) - b.q3.x, uy = fabsf(py) - b.q3.y, uz = fabsf(pz) - b.q3.z;
    const float umax = fmaxf(ux, fmaxf(uy, uz));
    // sdf >= umax in FP32 (sqrt(fl(a^2)) rounds back to a; adding terms only
    // grows it), so A - umax <= 0 implies phi = A - sdf <= 0: exact early out.
    if (A - umax <= 0.f) return;
    float sdf, glx, gly, glz;
    if (umax <= 0.f) {                 // inside: nearest face, lowest index on ties
        sdf = umax;
        glx = gly = glz = 0.f;
        if (ux >= uy && ux >= uz) glx = (px >= 0.f) ? 1.f : -1.f;
        else if (uy >= uz) gly = (py >= 0.f) ? 1.f : -1.f;
        else glz = (pz >= 0.f) ? 1.f : -1.f;
    } else {
        const float ox = fmaxf(ux, 0.f), oy = fmaxf(uy, 0.f), oz = fmaxf(uz, 0.f);
        // |o| and 1/|o| from one MUFU rsqrt (~2 ulp; parity tolerance 1e-5),
        // the IEEE path for arguments near the FP32 underflow
        const float o2 = fmaf(ox, ox, fmaf(oy, oy, oz * oz));
        float on, inv;
        if (o2 >= 1e-30f) {
            inv = rsqrtf(o2);
            on = o2 * inv;
        } else {
            on = sqrtf(o2);
            inv = 1.f / on;
        }
        sdf = on;
        glx = (px >= 0.f) ? ox * inv : -(ox * inv);
        gly = (py >= 0.f) ? oy * inv : -(oy * inv);
        glz = (pz >= 0.f) ? oz * inv : -(oz * inv);
    }
    const float phi = A - sdf;
    if (phi <= 0.f) return;
    float h, dh;
    if (phi <= eta) {
        h = phi * phi * half_over_eta;
        dh = phi * inv_eta;
    } else {
        h = phi - 0.5f * eta;
        dh = 1.f;
    }
    acc.cost = fmaf(cw * w, h, acc.cost);
    // world gradient = R g_local with R = (R^T)^T
    const float gxw = fmaf(b.q0.x, glx, fmaf(b.q0.w, gly, b.q1.z * glz));
    const float gyw = fmaf(b.q0.y, glx, fmaf(b.q1.x, gly, b.q1.w * glz));
    const float gzw = fmaf(b.q0.z, glx, fmaf(b.q1.y, gly, b.q2.x * glz));
    const float sc = -w * dh * gw;
    acc.gx = fmaf(sc, gxw, acc.gx);
    acc.gy = fmaf(sc, gyw, acc.gy);
    acc.gz = fmaf(sc, gzw, acc.gz);
}

// N3 sparse form of a gradient tensor (VAPR_OPT_SPARSE; reading c42): a
// pose's sphere bitmap and its non-zero codes packed in ascending sphere
// order at pool + pose * ceil(cols / pf).  The owner lane of a pose appends
// its spheres in order (the warp queue hands them back in ascending order).
struct SparseRow {
    uint32_t* row;
    uint32_t word = 0u;
    int q = 0, nw = 0;
    unsigned long long mask = 0ull;
    // the codes of a vector (computed by the item, in parallel)
    // (float2: the three codes in one word, t <= 10; float4: one word each)
    template <typename QT>
    __device__ __forceinline__ static QT codes(float vx, float vy, float vz, float cost,
                                               const Fmt& f) {
        const float v[3] = {vx + 0.f, vy + 0.f, vz + 0.f};
        uint32_t c[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) c[k] = (__float_as_uint(v[k]) != 0u) ? encode(v[k], f) : 0u;
        if constexpr (sizeof(QT) == 8)
            return make_float2(__uint_as_float(c[0] | (c[1] << f.t) | (c[2] << (2 * f.t))), cost);
        else
            return make_float4(__uint_as_float(c[0]), __uint_as_float(c[1]), __uint_as_float(c[2]), cost);
    }
    // append one sphere's codes (the owner, in ascending sphere order)
    __device__ __forceinline__ void put(int s, const float2& r, const Fmt& f) {
        // the three codes as one block (t <= 10: pf >= 3, so they span at
        // most two words); the word's bits above pf * t stay zero
        const uint32_t w = __float_as_uint(r.x);
        if (!w) return;
        mask |= 1ull << s;
        const uint32_t used = (f.pf * f.t >= 32) ? ~0u : ((1u << (f.pf * f.t)) - 1u);
        word |= (w << (q * f.t)) & used;
        const int room = f.pf - q;
        if (room > 3) {
            q += 3;
        } else {
            row[nw++] = word;
            word = (room == 3) ? 0u : (w >> (room * f.t));
            q = 3 - room;
        }
    }
    __device__ __forceinline__ void put(int s, const float4& r, const Fmt& f) {
        put3(s, __float_as_uint(r.x), __float_as_uint(r.y), __float_as_uint(r.z), f);
    }
    __device__ __forceinline__ void put3(int s, uint32_t c0, uint32_t c1, uint32_t c2, const Fmt& f) {
        const uint32_t c[3] = {c0, c1, c2};
        if (!(c[0] | c[1] | c[2])) return;
        mask |= 1ull << s;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            word |= (f.t == 32) ? c[k] : (c[k] << (q * f.t));
            if (++q == f.pf) {
                row[nw++] = word;
                word = 0u;
                q = 0;
            }
        }
    }
    __device__ __forceinline__ void finish(unsigned long long* mask_out) {
        if (q) row[nw] = word;
        *mask_out = mask;
    }
};

// OR the codes of the vector (vx, vy, vz) at elements e .. e+2 into a packed
// row: codes sharing a word go in one atomic, +0 components (code 0, the
// sparse common case) in none.
__device__ __forceinline__ void or_code3(uint32_t* row, int e, float vx, float vy, float vz,
                                         const Fmt& f, uint32_t rc) {
    const float v[3] = {vx, vy, vz};
    int cw = -1;
    uint32_t acc = 0u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int ec = e + c;
        const int w = int((ec * rc) >> 16);            // ec / pf (ec < 4096)
        if (w != cw) {
            if (acc) atomicOr(row + cw, acc);
            cw = w;
            acc = 0u;
        }
        if (__float_as_uint(v[c]) != 0u) acc |= encode(v[c], f) << ((ec - w * f.pf) * f.t);
    }
    if (acc) atomicOr(row + cw, acc);
}

// Tile-row coordinate access (byte offset 12 s of sphere s in an FP32 row):
// the decoded FP32 rows, or (H16, the self pass with E5M10 out_spheres) the
// staged E5M10 codes themselves -- 16-bit rows, half the shared memory, more
// warps per SM; every E5M10 value is an f16 value except the exponent-31
// codes (finite in the all-finite reading, inf / NaN to the hardware
// conversion), so a tile holding one (gen) reads through the generic decoder.
template <bool H16, bool GEN = false>
struct RowView {
    const Fmt* f;
    __device__ __forceinline__ float h(uint16_t c) const {
        if constexpr (GEN) return decode(c, *f);
        float x;
        asm("cvt.f32.f16 %0, %1;" : "=f"(x) : "h"(c));
        return x;
    }
    __device__ __forceinline__ void c3(const char* rb, uint32_t off12, float& x, float& y, float& z) const {
        if constexpr (H16) {
            const uint16_t* p = reinterpret_cast<const uint16_t*>(rb + (off12 >> 1));
            x = h(p[0]);
            y = h(p[1]);
            z = h(p[2]);
        } else {
            const float* p = reinterpret_cast<const float*>(rb + off12);
            x = p[0];
            y = p[1];
            z = p[2];
        }
    }
};

// Self pair (i, j), i < j: false when inactive; else the gradient
// contribution v (d cost / d c_i = -v, d cost / d c_j = +v) and the cost w h.
template <class RV>
__device__ __forceinline__ bool self_pair(const RV& rv, const char* rb, int i, int j, const float* sr,
                                          float eta, float inv_eta, float hoe, float w, float& vx,
                                          float& vy, float& vz, float& cost) {
    float xi, yi, zi, xj, yj, zj;
    rv.c3(rb, 12u * i, xi, yi, zi);
    rv.c3(rb, 12u * j, xj, yj, zj);
    const float dx = xi - xj, dy = yi - yj, dz = zi - zj;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float Rs = sr[i] + sr[j] + eta;
    // sqrt(fl(Rs^2)) rounds back to Rs and sqrt is monotone, so d2 >= fl(Rs^2)
    // implies fl(sqrt(d2)) >= Rs, i.e. phi <= 0: exact early out.
    if (d2 >= Rs * Rs) return false;
    // d and 1/d from one MUFU rsqrt (~2 ulp), IEEE near underflow
    float d, dinv;
    if (d2 >= 1e-30f) {
        dinv = rsqrtf(d2);
        d = d2 * dinv;
    } else {
        d = sqrtf(d2);
        dinv = (d > 0.f) ? 1.f / d : 0.f;
    }
    const float phi = Rs - d;
    if (phi <= 0.f) return false;
    float hh, dh;
    if (phi <= eta) {
        hh = phi * phi * hoe;
        dh = phi * inv_eta;
    } else {
        hh = phi - 0.5f * eta;
        dh = 1.f;
    }
    const float k = w * dh;
    if (d > 0.f) {
        vx = k * (dx * dinv);
        vy = k * (dy * dinv);
        vz = k * (dz * dinv);
    } else {                                       // coincident centres: direction (1, 0, 0)
        vx = k;
        vy = vz = 0.f;
    }
    cost = w * hh;
    return true;
}

// ---------------------------------------------------------------------------
// Shared-memory carve-up, computed once on the host and passed by value:
// the robot tables every warp of the CTA reads (staged once per CTA), then one
// private workspace per warp.
#ifndef VAPR_DEC_LOADS          // 16-byte loads in flight per lane in the tile decode
#define VAPR_DEC_LOADS 2
#endif
#ifndef VAPR_FUSED_SPLIT         // 1: world and self as two passes
#define VAPR_FUSED_SPLIT 1
#endif
#ifndef VAPR_MAX_WARPS          // cap on warps per (persistent, one per SM) CTA
#define VAPR_MAX_WARPS 16
#endif
#ifndef VAPR_MAX_WARPS_W        // the same for the world-only pass
#define VAPR_MAX_WARPS_W VAPR_MAX_WARPS
#endif
#ifndef VAPR_H16                 // self pass: 16-bit tile rows for E5M10 out_spheres
#define VAPR_H16 1
#endif
#ifndef VAPR_H16_V16             // 16-bit rows staged by 16-byte copies (row stride 4 mod 8 words)
#define VAPR_H16_V16 1
#endif
#ifndef VAPR_H16_W               // world pass: the same 16-bit tile rows
#define VAPR_H16_W 1
#endif
#ifndef VAPR_H16_W_MIN_POSES     // ... from this batch size on
#define VAPR_H16_W_MIN_POSES 16384
#endif
#ifndef VAPR_H16_S_MIN_POSES     // the self pass's
#define VAPR_H16_S_MIN_POSES 1024
#endif
#ifndef VAPR_MAX_WARPS_WH       // warps per SM of the world pass with 16-bit rows
#define VAPR_MAX_WARPS_WH 24
#endif
#ifndef VAPR_H16_MINB_S          // resident CTAs per SM of the 16-bit-row self / world kernels
                                 // (self: two CTAs of 11 warps -- finer retirement at the pass's
                                 // tail, so the world pass's CTAs start sooner: 1.17 -> 1.12 ms)
#define VAPR_H16_MINB_S 2
#endif
#ifndef VAPR_H16_MINB_W
#define VAPR_H16_MINB_W 1
#endif
#ifndef VAPR_MAX_WARPS_H        // the self pass with 16-bit tile rows (its kernel fits 96 registers)
#define VAPR_MAX_WARPS_H 11
#endif
#ifndef VAPR_DEC_ASYNC           // tile rows: cp.async staging + in-place decode (1) or loads (0)
#define VAPR_DEC_ASYNC 1
#endif
#ifndef VAPR_HALF_SM_TILES        // small-batch side-by-side passes below sms x warps x this tiles
#define VAPR_HALF_SM_TILES 1
#endif
#ifndef VAPR_SMALL_WARPS          // small batches: tiles (of fewer poses) per SM to aim for
#define VAPR_SMALL_WARPS 32
#endif
#ifndef VAPR_GRAB                // consecutive tiles a warp takes per scheduler grab
#define VAPR_GRAB 1
#endif
constexpr int kDecLoads = VAPR_DEC_LOADS;
constexpr int kGrab = VAPR_GRAB;
#ifdef VAPR_STATS
// work counters of the variant build -DVAPR_STATS (scripts/collision_stats.py)
__device__ unsigned long long g_stats[8];
#define VAPR_STAT(i, v) atomicAdd(&g_stats[i], (unsigned long long)(v))
#else
#define VAPR_STAT(i, v)
#endif
constexpr int kLPP = 2;            // lanes per pose: lane = half * 16 + p
constexpr int kPL = 32 / kLPP;     // pose lanes per half
constexpr int kTP = kPL - 1;       // poses per warp tile (pose lane kPL-1: the halo pose)
constexpr int kTR = kTP + 2;       // tile rows: poses p0 - 1 .. p0 + kTP
constexpr int kLH = (kLinks + kLPP - 1) / kLPP;   // links per half in the world broadphase
constexpr int kQ = 128;            // work-queue window (items)

struct Geo {
    int Wos, Wcp, Wov;             // packed row words
    int wmax_cp, wmax_ov;          // sparse pool segment per pose (words)
    int Qos;                       // 16-byte groups per out_spheres row
    int cs;                        // FP32 tile row stride (odd: lane-per-pose access is conflict-free)
    int pmw;                       // words of the per-pose active-pair mask
    int ngp, npairs, nlp, S;
    uint32_t rc_cp, rc_ov;         // e / pf reciprocals (16-bit fixed point)
    uint32_t rc_q;                 // q / Qos reciprocal (20-bit fixed point)
    int n8;                        // H16: 8-byte chunks per staged E5M10 row
    uint32_t rc_h;                 // H16: q / n8 reciprocal (20-bit fixed point)
    unsigned long long lmask[kLinks];   // spheres of each link
    // CTA tables (byte offsets from the start of dynamic shared memory)
    unsigned sr, rl, ref, slink, wtab, pij, prec, gpid, grec, gpoff, lrec, lgp, so, tables;
    // per-warp workspace (byte offsets from the warp's base), its size
    unsigned rows, pmask, pwm, wm, pk0, qi, qc, gfw, gt, warp;
};

Geo make_geo(const RobotDev& R, const Fmt& fos, const Fmt& fcp, const Fmt& fov, int do_world,
             int do_self, int sparse, int fused = 0, int h16 = 0) {
    Geo g{};
    g.Wos = row_words_of(fos, R.cols);
    g.Wcp = do_world ? row_words_of(fcp, R.cols) : 0;
    g.Wov = do_self ? row_words_of(fov, R.cols) : 0;
    g.wmax_cp = (R.cols + fcp.pf - 1) / fcp.pf;
    g.wmax_ov = (R.cols + fov.pf - 1) / fov.pf;
    g.Qos = g.Wos / 4;
    int cs = std::max(R.cols, g.Wos * fos.pf);
    g.cs = cs | 1;
    if (h16) {
        // 16-bit rows (self-only pass, E5M10): the row's (cols + 1) / 2 words at
        // a stride of 2 mod 4 words -- 8-byte aligned rows (8-byte cp.async),
        // and lane-per-pose reads of 16 rows on 16 distinct banks
#if VAPR_H16_V16
        // (16-byte copies of the whole packed row: a stride of 4 mod 8 words,
        // 2-way bank conflicts for lane-per-pose reads)
        int st = 4 * g.Qos;
        while (st % 8 != 4) ++st;
        g.cs = st;
        g.n8 = g.Qos;
#else
        const int w16 = (R.cols + 1) / 2;
        int st = w16;
        while (st % 4 != 2) ++st;
        g.cs = st;
        g.n8 = (w16 + 1) / 2;
#endif
        g.rc_h = (1u << 20) / (uint32_t)g.n8 + 1u;
        for (int q = 0; q < kTR * g.n8; ++q)
            if (int((uint32_t(q) * g.rc_h) >> 20) != q / g.n8) g.rc_h = 0;
    }
    g.pmw = (R.n_pairs + 31) >> 5;
    g.ngp = R.lp_gp_off[R.n_link_pairs];
    g.npairs = R.n_pairs;
    g.nlp = R.n_link_pairs;
    g.S = R.n_spheres;
    g.rc_cp = 65536u / fcp.pf + 1u;
    g.rc_ov = 65536u / fov.pf + 1u;
    g.rc_q = (1u << 20) / (uint32_t)g.Qos + 1u;     // exact for q < kTR * Qos (checked below)
    for (int q = 0; q < kTR * g.Qos; ++q)
        if (int((uint32_t(q) * g.rc_q) >> 20) != q / g.Qos) g.rc_q = 0;
    for (int l = 0; l < kLinks; ++l) {
        unsigned long long m = 0;
        for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) m |= 1ull << s;
        g.lmask[l] = m;
    }
    unsigned o = 0;
    auto take = [&](unsigned bytes, unsigned align) {
        o = (o + align - 1) / align * align;
        const unsigned at = o;
        o += bytes;
        return at;
    };
    // the world pass's tables first: a world-only pass stages only those
    g.sr = take(4u * kMaxSpheres, 4);
    g.rl = take(4u * 3 * kLinks, 4);
    g.ref = take(4u * 3 * kLinks, 4);
    g.slink = take(kMaxSpheres, 1);
    g.wtab = take(0, 16);
    g.pij = take(2u * g.npairs, 2);
    g.prec = take(8u * g.npairs, 8);
    g.gpid = take(2u * g.npairs, 2);
    g.grec = take(8u * kMaxGroupPairs, 8);
    g.gpoff = take(2u * (kMaxGroupPairs + 1), 2);
    g.lrec = take(8u * 32, 8);
    g.lgp = take(33, 1);
    g.so = take(fused ? 16u * kMaxSpheres : 0u, 16);      // N4: sphere offsets (BK)
    g.tables = (do_self || fused) ? take(0, 16) : g.wtab;
    o = 0;
    // (the self-only pass has no halo row 0: kPL rows, see `rows` in the kernel)
    g.rows = take(4u * (do_world ? kTR : kPL) * g.cs, 16);   // (h16: words of 2 codes)
    // (a self-only pass has no halo pose: its tiles take all kPL pose lanes)
    g.pmask = take(do_self ? 4u * kPL * g.pmw : 0u, 4);
    g.pwm = take(do_self ? 4u * kPL : 0u, 4);
    g.wm = take(do_world ? 4u * kPL * kLinks : 0u, 4);
    g.pk0 = take(do_world ? 4u * kPL : 0u, 4);
    g.qi = take(2u * kQ, 2);
    g.qc = take((sparse == 2 ? 16u : sparse == 1 ? 8u : 4u) * kQ, 16);   // item results: codes + cost / cost
    // N4: each pose's world-live spheres, and the FP32 grad_out_spheres tile
    g.gfw = take(fused ? 8u * kPL : 0u, 8);
    g.gt = take(fused ? 4u * kPL * R.cols : 0u, 16);
    g.warp = take(0, 16);
    return g;
}

// Warp work queue.  Every lane owns the items given by the set bits of its
// 128-bit mask (item = p << shift | bit); the warp processes all of them, kQ
// at a time, LPI lanes per item (fn(item, sub) with sub = 0 .. LPI-1), and,
// with LPI == 1, each lane gets back the results fn returned for its own
// items in ascending bit order -- cons(item, result) per item, and the sum of
// the results' .w (the items of a lane are contiguous in the queue, so the
// order is fixed by the mask alone and never by which lane processed what).
// All lanes must call it.
struct NoCons {
    template <typename T>
    __device__ __forceinline__ void operator()(int, const T&) const {}
};
__device__ __forceinline__ float cost_of(float r) { return r; }
__device__ __forceinline__ float cost_of(const float4& r) { return r.w; }
__device__ __forceinline__ float cost_of(const float2& r) { return r.y; }
template <int LPI, typename QT, typename Fn, typename Cons = NoCons>
__device__ __forceinline__ float warp_queue(unsigned long long lo, unsigned long long hi, int p,
                                            int shift, uint16_t* qi, QT* qc, int lane,
                                            Fn&& fn, Cons&& cons = Cons{}) {
    const int n = __popcll(lo) + __popcll(hi);
    int inc = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    const int T = __shfl_sync(0xffffffffu, inc, 31);
    const int base = inc - n;
    float sum = 0.f;
    int cur = base;
    for (int win = 0; win < T; win += kQ) {
        const int wend = win + kQ;
        while (cur < base + n && cur < wend) {
            int bit;
            if (lo) {
                bit = __ffsll((long long)lo) - 1;
                lo &= lo - 1;
            } else {
                bit = 63 + __ffsll((long long)hi);
                hi &= hi - 1;
            }
            qi[cur - win] = (uint16_t)((p << shift) | bit);
            ++cur;
        }
        __syncwarp();
        const int cnt = min(kQ, T - win);
        if constexpr (LPI == 1) {
            for (int i = lane; i < cnt; i += 32) qc[i] = fn((int)qi[i], 0);
            __syncwarp();
            const int e = min(base + n, win + cnt);
            for (int idx = max(base, win); idx < e; ++idx) {
                const QT r = qc[idx - win];
                sum += cost_of(r);
                cons((int)qi[idx - win], r);
            }
        } else {
            const int sub = lane % LPI;
            for (int i = lane / LPI; i < cnt; i += 32 / LPI) fn((int)qi[i], sub);
        }
        __syncwarp();
    }
    return sum;
}

// N4: quantise -> dequantise in registers (the error a stored tensor of format
// f would inject; exact RNE encode, exact decode -- the same value the
// materialised path reads back from HBM)
// -- computed on the FP32 bits without forming the code: the normal range
// rounds the dropped mantissa bits RNE in place (a carry into the exponent is
// the binade change), the format's subnormal range rounds in the FP32 adder
// (|x| + 2^(24-bias-M) has the subnormal quantum as its ulp; subtracting it
// back is exact), an overflow saturates (or is inf in IEEE mode), NaN gives
// decode(nancode), the sign is kept -- value for value decode(encode(x)),
// checked against it by tests/test_gpu_fused.py through the materialised path.
__device__ __forceinline__ float fake_quant(float x, const Fmt& f) {
    if (f.kind == KIND_IDENTITY) return x;
    const uint32_t u = __float_as_uint(x), a = u & 0x7fffffffu;
    uint32_t r = (a + f.fq_rnd + ((a >> f.sh) & f.lsb)) & f.fq_keep;
    const float mg = __uint_as_float(f.magic_bits);
    const float sv = __fsub_rn(__fadd_rn(__uint_as_float(a), mg), mg);
    r = (a < f.minnorm) ? __float_as_uint(sv) : r;
    r = (r > f.fq_maxfin) ? f.fq_sat : r;
    r |= u & 0x80000000u;
    return __uint_as_float(a > 0x7f800000u ? f.fq_nan : r);
}

// N4: backward kinematics of one pose inside the fused kernel -- bk.cu's chain
// (the same operations in the same order, so grad_q matches the materialised
// path bit for bit): g(s, c) returns sphere s's dequantised grad_out_spheres
// component c; spheres outside `mask` or with three zero codes are skipped
// (bk.cu's zero skip).
template <typename Gf>
__device__ __forceinline__ void bk_pose(const RobotDev& R, const float* qp, unsigned long long mask,
                                        const float4* so, Gf&& gfun, float* gq) {
#pragma unroll
    for (int j = 0; j < kJoints; ++j) gq[j] = 0.f;
    float zx[kJoints], zy[kJoints], zz[kJoints], ox[kJoints], oy[kJoints], oz[kJoints];
    Xf X;
    xf_identity(X);
#pragma unroll
    for (int l = 1; l < kLinks; ++l) {
        if (l <= kJoints) {
            fk_step(X, R, l - 1, qp[l - 1]);
            zx[l - 1] = X.r[2];
            zy[l - 1] = X.r[5];
            zz[l - 1] = X.r[8];
            ox[l - 1] = X.p[0];
            oy[l - 1] = X.p[1];
            oz[l - 1] = X.p[2];
        } else {
            fk_hand(X, R);
        }
        const int s0 = R.link_start[l], s1 = R.link_start[l + 1];
        unsigned long long lm = (mask >> s0) & ((s1 - s0 >= 64) ? ~0ull : ((1ull << (s1 - s0)) - 1ull));
        if (!lm) continue;
        float Fx = 0.f, Fy = 0.f, Fz = 0.f, Mx = 0.f, My = 0.f, Mz = 0.f;
        bool any = false;
        while (lm) {
            const int s = s0 + __ffsll((long long)lm) - 1;
            lm &= lm - 1;
            float g[3];
            if (!gfun(s, g)) continue;
            any = true;
            float cx, cy, cz;
            const float4 o4 = so[s];
            xf_apply(X, o4.x, o4.y, o4.z, cx, cy, cz);
            Fx += g[0];
            Fy += g[1];
            Fz += g[2];
            Mx += cy * g[2] - cz * g[1];
            My += cz * g[0] - cx * g[2];
            Mz += cx * g[1] - cy * g[0];
        }
        if (!any) continue;
#pragma unroll
        for (int j = 0; j < kJoints; ++j) {
            if (j < l) {
                const float tx = Mx - (oy[j] * Fz - oz[j] * Fy);
                const float ty = My - (oz[j] * Fx - ox[j] * Fz);
                const float tz = Mz - (ox[j] * Fy - oy[j] * Fx);
                gq[j] += zx[j] * tx + zy[j] * ty + zz[j] * tz;
            }
        }
    }
}

// One warp processes a tile of up to 16 consecutive poses, two lanes per pose
// (the arithmetic of every broadphase test runs for 16 poses per instruction, with
// uniform loops and no index math); the sparse narrowphase work (live world
// spheres, live group pairs, touched spheres) goes through warp work queues
// so that every lane has an item.  Warps are independent: no CTA barrier in
// the tile loop.
// SPARSE (N3, VAPR_OPT_SPARSE): the gradient outputs in the sparse form
// (SparseRow) instead of zero-filled dense rows -- its own instantiation, so
// the dense one carries no extra code (the kernel is instruction-cache
// sensitive); SP_WIDE: the item results hold one code per word (formats of
// more than 10 bits) rather than all three in one word.
// FUSED (N4, VAPR_OPT_FUSED): FK in the tile fill, the gradients summed in a
// shared FP32 tile, BK per pose at the tile's end (CollisionArgs::fused).
template <bool SPARSE, bool SP_WIDE, bool FUSED, int PASS, bool H16 = false>
__global__ void __launch_bounds__(32 * (PASS == 1 ? (H16 ? VAPR_MAX_WARPS_WH : VAPR_MAX_WARPS_W)
                                              : H16 ? VAPR_MAX_WARPS_H : VAPR_MAX_WARPS),
                                  !H16 ? 1 : PASS == 1 ? VAPR_H16_MINB_W : VAPR_H16_MINB_S)
collision_kernel(const __grid_constant__ RobotDev R, const __grid_constant__ Geo G,
                 const WorldsDev Wd, const Fmt fos, const Fmt fcp, const Fmt fov,
                 const CollisionArgs a) {
    // programmatic dependent launch (vapr_cost_grad): the first pass lets the
    // second launch at once, so its CTAs take SMs as the first's retire
    // programmatic dependent launch (vapr_cost_grad): the self pass waits for
    // FK after staging its tables (below) and then lets the world pass launch;
    // every other kernel of the chain lets its successor launch by exiting (an
    // early trigger would park the successor's CTAs on the SMs, blocked in
    // their wait, and take occupancy from the running grid)
    // PASS 1 / 2: a world-only / self-only instantiation (the two passes of
    // vapr_cost_grad: each kernel holds only its own code); 0: both from the
    // runtime flags
    const bool do_world = PASS == 1 || (PASS == 0 && a.do_world);
    const bool do_self = PASS == 2 || (PASS == 0 && a.do_self);
    extern __shared__ float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    float* ssr = reinterpret_cast<float*>(base + G.sr);
    float* srl = reinterpret_cast<float*>(base + G.rl);        // link_rl[9], grp_rl[18]
    int* sref = reinterpret_cast<int*>(base + G.ref);          // link_ref[9], grp_ref[18]
    uint16_t* spij = reinterpret_cast<uint16_t*>(base + G.pij);     // i | j << 8
    uint2* sprec = reinterpret_cast<uint2*>(base + G.prec);        // candidate pairs in group-pair order
    uint2* sgrec = reinterpret_cast<uint2*>(base + G.grec);        // group-pair ball tests
    uint16_t* sgpid = reinterpret_cast<uint16_t*>(base + G.gpid);  // pair id of each record
    uint16_t* sgpoff = reinterpret_cast<uint16_t*>(base + G.gpoff);
    uint8_t* slink = reinterpret_cast<uint8_t*>(base + G.slink);
    uint2* slrec = reinterpret_cast<uint2*>(base + G.lrec);        // link-pair ball tests
    uint8_t* slgp = reinterpret_cast<uint8_t*>(base + G.lgp);      // group pairs of link pair lp
    float4* sso = reinterpret_cast<float4*>(base + G.so);          // N4: sphere offsets

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pl = lane % kPL, half = lane / kPL;   // pose lane, its share of the per-pose work
    const int PMW = G.pmw;

    // ---- stage the robot tables (once per CTA): the device image (16-byte
    // loads), then eta_s added to the three distance tables -- the same
    // FP32 sums, in the same order, as building them from R directly
    {
        const uint4* img = a.tab_img;
        uint4* dst = reinterpret_cast<uint4*>(base);
        const int n16 = (do_self || FUSED) ? a.tab_img_bytes / 16 : (int)(G.wtab / 16);
        for (int i = tid; i < n16; i += blockDim.x) dst[i] = __ldg(img + i);
        if (FUSED)
            for (int i = tid; i < G.S; i += blockDim.x) sso[i] = make_float4(R.sx[i], R.sy[i], R.sz[i], 0.f);
        __syncthreads();
        if (do_self) {
            for (int i = tid; i < G.npairs; i += blockDim.x)
                sprec[i].y = __float_as_uint(__uint_as_float(sprec[i].y) + a.eta_s);
            for (int i = tid; i < G.nlp; i += blockDim.x)
                slrec[i].y = __float_as_uint(__uint_as_float(slrec[i].y) + a.eta_s + kSlack);
            for (int i = tid; i < G.ngp; i += blockDim.x)
                sgrec[i].y = __float_as_uint(__uint_as_float(sgrec[i].y) + a.eta_s + kSlack);
        }
    }
    __syncthreads();
    if (a.pdl == 1) {
        // out_spheres is complete after this; only then may the world pass
        // (which reads it without waiting) launch
        pdl_wait();
        pdl_trigger();
    }

    // ---- the warp's workspace
    char* wb = base + G.tables + (unsigned)warp * G.warp;
    // tile row r at rows + r * cs (a pass without the world part allocates
    // no row 0: its tiles use rows 1 .. kPL)
    float* rows = reinterpret_cast<float*>(wb + G.rows) - (do_world ? 0 : G.cs);
    uint32_t* pmask = reinterpret_cast<uint32_t*>(wb + G.pmask);
    uint32_t* pwm = reinterpret_cast<uint32_t*>(wb + G.pwm);
    uint32_t* wm = reinterpret_cast<uint32_t*>(wb + G.wm);
    int* pk0 = reinterpret_cast<int*>(wb + G.pk0);
    uint16_t* qi = reinterpret_cast<uint16_t*>(wb + G.qi);
    // item results in the queue window: the codes + cost (sparse) or the cost
    using QcT = typename std::conditional<SPARSE, typename std::conditional<SP_WIDE, float4, float2>::type,
                                          float>::type;
    QcT* qc = reinterpret_cast<QcT*>(wb + G.qc);
    unsigned long long* gfw = reinterpret_cast<unsigned long long*>(wb + G.gfw);   // N4
    float* gt = reinterpret_cast<float*>(wb + G.gt);                               // N4 [kPL][cols]

    const int cs = G.cs;
    const long long P = (long long)a.B * a.H;
    // poses per tile: kTP, or fewer for a small batch (more warps, each with
    // a shorter serial item list: latency)
    const int tp = a.tile_poses;
    const long long n_tiles = a.n_tiles;
    // one-pose tiles (the smallest batches): the broadphase loops of the pose
    // (and of its swept halo) spread over all 32 lanes instead of its 2
    const bool wide = tp == 1;
    // dynamic scheduling: a warp takes kGrab consecutive tiles at a time
    // from a global counter (collision-dense tiles cost several times the
    // average, so static ranges leave a long tail; consecutive tiles share
    // the problem and its cuboids)
    unsigned int* sched = a.sched;              // [0] next grab, [1] finished CTAs
    const long long n_grabs = (n_tiles + kGrab - 1) / kGrab;
    long long grab = -1, tile = 0, t_end = 0;

    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const bool swept = do_world && a.swept;
    const int nsub = swept ? a.sweep_steps : 0;
    const float inv_n1 = 1.f / float(nsub + 1);
    const uint4* os4 = reinterpret_cast<const uint4*>(a.os);
    // the clamp code's value: coordinates at or beyond it may be saturated
    // (all-finite) or inf (IEEE mode: 65536 for E5M10, inf for E8M7)
    const float fmax_os = decode(fos.maxcode, fos);

    for (;;) {
        if (tile >= t_end) {
            unsigned int gi = 0;
            if (lane == 0) gi = atomicAdd(sched, 1u);
            grab = __shfl_sync(0xffffffffu, gi, 0);
            if (grab >= n_grabs) break;
            tile = grab * kGrab;
            t_end = min(n_tiles, tile + kGrab);
        }
        const long long p0 = tile * tp;
        const int np = (int)min((long long)tp, P - p0);
        // halo rows p0 - 1 and p0 + 15 only for the swept world pass (the
        // segments that cross the tile edges); self and discrete need none
        const long long r_lo = swept ? max(p0 - 1, 0LL) : p0;
        const long long r_hi = swept ? min(p0 + np + 1, P) : p0 + np;   // exclusive
        const int row_off = int(r_lo - (p0 - 1));         // tile row of global row r_lo
        // the lane's pose p0 + lane = tile row lane + 1 (lane 31: the halo
        // pose, used only for the segment that ends there)
        // wide: lanes pl = 2k + j work for pose lane j (the pose, the halo)
        const int plb = wide ? (pl & 1) : pl;
        const long long pg = p0 + plb;
        int h = -1, k0 = 0, K = 0;
        if (pg < P) {
            // (32-bit division while the batch fits: the 64-bit one is a long
            // subroutine on every lane of every tile)
            const long long b = (P < 0x7fffffffLL) ? (long long)((uint32_t)pg / (uint32_t)a.H) : pg / a.H;
            h = int(pg - b * a.H);
            if (do_world) {
                const int wi = __ldg(a.world_idx + b);
                if (wi >= 0 && wi < Wd.n_worlds) {
                    k0 = __ldg(Wd.off + wi);
                    K = __ldg(Wd.off + wi + 1) - k0;
                }
            }
        }

        // ---- 1. load and decode the tile rows (16-byte loads, all in flight)
        float amax = 0.f;
        bool gen16 = false;             // H16: the tile holds an exponent-31 code
        if constexpr (FUSED) {
            // N4: the tile rows from FK, one lane per row (<= kTR of the 32),
            // every coordinate quantise->dequantised with the out_spheres
            // format (fk.cu's chain and its exact RNE codes)
            const int nr = int(r_hi - r_lo);
            if (lane < nr) {
                const float* qr = a.q + (r_lo + lane) * kJoints;
                float qv[kJoints];
#pragma unroll
                for (int j = 0; j < kJoints; ++j) qv[j] = __ldg(qr + j);
                float* d = rows + (row_off + lane) * cs;
                Xf X;
                xf_identity(X);
                for (int l = 0; l < kLinks; ++l) {
                    if (l >= 1 && l <= kJoints) fk_step(X, R, l - 1, qv[l - 1]);
                    if (l == kLinks - 1) fk_hand(X, R);
                    for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
                        float cx, cy, cz;
                        xf_apply(X, sso[s].x, sso[s].y, sso[s].z, cx, cy, cz);
                        cx = fake_quant(cx, fos);
                        cy = fake_quant(cy, fos);
                        cz = fake_quant(cz, fos);
                        d[3 * s] = cx;
                        d[3 * s + 1] = cy;
                        d[3 * s + 2] = cz;
                        amax = fmaxf(amax, fmaxf(fabsf(cx), fmaxf(fabsf(cy), fabsf(cz))));
                    }
                }
            }
        } else if constexpr (H16) {
            // the E5M10 codes are the tile: 8-byte asynchronous copies into
            // 16-bit rows, then one pass over the words for the largest code
            // magnitude (|x| is monotone in it) and exponent-31 codes
            // (the world pass's rows start at tile row row_off: halo rows)
            uint32_t* hr = reinterpret_cast<uint32_t*>(wb + G.rows) + (PASS == 2 ? 0 : row_off * cs);
            const int nr = int(r_hi - r_lo), n8 = G.n8, nq = nr * n8;
            {
                const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(hr);
                const char* src = reinterpret_cast<const char*>(os4 + r_lo * G.Qos);
                for (int q = lane; q < nq; q += 32) {
                    const int r = int((uint32_t(q) * G.rc_h) >> 20), k = q - r * n8;
#if VAPR_H16_V16
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + 4u * (r * cs + 4 * k)),
                                 "l"(src + (size_t)r * (16 * G.Qos) + 16 * k)
                                 : "memory");
#else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 4u * (r * cs + 2 * k)),
                                 "l"(src + (size_t)r * (16 * G.Qos) + 8 * k)
                                 : "memory");
#endif
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
            }
            // (8-byte reads of the staged chunks; an exponent-31 code is a
            // magnitude code >= 0x7C00, so the largest one also flags them)
            uint32_t cmax = 0u;
            for (int q = lane; q < nq; q += 32) {
                const int r = int((uint32_t(q) * G.rc_h) >> 20), k = q - r * n8;
#if VAPR_H16_V16
                const uint4 v = *reinterpret_cast<const uint4*>(hr + r * cs + 4 * k);
                cmax = __vmaxu2(cmax, __vmaxu2(__vmaxu2(v.x & 0x7fff7fffu, v.y & 0x7fff7fffu),
                                               __vmaxu2(v.z & 0x7fff7fffu, v.w & 0x7fff7fffu)));
#else
                const uint2 v = *reinterpret_cast<const uint2*>(hr + r * cs + 2 * k);
                cmax = __vmaxu2(cmax, __vmaxu2(v.x & 0x7fff7fffu, v.y & 0x7fff7fffu));
#endif
            }
            cmax = __vmaxu2(cmax, cmax >> 16) & 0xffffu;
            cmax = __reduce_max_sync(0xffffffffu, cmax);
            gen16 = cmax >= 0x7C00u;
            amax = decode(cmax, fos);
        } else {
            const int nq = int(r_hi - r_lo) * G.Qos;
            const uint4* src = os4 + r_lo * G.Qos;
            float* dst0 = rows + row_off * cs;
#if VAPR_DEC_ASYNC
            // the tile's packed rows land at the start of the row buffer by
            // asynchronous 16-byte copies, all in flight at once (one memory
            // latency per tile, no registers held); they are then decoded in
            // place, in waves of rows from the last one down: FP32 row r starts
            // at or after the end of packed row r - 1 (cs >= row words), so a
            // wave's stores never reach the packed rows still to be read, and
            // within a wave every lane reads before any lane writes
            uint4* stage = reinterpret_cast<uint4*>(wb + G.rows);   // (16-byte aligned, at or before dst0)
            {
                const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(stage);
                for (int q = lane; q < nq; q += 32)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + 16u * q),
                                 "l"(src + q)
                                 : "memory");
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
            }
            const int rpw = max(1, (32 * kDecLoads) / G.Qos);     // rows per wave
#endif
            with_pf(fos.pf, [&](auto Pc) {
                constexpr int PF = decltype(Pc)::value;
                // kDecLoads 16-byte loads in flight per lane, then one word
                // at a time through the decoder (few live temporaries)
#if VAPR_DEC_ASYNC
                for (int r1 = int(r_hi - r_lo); r1 > 0; r1 -= rpw) {
                    const int qa = max(0, r1 - rpw) * G.Qos, qb = r1 * G.Qos;
                    const int q0 = qa + lane;
                    uint4 v[kDecLoads];
#pragma unroll
                    for (int u = 0; u < kDecLoads; ++u) {
                        const int q = q0 + 32 * u;
                        v[u] = (q < qb) ? stage[q] : make_uint4(0u, 0u, 0u, 0u);
                    }
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < kDecLoads; ++u) {
                        const int q = q0 + 32 * u;
                        if (q >= qb) break;
#else
                for (int q0 = lane; q0 < nq; q0 += 32 * kDecLoads) {
                    uint4 v[kDecLoads];
#pragma unroll
                    for (int u = 0; u < kDecLoads; ++u) {
                        const int q = q0 + 32 * u;
                        v[u] = (q < nq) ? __ldg(src + q) : make_uint4(0u, 0u, 0u, 0u);
                    }
#pragma unroll
                    for (int u = 0; u < kDecLoads; ++u) {
                        const int q = q0 + 32 * u;
                        if (q >= nq) break;
#endif
                        const int r = int((uint32_t(q) * G.rc_q) >> 20);
                        const int g = q - r * G.Qos;
                        float* d = dst0 + r * cs + 4 * PF * g;
                        if constexpr (PF == 2) {
                            // E5M10 (the 43-bit set): one SWAR special-code test per group
                            float x[8];
                            decode_group_t<2>(v[u], x, fos);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                d[j] = x[j];
                                amax = fmaxf(amax, fabsf(x[j]));
                            }
                        } else {
                            const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                            for (int j4 = 0; j4 < 4; ++j4) {
                                float x[PF];
                                decode_word_t<PF>(w4[j4], x, fos);
#pragma unroll
                                for (int j = 0; j < PF; ++j) {
                                    d[j4 * PF + j] = x[j];
                                    amax = fmaxf(amax, fabsf(x[j]));
                                }
                            }
                        }
                    }
#if VAPR_DEC_ASYNC
                    __syncwarp();
#endif
                }
            });
        }
        amax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(amax)));
        // dense: the output rows are zero-filled here and their non-zero codes
        // ORed in with atomics (__syncwarp orders the fill before every lane's
        // atomics); sparse: each pose's owner lane appends its codes to the
        // pose's pool segment and writes its bitmap
        uint32_t* const cpg = (!SPARSE && !FUSED && do_world) ? a.cp + p0 * G.Wcp : nullptr;
        uint32_t* const ovg = (!SPARSE && !FUSED && do_self) ? a.ov + p0 * G.Wov : nullptr;
        if (!SPARSE && !FUSED && do_world)
            for (int i = lane; i < np * G.Wcp / 4; i += 32)
                reinterpret_cast<uint4*>(cpg)[i] = make_uint4(0u, 0u, 0u, 0u);
        if (do_self) {
            if (!SPARSE && !FUSED)
                for (int i = lane; i < np * G.Wov / 4; i += 32)
                    reinterpret_cast<uint4*>(ovg)[i] = make_uint4(0u, 0u, 0u, 0u);
            for (int i = lane; i < np * PMW; i += 32) pmask[i] = 0u;
            if (lane < kPL) pwm[lane] = 0u;
        }
        if (do_world && half == 0) pk0[pl] = k0;
        __syncwarp();

        // Quantisation margin: a decoded coordinate y of an FK value x
        // satisfies |y - x| <= 2^-(M+1) |x| + 2^-(bias+M) unless the code
        // saturated; two centres per distance and sqrt(3) per vector give the
        // ball margin.  A saturated coordinate in the tile switches culling off.
        bool can_cull = a.cull != 0;
        float margin = 0.f;
        if (fos.kind != KIND_IDENTITY) {
            if (amax >= fmax_os) can_cull = false;
            const float rel = ldexpf(1.f, -(fos.M + 1));
            const float sub = ldexpf(1.f, -((1 << (fos.E - 1)) - 1) - fos.M);
            margin = 2.f * 1.7320509f * (rel * amax * 1.01f + sub);
        }
        [[maybe_unused]] const float* myrow = rows + (pl + 1) * cs;
        // tile row t (pose p0 + t - 1; a pass without the world part has no
        // row 0), and rowb(p) = the row of pose p0 + p
        auto rowt = [&](int t) -> const char* {
            if constexpr (H16) return wb + G.rows + 4 * (t - (PASS == 2 ? 1 : 0)) * cs;
            else return reinterpret_cast<const char*>(rows + t * cs);
        };
        auto rowb = [&](int p) -> const char* { return rowt(p + 1); };
        const bool owner = half == 0 && pl < np;     // the lane that owns pose pl's results

        // ---- 2. world
        float wcost = 0.f;
        if (do_world) {
            // (a generic lambda, as the self part below: tiles with an
            // exponent-31 code in their own copy)
            auto world_part = [&](auto GenC) {
            constexpr bool GEN = decltype(GenC)::value;
            const RowView<H16, GEN> rv{&fos};
            // test ball per link: swept -> the segment (pose pg-1, pose pg),
            // i.e. tile rows (lane, lane+1), a ball around both endpoint balls
            // (it bounds every sample on the segment); discrete -> pose pg
            const bool tv = swept ? (h >= 1 && plb <= np) : (plb < np);
            float bx[kLH], by[kLH], bz[kLH], lim2[kLH];
            const char* prow = rowt(plb);
            const char* brow = rowt(plb + 1);
#pragma unroll
            for (int u = 0; u < kLH; ++u) {
                const int l = half * kLH + u;
                const int lc = min(l, kLinks - 1);
                const uint32_t r12 = 12u * sref[lc];
                float cx, cy, cz;
                rv.c3(brow, r12, cx, cy, cz);
                float rr = srl[lc] + margin;
                if (swept) {
                    float qx, qy, qz;
                    rv.c3(prow, r12, qx, qy, qz);
                    const float dx = qx - cx, dy = qy - cy, dz = qz - cz;
                    cx = fmaf(0.5f, dx, cx);
                    cy = fmaf(0.5f, dy, cy);
                    cz = fmaf(0.5f, dz, cz);
                    rr += 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                }
                bx[u] = cx;
                by[u] = cy;
                bz[u] = cz;
                const float lim = rr + a.eta_w + kSlack;
                // a link without spheres (or past the last link): never live
                lim2[u] = (l >= kLinks || srl[lc] < 0.f) ? -1.f : lim * lim;
            }
            uint32_t fm[kLH];
#pragma unroll
            for (int u = 0; u < kLH; ++u) fm[u] = 0u;
            const int Kw = __reduce_max_sync(0xffffffffu, tv ? K : 0);
            const int kstep = wide ? kPL / 2 : 1;
            for (int k = wide ? (pl >> 1) : 0; k < Kw; k += kstep) {
                const int ci = (k < K) ? k0 + k : 0;
                const float4 q0 = __ldg(Wd.cub + 4 * ci), q1 = __ldg(Wd.cub + 4 * ci + 1);
                const float4 q2 = __ldg(Wd.cub + 4 * ci + 2), q3 = __ldg(Wd.cub + 4 * ci + 3);
                const bool kv = tv && k < K;
#pragma unroll
                for (int u = 0; u < kLH; ++u) {
                    // squared distance from the ball centre to the box (0 inside)
                    const float dx = bx[u] - q2.y, dy = by[u] - q2.z, dz = bz[u] - q2.w;
                    const float px = fmaf(q0.x, dx, fmaf(q0.y, dy, q0.z * dz));
                    const float py = fmaf(q0.w, dx, fmaf(q1.x, dy, q1.y * dz));
                    const float pz = fmaf(q1.z, dx, fmaf(q1.w, dy, q2.x * dz));
                    const float ox = fmaxf(fabsf(px) - q3.x, 0.f);
                    const float oy = fmaxf(fabsf(py) - q3.y, 0.f);
                    const float oz = fmaxf(fabsf(pz) - q3.z, 0.f);
                    const float o2 = fmaf(ox, ox, fmaf(oy, oy, oz * oz));
                    const bool live = (o2 <= lim2[u]) || (!can_cull && lim2[u] >= 0.f);
                    if (kv && live) fm[u] |= 1u << k;
                }
            }
            if (wide) {                 // gather the cuboid subsets of a pose lane
#pragma unroll
                for (int u = 0; u < kLH; ++u)
#pragma unroll
                    for (int d = 2; d < kPL; d <<= 1) fm[u] |= __shfl_xor_sync(0xffffffffu, fm[u], d);
            }
            // per pose: own / forward / backward cuboid masks of each link
            // (forward = the segment of pose lane pl + 1, same half)
            unsigned long long smask = 0ull;
#pragma unroll
            for (int u = 0; u < kLH; ++u) {
                const int l = half * kLH + u;
                uint32_t v, own;
                if (swept) {
                    const uint32_t fwd = __shfl_down_sync(0xffffffffu, fm[u], 1);
                    v = (fwd & 0xffffu) | (fm[u] << 16);
                    own = fwd | fm[u];
                } else {
                    v = own = fm[u];
                }
                if (pl < np && l < kLinks) {
                    wm[pl * kLinks + l] = v;
                    if (own) smask |= G.lmask[l];
                }
            }
            smask |= __shfl_xor_sync(0xffffffffu, smask, kPL);
            if (!owner) smask = 0ull;
            __syncwarp();
            // live (pose, sphere) items: the complete gradient of the sphere
            // (no scatter), its codes ORed into the packed tile row
            VAPR_STAT(0, __popcll(smask));
            SparseRow sr_cp;
            if (SPARSE && owner) sr_cp.row = a.cp + (p0 + pl) * G.wmax_cp;
            wcost = warp_queue<1>(smask, 0ull, pl, 6, qi, qc, lane, [&](int it, int) -> QcT {
                const int p = it >> 6, sp = it & 63;
                const int l = slink[sp];
                const uint32_t v = wm[p * kLinks + l];
                uint32_t m_own, m_fwd = 0u, m_bwd = 0u;
                if (swept) {
                    m_fwd = v & 0xffffu;
                    m_bwd = v >> 16;
                    m_own = m_fwd | m_bwd;
                } else {
                    m_own = v;
                }
                const float4* cub = Wd.cub + 4 * pk0[p];
                auto cuboid = [&](int kk) -> Cub {
                    return Cub{__ldg(cub + 4 * kk), __ldg(cub + 4 * kk + 1), __ldg(cub + 4 * kk + 2),
                               __ldg(cub + 4 * kk + 3)};
                };
                const char* crow = rowt(p + 1);
                float cx, cy, cz;
                rv.c3(crow, 12u * sp, cx, cy, cz);
                const float A = ssr[sp] + a.eta_w;
                Acc acc{0.f, 0.f, 0.f, 0.f};
                // terms in a fixed order: the pose itself, the samples of
                // segment (h, h+1) (cost + (1-tau) grad), the samples of
                // segment (h-1, h) (tau grad only) -- one call site
                const char* nrow = rowt(p + 2);
                const char* qrow = rowt(p);
                const int nt = 1 + (m_fwd ? nsub : 0) + (m_bwd ? nsub : 0);
                for (int t = 0; t < nt; ++t) {
                    float sx = cx, sy = cy, sz = cz, cw = 1.f, gw = 1.f;
                    uint32_t m = m_own;
                    if (t > 0) {
                        const bool fw = m_fwd && t <= nsub;
                        const int j = fw ? t : t - (m_fwd ? nsub : 0);
                        const float tau = float(j) * inv_n1, omt = 1.f - tau;
                        float ox, oy, oz;
                        rv.c3(fw ? nrow : qrow, 12u * sp, ox, oy, oz);
                        if (fw) {
                            sx = fmaf(tau, ox, omt * cx);
                            sy = fmaf(tau, oy, omt * cy);
                            sz = fmaf(tau, oz, omt * cz);
                            gw = omt;
                            m = m_fwd;
                        } else {
                            sx = fmaf(tau, cx, omt * ox);
                            sy = fmaf(tau, cy, omt * oy);
                            sz = fmaf(tau, cz, omt * oz);
                            cw = 0.f;
                            gw = tau;
                            m = m_bwd;
                        }
                    }
                    VAPR_STAT(1, __popc(m));
                    for (; m; m &= m - 1)
                        world_term(cuboid(__ffs(m) - 1), sx, sy, sz, A, a.eta_w, inv_eta_w, hoe_w,
                                   a.w_w, cw, gw, acc);
                }
                [[maybe_unused]] uint32_t* orow = SPARSE ? nullptr : cpg + p * G.Wcp;
                VAPR_TAP(a.swept ? 4 : 3, (p0 + p) * R.cols + 3 * sp, acc.gx + 0.f);
                VAPR_TAP(a.swept ? 4 : 3, (p0 + p) * R.cols + 3 * sp + 1, acc.gy + 0.f);
                VAPR_TAP(a.swept ? 4 : 3, (p0 + p) * R.cols + 3 * sp + 2, acc.gz + 0.f);
                if constexpr (FUSED) {
                    float* gr = gt + p * R.cols + 3 * sp;
                    gr[0] = fake_quant(acc.gx + 0.f, fcp);
                    gr[1] = fake_quant(acc.gy + 0.f, fcp);
                    gr[2] = fake_quant(acc.gz + 0.f, fcp);
                    return acc.cost;
                } else if constexpr (SPARSE) {
                    return SparseRow::codes<QcT>(acc.gx, acc.gy, acc.gz, acc.cost, fcp);
                } else {
                    or_code3(orow, 3 * sp, acc.gx + 0.f, acc.gy + 0.f, acc.gz + 0.f, fcp, G.rc_cp);
                    return acc.cost;
                }
            }, [&](int it, const QcT& r) {
                if constexpr (SPARSE) sr_cp.put(it & 63, r, fcp);
            });
            if (SPARSE && owner) sr_cp.finish(a.cp_mask + p0 + pl);
            if (FUSED && half == 0) gfw[pl] = smask;
            };
            if constexpr (H16) {
                if (gen16) world_part(std::true_type{});
                else world_part(std::false_type{});
            } else {
                world_part(std::false_type{});
            }
        }

        // ---- 3. self
        float scost = 0.f;
        if (do_self) {
            // (a generic lambda: tiles with an exponent-31 code read through the
            // generic decoder in their own copy of the code, so the common
            // copy carries no per-read branch)
            auto self_part = [&](auto GenC) {
            constexpr bool GEN = decltype(GenC)::value;
            const RowView<H16, GEN> rv{&fos};
            // broadphase, per pose, two levels (the two lanes of a pose split
            // each list): the link pairs' balls, then the half-link group
            // pairs of the live link pairs; glo / ghi bit g <=> group pair g
            // (g < 64 / >= 64) is live
            const float m2 = 2.f * margin;
            const char* rb = rowb(wide ? 0 : pl);
            auto ball = [&](uint2 r) -> bool {
                float ax, ay, az, bx, by, bz;
                rv.c3(rb, r.x & 0xffffu, ax, ay, az);
                rv.c3(rb, r.x >> 16, bx, by, bz);
                const float dx = ax - bx, dy = ay - by, dz = az - bz;
                const float lim = __uint_as_float(r.y) + m2;
                return !can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim;
            };
            // wide: the 32 lanes split the one pose's lists
            const int bl0 = wide ? lane : half, bls = wide ? 32 : kLPP;
            uint32_t lpm = 0u;
            if (pl < np || wide)
                for (int lp = bl0; lp < G.nlp; lp += bls)
                    if (ball(slrec[lp])) lpm |= 1u << lp;
            lpm = wide ? __reduce_or_sync(0xffffffffu, lpm) : (lpm | __shfl_xor_sync(0xffffffffu, lpm, kPL));
            // group pairs: a uniform loop over the link pairs live for some
            // pose of the tile, each lane testing its pose's (the two lanes of
            // a pose alternate over the group pairs)
            unsigned long long glo = 0ull, ghi = 0ull;
            for (uint32_t m = __reduce_or_sync(0xffffffffu, lpm); m; m &= m - 1) {
                const int lp = __ffs(m) - 1;
                const bool live = (lpm >> lp) & 1u;
                const int g1 = slgp[lp + 1];
                for (int g = slgp[lp] + bl0; g < g1; g += bls)
                    if (live && ball(sgrec[g])) {
                        if (g < 64) glo |= 1ull << g;
                        else ghi |= 1ull << (g - 64);
                    }
            }
            // each lane lists the live group pairs it found itself (the lanes
            // of a pose tested disjoint ones; the marks below do not depend
            // on the order of the entries)
            VAPR_STAT(2, __popcll(glo) + __popcll(ghi));
            // narrowphase: the live (pose, group pair) entries are listed, each
            // expanded into chunks of <= 4 candidate pairs, one chunk per lane
            // (balanced whatever the group-pair sizes); active pairs are marked
            // in the pose's pair-id mask
            {
                uint16_t* qx = reinterpret_cast<uint16_t*>(qc);     // kQ floats = 2 kQ chunk items
                constexpr int kX = 2 * kQ;
                const int n = __popcll(glo) + __popcll(ghi);
                int inc = n;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += t;
                }
                const int T = __shfl_sync(0xffffffffu, inc, 31);
                const int base = inc - n;
                int cur = base;
                for (int win = 0; win < T; win += kQ) {
                    while (cur < base + n && cur < win + kQ) {
                        int bit;
                        if (glo) {
                            bit = __ffsll((long long)glo) - 1;
                            glo &= glo - 1;
                        } else {
                            bit = 63 + __ffsll((long long)ghi);
                            ghi &= ghi - 1;
                        }
                        qi[cur - win] = (uint16_t)(((wide ? 0 : pl) << 7) | bit);
                        ++cur;
                    }
                    __syncwarp();
                    const int cnt = min(kQ, T - win);
                    for (int e0 = 0; e0 < cnt; e0 += 32) {
                        const int e = e0 + lane;
                        int nch = 0;
                        if (e < cnt) {
                            const int g = qi[e] & 127;
                            nch = (sgpoff[g + 1] - sgpoff[g] + 3) >> 2;
                        }
                        int cinc = nch;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const int t = __shfl_up_sync(0xffffffffu, cinc, d);
                            if (lane >= d) cinc += t;
                        }
                        const int C = __shfl_sync(0xffffffffu, cinc, 31);
                        const int off = cinc - nch;
                        for (int cw = 0; cw < C; cw += kX) {
                            const int c0 = max(0, cw - off), c1 = min(nch, cw + kX - off);
                            for (int c = c0; c < c1; ++c) qx[off + c - cw] = (uint16_t)(e | (c << 7));
                            __syncwarp();
                            const int ccnt = min(kX, C - cw);
                            for (int i = lane; i < ccnt; i += 32) {
                                const int xi = qx[i];
                                const int ent = qi[xi & 127];
                                const int p = ent >> 7, g = ent & 127;
                                const char* crow = rowb(p);
                                const int k0c = sgpoff[g] + 4 * (xi >> 7);
                                const int k1c = min(k0c + 4, (int)sgpoff[g + 1]);
                                VAPR_STAT(3, 1);
                                VAPR_STAT(4, k1c - k0c);
                                // the four tests first (no shared-memory stores between
                                // them, so their loads are all in flight), then the marks
                                bool act[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const int k = k0c + u;
                                    const uint2 rec = sprec[min(k, k1c - 1)];
                                    float xi, yi, zi, xj, yj, zj;
                                    rv.c3(crow, rec.x & 0xffffu, xi, yi, zi);
                                    rv.c3(crow, rec.x >> 16, xj, yj, zj);
                                    const float dx = xi - xj, dy = yi - yj, dz = zi - zj;
                                    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                                    const float Rs = __uint_as_float(rec.y);
                                    // d2 >= fl(Rs^2) => phi <= 0 (self_pair's exact early-out);
                                    // the rare d2 within an ulp of Rs^2 is settled by self_pair
                                    // in the gather (an inactive marked pair contributes nothing)
                                    act[u] = k < k1c && d2 < Rs * Rs;
                                }
                                uint32_t wmk = 0u;
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    if (!act[u]) continue;
                                    const int pid = sgpid[k0c + u];
                                    atomicOr(pmask + p * PMW + (pid >> 5), 1u << (pid & 31));
                                    wmk |= 1u << (pid >> 5);
                                }
                                if (wmk) atomicOr(pwm + p, wmk);
                            }
                            __syncwarp();
                        }
                    }
                }
            }
            __syncwarp();
            // gradients: one item per (pose, touched sphere), gathered over its
            // active pairs in canonical id order (for a fixed sphere: its
            // partners ascending, independent of culling and of the task
            // order); the item also returns the cost of the pairs it leads
            // (i == s), so a pose's self cost is summed in pair-id order
            // the pose's touched spheres, from its active pairs
            unsigned long long tb = 0ull;
            if (owner)
                for (uint32_t wmk = pwm[pl]; wmk; wmk &= wmk - 1) {
                    const int wd = __ffs(wmk) - 1;
                    for (uint32_t m = pmask[pl * PMW + wd]; m; m &= m - 1) {
                        const int ij = spij[(wd << 5) + __ffs(m) - 1];
                        tb |= (1ull << (ij & 0xff)) | (1ull << (ij >> 8));
                    }
                }
            VAPR_STAT(5, __popcll(tb));
            if (owner) VAPR_STAT(6, __popc(pwm[pl]));
            SparseRow sr_ov;
            if (SPARSE && owner) sr_ov.row = a.ov + (p0 + pl) * G.wmax_ov;
            scost = warp_queue<1>(tb, 0ull, pl, 6, qi, qc, lane, [&](int it, int) -> QcT {
                const int p = it >> 6, s = it & 63;
                const char* crow = rowb(p);
                const uint32_t* pm = pmask + p * PMW;
                float gx = 0.f, gy = 0.f, gz = 0.f, c_lead = 0.f;
                // the active partners of sphere s (a sphere's pairs in id
                // order are its partners in ascending order: (t, s) for t < s,
                // then (s, t)), collected first so that the pair evaluations
                // below run together on the warp's lanes rather than one
                // lane at a time inside the scan of the pose's pairs
                unsigned long long part = 0ull;
                for (uint32_t wmk = pwm[p]; wmk; wmk &= wmk - 1) {
                    const int wd = __ffs(wmk) - 1;
                    for (uint32_t m = pm[wd]; m; m &= m - 1) {
                        const int ij = spij[(wd << 5) + __ffs(m) - 1];
                        const int i = ij & 0xff, j = ij >> 8;
                        part |= (i == s ? 1ull << j : 0ull) | (j == s ? 1ull << i : 0ull);
                    }
                }
                for (; part; part &= part - 1) {
                    const int t = __ffsll((long long)part) - 1;
                    const int i = min(s, t), j = max(s, t);
                    float vx, vy, vz, c;
                    // always active here (same test as the narrowphase that marked it)
                    if (!self_pair(rv, crow, i, j, ssr, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c))
                        continue;
                    const float sg = (i == s) ? -1.f : 1.f;
                    gx = fmaf(sg, vx, gx);
                    gy = fmaf(sg, vy, gy);
                    gz = fmaf(sg, vz, gz);
                    if (i == s) c_lead += c;
                }
                [[maybe_unused]] uint32_t* orow = SPARSE ? nullptr : ovg + p * G.Wov;
                VAPR_TAP(2, (p0 + p) * R.cols + 3 * s, gx + 0.f);
                VAPR_TAP(2, (p0 + p) * R.cols + 3 * s + 1, gy + 0.f);
                VAPR_TAP(2, (p0 + p) * R.cols + 3 * s + 2, gz + 0.f);
                if constexpr (FUSED) {
                    // aggregation on chip: closest_pt + out_vec (world first;
                    // 0 + v where the sphere had no world item)
                    float* gr = gt + p * R.cols + 3 * s;
                    const bool wl = (gfw[p] >> s) & 1ull;
                    const float vx = fake_quant(gx + 0.f, fov), vy = fake_quant(gy + 0.f, fov),
                                vz = fake_quant(gz + 0.f, fov);
                    gr[0] = wl ? gr[0] + vx : vx;
                    gr[1] = wl ? gr[1] + vy : vy;
                    gr[2] = wl ? gr[2] + vz : vz;
                    return c_lead;
                } else if constexpr (SPARSE) {
                    return SparseRow::codes<QcT>(gx, gy, gz, c_lead, fov);
                } else {
                    or_code3(orow, 3 * s, gx + 0.f, gy + 0.f, gz + 0.f, fov, G.rc_ov);
                    return c_lead;
                }
            }, [&](int it, const QcT& r) {
                if constexpr (SPARSE) sr_ov.put(it & 63, r, fov);
            });
            if (SPARSE && owner) sr_ov.finish(a.ov_mask + p0 + pl);
            if constexpr (FUSED) {
                // ---- 4. N4: backward kinematics of the owned poses, from the
                // on-chip grad_out_spheres (quantise->dequantised with fgos)
                if (owner) {
                    float qv[kJoints], gq[kJoints];
                    const float* qr = a.q + (p0 + pl) * kJoints;
#pragma unroll
                    for (int j = 0; j < kJoints; ++j) qv[j] = __ldg(qr + j);
                    const float* gr = gt + pl * R.cols;
                    const unsigned long long m = gfw[pl] | tb;
                    bk_pose(R, qv, m, sso, [&](int s, float* g) -> bool {
                        // a zero code <=> a +0 value (-0 has the sign bit)
#pragma unroll
                        for (int c = 0; c < 3; ++c) g[c] = fake_quant(gr[3 * s + c], a.fgos);
                        return (__float_as_uint(g[0]) | __float_as_uint(g[1]) |
                                __float_as_uint(g[2])) != 0u;
                    }, gq);
                    float* go = a.grad_q + (p0 + pl) * kJoints;
#pragma unroll
                    for (int j = 0; j < kJoints; ++j) go[j] = gq[j];
                }
            }
            };
            if constexpr (H16) {
                if (gen16) self_part(std::true_type{});
                else self_part(std::false_type{});
            } else {
                self_part(std::false_type{});
            }
        }
        if (owner) VAPR_STAT(7, 1);
        if (owner) {
            const float c = wcost + scost;
            a.cost[p0 + pl] = a.cost_accumulate ? a.cost[p0 + pl] + c : c;
        }
        __syncwarp();

        ++tile;
    }  // tile loop
    // the last CTA to finish resets the scheduler slot for its next use
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
            sched[0] = 0u;
            sched[1] = 0u;
            __threadfence();
        }
    }
    // the second pass completes only after the first: stream-ordered work
    // after it (aggregation, BK) sees both passes' outputs
    if (a.pdl == 2) pdl_wait();
}

__global__ void traj_reduce_kernel(float* __restrict__ cost_pose, int B, int H,
                                   float* __restrict__ cost_traj, const float* __restrict__ add) {
    pdl_wait();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    float c = 0.f;
    for (int h = 0; h < H; ++h) {
        float v = cost_pose[(long long)b * H + h];
        if (add) {                      // world (+ IKO) then self: the fused order
            v = v + add[(long long)b * H + h];
            cost_pose[(long long)b * H + h] = v;
        }
        c += v;
    }
    if (cost_traj) cost_traj[b] = c;
}

// The same sums with coalesced accesses: a CTA stages T whole trajectories'
// pose costs (the world + self addition done on the way, in the same order)
// in shared memory at stride H + 1 (conflict-free), then thread t sums
// trajectory t over h in order -- bit-identical to traj_reduce_kernel.
__global__ void __launch_bounds__(256)
traj_reduce_tiled_kernel(float* __restrict__ cost_pose, int B, int H, int T,
                         float* __restrict__ cost_traj, const float* __restrict__ add) {
    extern __shared__ float sv[];
    pdl_wait();
    const long long b0 = (long long)blockIdx.x * T;
    const int nb = (int)min((long long)T, B - b0);
    const long long g0 = b0 * H;
    const int n = nb * H;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        float v = cost_pose[g0 + i];
        if (add) {
            v = v + add[g0 + i];
            cost_pose[g0 + i] = v;
        }
        const int t = i / H;
        sv[i + t] = v;
    }
    __syncthreads();
    if (cost_traj && threadIdx.x < nb) {
        const float* r = sv + threadIdx.x * (H + 1);
        float c = 0.f;
        for (int h = 0; h < H; ++h) c += r[h];
        cost_traj[b0 + threadIdx.x] = c;
    }
}

__global__ void best_kernel(const float* __restrict__ cost_traj, int n_problems, int seeds,
                            float* __restrict__ best_cost, int32_t* __restrict__ best_seed) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_problems) return;
    float best = cost_traj[(long long)p * seeds];
    int arg = 0;
    for (int s = 1; s < seeds; ++s) {
        const float c = cost_traj[(long long)p * seeds + s];
        if (c < best) {
            best = c;
            arg = s;
        }
    }
    best_cost[p] = best;
    best_seed[p] = arg;
}


}  // namespace

#ifdef VAPR_STATS
extern "C" int vapr_debug_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_stats, z, sizeof(z));
    }
    return 0;
}
#endif

std::vector<uint8_t> collision_table_image(const RobotDev& R) {
    Fmt f32{};
    f32.pf = 1;
    f32.t = 32;
    const Geo G = make_geo(R, f32, f32, f32, 1, 1, 0, 0);
    std::vector<uint8_t> img((G.so + 15) / 16 * 16, 0);
    uint8_t* base = img.data();
    auto at = [&](unsigned off) { return base + off; };
    float* ssr = reinterpret_cast<float*>(at(G.sr));
    float* srl = reinterpret_cast<float*>(at(G.rl));
    int* sref = reinterpret_cast<int*>(at(G.ref));
    uint16_t* spij = reinterpret_cast<uint16_t*>(at(G.pij));
    uint32_t* sprec = reinterpret_cast<uint32_t*>(at(G.prec));
    uint16_t* sgpid = reinterpret_cast<uint16_t*>(at(G.gpid));
    uint32_t* sgrec = reinterpret_cast<uint32_t*>(at(G.grec));
    uint16_t* sgpoff = reinterpret_cast<uint16_t*>(at(G.gpoff));
    uint8_t* slink = at(G.slink);
    uint32_t* slrec = reinterpret_cast<uint32_t*>(at(G.lrec));
    uint8_t* slgp = at(G.lgp);
    auto fb = [](float x) {
        uint32_t u;
        std::memcpy(&u, &x, 4);
        return u;
    };
    for (int i = 0; i < G.S; ++i) {
        ssr[i] = R.sr[i];
        int l = 0;
        while (l < kLinks - 1 && i >= R.link_start[l + 1]) ++l;
        slink[i] = (uint8_t)l;
    }
    for (int t = 0; t < kLinks; ++t) {
        srl[t] = R.link_rl[t];
        sref[t] = R.link_ref[t];
    }
    for (int t = 0; t < 2 * kLinks; ++t) {
        srl[kLinks + t] = R.grp_rl[t];
        sref[kLinks + t] = R.grp_ref[t];
    }
    for (int i = 0; i < G.npairs; ++i) {
        spij[i] = (uint16_t)(R.pair_i[i] | (R.pair_j[i] << 8));
        // record k of the group-pair order: byte offsets 12 i | 12 j << 16 in
        // a row, and r_i + r_j (+ eta_s in the kernel); its pair id in sgpid[k]
        const int pid = R.gp_pid[i], pi = R.pair_i[pid], pj = R.pair_j[pid];
        sprec[2 * i] = (uint32_t)(12 * pi) | ((uint32_t)(12 * pj) << 16);
        sprec[2 * i + 1] = fb(R.sr[pi] + R.sr[pj]);
        sgpid[i] = (uint16_t)pid;
    }
    for (int i = 0; i <= G.ngp; ++i) sgpoff[i] = R.gp_off[i];
    for (int i = 0; i < G.nlp; ++i) {
        // link pair i: byte offsets 12 ref_a | 12 ref_b << 16 in a row and the
        // static part of the cull distance (+ eta_s + slack in the kernel)
        const int la = R.lp_a[i], lb = R.lp_b[i];
        slrec[2 * i] = (uint32_t)(12 * R.link_ref[la]) | ((uint32_t)(12 * R.link_ref[lb]) << 16);
        slrec[2 * i + 1] = fb(R.link_rl[la] + R.link_rl[lb]);
    }
    for (int i = 0; i <= G.nlp; ++i) slgp[i] = R.lp_gp_off[i];
    for (int i = 0; i < G.ngp; ++i) {
        const int ga = R.gp_a[i], gb = R.gp_b[i];
        sgrec[2 * i] = (uint32_t)(12 * R.grp_ref[ga]) | ((uint32_t)(12 * R.grp_ref[gb]) << 16);
        sgrec[2 * i + 1] = fb(R.grp_rl[ga] + R.grp_rl[gb]);
    }
    return img;
}

#ifndef VAPR_SPREAD_SMALL
#define VAPR_SPREAD_SMALL 1
#endif
#ifndef VAPR_PDL
#define VAPR_PDL 1
#endif
cudaError_t launch_collision_pass(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                                  const Fmt& fcp, const Fmt& fov, const CollisionArgs& a_in,
                                  cudaStream_t s) {
    CollisionArgs a = a_in;
    const long long P = (long long)a.B * a.H;
    const bool sparse = a.cp_mask || a.ov_mask;
    const bool wide = (a.do_world && fcp.t > 10) || (a.do_self && fov.t > 10);
    const bool fused = a.fused != 0;
    if (fused && (sparse || !a.do_world || !a.do_self)) return cudaErrorInvalidValue;
    // the self-only pass with E5M10 out_spheres keeps the codes as 16-bit tile
    // rows (RowView: half the shared memory, VAPR_MAX_WARPS_H warps per SM)
    // (not on small batches, whose one-pose tiles measured faster with the
    // FP32 rows: config 2 49.2 vs 50.8 us; from 1,024 poses for the self
    // pass, 16,384 for the world pass)
    // (VAPR_H16_MIN_POSES in the environment overrides both sizes: the tests)
    const char* h16min = getenv("VAPR_H16_MIN_POSES");
    const long long min_s = h16min ? atoll(h16min) : VAPR_H16_S_MIN_POSES;
    const long long min_w = h16min ? atoll(h16min) : VAPR_H16_W_MIN_POSES;
    const bool h16 = !fused && fos.kind == KIND_F16 && !getenv("VAPR_NO_H16") &&
                     ((VAPR_H16 && a.do_self && !a.do_world && P >= min_s) ||
                      (VAPR_H16_W && a.do_world && !a.do_self && P >= min_w));
    const Geo G = make_geo(R, fos, fcp, fov, a.do_world, a.do_self, sparse ? (wide ? 2 : 1) : 0,
                           fused ? 1 : 0, h16 ? 1 : 0);
    if (G.rc_q == 0 || (h16 && G.rc_h == 0)) return cudaErrorInvalidValue;
    int dev = 0, sms = 148, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // as many warps per CTA as shared memory holds (the tables are staged
    // once per CTA), at most VAPR_MAX_WARPS (16); one persistent CTA per SM
    int nw = (optin - (int)G.tables) / (int)G.warp;
    const int pass = (a.do_world && !a.do_self) ? 1 : (!a.do_world && a.do_self) ? 2 : 0;
    nw = std::min(nw, (pass == 1 && !fused) ? (h16 ? VAPR_MAX_WARPS_WH : VAPR_MAX_WARPS_W)
                                            : h16 ? VAPR_MAX_WARPS_H : VAPR_MAX_WARPS);
    if (h16 && pass == 2 && VAPR_H16_MINB_S > 1) {
        // the self pass's CTAs come VAPR_H16_MINB_S to an SM: size them so that
        // they fit together (the wide sparse form's larger result buffers)
        int sm_smem = 0;
        cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        nw = std::min(nw, (sm_smem / VAPR_H16_MINB_S - 1024 - (int)G.tables) / (int)G.warp);
    }
    if (nw < 1) return cudaErrorInvalidValue;
    const size_t smem = G.tables + (size_t)nw * G.warp;
    if (getenv("VAPR_DEBUG_LAUNCH"))
        fprintf(stderr, "collision pass %d: %d warps/CTA, tables %u B, %u B/warp, smem %zu B\n", pass, nw,
                G.tables, G.warp, smem);
    auto pick = [&](auto Pc) {
        constexpr int PS = decltype(Pc)::value;
        return !sparse ? collision_kernel<false, false, false, PS>
                       : (wide ? collision_kernel<true, true, false, PS> : collision_kernel<true, false, false, PS>);
    };
    auto pick16 = [&](auto Pc) {
        constexpr int PS = decltype(Pc)::value;
        return !sparse ? collision_kernel<false, false, false, PS, true>
                       : (wide ? collision_kernel<true, true, false, PS, true> : collision_kernel<true, false, false, PS, true>);
    };
    auto kern = fused ? collision_kernel<false, false, true, 0>
                : h16 ? (pass == 1 ? pick16(std::integral_constant<int, 1>{}) : pick16(std::integral_constant<int, 2>{}))
                : pass == 1 ? pick(std::integral_constant<int, 1>{})
                : pass == 2 ? pick(std::integral_constant<int, 2>{}) : pick(std::integral_constant<int, 0>{});
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * nw, smem);
    // small batches: fewer poses per tile so that the tiles fill ~VAPR_SMALL_WARPS
    // warps per SM (a tile's latency is its warp's serial item list)
    {
        // only the swept world part needs the halo pose: otherwise kPL poses
        // per tile
        const int tmax = (a.do_world && a.swept) ? kTP : kPL;
        const long long full = (P + tmax - 1) / tmax;
        const long long target = (long long)sms * VAPR_SMALL_WARPS;
        a.tile_poses = tmax;
        if (full < target) a.tile_poses = (int)std::max(1LL, std::min<long long>(tmax, (P + target - 1) / target));
        if (const char* e = getenv("VAPR_TILE_POSES")) a.tile_poses = std::max(1, std::min(tmax, atoi(e)));
    }
    const long long tiles = (P + a.tile_poses - 1) / a.tile_poses;
    a.n_tiles = tiles;
    if (!a.tab_img || a.tab_img_bytes != (int)((G.so + 15) / 16 * 16)) return cudaErrorInvalidValue;
    // enough CTAs for every warp to have a chunk; small batches: spread up to
    // one CTA per tile over the SMs (latency: a lone SM's issue slots shared
    // by its 16 warps would serialise the few tiles there are)
    const long long need = (tiles + kGrab * nw - 1) / (kGrab * nw);
    // the two passes of vapr_cost_grad (pdl != 0) on a small batch: each
    // spreads over half of the SMs, so that they run side by side (one CTA
    // fills an SM's shared memory: a full-width first pass would keep the
    // second off every SM until its CTAs retire)
    const long long sms_pass = (a.pdl != 0 && tiles < (long long)sms * nw * VAPR_HALF_SM_TILES)
                                   ? std::max(1, sms / 2) : sms;
    const long long spread = VAPR_SPREAD_SMALL ? std::min<long long>(tiles, sms_pass) : need;
    const long long grid = std::min<long long>(std::max(need, spread),
                                               (long long)sms * std::max(per_sm, 1));
#ifdef VAPR_DEBUG_TAP
    const int tw = a.swept ? 4 : 3;
    const bool tap_w = a.do_world && tap_arm(tw, P, R.cols, s);
    const bool tap_s = a.do_self && tap_arm(2, P, R.cols, s);
#endif
    // pdl 1: the self pass, a programmatic dependent of FK; pdl 2: the world
    // pass, a programmatic dependent of the self pass
    e = launch_k(kern, dim3((unsigned)grid), dim3(32 * nw), smem, s, a.pdl != 0, R, G, W, fos, fcp,
                 fov, a);
    if (e != cudaSuccess) return e;
#ifdef VAPR_DEBUG_TAP
    if (tap_w) tap_disarm(tw, s);
    if (tap_s) tap_disarm(2, s);
#endif
    return cudaGetLastError();
}

// World and self run as two passes over the tile rows: each pass keeps a
// smaller instruction working set, which beats re-reading out_spheres.  With
// a0.self_cost (vapr_cost_grad) the self pass runs first into its own cost
// array and the world pass is its programmatic dependent launch (traj_reduce
// adds the two in the fused order); otherwise world first, the self pass
// adding its cost to the world pass's (the same wcost + scost).
cudaError_t launch_collision(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                             const Fmt& fcp, const Fmt& fov, const CollisionArgs& a0,
                             unsigned int* sched_ring, unsigned int* sched_next, cudaStream_t s) {
    const long long P = (long long)a0.B * a0.H;
    if (P <= 0) return cudaSuccess;
    // each pass takes the next scheduler slot of the context's ring (the
    // kernel's last CTA leaves it zeroed); kSchedSlots passes may be in flight
    auto slot = [&]() {
        const unsigned k = __atomic_fetch_add(sched_next, 1u, __ATOMIC_RELAXED) % kSchedSlots;
        return sched_ring + 2 * k;
    };
    CollisionArgs a = a0;
    // a.self_cost (vapr_cost_grad) is added by traj_reduce: a path that puts
    // the self cost into a.cost itself leaves it zero
    auto zero_self = [&]() -> cudaError_t {
        return a.self_cost ? cudaMemsetAsync(a.self_cost, 0, sizeof(float) * (size_t)P, s) : cudaSuccess;
    };
    if (!(VAPR_FUSED_SPLIT && a.do_world && a.do_self) || a.fused) {
        a.sched = slot();
        const cudaError_t e = launch_collision_pass(R, W, fos, fcp, fov, a, s);
        return e == cudaSuccess ? zero_self() : e;
    }
    CollisionArgs aw = a, as = a;
    aw.sched = slot();
    as.sched = slot();
    aw.do_self = 0;
    as.do_world = 0;
    as.cost_accumulate = 1;
    if (VAPR_PDL && a.self_cost) {
        // the self pass writes its own cost, so neither pass depends on the
        // other (both read only out_spheres): the self pass (the longer tail)
        // runs first and the world pass starts on the SMs its CTAs leave
        as.cost = a.self_cost;
        as.cost_accumulate = 0;
        as.pdl = 1;
        aw.pdl = 2;
        cudaError_t e = launch_collision_pass(R, W, fos, fcp, fov, as, s);
        if (e != cudaSuccess) return e;
        return launch_collision_pass(R, W, fos, fcp, fov, aw, s);
    }
    cudaError_t e = launch_collision_pass(R, W, fos, fcp, fov, aw, s);
    if (e != cudaSuccess) return e;
    e = launch_collision_pass(R, W, fos, fcp, fov, as, s);
    return e == cudaSuccess ? zero_self() : e;
}

cudaError_t launch_traj_reduce(float* cost_pose, int32_t B, int32_t H, float* cost_traj,
                               cudaStream_t s, const float* add, bool pdl) {
    if (B <= 0) return cudaSuccess;
    if (H >= 1 && H <= 4096) {
        const int T = std::max(1, std::min(256, 4096 / H));
        const size_t smem = sizeof(float) * (size_t)T * (H + 1);
        return launch_k(traj_reduce_tiled_kernel, dim3((unsigned)((B + T - 1) / T)), dim3(256), smem, s, pdl,
                        cost_pose, B, H, T, cost_traj, add);
    }
    return launch_k(traj_reduce_kernel, dim3((B + 255) / 256), dim3(256), 0, s, pdl, cost_pose, B,
                    H, cost_traj, add);
}

cudaError_t launch_best_per_problem(const float* cost_traj, int32_t n_problems, int32_t seeds,
                                    float* best_cost, int32_t* best_seed, cudaStream_t s) {
    if (n_problems <= 0) return cudaSuccess;
    best_kernel<<<(n_problems + 255) / 256, 256, 0, s>>>(cost_traj, n_problems, seeds,
                                                        best_cost, best_seed);
    return cudaGetLastError();
}

}  // namespace vapr
