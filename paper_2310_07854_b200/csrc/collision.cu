// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients, reading packed
// out_spheres and writing packed closest_pt[_swept] / out_vec.
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// Execution model: persistent CTAs whose WARPS are independent workers.  Each
// warp streams a contiguous range of poses (whole trajectories in practice)
// and keeps everything it needs in warp-private shared memory: a ring of three
// decoded rows (poses h-1, h, h+1 for the swept samples), their link balls,
// the segment cull masks and the current world's cuboids.  There is no
// CTA-wide barrier: latency is hidden by the other warps.  Per pose:
//  1. decode the next row (16-byte loads, one per lane), its link balls and
//     largest coordinate (quantisation margin), and the cull masks of the
//     segment (h, h+1) -- or of pose h for the discrete cost;
//  2. world: one lane per sphere whose link has a live cuboid gathers its
//     complete gradient (pose terms, then the samples of both adjacent
//     segments) into an FP32 row; cost summed by a fixed shuffle tree;
//  3. self: lanes test the link pairs (balls), then the <= 4 half-link group
//     pairs of each live link pair, then the sphere pairs of each live group
//     pair (one pair per lane); active pairs are appended in (group pair,
//     pair id) order -- an order culling does not change -- and accumulated
//     in that order into an FP32 row;
//  4. lanes encode the packed output words from the FP32 rows (hardware cvt
//     fast paths) and store them with 16-byte coalesced stores.
//
// Culling is exact: a (ball, cuboid) or (ball, ball) combination is skipped
// only when its bound clears the activation distance by kSlack = 1e-4 m,
// orders of magnitude above the FP32 evaluation error of the distances for
// workspace-scale coordinates (|x| < 100 m), so every skipped term would
// evaluate to phi <= 0, i.e. to exactly 0; surviving terms are accumulated in
// the same order with and without culling, so VAPR_OPT_CULL on and off give
// bit-identical results (tests/test_gpu_parity.py::test_cull_is_exact).
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kListCap = 64;        // active self pairs buffered per round
constexpr float kSlack = 1e-4f;

struct Acc {
    float cost, gx, gy, gz;
};



struct Cub {
    float4 q0, q1, q2, q3;   // R^T (9), t (3), h (3), pad
};

// Lower bound of the box signed distance at c (the exact value outside, the
// face distance max_k(|p_k| - h_k) inside).
__device__ __forceinline__ float box_sdf_lb(const Cub& b, float cx, float cy, float cz) {
    const float dx = cx - b.q2.y, dy = cy - b.q2.z, dz = cz - b.q2.w;
    const float px = fmaf(b.q0.x, dx, fmaf(b.q0.y, dy, b.q0.z * dz));
    const float py = fmaf(b.q0.w, dx, fmaf(b.q1.x, dy, b.q1.y * dz));
    const float pz = fmaf(b.q1.z, dx, fmaf(b.q1.w, dy, b.q2.x * dz));
    const float ux = fabsf(px) - b.q3.x, uy = fabsf(py) - b.q3.y, uz = fabsf(pz) - b.q3.z;
    const float umax = fmaxf(ux, fmaxf(uy, uz));
    const float ox = fmaxf(ux, 0.f), oy = fmaxf(uy, 0.f), oz = fmaxf(uz, 0.f);
    const float out = sqrtf(fmaf(ox, ox, fmaf(oy, oy, oz * oz)));
    return (umax <= 0.f) ? umax : out;          // branch-free: independent tests interleave
}

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
        const float on = sqrtf(fmaf(ox, ox, fmaf(oy, oy, oz * oz)));
        sdf = on;
        const float inv = 1.f / on;
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

__device__ __forceinline__ void or_code(uint32_t* row, int e, float v, const Fmt& f,
                                        uint32_t rc) {
    if (__float_as_uint(v) == 0u) return;          // +0 -> code 0 (the sparse common case)
    const uint32_t c = encode(v, f);
    const int w = int((e * rc) >> 16);             // e / pf (e < 4096)
    atomicOr(row + w, c << ((e - w * f.pf) * f.t));
}

// Self pair (i, j), i < j: false when inactive; else the gradient
// contribution v (d cost / d c_i = -v, d cost / d c_j = +v) and the cost w h.
__device__ __forceinline__ bool self_pair(const float* crow, int i, int j, const float* sr,
                                          float eta, float inv_eta, float hoe, float w, float& vx,
                                          float& vy, float& vz, float& cost) {
    const float dx = crow[3 * i] - crow[3 * j], dy = crow[3 * i + 1] - crow[3 * j + 1],
                dz = crow[3 * i + 2] - crow[3 * j + 2];
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float Rs = sr[i] + sr[j] + eta;
    // sqrt(fl(Rs^2)) rounds back to Rs and sqrt is monotone, so d2 >= fl(Rs^2)
    // implies fl(sqrt(d2)) >= Rs, i.e. phi <= 0: exact early out.
    if (d2 >= Rs * Rs) return false;
    const float d = sqrtf(d2);
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
        const float inv = 1.f / d;
        vx = k * (dx * inv);
        vy = k * (dy * inv);
        vz = k * (dz * inv);
    } else {                                       // coincident centres: direction (1, 0, 0)
        vx = k;
        vy = vz = 0.f;
    }
    cost = w * hh;
    return true;
}

// Per-CTA shared tables + per-warp workspaces; offsets computed on the host.
struct Geo {
    int Wos, Wcp, Wov, Qos, Qcp, Qov;  // packed row words and 16-byte groups
    int RS;                            // FP32 row stride (floats)
    int npairs, nlp, ngp, S;
    // per-CTA tables (bytes)
    unsigned sr, rl, ref, slink, pij, gpid, gpoff, gpab, lpab, lpgp, tables;
    // per-warp workspace (bytes, relative to the warp's base)
    unsigned rows, balls, amax, cub, wg, sg, lpid, lval, masks, wtotal;
    unsigned total;
};

Geo make_geo(const RobotDev& R, const Fmt& fos, const Fmt& fcp, const Fmt& fov, int do_world,
             int do_self) {
    Geo g{};
    g.Wos = row_words_of(fos, R.cols);
    g.Wcp = do_world ? row_words_of(fcp, R.cols) : 0;
    g.Wov = do_self ? row_words_of(fov, R.cols) : 0;
    g.Qos = g.Wos / 4;
    g.Qcp = g.Wcp / 4;
    g.Qov = g.Wov / 4;
    int rs = (R.cols + 3) & ~3;
    rs = std::max(rs, g.Wos * fos.pf);
    if (do_world) rs = std::max(rs, g.Wcp * fcp.pf);
    if (do_self) rs = std::max(rs, g.Wov * fov.pf);
    g.RS = rs;
    g.npairs = R.n_pairs;
    g.nlp = R.n_link_pairs;
    g.ngp = R.lp_gp_off[R.n_link_pairs];
    g.S = R.n_spheres;
    unsigned o = 0;
    auto take = [&](unsigned bytes, unsigned align) {
        o = (o + align - 1) / align * align;
        const unsigned at = o;
        o += bytes;
        return at;
    };
    g.sr = take(4u * kMaxSpheres, 4);
    g.rl = take(4u * 3 * kLinks, 4);
    g.ref = take(4u * 3 * kLinks, 4);
    g.slink = take(kMaxSpheres, 1);
    g.pij = take(2u * std::max(g.npairs, 1), 2);
    g.gpid = take(2u * std::max(g.npairs, 1), 2);
    g.gpoff = take(2u * (kMaxGroupPairs + 1), 2);
    g.gpab = take(2u * kMaxGroupPairs, 2);
    g.lpab = take(2u * 33, 2);
    g.lpgp = take(2u * 33, 2);
    g.tables = (o + 15) & ~15u;
    unsigned w = 0;
    auto wtake = [&](unsigned bytes, unsigned align) {
        w = (w + align - 1) / align * align;
        const unsigned at = w;
        w += bytes;
        return at;
    };
    g.rows = wtake(4u * 3 * g.RS, 16);            // decoded rows, ring of 3
    g.balls = wtake(16u * 3 * kLinks, 16);        // link balls of the 3 rows
    g.amax = wtake(4u * 4, 4);                    // per-row largest |coordinate|
    g.cub = wtake(64u * kMaxCuboids, 16);         // current world's cuboids
    g.wg = wtake(4u * g.RS, 16);                  // world gradient row (FP32)
    g.sg = wtake(4u * g.RS, 16);                  // self gradient row (FP32)
    g.lpid = wtake(2u * kListCap, 2);             // active self pairs (ids)
    g.lval = wtake(16u * kListCap, 16);           // ... their (v, cost)
    g.masks = wtake(4u * 2 * kLinks, 4);          // cull words: [2][link] (ping-pong)
    g.wtotal = (w + 15) & ~15u;
    g.total = g.tables + kWarps * g.wtotal + 16;
    return g;
}

struct Seg {                     // cull masks of a segment, one word per link
    uint32_t m[kLinks];
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kThreads)
collision_kernel(const __grid_constant__ RobotDev R, const __grid_constant__ Geo G,
                 const WorldsDev Wd, const Fmt fos, const Fmt fcp, const Fmt fov,
                 const CollisionArgs a) {
    extern __shared__ float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    float* ssr = reinterpret_cast<float*>(base + G.sr);
    float* link_rl = reinterpret_cast<float*>(base + G.rl);
    float* grp_rl = link_rl + kLinks;
    int* link_ref = reinterpret_cast<int*>(base + G.ref);
    int* grp_ref = link_ref + kLinks;
    uint8_t* slink = reinterpret_cast<uint8_t*>(base + G.slink);
    uint16_t* spij = reinterpret_cast<uint16_t*>(base + G.pij);     // i | j << 8
    uint16_t* sgpid = reinterpret_cast<uint16_t*>(base + G.gpid);
    uint16_t* sgpoff = reinterpret_cast<uint16_t*>(base + G.gpoff);
    uint16_t* sgpab = reinterpret_cast<uint16_t*>(base + G.gpab);   // a | b << 8
    uint16_t* slpab = reinterpret_cast<uint16_t*>(base + G.lpab);
    uint16_t* slpgp = reinterpret_cast<uint16_t*>(base + G.lpgp);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    char* wbase = base + G.tables + warp * G.wtotal;
    float* rows = reinterpret_cast<float*>(wbase + G.rows);
    float4* balls = reinterpret_cast<float4*>(wbase + G.balls);
    float* ramax = reinterpret_cast<float*>(wbase + G.amax);
    Cub* cub = reinterpret_cast<Cub*>(wbase + G.cub);
    float* wg = reinterpret_cast<float*>(wbase + G.wg);
    float* sg = reinterpret_cast<float*>(wbase + G.sg);
    uint16_t* lpid = reinterpret_cast<uint16_t*>(wbase + G.lpid);
    float4* lval = reinterpret_cast<float4*>(wbase + G.lval);
    uint32_t* masks = reinterpret_cast<uint32_t*>(wbase + G.masks);   // [2][kLinks]

    // ---- stage the divergently-indexed tables once per CTA
    for (int i = tid; i < G.S; i += kThreads) ssr[i] = R.sr[i];
    if (tid < kLinks) {
        link_rl[tid] = R.link_rl[tid];
        link_ref[tid] = R.link_ref[tid];
        for (int s2 = R.link_start[tid]; s2 < R.link_start[tid + 1]; ++s2) slink[s2] = (uint8_t)tid;
    }
    if (tid < 2 * kLinks) {
        grp_rl[tid] = R.grp_rl[tid];
        grp_ref[tid] = R.grp_ref[tid];
    }
    if (a.do_self) {
        for (int i = tid; i < G.npairs; i += kThreads) {
            spij[i] = (uint16_t)(R.pair_i[i] | (R.pair_j[i] << 8));
            sgpid[i] = R.gp_pid[i];
        }
        for (int i = tid; i <= G.ngp; i += kThreads) sgpoff[i] = R.gp_off[i];
        for (int i = tid; i < G.ngp; i += kThreads)
            sgpab[i] = (uint16_t)(R.gp_a[i] | (R.gp_b[i] << 8));
        for (int i = tid; i < G.nlp; i += kThreads)
            slpab[i] = (uint16_t)(R.lp_a[i] | (R.lp_b[i] << 8));
        for (int i = tid; i <= G.nlp; i += kThreads) slpgp[i] = R.lp_gp_off[i];
    }
    __syncthreads();                       // the only CTA barrier

    const long long P = (long long)a.B * a.H;
    const long long gw = (long long)blockIdx.x * kWarps + warp;
    const long long GW = (long long)gridDim.x * kWarps;
    const long long q0 = P * gw / GW, q1 = P * (gw + 1) / GW;   // this warp's poses
    if (q0 >= q1) return;

    const int RS = G.RS, S = G.S;
    const int nsub = (a.do_world && a.swept) ? a.sweep_steps : 0;
    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const float inv_n1 = 1.f / float(nsub + 1);
    const float maxfin = (fos.kind == KIND_IDENTITY) ? 3.0e38f : decode(fos.maxcode, fos);
    const float rel = ldexpf(1.f, -(fos.M + 1));
    const float sub = ldexpf(1.f, -((1 << (fos.E - 1)) - 1) - fos.M);

    // decode row pg into ring slot pg % 3 (+ its link balls and |x|max)
    auto decode_row = [&](long long pg) {
        const int slot = int(pg % 3);
        float* dst = rows + slot * RS;
        const uint4* src = reinterpret_cast<const uint4*>(a.os + pg * G.Wos);
        float am = 0.f;
        with_pf(fos.pf, [&](auto Pc) {
            constexpr int PF = decltype(Pc)::value;
            for (int q = lane; q < G.Qos; q += 32) {
                const uint4 v = __ldcs(src + q);
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                float x[4 * PF];
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) decode_word_t<PF>(w4[j4], x + j4 * PF, fos);
                float4* d4 = reinterpret_cast<float4*>(dst + 4 * PF * q);
#pragma unroll
                for (int j = 0; j < PF; ++j) {
                    d4[j] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
                    am = fmaxf(am, fmaxf(fmaxf(fabsf(x[4 * j]), fabsf(x[4 * j + 1])),
                                         fmaxf(fabsf(x[4 * j + 2]), fabsf(x[4 * j + 3]))));
                }
            }
        });
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
        __syncwarp();
        // Quantisation margin: a decoded coordinate y of an FK value x is
        // within 2^-(M+1)|x| + 2^-(bias+M) of it unless the code saturated
        // (|y| == max_finite: no bound, culling off for this row); two centres
        // per distance and sqrt(3) per vector give the ball margin.
        float margin = 0.f;
        if (fos.kind != KIND_IDENTITY) margin = 2.f * 1.7320509f * (rel * am * 1.01f + sub);
        if (lane < kLinks) {
            const float* c = dst + 3 * link_ref[lane];
            balls[slot * kLinks + lane] = make_float4(c[0], c[1], c[2], link_rl[lane] + margin);
        }
        if (lane == 0) ramax[slot] = (am >= maxfin) ? -1.f : margin;   // -1: saturated
        __syncwarp();
    };
    long long b = q0 / a.H;
    int h = int(q0 - b * a.H);
    int cur_world = -2, K = 0;
    long long have_lo = -1, have_hi = -1;          // decoded rows [have_lo, have_hi]
    int par = 0;                                   // masks + par*9: segment (pg-1, pg)
    if (lane < 2 * kLinks) masks[lane] = 0u;
    for (int e = lane; e < RS; e += 32) sg[e] = 0.f;
    __syncwarp();

    for (long long pg = q0; pg < q1; ++pg) {
        // ---- world of this trajectory: (re)load the cuboid cache
        if (a.do_world) {
            int wi = __ldg(a.world_idx + b);
            if (wi < 0 || wi >= Wd.n_worlds) wi = -1;
            if (wi != cur_world) {
                cur_world = wi;
                K = 0;
                if (wi >= 0) {
                    const int c0 = __ldg(Wd.off + wi);
                    K = __ldg(Wd.off + wi + 1) - c0;
                    for (int i = lane; i < 4 * K; i += 32)
                        reinterpret_cast<float4*>(cub)[i] = __ldg(Wd.cub + 4 * c0 + i);
                }
                __syncwarp();
            }
        }
        // ---- rows: pg-1 (swept, h > 0), pg, pg+1 (swept, h < H-1)
        const bool need_prev = nsub > 0 && h > 0;
        const bool need_next = nsub > 0 && h + 1 < a.H;
        if (need_prev && !(have_lo <= pg - 1 && pg - 1 <= have_hi)) {
            decode_row(pg - 1);
            have_lo = pg - 1;
            have_hi = pg - 1;
        }
        if (!(have_lo <= pg && pg <= have_hi)) {
            decode_row(pg);
            if (have_hi != pg - 1) have_lo = pg;
            have_hi = pg;
        }
        if (need_next) {
            decode_row(pg + 1);
            have_hi = pg + 1;
        }
        have_lo = max(have_lo, pg - 1);
        const int sc = int(pg % 3), sp_ = int((pg + 2) % 3), sn = int((pg + 1) % 3);
        const float* crow = rows + sc * RS;
        const bool cull_cur = a.cull && ramax[sc] >= 0.f;

        // ---- world cull masks: one word per link, bit k = cuboid k live.
        //      swept: mnext = segment (pg, pg+1), mprev = segment (pg-1, pg)
        //      (the previous pose's mnext); discrete: mnext = pose pg.
        uint32_t* mprev = masks + par * kLinks;
        uint32_t* mnext = masks + (par ^ 1) * kLinks;
        if (lane < kLinks) mnext[lane] = 0u;
        if (a.do_world && nsub > 0 && (h == 0 || pg == q0) && lane < kLinks) mprev[lane] = 0u;
        __syncwarp();
        if (a.do_world && K > 0) {
            auto test = [&](int s0, int s1, bool seg, bool ok, uint32_t* out) {
                for (int it = lane; it < kLinks * K; it += 32) {
                    const int l = it / K, k = it - l * K;
                    if (link_rl[l] < 0.f) continue;
                    const float4 b0 = balls[s0 * kLinks + l];
                    float mx = b0.x, my = b0.y, mz = b0.z, rs = b0.w;
                    if (seg) {
                        const float4 b1 = balls[s1 * kLinks + l];
                        const float dx = b1.x - b0.x, dy = b1.y - b0.y, dz = b1.z - b0.z;
                        mx += 0.5f * dx;
                        my += 0.5f * dy;
                        mz += 0.5f * dz;
                        rs = fmaxf(b0.w, b1.w) + 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    }
                    if (!ok || box_sdf_lb(cub[k], mx, my, mz) - rs - a.eta_w <= kSlack)
                        atomicOr(out + l, 1u << k);
                }
            };
            if (nsub > 0) {
                if (h > 0 && pg == q0)     // range starts mid-trajectory: segment (pg-1, pg)
                    test(sp_, sc, true, a.cull && ramax[sp_] >= 0.f && ramax[sc] >= 0.f, mprev);
                if (need_next) test(sc, sn, true, a.cull && ramax[sc] >= 0.f && ramax[sn] >= 0.f, mnext);
            } else {
                test(sc, sc, false, cull_cur, mnext);
            }
        }
        __syncwarp();

        // ---- world: one lane per sphere; gradient into wg, cost by a fixed tree
        float wcost = 0.f;
        bool wany = false;
        if (a.do_world) {
            for (int s0 = 0; s0 < S; s0 += 32) {
                const int sp = s0 + lane;
                float gx = 0.f, gy = 0.f, gz = 0.f, c = 0.f;
                if (sp < S) {
                    const int l = slink[sp];
                    uint32_t own, fwd = 0u, bwd = 0u;
                    if (nsub > 0) {
                        fwd = mnext[l];
                        bwd = (h > 0) ? mprev[l] : 0u;
                        own = fwd | bwd;   // a segment ball contains both endpoint balls
                    } else {
                        own = mnext[l];
                    }
                    if (own) {
                        const float cx = crow[3 * sp], cy = crow[3 * sp + 1], cz = crow[3 * sp + 2];
                        const float A = ssr[sp] + a.eta_w;
                        Acc acc{0.f, 0.f, 0.f, 0.f};
                        for (uint32_t m = own; m; m &= m - 1)
                            world_term(cub[__ffs(m) - 1], cx, cy, cz, A, a.eta_w, inv_eta_w, hoe_w,
                                       a.w_w, 1.f, 1.f, acc);
                        if (fwd) {          // samples of segment (h, h+1): cost + (1-tau) grad
                            const float* nrow = rows + sn * RS;
                            const float nx = nrow[3 * sp], ny = nrow[3 * sp + 1], nz = nrow[3 * sp + 2];
                            for (int j = 1; j <= nsub; ++j) {
                                const float tau = float(j) * inv_n1, omt = 1.f - tau;
                                const float sx = fmaf(tau, nx, omt * cx), sy = fmaf(tau, ny, omt * cy),
                                            sz = fmaf(tau, nz, omt * cz);
                                for (uint32_t m = fwd; m; m &= m - 1)
                                    world_term(cub[__ffs(m) - 1], sx, sy, sz, A, a.eta_w, inv_eta_w,
                                               hoe_w, a.w_w, 1.f, omt, acc);
                            }
                        }
                        if (bwd) {          // samples of segment (h-1, h): tau grad only
                            const float* prow = rows + sp_ * RS;
                            const float qx = prow[3 * sp], qy = prow[3 * sp + 1], qz = prow[3 * sp + 2];
                            for (int j = 1; j <= nsub; ++j) {
                                const float tau = float(j) * inv_n1, omt = 1.f - tau;
                                const float sx = fmaf(tau, cx, omt * qx), sy = fmaf(tau, cy, omt * qy),
                                            sz = fmaf(tau, cz, omt * qz);
                                for (uint32_t m = bwd; m; m &= m - 1)
                                    world_term(cub[__ffs(m) - 1], sx, sy, sz, A, a.eta_w, inv_eta_w,
                                               hoe_w, a.w_w, 0.f, tau, acc);
                            }
                        }
                        gx = acc.gx + 0.f;
                        gy = acc.gy + 0.f;
                        gz = acc.gz + 0.f;
                        c = acc.cost;
                    }
                    wg[3 * sp] = gx;
                    wg[3 * sp + 1] = gy;
                    wg[3 * sp + 2] = gz;
                }
                wcost += c;
                wany |= __any_sync(0xffffffffu, (__float_as_uint(gx) | __float_as_uint(gy) |
                                                 __float_as_uint(gz)) != 0u);
            }
            wcost = warp_sum(wcost);       // fixed shuffle tree: deterministic
        }

        // ---- self: link pairs -> group pairs -> sphere pairs (list order:
        //      group pair, then pair id), accumulated in list order into sg
        float scost = 0.f;
        bool sany = false;
        if (a.do_self) {
            bool live_lp = false;
            uint32_t gpbits = 0u;          // live group pairs of this lane's link pair
            if (lane < G.nlp) {
                const int la = slpab[lane] & 0xff, lb = slpab[lane] >> 8;
                const float4 A4 = balls[sc * kLinks + la], B4 = balls[sc * kLinks + lb];
                const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                const float lim = A4.w + B4.w + a.eta_s + kSlack;
                live_lp = !cull_cur || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim;
                if (live_lp) {
                    const float margin = fmaxf(ramax[sc], 0.f);
                    for (int g = slpgp[lane]; g < slpgp[lane + 1]; ++g) {
                        const int ga = sgpab[g] & 0xff, gb = sgpab[g] >> 8;
                        const float* ca = crow + 3 * grp_ref[ga];
                        const float* cb = crow + 3 * grp_ref[gb];
                        const float ex = ca[0] - cb[0], ey = ca[1] - cb[1], ez = ca[2] - cb[2];
                        const float gl = grp_rl[ga] + grp_rl[gb] + 2.f * margin + a.eta_s + kSlack;
                        if (!cull_cur || fmaf(ex, ex, fmaf(ey, ey, ez * ez)) <= gl * gl)
                            gpbits |= 1u << (g - slpgp[lane]);
                    }
                }
            }
            const uint32_t lpmask = __ballot_sync(0xffffffffu, gpbits != 0u);
            int n = 0;                     // active pairs buffered in the list
            auto flush = [&]() {           // accumulate the buffered pairs in order
                __syncwarp();
                if (lane == 0) {
                    for (int k = 0; k < n; ++k) {
                        const int pid = lpid[k];
                        const int i = spij[pid] & 0xff, j = spij[pid] >> 8;
                        const float4 v = lval[k];
                        sany = true;       // sg is all +0 at the start of every pose
                        sg[3 * i] -= v.x;
                        sg[3 * i + 1] -= v.y;
                        sg[3 * i + 2] -= v.z;
                        sg[3 * j] += v.x;
                        sg[3 * j + 1] += v.y;
                        sg[3 * j + 2] += v.z;
                        scost += v.w;
                    }
                }
                sany = __shfl_sync(0xffffffffu, sany, 0);
                n = 0;
                __syncwarp();
            };
            for (uint32_t lm = lpmask; lm; lm &= lm - 1) {
                const int lp = __ffs(lm) - 1;
                const uint32_t gbits = __shfl_sync(0xffffffffu, gpbits, lp);
                for (uint32_t gm = gbits; gm; gm &= gm - 1) {
                    const int g = slpgp[lp] + __ffs(gm) - 1;
                    const int k0 = sgpoff[g], k1 = sgpoff[g + 1];
                    for (int kb = k0; kb < k1; kb += 32) {
                        const int k = kb + lane;
                        bool act = false;
                        int pid = 0;
                        float vx = 0.f, vy = 0.f, vz = 0.f, c = 0.f;
                        if (k < k1) {
                            pid = sgpid[k];
                            act = self_pair(crow, spij[pid] & 0xff, spij[pid] >> 8, ssr, a.eta_s,
                                            inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c);
                        }
                        const uint32_t am = __ballot_sync(0xffffffffu, act);
                        if (n + __popc(am) > kListCap) flush();
                        if (act) {
                            const int slot = n + __popc(am & ((1u << lane) - 1u));
                            lpid[slot] = (uint16_t)pid;
                            lval[slot] = make_float4(vx, vy, vz, c);
                        }
                        n += __popc(am);
                    }
                }
            }
            if (n) flush();
            scost = __shfl_sync(0xffffffffu, scost, 0);
        }

        // ---- encode and store the packed rows; the pose cost
        if (a.do_world) {
            uint4* dst = reinterpret_cast<uint4*>(a.cp + pg * G.Wcp);
            with_pf(fcp.pf, [&](auto Pc) {
                constexpr int PF = decltype(Pc)::value;
                for (int q = lane; q < G.Qcp; q += 32) {
                    uint32_t w[4] = {0u, 0u, 0u, 0u};
                    if (wany) {
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            float x[PF];
                            const int e0 = (4 * q + j4) * PF;
#pragma unroll
                            for (int j = 0; j < PF; ++j) x[j] = (e0 + j < 3 * S) ? wg[e0 + j] : 0.f;
                            w[j4] = encode_word_t<PF>(x, fcp);
                        }
                    }
                    __stcs(dst + q, make_uint4(w[0], w[1], w[2], w[3]));
                }
            });
        }
        if (a.do_self) {
            uint4* dst = reinterpret_cast<uint4*>(a.ov + pg * G.Wov);
            with_pf(fov.pf, [&](auto Pc) {
                constexpr int PF = decltype(Pc)::value;
                for (int q = lane; q < G.Qov; q += 32) {
                    uint32_t w[4] = {0u, 0u, 0u, 0u};
                    if (sany) {
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            float x[PF];
                            const int e0 = (4 * q + j4) * PF;
#pragma unroll
                            for (int j = 0; j < PF; ++j) x[j] = (e0 + j < 3 * S) ? sg[e0 + j] + 0.f : 0.f;
                            w[j4] = encode_word_t<PF>(x, fov);
                        }
                    }
                    __stcs(dst + q, make_uint4(w[0], w[1], w[2], w[3]));
                }
            });
        }
        if (lane == 0) a.cost[pg] = wcost + scost;
        __syncwarp();
        if (sany)                          // restore the all-zero self row
            for (int e = lane; e < 3 * S; e += 32) sg[e] = 0.f;

        // ---- advance: segment (pg, pg+1) becomes the previous segment
        par ^= 1;
        if (++h == a.H) {
            h = 0;
            ++b;
        }
    }
}

__global__ void traj_reduce_kernel(const float* __restrict__ cost_pose, int B, int H,
                                   float* __restrict__ cost_traj) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    float c = 0.f;
    for (int h = 0; h < H; ++h) c += cost_pose[(long long)b * H + h];
    cost_traj[b] = c;
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

cudaError_t launch_collision(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                             const Fmt& fcp, const Fmt& fov, const CollisionArgs& a,
                             cudaStream_t s) {
    const long long P = (long long)a.B * a.H;
    if (P <= 0) return cudaSuccess;
    const Geo G = make_geo(R, fos, fcp, fov, a.do_world, a.do_self);
    const size_t smem = G.total;
    cudaError_t e = cudaFuncSetAttribute(collision_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // persistent CTAs: as many as fit; every warp streams a contiguous range
    // of poses (at least ~8 poses per warp so the ring of rows pays off)
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, collision_kernel, kThreads, smem);
    long long grid = (long long)sms * std::max(per_sm, 1);
    const long long max_grid = std::max(1LL, P / (8LL * kWarps));
    grid = std::max(1LL, std::min(grid, max_grid));
    collision_kernel<<<(unsigned)grid, kThreads, smem, s>>>(R, G, W, fos, fcp, fov, a);
    return cudaGetLastError();
}

cudaError_t launch_traj_reduce(const float* cost_pose, int32_t B, int32_t H, float* cost_traj,
                               cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    traj_reduce_kernel<<<(B + 255) / 256, 256, 0, s>>>(cost_pose, B, H, cost_traj);
    return cudaGetLastError();
}

cudaError_t launch_best_per_problem(const float* cost_traj, int32_t n_problems, int32_t seeds,
                                    float* best_cost, int32_t* best_seed, cudaStream_t s) {
    if (n_problems <= 0) return cudaSuccess;
    best_kernel<<<(n_problems + 255) / 256, 256, 0, s>>>(cost_traj, n_problems, seeds,
                                                        best_cost, best_seed);
    return cudaGetLastError();
}

}  // namespace vapr
