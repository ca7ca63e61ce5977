// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients in ONE pass over the
// packed out_spheres, writing packed closest_pt[_swept] / out_vec (dense rows,
// or the N3 sparse form).
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// Lane = pose.  A warp owns a tile of 32 consecutive poses (31 plus a halo
// pose when trajectories do not align with 32-pose tiles), decodes their
// packed rows once into an FP32 tile in shared memory laid out [element][33]
// (a uniform element index across the lanes is a conflict-free read), and
// then every lane evaluates its own pose with warp-uniform loops:
//  1. world broadphase: the spheres of a link lie in a ball around a
//     reference sphere (rigid radius, host-computed, plus the quantisation
//     margin); per (link, cuboid) a ball-box distance test -- for the swept
//     cost a ball around the segment (pose, next pose) -- gives per-lane
//     cuboid masks;
//  2. world narrowphase over the links some lane has live, sphere by sphere:
//     the pose's own term and, swept, the samples of its forward segment,
//     each sample evaluated ONCE: the lane keeps (1 - tau) of its gradient
//     and hands tau of it to the next pose's lane (shuffle); a sample is
//     skipped when the endpoint SDFs already prove it inactive (the box SDF
//     is 1-Lipschitz: sdf(p_j) >= sdf(c_h) - tau |c_h+1 - c_h|, and from the
//     other end);
//  3. self broadphase: link pairs (link balls), group pairs (balls of runs of
//     <= 5 spheres), then sphere-vs-group-ball, then the listed sphere pairs;
//     active pairs are marked in a per-pose pair-id bitmask;
//  4. self gradients: per touched sphere, the active pairs in pair-id order.
// Every lane writes its own pose's outputs (no atomics).
//
// Culling is exact: a term is skipped only when its bound clears the
// activation distance by kSlack = 1e-4 m, orders of magnitude above the FP32
// evaluation error of the distances for workspace-scale coordinates
// (|x| < 100 m), so every skipped term would evaluate to phi <= 0, i.e. to
// exactly 0; surviving terms are accumulated in the same order with and
// without culling, so VAPR_OPT_CULL on and off give bit-identical results
// (tests/test_gpu_parity.py::test_cull_is_exact).
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "tap.cuh"

namespace vapr {

namespace {

constexpr float kSlack = 1e-4f;
constexpr int kTS = 33;            // FP32 tile row stride (lanes 0..31 + the halo pose)

#ifndef VAPR_COLL_WARPS           // warps per CTA
#define VAPR_COLL_WARPS 4
#endif
#ifndef VAPR_COLL_MINB_W          // CTAs per SM the register allocation targets (world, self)
#define VAPR_COLL_MINB_W 2
#endif
#ifndef VAPR_COLL_MINB_S
#define VAPR_COLL_MINB_S 2
#endif
constexpr int kWarps = VAPR_COLL_WARPS;

struct Cub {
    float4 q0, q1, q2, q3;   // R^T (9), t (3), h (3), pad
};

__device__ __forceinline__ Cub load_cub(const float4* c) {
    return Cub{__ldg(c), __ldg(c + 1), __ldg(c + 2), __ldg(c + 3)};
}

struct WTerm {
    float sdf;               // the box SDF, or a lower bound of it when inactive
    float h, s;              // hinge value and -w h'(phi) (0 when inactive)
    float gx, gy, gz;        // world-frame SDF gradient (valid when s != 0)
};

// One sphere-vs-cuboid term at centre c with activation distance A = r + eta.
__device__ __forceinline__ WTerm world_term(const Cub& b, float cx, float cy, float cz, float A,
                                            float eta, float inv_eta, float hoe, float w) {
    WTerm t;
    t.h = 0.f;
    t.s = 0.f;
    t.gx = t.gy = t.gz = 0.f;
    const float dx = cx - b.q2.y, dy = cy - b.q2.z, dz = cz - b.q2.w;
    const float px = fmaf(b.q0.x, dx, fmaf(b.q0.y, dy, b.q0.z * dz));
    const float py = fmaf(b.q0.w, dx, fmaf(b.q1.x, dy, b.q1.y * dz));
    const float pz = fmaf(b.q1.z, dx, fmaf(b.q1.w, dy, b.q2.x * dz));
    const float ux = fabsf(px) - b.q3.x, uy = fabsf(py) - b.q3.y, uz = fabsf(pz) - b.q3.z;
    const float umax = fmaxf(ux, fmaxf(uy, uz));
    // sdf >= umax in FP32 (sqrt(fl(a^2)) rounds back to a; adding terms only
    // grows it), so A - umax <= 0 implies phi = A - sdf <= 0: exact early out,
    // and umax is a valid lower bound of the SDF for the swept sample cull
    t.sdf = umax;
    if (A - umax <= 0.f) return t;
    float glx, gly, glz;
    if (umax <= 0.f) {                 // inside: nearest face, lowest index on ties
        glx = gly = glz = 0.f;
        if (ux >= uy && ux >= uz) glx = (px >= 0.f) ? 1.f : -1.f;
        else if (uy >= uz) gly = (py >= 0.f) ? 1.f : -1.f;
        else glz = (pz >= 0.f) ? 1.f : -1.f;
    } else {
        const float ox = fmaxf(ux, 0.f), oy = fmaxf(uy, 0.f), oz = fmaxf(uz, 0.f);
        // |o| and 1/|o| from one MUFU rsqrt (~2 ulp; parity tolerance), the
        // IEEE path for arguments near the FP32 underflow
        const float o2 = fmaf(ox, ox, fmaf(oy, oy, oz * oz));
        float on, inv;
        if (o2 >= 1e-30f) {
            inv = rsqrtf(o2);
            on = o2 * inv;
        } else {
            on = sqrtf(o2);
            inv = 1.f / on;
        }
        t.sdf = on;
        glx = (px >= 0.f) ? ox * inv : -(ox * inv);
        gly = (py >= 0.f) ? oy * inv : -(oy * inv);
        glz = (pz >= 0.f) ? oz * inv : -(oz * inv);
    }
    const float phi = A - t.sdf;
    if (phi <= 0.f) return t;
    float dh;
    if (phi <= eta) {
        t.h = phi * phi * hoe;
        dh = phi * inv_eta;
    } else {
        t.h = phi - 0.5f * eta;
        dh = 1.f;
    }
    t.s = -w * dh;
    // world gradient = R g_local with R = (R^T)^T
    t.gx = fmaf(b.q0.x, glx, fmaf(b.q0.w, gly, b.q1.z * glz));
    t.gy = fmaf(b.q0.y, glx, fmaf(b.q1.x, gly, b.q1.w * glz));
    t.gz = fmaf(b.q0.z, glx, fmaf(b.q1.y, gly, b.q2.x * glz));
    return t;
}

// Self pair (i, j), i < j, at centres ci, cj: false when inactive; else the
// gradient contribution v (d cost / d c_i = -v, d cost / d c_j = +v) and the
// cost w h.  Rs = r_i + r_j + eta.
__device__ __forceinline__ bool self_pair(float ix, float iy, float iz, float jx, float jy, float jz,
                                          float Rs, float eta, float inv_eta, float hoe, float w,
                                          float& vx, float& vy, float& vz, float& cost) {
    const float dx = ix - jx, dy = iy - jy, dz = iz - jz;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
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
// Per-pose output of one gradient tensor: dense rows (zero-filled per tile,
// then the words holding non-zero codes rewritten) or the N3 sparse form (the
// row's sphere bitmap and its non-zero codes packed in ascending sphere order
// at pool + pose * wmax; reading c42).  Spheres arrive in ascending order; one
// writer per pose at a time.
struct RowOut {
    uint32_t word;        // sparse: the word being filled
    uint32_t qnw;         // sparse: codes in `word` (low 8 bits), words written (<< 8)
    unsigned long long mask;
    float cost;           // the pose's cost terms carried with its codes (world)
    uint32_t pad;
};

__device__ __forceinline__ void out_put(RowOut& o, uint32_t* row, bool sparse, int s, float vx,
                                        float vy, float vz, const Fmt& f, uint32_t rc) {
    const float v[3] = {vx + 0.f, vy + 0.f, vz + 0.f};
    uint32_t c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = (__float_as_uint(v[k]) != 0u) ? encode(v[k], f) : 0u;
    if (!(c[0] | c[1] | c[2])) return;
    if (sparse) {
        o.mask |= 1ull << s;
        int q = int(o.qnw & 0xffu), nw = int(o.qnw >> 8);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            o.word |= (f.t == 32) ? c[k] : (c[k] << (q * f.t));
            if (++q == f.pf) {
                row[nw++] = o.word;
                o.word = 0u;
                q = 0;
            }
        }
        o.qnw = uint32_t(q) | (uint32_t(nw) << 8);
    } else {
        // the row was zero-filled at the tile start: OR the codes into the
        // words holding them (one writer per pose)
        int cw = -1;
        uint32_t acc = 0u;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int e = 3 * s + k;
            const int w = int((uint32_t(e) * rc) >> 16);      // e / pf (e < 4096)
            if (w != cw) {
                if (acc) row[cw] |= acc;
                cw = w;
                acc = 0u;
            }
            acc |= (f.t == 32) ? c[k] : (c[k] << ((e - w * f.pf) * f.t));
        }
        if (acc) row[cw] |= acc;
    }
}

__device__ __forceinline__ void out_finish(RowOut& o, uint32_t* row, bool sparse,
                                           unsigned long long* mask_out) {
    if (!sparse) return;
    const int q = int(o.qnw & 0xffu), nw = int(o.qnw >> 8);
    if (q) row[nw] = o.word;
    *mask_out = o.mask;
}

// ---------------------------------------------------------------------------
// The pose tile: FP32 values [E][kTS] (element e of the pose in column col at
// e * kTS + col), E = Wos * pf (padded rows: the decode needs no bounds checks).
__device__ __forceinline__ void tsph(const float* T, int s, int col, float& x, float& y, float& z) {
    const float* c = T + 3 * s * kTS + col;
    x = c[0];
    y = c[kTS];
    z = c[2 * kTS];
}

// Warp pairs: the two warps of a pair share one 32-pose tile.  The even warp
// (W) runs the world cost, the odd warp (S) the self cost and writes the
// pose's total; both unpack the tile.  Shared-memory carve-up (bytes): CTA
// tables (pair table, sphere radii), then per pair: the tile; W's region (link
// masks [kLinks][32], world of each pose, link blocks, per-pose output
// states, item window, world costs); S's region (active-pair bitmask
// [pmw][32], live group pairs, touched / word masks, item window); the pair's
// exchange words.  The unpacking's staging (kStage 16-byte groups per thread
// in flight) spans W's and S's regions.
constexpr int kStage = 7;
constexpr int kPairs = kWarps / 2;
struct LinkBlk {
    uint32_t pm;          // poses (lanes) with a live cuboid for the link
    int start, cnt;       // first item, poses
    float rcp;            // 1 / cnt
};
struct PairX {
    long long tile;
    float amax[2];
};
struct CGeo {
    int Wos;                      // packed out_spheres row words
    int Qos;                      // 16-byte groups per row
    uint32_t rc_q;                // q / Qos reciprocal (20-bit fixed point)
    int Wcp, Wov;                 // dense output row words
    int wmax_cp, wmax_ov;         // sparse output row capacity (words)
    uint32_t rc_cp, rc_ov;        // e / pf reciprocals (16-bit fixed point)
    int pmw;                      // active-pair bitmask words per pose
    int own0;                     // 1: lane 0 is the halo pose p0 - 1 (swept, unaligned H)
    unsigned off_sr, cta_bytes;   // CTA tables: pair table at 0, radii at off_sr
    // per pair
    unsigned off_wm, off_kk, off_lb, off_rs, off_qdw, off_qrw, off_wc;
    unsigned off_pm, off_gl, off_tc, off_wk, off_qds, off_qrs, off_x, w_bytes, s_bytes;
};

CGeo make_cgeo(const RobotDev& R, const SelfDev& SD, const Fmt& fos, const Fmt& fcp,
               const Fmt& fov, const CollisionArgs& a) {
    CGeo g{};
    g.Wos = row_words_of(fos, R.cols);
    g.Qos = g.Wos / 4;
    g.rc_q = (1u << 20) / (uint32_t)g.Qos + 1u;      // exact for q < kTS * Qos (checked)
    for (int q = 0; q < kTS * g.Qos; ++q)
        if (int((uint32_t(q) * g.rc_q) >> 20) != q / g.Qos) g.rc_q = 0;
    g.Wcp = row_words_of(fcp, R.cols);
    g.Wov = row_words_of(fov, R.cols);
    g.wmax_cp = (R.cols + fcp.pf - 1) / fcp.pf;
    g.wmax_ov = (R.cols + fov.pf - 1) / fov.pf;
    g.rc_cp = 65536u / fcp.pf + 1u;
    g.rc_ov = 65536u / fov.pf + 1u;
    g.pmw = a.do_self ? (SD.n_pairs + 31) / 32 : 0;
    // swept tiles must hold whole segments: 32 poses per tile when every
    // trajectory boundary is a tile boundary, else 31 plus the halo pose
    g.own0 = (a.do_world && a.swept && (32 % a.H) != 0) ? 1 : 0;
    g.off_sr = (unsigned)((2 * SD.n_pairs + 15) & ~15);
    g.cta_bytes = g.off_sr + 4u * kMaxSpheres;
    unsigned o = (unsigned)(4 * g.Wos * fos.pf * kTS);
    auto take = [&](unsigned bytes) {
        o = (o + 15u) & ~15u;
        const unsigned at = o;
        o += bytes;
        return at;
    };
    const unsigned t_end = o;
    // W (world kernel)
    g.off_wm = take(4u * kLinks * 32u);
    g.off_kk = take(4u * 32u);
    g.off_lb = take((unsigned)sizeof(LinkBlk) * kLinks);
    g.off_rs = take((unsigned)sizeof(RowOut) * 32u);
    g.off_qdw = take(4u * 32u);
    g.off_qrw = take(16u * 32u);
    g.off_wc = take(4u * 32u);
    g.w_bytes = std::max(o, t_end + 16u * kStage * 32u);
    // S (self kernel), from the tile's end again
    o = t_end;
    g.off_pm = take(4u * g.pmw * 32u);
    g.off_gl = take(8u * (SD.n_gp + 1));
    g.off_tc = take(8u * 32u);
    g.off_wk = take(4u * 32u);
    g.off_qds = take(4u * 32u);
    g.off_qrs = take(16u * 32u);
    g.s_bytes = std::max(o, t_end + 16u * kStage * 32u);
    g.off_x = 0;
    g.w_bytes = (g.w_bytes + 15u) & ~15u;
    g.s_bytes = (g.s_bytes + 15u) & ~15u;
    return g;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// the two warps of a pair (named barrier 1 + pair; constant ids)
__device__ __forceinline__ void pair_sync(int pair) {
    static_assert(kPairs <= 4, "named barriers 1..4");
    if (pair == 0) asm volatile("bar.sync 1, 64;" ::: "memory");
    else if (pair == 1) asm volatile("bar.sync 2, 64;" ::: "memory");
    else if (pair == 2) asm volatile("bar.sync 3, 64;" ::: "memory");
    else asm volatile("bar.sync 4, 64;" ::: "memory");
}

// ---------------------------------------------------------------------------
template <bool SWEPT, int ROLE>
__global__ void __launch_bounds__(32 * kWarps, ROLE == 0 ? VAPR_COLL_MINB_W : VAPR_COLL_MINB_S)
collision_kernel(const __grid_constant__ RobotDev R, const SelfDev* __restrict__ SD,
                 const CGeo G, const WorldsDev Wd, const Fmt fos, const Fmt fcp, const Fmt fov,
                 const CollisionArgs a) {
    extern __shared__ float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    uint16_t* spij = reinterpret_cast<uint16_t*>(base);            // pair id -> i | j << 8
    float* ssr = reinterpret_cast<float*>(base + G.off_sr);         // sphere radii
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int role = ROLE;                                      // 0: world, 1: self
    char* wb = base + G.cta_bytes + (unsigned)warp * (ROLE == 0 ? G.w_bytes : G.s_bytes);
    float* T = reinterpret_cast<float*>(wb);                        // the tile [E][kTS]
    uint4* stage = reinterpret_cast<uint4*>(wb + (ROLE == 0 ? G.off_wm : G.off_pm));  // [kStage][32]
    uint32_t* WM = reinterpret_cast<uint32_t*>(wb + G.off_wm);      // W: [kLinks][32]
    uint32_t* KK = reinterpret_cast<uint32_t*>(wb + G.off_kk);      // W: [32] k0 | K << 16
    LinkBlk* LB = reinterpret_cast<LinkBlk*>(wb + G.off_lb);        // W: [kLinks]
    RowOut* RS = reinterpret_cast<RowOut*>(wb + G.off_rs);          // W: [32] per-pose output
    float* WC = reinterpret_cast<float*>(wb + G.off_wc);            // W: [32] world cost
    uint32_t* PM = reinterpret_cast<uint32_t*>(wb + G.off_pm);      // S: [pmw][32]
    uint2* GL = reinterpret_cast<uint2*>(wb + G.off_gl);            // S: live group pairs
    unsigned long long* TC = reinterpret_cast<unsigned long long*>(wb + G.off_tc);  // S: touched
    uint32_t* WK = reinterpret_cast<uint32_t*>(wb + G.off_wk);      // S: pair-mask words
    uint32_t* QD = reinterpret_cast<uint32_t*>(wb + (role ? G.off_qds : G.off_qdw));  // window items
    float4* QR = reinterpret_cast<float4*>(wb + (role ? G.off_qrs : G.off_qrw));      // their results

    const int npairs = a.do_self ? __ldg(&SD->n_pairs) : 0;
    for (int i = tid; i < npairs; i += blockDim.x) spij[i] = __ldg(&SD->pij[i]);
    for (int i = tid; i < R.n_spheres; i += blockDim.x) ssr[i] = R.sr[i];
    __syncthreads();

    const int cols = R.cols;       // (the debug tap's row stride)
    (void)cols;
    const long long P = (long long)a.B * a.H;
    const int own0 = G.own0;
    const int TP = 32 - own0;                     // poses owned per tile
    const long long n_tiles = (P + TP - 1) / TP;
    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const int nsub = SWEPT ? a.sweep_steps : 0;
    const float inv_n1 = 1.f / float(nsub + 1);
    const uint4* os4 = reinterpret_cast<const uint4*>(a.os);
    // the clamp code's value: coordinates at or beyond it may be saturated
    // (all-finite) or inf (IEEE mode: 65536 for E5M10, inf for E8M7)
    const float fmax_os = decode(fos.maxcode, fos);
    const bool sp_cp = a.cp_mask != nullptr, sp_ov = a.ov_mask != nullptr;
    unsigned int* sched = a.sched;                // [0] next tile, [1] finished CTAs

    for (;;) {
        unsigned int ti = 0;
        if (lane == 0) ti = atomicAdd(sched, 1u);
        const long long tile = __shfl_sync(0xffffffffu, ti, 0);
        if (tile >= n_tiles) break;
        const long long p0 = tile * TP - own0;     // pose of lane 0
        const long long pg = p0 + lane;
        const bool valid = pg >= 0 && pg < P;
        const bool owner = valid && lane >= own0;
        int h = 0;
        long long b = 0;
        if (valid) {
            b = pg / a.H;
            h = int(pg - b * a.H);
        }
        // tile rows: poses p0 .. p0 + 32 (row 32 = the pose after lane 31,
        // needed only by a swept segment crossing the tile end)
        const bool need_hi = SWEPT && own0 && (p0 + 32 < P);
        const long long r_lo = max(p0, 0LL);
        const long long r_hi = min(p0 + (need_hi ? 33 : 32), P);      // exclusive
        const int row_off = int(r_lo - p0);

        // ---- 1. the tile rows into T[e][row]: kStage 16-byte groups per lane
        // in flight (cp.async into the staging region), unpacked one group at
        // a time (a compact loop: the kernels are instruction-cache sensitive)
        float amax = 0.f;
        {
            const int nq = int(r_hi - r_lo) * G.Qos;
            const uint4* src = os4 + r_lo * G.Qos;
            with_pf(fos.pf, [&](auto Pc) {
                constexpr int PF = decltype(Pc)::value;
                for (int q0 = 0; q0 < nq; q0 += 32 * kStage) {
#pragma unroll
                    for (int u = 0; u < kStage; ++u) {
                        const int q = q0 + 32 * u + lane;
                        if (q < nq) cp_async16(stage + 32 * u + lane, src + q);
                    }
                    cp_async_wait_all();
#pragma unroll 1
                    for (int u = 0; u < kStage; ++u) {
                        const int q = q0 + 32 * u + lane;
                        if (q >= nq) break;
                        const uint4 v = stage[32 * u + lane];
                        const int r = int((uint32_t(q) * G.rc_q) >> 20);
                        const int g = q - r * G.Qos;
                        float* d = T + row_off + r + (4 * PF * g) * kTS;
                        float x[4 * PF];
                        if constexpr (PF == 2) {
                            decode_group_t<2>(v, x, fos);
                        } else {
                            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int j4 = 0; j4 < 4; ++j4) decode_word_t<PF>(w4[j4], x + j4 * PF, fos);
                        }
#pragma unroll
                        for (int j = 0; j < 4 * PF; ++j) {
                            d[j * kTS] = x[j];
                            amax = fmaxf(amax, fabsf(x[j]));
                        }
                    }
                }
            });
            amax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(amax)));
        }
        // dense outputs: zero-fill the tile's owned rows (coalesced); the pose
        // writers then OR in their non-zero codes
        const long long o_lo = p0 + own0;
        const int n_own = (int)max(0LL, min((long long)TP, P - o_lo));
        if (role == 0 && a.do_world && !sp_cp)
            for (int i = lane; i < n_own * G.Wcp / 4; i += 32)
                reinterpret_cast<uint4*>(a.cp + o_lo * G.Wcp)[i] = make_uint4(0u, 0u, 0u, 0u);
        if (role == 1 && a.do_self && !sp_ov)
            for (int i = lane; i < n_own * G.Wov / 4; i += 32)
                reinterpret_cast<uint4*>(a.ov + o_lo * G.Wov)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        if (role == 0) RS[lane] = RowOut{0u, 0u, 0ull, 0.f, 0u};   // (after the staging's last read)

        // Quantisation margin: a decoded coordinate y of an FK value x
        // satisfies |y - x| <= 2^-(M+1) |x| + 2^-(bias+M) unless the code
        // saturated; two centres per distance and sqrt(3) per vector give the
        // ball margin.  A saturated coordinate in the tile switches culling off.
        bool can_cull = a.cull != 0;
        float margin = 0.f;
        if (fos.kind != KIND_IDENTITY) {
            if (!(amax < fmax_os)) can_cull = false;
            const float rel = ldexpf(1.f, -(fos.M + 1));
            const float sub = ldexpf(1.f, -((1 << (fos.E - 1)) - 1) - fos.M);
            margin = 2.f * 1.7320509f * (rel * amax * 1.01f + sub);
        }

        // link reference spheres of the lane's pose (registers, static index)
        float rx[kLinks], ry[kLinks], rz[kLinks];
#pragma unroll
        for (int l = 0; l < kLinks; ++l)
            tsph(T, min(max(R.link_ref[l], 0), R.n_spheres - 1), lane, rx[l], ry[l], rz[l]);

        // self broadphase, link level (needs the reference spheres, which die
        // after the world broadphase)
        const float m2 = 2.f * margin + kSlack + a.eta_s;
        unsigned long long lpm = 0ull;
        if (role == 1 && a.do_self) {
            // link pairs: bit i <=> link pair i's balls are within reach (the
            // reference spheres in registers: a static loop over link pairs)
#pragma unroll
            for (int la = 0; la < kLinks; ++la)
#pragma unroll
                for (int lb = la; lb < kLinks; ++lb) {
                    const int i = __ldg(&SD->lp_of[la][lb]);
                    if (i < 0) continue;
                    const float dx = rx[la] - rx[lb], dy = ry[la] - ry[lb], dz = rz[la] - rz[lb];
                    const float lim = R.link_rl[la] + R.link_rl[lb] + m2;
                    if (owner && (!can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim))
                        lpm |= 1ull << i;
                }
        }
        float wcost = 0.f, scost = 0.f;
        // ---- 2. world (W)
        if (role == 0 && a.do_world) {
            int k0 = 0, K = 0;
            if (valid) {
                const int wi = __ldg(a.world_idx + b);
                if (wi >= 0 && wi < Wd.n_worlds) {
                    k0 = __ldg(Wd.off + wi);
                    K = __ldg(Wd.off + wi + 1) - k0;
                }
            }
            KK[lane] = uint32_t(k0) | (uint32_t(K) << 16);
            // test balls per link: swept -> the forward segment (pose, next
            // pose), a ball around both endpoint balls (it bounds every sample
            // on the segment); discrete -> the pose's own ball
            const bool has_fwd = SWEPT && valid && h < a.H - 1;
            const bool tv = SWEPT ? has_fwd : valid;
            float bx[kLinks], by[kLinks], bz[kLinks], lim2[kLinks];
#pragma unroll
            for (int l = 0; l < kLinks; ++l) {
                float cx = rx[l], cy = ry[l], cz = rz[l];
                float rr = R.link_rl[l] + margin;
                if (SWEPT) {
                    float nx = __shfl_down_sync(0xffffffffu, cx, 1);
                    float ny = __shfl_down_sync(0xffffffffu, cy, 1);
                    float nz = __shfl_down_sync(0xffffffffu, cz, 1);
                    if (lane == 31 && has_fwd)       // the halo row
                        tsph(T, min(max(R.link_ref[l], 0), R.n_spheres - 1), 32, nx, ny, nz);
                    if (!has_fwd) nx = cx, ny = cy, nz = cz;
                    const float dx = nx - cx, dy = ny - cy, dz = nz - cz;
                    cx = fmaf(0.5f, dx, cx);
                    cy = fmaf(0.5f, dy, cy);
                    cz = fmaf(0.5f, dz, cz);
                    rr += 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                }
                bx[l] = cx;
                by[l] = cy;
                bz[l] = cz;
                const float lim = rr + a.eta_w + kSlack;
                // a link without spheres: never live
                lim2[l] = (R.link_rl[l] < 0.f) ? -1.f : lim * lim;
            }
            uint32_t fm[kLinks];
#pragma unroll
            for (int l = 0; l < kLinks; ++l) fm[l] = 0u;
            const int Kw = __reduce_max_sync(0xffffffffu, tv ? K : 0);
            for (int k = 0; k < Kw; ++k) {
                const Cub c = load_cub(Wd.cub + 4 * ((k < K) ? k0 + k : 0));
                const bool kv = tv && k < K;
#pragma unroll
                for (int l = 0; l < kLinks; ++l) {
                    // squared distance from the ball centre to the box (0 inside)
                    const float dx = bx[l] - c.q2.y, dy = by[l] - c.q2.z, dz = bz[l] - c.q2.w;
                    const float px = fmaf(c.q0.x, dx, fmaf(c.q0.y, dy, c.q0.z * dz));
                    const float py = fmaf(c.q0.w, dx, fmaf(c.q1.x, dy, c.q1.y * dz));
                    const float pz = fmaf(c.q1.z, dx, fmaf(c.q1.w, dy, c.q2.x * dz));
                    const float ox = fmaxf(fabsf(px) - c.q3.x, 0.f);
                    const float oy = fmaxf(fabsf(py) - c.q3.y, 0.f);
                    const float oz = fmaxf(fabsf(pz) - c.q3.z, 0.f);
                    const float o2 = fmaf(ox, ox, fmaf(oy, oy, oz * oz));
                    const bool live = (o2 <= lim2[l]) || (!can_cull && lim2[l] >= 0.f);
                    if (kv && live) fm[l] |= 1u << k;
                }
            }
            // per pose and link: forward-segment mask (low 16 bits) and the
            // backward segment's (the previous pose's forward mask, high 16);
            // the link blocks of the item stream: item = (link, sphere, pose)
            // for every pose with a live cuboid, sphere-major -- so the pose
            // after a segment's start holds the next item of the same sphere
            int tot = 0;
#pragma unroll
            for (int l = 0; l < kLinks; ++l) {
                if (SWEPT) {
                    const uint32_t bwd = __shfl_up_sync(0xffffffffu, fm[l], 1);
                    fm[l] |= (lane > 0 && valid && h > 0 ? bwd : 0u) << 16;
                }
                WM[32 * l + lane] = fm[l];
                const uint32_t pm = __ballot_sync(0xffffffffu, fm[l] != 0u);
                const int cnt = __popc(pm);
                if (lane == l)
                    LB[l] = LinkBlk{pm, tot, cnt, cnt ? 1.f / float(cnt) : 0.f};
                tot += cnt * (R.link_start[l + 1] - R.link_start[l]);
            }
            __syncwarp();
            // the item stream, 32 items per window
            float carry_x = 0.f, carry_y = 0.f, carry_z = 0.f;
            uint32_t carry_id = 0xffffffffu;      // (sphere << 8 | pose) of the window's last item
            for (int w0 = 0; w0 < tot; w0 += 32) {
                const int idx = w0 + lane;
                const bool have = idx < tot;
                int l = 0;
#pragma unroll
                for (int q = 1; q < kLinks; ++q)
                    if (idx >= LB[q].start) l = q;
                const LinkBlk lb = LB[l];
                const int r = idx - lb.start;
                const int qs = int((float(r) + 0.5f) * lb.rcp);      // exact: r < 2^10, cnt <= 32
                const int rank = r - qs * lb.cnt;
                const int s = R.link_start[l] + qs;
                const int pl = have ? __fns(lb.pm, 0, rank + 1) : 0;
                float gx = 0.f, gy = 0.f, gz = 0.f, sx = 0.f, sy = 0.f, sz = 0.f, icost = 0.f;
                if (have) {
                    const uint32_t m = WM[32 * l + pl];
                    const uint32_t fwd = m & 0xffffu, own = fwd | (m >> 16);
                    const uint32_t kk = KK[pl];
                    const int k0i = int(kk & 0xffffu), Ki = int(kk >> 16);
                    float cx, cy, cz, nx, ny, nz, L = 0.f;
                    tsph(T, s, pl, cx, cy, cz);
                    nx = cx, ny = cy, nz = cz;
                    if (SWEPT && fwd) {
                        tsph(T, s, pl + 1, nx, ny, nz);   // pl = 31: the halo row
                        const float dx = nx - cx, dy = ny - cy, dz = nz - cz;
                        L = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    }
                    const float A = ssr[s] + a.eta_w;
                    for (uint32_t mk = own; mk; mk &= mk - 1) {
                        const int k = __ffs(mk) - 1;
                        const bool fw = (fwd >> k) & 1u;
                        const Cub c = load_cub(Wd.cub + 4 * ((k < Ki) ? k0i + k : 0));
                        // the SDF at the pose bounds each forward sample's from
                        // below (1-Lipschitz: sdf(p_j) >= sdf(c_h) - tau |c_h+1 - c_h|)
                        float sdf0 = -3.0e38f;
                        // term t = 0: the pose itself (weight 1); t = j >= 1:
                        // forward sample j, (1 - tau) kept, tau sent to the
                        // next pose -- one world_term call site
                        const int nt = (SWEPT && fw) ? nsub : 0;
                        for (int t = 0; t <= nt; ++t) {
                            float qx = cx, qy = cy, qz = cz, wo = 1.f, wsend = 0.f;
                            if (SWEPT && t > 0) {
                                const float tau = float(t) * inv_n1, omt = 1.f - tau;
                                if (can_cull && sdf0 - tau * L - A > kSlack) continue;
                                qx = fmaf(tau, nx, omt * cx);
                                qy = fmaf(tau, ny, omt * cy);
                                qz = fmaf(tau, nz, omt * cz);
                                wo = omt;
                                wsend = tau;
                            }
                            const WTerm tm = world_term(c, qx, qy, qz, A, a.eta_w, inv_eta_w, hoe_w, a.w_w);
                            if (t == 0) sdf0 = tm.sdf;
                            if (tm.s == 0.f) continue;
                            icost = fmaf(a.w_w, tm.h, icost);
                            const float so = tm.s * wo, st = tm.s * wsend;
                            gx = fmaf(so, tm.gx, gx);
                            gy = fmaf(so, tm.gy, gy);
                            gz = fmaf(so, tm.gz, gz);
                            sx = fmaf(st, tm.gx, sx);
                            sy = fmaf(st, tm.gy, sy);
                            sz = fmaf(st, tm.gz, sz);
                        }
                    }
                }
                // the tau parts of the previous item's forward samples: it is
                // the same sphere at the previous pose when that pose's segment
                // ends here (a sent part is then always non-zero only for such)
                const uint32_t id = have ? (uint32_t(s) << 8) | uint32_t(pl) : 0xffffffffu;
                float rxs = __shfl_up_sync(0xffffffffu, sx, 1);
                float rys = __shfl_up_sync(0xffffffffu, sy, 1);
                float rzs = __shfl_up_sync(0xffffffffu, sz, 1);
                uint32_t pid_ = __shfl_up_sync(0xffffffffu, id, 1);
                if (lane == 0) {
                    rxs = carry_x, rys = carry_y, rzs = carry_z;
                    pid_ = carry_id;
                }
                carry_x = __shfl_sync(0xffffffffu, sx, 31);
                carry_y = __shfl_sync(0xffffffffu, sy, 31);
                carry_z = __shfl_sync(0xffffffffu, sz, 31);
                carry_id = __shfl_sync(0xffffffffu, id, 31);
                if (SWEPT && have && pid_ + 1u == id) {
                    gx += rxs;
                    gy += rys;
                    gz += rzs;
                }
                // outputs: per pose, its items of the window in ascending lane
                // (= sphere) order, through its output state
                QR[lane] = make_float4(gx, gy, gz, icost);
                QD[lane] = uint32_t(s);
                const uint32_t grp = __match_any_sync(0xffffffffu, have ? pl : 64 + lane);
                __syncwarp();
                if (have && lane == __ffs(grp) - 1) {
                    RowOut o = RS[pl];
                    uint32_t* row = sp_cp ? a.cp + (p0 + pl) * G.wmax_cp : a.cp + (p0 + pl) * G.Wcp;
                    const bool own_p = pl >= own0;
                    for (uint32_t gm = grp; gm; gm &= gm - 1) {
                        const int j = __ffs(gm) - 1;
                        const float4 rv = QR[j];
                        const int sj = int(QD[j]);
                        o.cost += rv.w;
                        if (own_p) {
                            VAPR_TAP(a.swept ? 4 : 3, (p0 + pl) * cols + 3 * sj, rv.x + 0.f);
                            VAPR_TAP(a.swept ? 4 : 3, (p0 + pl) * cols + 3 * sj + 1, rv.y + 0.f);
                            VAPR_TAP(a.swept ? 4 : 3, (p0 + pl) * cols + 3 * sj + 2, rv.z + 0.f);
                            out_put(o, row, sp_cp, sj, rv.x, rv.y, rv.z, fcp, G.rc_cp);
                        }
                    }
                    RS[pl] = o;
                }
                __syncwarp();
            }
            {
                RowOut o = RS[lane];
                wcost = o.cost;
                if (owner) out_finish(o, a.cp + pg * G.wmax_cp, sp_cp, a.cp_mask + pg);
            }
        }


        // ---- 3. self (S)
        if (role == 1 && a.do_self) {
            TC[lane] = 0ull;
            WK[lane] = 0u;
            for (int w = 0; w < G.pmw; ++w) PM[32 * w + lane] = 0u;
            __syncwarp();
            // group pairs of the link pairs some pose has live (uniform
            // loops, lane = pose): the group-ball test; the group pairs live
            // for some pose are listed with their poses (a ballot)
            int ngl = 0, tot = 0;
            const unsigned long long ulp =
                ((unsigned long long)__reduce_or_sync(0xffffffffu, (uint32_t)(lpm >> 32)) << 32) |
                __reduce_or_sync(0xffffffffu, (uint32_t)lpm);
            for (unsigned long long ul = ulp; ul; ul &= ul - 1) {
                const int i = __ffsll((long long)ul) - 1;
                const bool lp_live = (lpm >> i) & 1ull;
                const int g1 = __ldg(&SD->lp_gp0[i + 1]);
                for (int gp = __ldg(&SD->lp_gp0[i]); gp < g1; ++gp) {
                    const int ga = __ldg(&SD->gp_a[gp]), gb = __ldg(&SD->gp_b[gp]);
                    float ax0, ay0, az0, bx0, by0, bz0;
                    tsph(T, __ldg(&SD->g_ref[ga]), lane, ax0, ay0, az0);
                    tsph(T, __ldg(&SD->g_ref[gb]), lane, bx0, by0, bz0);
                    const float dx = ax0 - bx0, dy = ay0 - by0, dz = az0 - bz0;
                    const float lim = __ldg(&SD->g_rl[ga]) + __ldg(&SD->g_rl[gb]) + m2;
                    const bool gl = lp_live && (!can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim);
                    const uint32_t bm = __ballot_sync(0xffffffffu, gl);
                    if (bm) {
                        if (lane == 0) GL[ngl] = make_uint2(uint32_t(gp) | (uint32_t(tot) << 16), bm);
                        ++ngl;
                        tot += __popc(bm);
                    }
                }
            }
            if (lane == 0) GL[ngl] = make_uint2(uint32_t(tot) << 16, 0u);
            __syncwarp();
            // items = (live group pair, pose), group-pair-major, 32 per window
            // (neighbouring lanes share the group pair's loops): each sphere
            // vs the other group's ball, then the listed sphere pairs; active
            // pairs go to the pose's pair-id bitmask
            {
                int e = 0;
                for (int w0 = 0; w0 < tot; w0 += 32) {
                    const int idx = w0 + lane;
                    const bool have = idx < tot;
                    if (have)
                        while (idx >= int(GL[e + 1].x >> 16)) ++e;
                    // explicit reconvergence after each divergent loop: the
                    // item body is the same code for every lane
                    __syncwarp();
                    const uint2 ent = GL[e];
                    const int gp = int(ent.x & 0xffffu);
                    const int pl = have ? __fns(ent.y, 0, idx - int(ent.x >> 16) + 1) : 0;
                    const int ga = __ldg(&SD->gp_a[gp]), gb = __ldg(&SD->gp_b[gp]);
                    const float rla = __ldg(&SD->g_rl[ga]), rlb = __ldg(&SD->g_rl[gb]);
                    float ax0, ay0, az0, bx0, by0, bz0;
                    tsph(T, __ldg(&SD->g_ref[ga]), pl, ax0, ay0, az0);
                    tsph(T, __ldg(&SD->g_ref[gb]), pl, bx0, by0, bz0);
                    const int sa = __ldg(&SD->g_start[ga]), na = have ? __ldg(&SD->g_n[ga]) : 0;
                    const int sb = __ldg(&SD->g_start[gb]), nb = have ? __ldg(&SD->g_n[gb]) : 0;
                    uint32_t ma = 0u, mb = 0u;
                    // each sphere vs the other group's ball
#pragma unroll 1
                    for (int u = 0; u < na; ++u) {
                        float x, y, z;
                        tsph(T, sa + u, pl, x, y, z);
                        const float dx = x - bx0, dy = y - by0, dz = z - bz0;
                        const float lim = ssr[sa + u] + rlb + m2;
                        if (!can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim) ma |= 1u << u;
                    }
                    __syncwarp();
#pragma unroll 1
                    for (int v = 0; v < nb; ++v) {
                        float x, y, z;
                        tsph(T, sb + v, pl, x, y, z);
                        const float dx = x - ax0, dy = y - ay0, dz = z - az0;
                        const float lim = ssr[sb + v] + rla + m2;
                        if (!can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim) mb |= 1u << v;
                    }
                    __syncwarp();
                    uint32_t cand = 0u;
#pragma unroll
                    for (int u = 0; u < kGMax; ++u)
                        if ((ma >> u) & 1u) cand |= mb << (kGMax * u);
                    cand &= __ldg(&SD->gp_L[gp]);
                    // the listed sphere pairs that survive (per lane)
                    for (; cand; cand &= cand - 1) {
                        const int bit = __ffs(cand) - 1;
                        const int u = (bit * 205) >> 10, v = bit - kGMax * u;  // bit / 5, bit % 5
                        float xi, yi, zi, xj, yj, zj;
                        tsph(T, sa + u, pl, xi, yi, zi);
                        tsph(T, sb + v, pl, xj, yj, zj);
                        const float dx = xi - xj, dy = yi - yj, dz = zi - zj;
                        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                        const float Rs = ssr[sa + u] + ssr[sb + v] + a.eta_s;
                        // d2 >= fl(Rs^2) => phi <= 0 (self_pair's exact early
                        // out); the rare d2 within an ulp of Rs^2 is settled by
                        // self_pair in the gather
                        if (d2 >= Rs * Rs) continue;
                        const int pid = __ldg(&SD->gp_pid[gp][bit]);
                        atomicOr(PM + 32 * (pid >> 5) + pl, 1u << (pid & 31));
                        atomicOr(WK + pl, 1u << (pid >> 5));
                        atomicOr(TC + pl, (1ull << (sa + u)) | (1ull << (sb + v)));
                    }
                    __syncwarp();
                }
            }
            // gradients, warp-cooperatively: items = (pose, touched sphere) in
            // (lane, sphere) order, 32 per window; an item sums its sphere's
            // active pairs in pair-id order (and the cost of the pairs it
            // leads, i == s), then each pose's owner takes its items' results
            // in ascending sphere order -- so the pose's self cost is summed in
            // pair-id order and its codes leave in ascending sphere order
            const unsigned long long touched = owner ? TC[lane] : 0ull;
            const int nt = __popcll(touched);
            int incl = nt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int ibase = incl - nt;
            RowOut oo{};
            uint32_t* orow = sp_ov ? a.ov + pg * G.wmax_ov : a.ov + pg * G.Wov;
            unsigned long long tb = touched;
            int cur = ibase;
            for (int w0 = 0; w0 < total; w0 += 32) {
                for (; tb && cur < w0 + 32; ++cur, tb &= tb - 1)
                    QD[cur - w0] = uint32_t(lane) | (uint32_t(__ffsll((long long)tb) - 1) << 8);
                __syncwarp();
                if (w0 + lane < total) {
                    const uint32_t d = QD[lane];
                    const int pl = int(d & 0xffu), s = int(d >> 8);
                    const uint32_t* pmp = PM + pl;
                    float gx = 0.f, gy = 0.f, gz = 0.f, c_lead = 0.f;
                    for (uint32_t wm = WK[pl]; wm; wm &= wm - 1) {
                        const int wd = __ffs(wm) - 1;
                        for (uint32_t m = pmp[wd * 32]; m; m &= m - 1) {
                            const int pid = (wd << 5) + __ffs(m) - 1;
                            const int ij = spij[pid];
                            const int i = ij & 0xff, j = ij >> 8;
                            if (i != s && j != s) continue;
                            float xi, yi, zi, xj, yj, zj;
                            tsph(T, i, pl, xi, yi, zi);
                            tsph(T, j, pl, xj, yj, zj);
                            float vx, vy, vz, c;
                            if (!self_pair(xi, yi, zi, xj, yj, zj, ssr[i] + ssr[j] + a.eta_s, a.eta_s,
                                           inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c))
                                continue;
                            const float sg = (i == s) ? -1.f : 1.f;
                            gx = fmaf(sg, vx, gx);
                            gy = fmaf(sg, vy, gy);
                            gz = fmaf(sg, vz, gz);
                            if (i == s) c_lead += c;
                        }
                    }
                    QR[lane] = make_float4(gx, gy, gz, c_lead);
                }
                __syncwarp();
                const int lo = max(ibase, w0), hi = min(incl, w0 + 32);
                for (int idx = lo; idx < hi; ++idx) {
                    const float4 rv = QR[idx - w0];
                    const int sq = int(QD[idx - w0] >> 8);
                    scost += rv.w;
                    VAPR_TAP(2, pg * cols + 3 * sq, rv.x + 0.f);
                    VAPR_TAP(2, pg * cols + 3 * sq + 1, rv.y + 0.f);
                    VAPR_TAP(2, pg * cols + 3 * sq + 2, rv.z + 0.f);
                    out_put(oo, orow, sp_ov, sq, rv.x, rv.y, rv.z, fov, G.rc_ov);
                }
                __syncwarp();
            }
            if (owner) out_finish(oo, orow, sp_ov, a.ov_mask + pg);
        }
        if (owner) {
            const float c = role == 0 ? wcost : scost;
            a.cost[pg] = a.cost_accumulate ? a.cost[pg] + c : c;
        }
        __syncwarp();
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

// World and self as two kernels over the tile rows (each keeps a small
// instruction working set; out_spheres is read twice).  The CTAs are
// persistent: as many as fit on the SMs, each warp taking 32-pose tiles from
// the context's scheduler slot.
static cudaError_t launch_role(int role, const RobotDev& R, const SelfDev* SD_dev, const SelfDev& SD,
                               const WorldsDev& W, const Fmt& fos, const Fmt& fcp, const Fmt& fov,
                               const CollisionArgs& a0, unsigned int* sched_ring,
                               unsigned int* sched_next, cudaStream_t s) {
    const long long P = (long long)a0.B * a0.H;
    CollisionArgs a = a0;
    // each launch takes the next scheduler slot of the context's ring (the
    // kernel's last CTA leaves it zeroed); kSchedSlots launches may be in flight
    const unsigned k = __atomic_fetch_add(sched_next, 1u, __ATOMIC_RELAXED) % kSchedSlots;
    a.sched = sched_ring + 2 * k;
    const CGeo G = make_cgeo(R, SD, fos, fcp, fov, a);
    if (G.rc_q == 0) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = G.cta_bytes + (size_t)kWarps * (role == 0 ? G.w_bytes : G.s_bytes);
    const bool sw = a.do_world && a.swept;
    auto kern = role == 0 ? (sw ? collision_kernel<true, 0> : collision_kernel<false, 0>)
                          : (sw ? collision_kernel<true, 1> : collision_kernel<false, 1>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kWarps, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const long long TP = 32 - G.own0;
    const long long tiles = (P + TP - 1) / TP;
    // enough CTAs for every warp to have a tile, at most the resident ones
    const long long grid = std::max(1LL, std::min<long long>((tiles + kWarps - 1) / kWarps,
                                                             (long long)sms * per_sm));
#ifdef VAPR_DEBUG_TAP
    const int tw = a.swept ? 4 : 3;
    const bool tapped = role == 0 ? tap_arm(tw, P, R.cols, s) : tap_arm(2, P, R.cols, s);
#endif
    kern<<<(unsigned)grid, 32 * kWarps, smem, s>>>(R, SD_dev, G, W, fos, fcp, fov, a);
#ifdef VAPR_DEBUG_TAP
    if (tapped) tap_disarm(role == 0 ? tw : 2, s);
#endif
    return cudaGetLastError();
}

cudaError_t launch_collision(const RobotDev& R, const SelfDev* SD_dev, const SelfDev& SD,
                             const WorldsDev& W, const Fmt& fos, const Fmt& fcp, const Fmt& fov,
                             const CollisionArgs& a0, unsigned int* sched_ring,
                             unsigned int* sched_next, cudaStream_t s) {
    const long long P = (long long)a0.B * a0.H;
    if (P <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (a0.do_world) {
        CollisionArgs aw = a0;
        aw.do_self = 0;
        e = launch_role(0, R, SD_dev, SD, W, fos, fcp, fov, aw, sched_ring, sched_next, s);
    }
    if (e == cudaSuccess && a0.do_self) {
        CollisionArgs as = a0;
        as.do_world = 0;
        as.swept = 0;
        as.cost_accumulate = a0.do_world ? 1 : a0.cost_accumulate;   // world + self
        e = launch_role(1, R, SD_dev, SD, W, fos, fcp, fov, as, sched_ring, sched_next, s);
    }
    return e;
}

cudaError_t launch_traj_reduce(const float* cost_pose, int32_t B, int32_t H, float* cost_traj,
                               cudaStream_t s) {
    if (B <= 0 || cost_traj == nullptr) return cudaSuccess;
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
