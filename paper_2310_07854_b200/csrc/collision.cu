// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients, reading packed
// out_spheres and writing packed closest_pt[_swept] / out_vec.
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// One CTA per tile of kTile consecutive poses (+1 halo pose on each side for
// the swept samples):
//  1. decode the packed rows into an FP32 shared tile (row stride 3S|1, odd),
//     tracking the largest decoded coordinate (quantisation-error bound);
//  2. broadphase.  The spheres of a link (or of a half-link group) lie in a
//     ball around a reference sphere whose radius is rigid (computed once on
//     the host) plus the quantisation-error margin.  World: per (segment,
//     link, cuboid) -- or per (pose, link, cuboid) for the discrete cost -- a
//     cull bit from a lower bound of the 1-Lipschitz box SDF at the ball
//     centre.  Self: per (pose, link pair) a ball-ball test, then per live
//     link pair its (<= 4) half-link group pairs;
//  3. the live (pose, link) world tasks and live (pose, group pair) self tasks
//     are compacted into shared task lists and processed by all threads;
//     world tasks gather the complete gradient of each sphere of the link (no
//     scatter) and OR its codes into shared packed rows (OR is
//     order-independent); self tasks mark the active sphere pairs of their
//     pose in a per-pose bitmask over canonical pair ids;
//  4. one item per (pose, touched sphere) gathers its self gradient over its
//     partners in ascending order; one thread per pose sums its costs in a
//     fixed order; the packed tiles are streamed out with coalesced stores.
//
// Culling is exact: a term is skipped only when its bound clears the
// activation distance by kSlack = 1e-4 m, orders of magnitude above the FP32
// evaluation error of the distances for workspace-scale coordinates
// (|x| < 100 m), so every skipped term would evaluate to phi <= 0, i.e. to
// exactly 0; surviving terms are accumulated in the same order with and
// without culling, so VAPR_OPT_CULL on and off give bit-identical results
// (tests/test_gpu_parity.py::test_cull_is_exact).
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kTile = 64;           // poses per CTA
constexpr int kRows = kTile + 2;    // with the two halo poses
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr float kSlack = 1e-4f;

struct Acc {
    float cost, gx, gy, gz;
};

struct Cub {
    float4 q0, q1, q2, q3;   // R^T (9), t (3), h (3), pad
};

__device__ __forceinline__ Cub load_cub(const float4* __restrict__ cub, int k) {
    return Cub{__ldg(cub + 4 * k), __ldg(cub + 4 * k + 1), __ldg(cub + 4 * k + 2),
               __ldg(cub + 4 * k + 3)};
}

// Lower bound of the box signed distance at c (the exact value outside, the
// face distance max_k(|p_k| - h_k) inside).
__device__ __forceinline__ float box_sdf_lb(const Cub& b, float cx, float cy, float cz) {
    const float dx = cx - b.q2.y, dy = cy - b.q2.z, dz = cz - b.q2.w;
    const float px = fmaf(b.q0.x, dx, fmaf(b.q0.y, dy, b.q0.z * dz));
    const float py = fmaf(b.q0.w, dx, fmaf(b.q1.x, dy, b.q1.y * dz));
    const float pz = fmaf(b.q1.z, dx, fmaf(b.q1.w, dy, b.q2.x * dz));
    const float ux = fabsf(px) - b.q3.x, uy = fabsf(py) - b.q3.y, uz = fabsf(pz) - b.q3.z;
    const float umax = fmaxf(ux, fmaxf(uy, uz));
    if (umax <= 0.f) return umax;
    const float ox = fmaxf(ux, 0.f), oy = fmaxf(uy, 0.f), oz = fmaxf(uz, 0.f);
    return sqrtf(fmaf(ox, ox, fmaf(oy, oy, oz * oz)));
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

// Append to a shared list with one atomic per warp; every lane of the warp
// must call it.  Returns the lane's slot (meaningful only when pred).
__device__ __forceinline__ int warp_append(int* counter, bool pred, int lane) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    return base + __popc(m & ((1u << lane) - 1u));
}

// Self pair (i, j), i < j: false when inactive; else the gradient
// contribution v (d cost / d c_i = -v, d cost / d c_j = +v) and the cost w h.
__device__ __forceinline__ bool self_pair(const float* crow, int i, int j, const RobotDev& R,
                                          float eta, float inv_eta, float hoe, float w, float& vx,
                                          float& vy, float& vz, float& cost) {
    const float dx = crow[3 * i] - crow[3 * j], dy = crow[3 * i + 1] - crow[3 * j + 1],
                dz = crow[3 * i + 2] - crow[3 * j + 2];
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float Rs = R.sr[i] + R.sr[j] + eta;
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

struct Smem {
    float* ctile;      // [kRows * cs], row 0 = pose p0-1
    uint32_t* wmask;   // [kRows * kLinks] bits 0-15 pose (discrete), 16-31 segment row->row+1
    uint32_t* smask;   // [kRows] live link pairs
    int2* krange;      // [kRows] cuboid range of the row's world
    int* hrow;         // [kRows] step index h, -1 when the row is absent
    float* wcost;      // [kTile * kLinks]
    unsigned long long* touched;   // [kTile] spheres with an active self pair
    int* counters;     // [8]: world tasks, self tasks, max-coordinate bits, live link
                       //      pairs, touched spheres
    uint16_t* wtask;   // [kTile * kLinks]
    uint16_t* stask;   // [kTile * n_group_pairs]
    uint16_t* l1;      // [kTile * 64] live (pose, link pair), later touched (pose, sphere)
    uint32_t* pmask;   // [kTile * PMW] active self pairs, bit = canonical pair id
    uint32_t* wcp;     // [kTile * (Wcp+1)]
    uint32_t* wov;     // [kTile * (Wov+1)]
};

__global__ void __launch_bounds__(kThreads, 2)
collision_kernel(const __grid_constant__ RobotDev R, const WorldsDev Wd, const Fmt fos,
                 const Fmt fcp, const Fmt fov, const CollisionArgs a, int Wos, int Wcp,
                 int Wov) {
    extern __shared__ float4 smem4[];
    const int cols = R.cols;
    const int cs = cols | 1;                       // odd fp32 row stride
    const long long P = (long long)a.B * a.H;
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;
    const int WcpS = Wcp + 1, WovS = Wov + 1;

    Smem sm;
    sm.wmask = reinterpret_cast<uint32_t*>(smem4);
    sm.smask = sm.wmask + kRows * kLinks;
    sm.krange = reinterpret_cast<int2*>(sm.smask + kRows + (kRows & 1));
    sm.hrow = reinterpret_cast<int*>(sm.krange + kRows);
    const int PMW = (R.n_pairs + 31) >> 5;
    sm.touched = reinterpret_cast<unsigned long long*>(sm.hrow + kRows + (kRows & 1));
    sm.wcost = reinterpret_cast<float*>(sm.touched + kTile);
    sm.counters = reinterpret_cast<int*>(sm.wcost + kTile * kLinks);
    sm.pmask = reinterpret_cast<uint32_t*>(sm.counters + 8);
    sm.wtask = reinterpret_cast<uint16_t*>(sm.pmask + kTile * PMW);
    sm.stask = sm.wtask + kTile * kLinks;
    sm.l1 = sm.stask + kTile * R.lp_gp_off[R.n_link_pairs];
    {
        const uintptr_t e = reinterpret_cast<uintptr_t>(sm.l1 + kTile * 64);
        sm.wcp = reinterpret_cast<uint32_t*>((e + 15) & ~uintptr_t(15));
    }
    sm.wov = sm.wcp + (a.do_world ? kTile * WcpS : 0);
    sm.ctile = reinterpret_cast<float*>(sm.wov + (a.do_self ? kTile * WovS : 0));

    // ---- 1. decode rows p0-1 .. p0+np into the FP32 tile; zero the outputs
    const long long r_lo = max(p0 - 1, 0LL);
    const long long r_hi = min(p0 + np + 1, P);           // exclusive
    const int row_off = int(r_lo - (p0 - 1));             // tile row of global row r_lo
    if (tid < 8) sm.counters[tid] = 0;
    __syncthreads();
    {
        const int nrows = int(r_hi - r_lo);
        const int nw = nrows * Wos;
        const uint32_t* src = a.os + r_lo * Wos;
        const int dr = kThreads / Wos, dw = kThreads % Wos;
        int r = tid / Wos, w = tid - (tid / Wos) * Wos;
        uint32_t amax = 0;
        with_pf(fos.pf, [&](auto Pc) {
            constexpr int PF = decltype(Pc)::value;
            for (int i = tid; i < nw; i += kThreads) {
                float x[PF];
                decode_word_t<PF>(__ldg(src + i), x, fos);
                float* dst = sm.ctile + (row_off + r) * cs + w * PF;
#pragma unroll
                for (int j = 0; j < PF; ++j)
                    if (w * PF + j < cols) {
                        dst[j] = x[j];
                        amax = max(amax, __float_as_uint(x[j]) & 0x7fffffffu);
                    }
                r += dr;
                w += dw;
                if (w >= Wos) {
                    w -= Wos;
                    ++r;
                }
            }
        });
        amax = __reduce_max_sync(0xffffffffu, amax);
        if ((tid & 31) == 0) atomicMax(reinterpret_cast<unsigned*>(sm.counters + 2), amax);
    }
    if (a.do_world)
        for (int i = tid; i < kTile * WcpS; i += kThreads) sm.wcp[i] = 0u;
    if (a.do_self)
        for (int i = tid; i < kTile * WovS; i += kThreads) sm.wov[i] = 0u;
    for (int i = tid; i < kTile * kLinks; i += kThreads) sm.wcost[i] = 0.f;
    if (a.do_self) {
        for (int i = tid; i < kTile * PMW; i += kThreads) sm.pmask[i] = 0u;
        if (tid < kTile) sm.touched[tid] = 0ull;
    }
    // world cuboid range and step index h of every tile row (the only 64-bit
    // divisions of the kernel: once per row)
    for (int row = tid; row < kRows; row += kThreads) {
        const long long pg = p0 - 1 + row;
        int2 kr = make_int2(0, 0);
        int hh = -1;
        if (pg >= 0 && pg < P) {
            const long long b = pg / a.H;
            hh = int(pg - b * a.H);
            if (a.do_world) {
                const int wi = __ldg(a.world_idx + b);
                if (wi >= 0 && wi < Wd.n_worlds)
                    kr = make_int2(__ldg(Wd.off + wi), __ldg(Wd.off + wi + 1));
            }
        }
        sm.krange[row] = kr;
        sm.hrow[row] = hh;
    }
    __syncthreads();

    // Quantisation margin: a decoded coordinate y of an FK value x satisfies
    // |y - x| <= 2^-(M+1) |x| + 2^-(bias+M) (half an ulp; the subnormal
    // quantum covers the bottom of the range) unless the code saturated; two
    // centres per distance and sqrt(3) per vector give the ball margin.  With
    // a saturated coordinate in the tile (|y| == max_finite) there is no bound
    // and culling is switched off for the tile.
    const float amaxf = __uint_as_float((uint32_t)sm.counters[2]);
    bool can_cull = a.cull != 0;
    float margin = 0.f;
    if (fos.kind != KIND_IDENTITY) {
        if (amaxf >= decode(fos.maxcode, fos)) can_cull = false;
        const float rel = ldexpf(1.f, -(fos.M + 1));
        const float sub = ldexpf(1.f, -((1 << (fos.E - 1)) - 1) - fos.M);
        margin = 2.f * 1.7320509f * (rel * amaxf * 1.01f + sub);
    }

    // ball of link / group `ref` in tile row `row`: (centre, radius)
    auto ball = [&](int row, int ref, float rl) {
        const float* c = sm.ctile + row * cs + 3 * ref;
        return make_float4(c[0], c[1], c[2], rl + margin);
    };

    // ---- 2b. world cull masks per (row, link); self link-pair masks per row
    const int nsub = (a.do_world && a.swept) ? a.sweep_steps : 0;
    for (int task = tid; task < kRows * kLinks; task += kThreads) {
        {
            const int row = task / kLinks, l = task - row * kLinks;
            uint32_t m = 0;
            const int2 kr = sm.krange[row];
            const int h = sm.hrow[row];
            if (a.do_world && h >= 0 && kr.y > kr.x && R.link_rl[l] >= 0.f) {
                const float4 b0 = ball(row, R.link_ref[l], R.link_rl[l]);
                if (nsub > 0) {
                    // segment row -> row+1 of the same trajectory: one ball
                    // around both endpoint balls bounds every sample
                    if (h + 1 < a.H && row + 1 < kRows && sm.hrow[row + 1] >= 0) {
                        const float4 b1 = ball(row + 1, R.link_ref[l], R.link_rl[l]);
                        const float dx = b1.x - b0.x, dy = b1.y - b0.y, dz = b1.z - b0.z;
                        const float half = 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                        const float mx = b0.x + 0.5f * dx, my = b0.y + 0.5f * dy,
                                    mz = b0.z + 0.5f * dz, rs = fmaxf(b0.w, b1.w) + half;
                        for (int k = kr.x; k < kr.y; ++k)
                            if (!can_cull ||
                                box_sdf_lb(load_cub(Wd.cub, k), mx, my, mz) - rs - a.eta_w <= kSlack)
                                m |= 1u << (16 + k - kr.x);
                    }
                } else {
                    for (int k = kr.x; k < kr.y; ++k)
                        if (!can_cull ||
                            box_sdf_lb(load_cub(Wd.cub, k), b0.x, b0.y, b0.z) - b0.w - a.eta_w <= kSlack)
                            m |= 1u << (k - kr.x);
                }
            }
            sm.wmask[task] = m;
        }
    }
    __syncthreads();

    // ---- 2c. task lists (dense, appended with one atomic per warp):
    //          live (pose, link) world tasks and live (pose, link pair) self
    //          candidates.  Loops run over whole warps so every lane votes.
    const int lane = tid & 31;
    if (a.do_world)
        for (int base = tid - lane; base < kTile * kLinks; base += kThreads) {
            const int task = base + lane;
            const int p = task / kLinks, l = task - p * kLinks;
            bool live = false;
            if (p < np) {
                const int row = p + 1, h = sm.hrow[row];
                uint32_t m;
                if (nsub > 0)
                    m = (sm.wmask[row * kLinks + l] >> 16) |
                        (h > 0 ? (sm.wmask[(row - 1) * kLinks + l] >> 16) : 0u);
                else
                    m = sm.wmask[row * kLinks + l] & 0xffffu;
                live = m != 0u;
            }
            const int slot = warp_append(sm.counters + 0, live, lane);
            if (live) sm.wtask[slot] = (uint16_t)task;
        }
    if (a.do_self)
        for (int base = tid - lane; base < kTile * R.n_link_pairs; base += kThreads) {
            const int task = base + lane;
            const int p = task / R.n_link_pairs, lp = task - p * R.n_link_pairs;
            bool live = false;
            if (p < np) {
                const int row = p + 1;
                const int la = R.lp_a[lp], lb = R.lp_b[lp];
                const float4 A4 = ball(row, R.link_ref[la], R.link_rl[la]);
                const float4 B4 = ball(row, R.link_ref[lb], R.link_rl[lb]);
                const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                live = !can_cull ||
                       sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - A4.w - B4.w - a.eta_s <= kSlack;
            }
            const int slot = warp_append(sm.counters + 3, live, lane);
            if (live) sm.l1[slot] = (uint16_t)(p * 32 + lp);
        }
    __syncthreads();
    // self level 2: the (<= 4) half-link group pairs of every live link pair
    if (a.do_self) {
        const int n1 = sm.counters[3];
        for (int base = tid - lane; base < n1 * 4; base += kThreads) {
            const int it = base + lane;
            bool live = false;
            int p = 0, g = 0;
            if (it < n1 * 4) {
                const int e = sm.l1[it >> 2];
                p = e >> 5;
                const int lp = e & 31;
                g = R.lp_gp_off[lp] + (it & 3);
                if (g < R.lp_gp_off[lp + 1]) {
                    const int row = p + 1;
                    const int ga = R.gp_a[g], gb = R.gp_b[g];
                    const float4 A4 = ball(row, R.grp_ref[ga], R.grp_rl[ga]);
                    const float4 B4 = ball(row, R.grp_ref[gb], R.grp_rl[gb]);
                    const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                    live = !can_cull ||
                           sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - A4.w - B4.w - a.eta_s <= kSlack;
                }
            }
            const int slot = warp_append(sm.counters + 1, live, lane);
            if (live) sm.stask[slot] = (uint16_t)(p * kMaxGroupPairs + g);
        }
    }
    __syncthreads();

    // ---- 3a. world tasks: all spheres of one link of one pose
    const uint32_t rc_cp = 65536u / fcp.pf + 1u, rc_ov = 65536u / fov.pf + 1u;
    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const float inv_n1 = 1.f / float(nsub + 1);
    const int n_wtask = sm.counters[0], n_stask = sm.counters[1];
    for (int t = tid; t < n_wtask; t += kThreads) {
        const int task = sm.wtask[t];
        const int p = task / kLinks, l = task - p * kLinks;
        const int row = p + 1, h = sm.hrow[row];
        const int k0 = sm.krange[row].x;
        uint32_t m_own, m_fwd = 0, m_bwd = 0;
        if (nsub > 0) {
            m_fwd = (h < a.H - 1) ? (sm.wmask[row * kLinks + l] >> 16) : 0u;
            m_bwd = (h > 0) ? (sm.wmask[(row - 1) * kLinks + l] >> 16) : 0u;
            m_own = m_fwd | m_bwd;     // a segment ball contains both endpoint balls
        } else {
            m_own = sm.wmask[row * kLinks + l] & 0xffffu;
        }
        const float* crow = sm.ctile + row * cs;
        uint32_t* orow = sm.wcp + p * WcpS;
        float lcost = 0.f;
        for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
            const float cx = crow[3 * s], cy = crow[3 * s + 1], cz = crow[3 * s + 2];
            const float A = R.sr[s] + a.eta_w;
            Acc acc{0.f, 0.f, 0.f, 0.f};
            for (uint32_t m = m_own; m; m &= m - 1)
                world_term(load_cub(Wd.cub, k0 + __ffs(m) - 1), cx, cy, cz, A, a.eta_w, inv_eta_w,
                           hoe_w, a.w_w, 1.f, 1.f, acc);
            if (m_fwd) {                // samples of segment (h, h+1): cost + (1-tau) grad
                const float* nrow = crow + cs;
                const float nx = nrow[3 * s], ny = nrow[3 * s + 1], nz = nrow[3 * s + 2];
                for (int j = 1; j <= nsub; ++j) {
                    const float tau = float(j) * inv_n1, omt = 1.f - tau;
                    const float sx = fmaf(tau, nx, omt * cx), sy = fmaf(tau, ny, omt * cy),
                                sz = fmaf(tau, nz, omt * cz);
                    for (uint32_t m = m_fwd; m; m &= m - 1)
                        world_term(load_cub(Wd.cub, k0 + __ffs(m) - 1), sx, sy, sz, A, a.eta_w,
                                   inv_eta_w, hoe_w, a.w_w, 1.f, omt, acc);
                }
            }
            if (m_bwd) {                // samples of segment (h-1, h): tau grad only
                const float* prow = crow - cs;
                const float qx = prow[3 * s], qy = prow[3 * s + 1], qz = prow[3 * s + 2];
                for (int j = 1; j <= nsub; ++j) {
                    const float tau = float(j) * inv_n1, omt = 1.f - tau;
                    const float sx = fmaf(tau, cx, omt * qx), sy = fmaf(tau, cy, omt * qy),
                                sz = fmaf(tau, cz, omt * qz);
                    for (uint32_t m = m_bwd; m; m &= m - 1)
                        world_term(load_cub(Wd.cub, k0 + __ffs(m) - 1), sx, sy, sz, A, a.eta_w,
                                   inv_eta_w, hoe_w, a.w_w, 0.f, tau, acc);
                }
            }
            lcost += acc.cost;
            or_code(orow, 3 * s + 0, acc.gx + 0.f, fcp, rc_cp);
            or_code(orow, 3 * s + 1, acc.gy + 0.f, fcp, rc_cp);
            or_code(orow, 3 * s + 2, acc.gz + 0.f, fcp, rc_cp);
        }
        sm.wcost[task] = lcost;
    }
    // ---- 3b. self tasks: the active sphere pairs of one group pair of one pose
    for (int t = tid; t < n_stask; t += kThreads) {
        const int task = sm.stask[t];
        const int p = task / kMaxGroupPairs, g = task - p * kMaxGroupPairs;
        const float* crow = sm.ctile + (p + 1) * cs;
        for (int k = R.gp_off[g]; k < R.gp_off[g + 1]; ++k) {
            const int pid = R.gp_pid[k];
            const int i = R.pair_i[pid], j = R.pair_j[pid];
            float vx, vy, vz, c;
            if (self_pair(crow, i, j, R, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c)) {
                atomicOr(sm.pmask + p * PMW + (pid >> 5), 1u << (pid & 31));
                atomicOr(sm.touched + p, (1ull << i) | (1ull << j));
            }
        }
    }
    __syncthreads();

    // ---- 4a. self gradients: one item per (pose, touched sphere), gathered
    //          over the pose's active pairs in canonical id order, which for a
    //          fixed sphere s is its partners in ascending order (independent
    //          of culling and of the task order).
    if (a.do_self) {
        for (int base = tid - lane; base < np * 64; base += kThreads) {
            const int it = base + lane;
            const int p = it >> 6, s = it & 63;
            const bool live = it < np * 64 && ((sm.touched[p] >> s) & 1ull);
            const int slot = warp_append(sm.counters + 4, live, lane);
            if (live) sm.l1[slot] = (uint16_t)it;        // l1 is free again
        }
        __syncthreads();
        const int nt = sm.counters[4];
        for (int t = tid; t < nt; t += kThreads) {
            const int it = sm.l1[t];
            const int p = it >> 6, s = it & 63;
            const float* crow = sm.ctile + (p + 1) * cs;
            const uint32_t* pm = sm.pmask + p * PMW;
            float gx = 0.f, gy = 0.f, gz = 0.f;
            for (int wd = 0; wd < PMW; ++wd)
                for (uint32_t m = pm[wd]; m; m &= m - 1) {
                    const int pid = (wd << 5) + __ffs(m) - 1;
                    const int i = R.pair_i[pid], j = R.pair_j[pid];
                    if (i != s && j != s) continue;
                    float vx, vy, vz, c;
                    self_pair(crow, i, j, R, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c);
                    const float sg = (i == s) ? -1.f : 1.f;
                    gx = fmaf(sg, vx, gx);
                    gy = fmaf(sg, vy, gy);
                    gz = fmaf(sg, vz, gz);
                }
            uint32_t* orow = sm.wov + p * WovS;
            or_code(orow, 3 * s + 0, gx + 0.f, fov, rc_ov);
            or_code(orow, 3 * s + 1, gy + 0.f, fov, rc_ov);
            or_code(orow, 3 * s + 2, gz + 0.f, fov, rc_ov);
        }
    }
    // ---- 4b. per-pose cost: world per link, then the active self pairs in id order
    if (tid < np) {
        const int p = tid;
        float cost = 0.f;
        for (int l = 0; l < kLinks; ++l) cost += sm.wcost[p * kLinks + l];
        if (a.do_self && sm.touched[p]) {
            const float* crow = sm.ctile + (p + 1) * cs;
            const uint32_t* pm = sm.pmask + p * PMW;
            float scost = 0.f;
            for (int wd = 0; wd < PMW; ++wd)
                for (uint32_t m = pm[wd]; m; m &= m - 1) {
                    const int pid = (wd << 5) + __ffs(m) - 1;
                    float vx, vy, vz, c;
                    self_pair(crow, R.pair_i[pid], R.pair_j[pid], R, a.eta_s, inv_eta_s, hoe_s,
                              a.w_s, vx, vy, vz, c);
                    scost += c;
                }
            cost += scost;
        }
        a.cost[p0 + p] = cost;
    }
    __syncthreads();

    // ---- 5. coalesced packed stores
    if (a.do_world) {
        const int n = np * Wcp;
        uint32_t* dst = a.cp + p0 * Wcp;
        const int dr = kThreads / Wcp, dw = kThreads % Wcp;
        int r = tid / Wcp, w = tid - (tid / Wcp) * Wcp;
        for (int i = tid; i < n; i += kThreads) {
            __stcs(dst + i, sm.wcp[r * WcpS + w]);
            r += dr;
            w += dw;
            if (w >= Wcp) {
                w -= Wcp;
                ++r;
            }
        }
    }
    if (a.do_self) {
        const int n = np * Wov;
        uint32_t* dst = a.ov + p0 * Wov;
        const int dr = kThreads / Wov, dw = kThreads % Wov;
        int r = tid / Wov, w = tid - (tid / Wov) * Wov;
        for (int i = tid; i < n; i += kThreads) {
            __stcs(dst + i, sm.wov[r * WovS + w]);
            r += dr;
            w += dw;
            if (w >= Wov) {
                w -= Wov;
                ++r;
            }
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

size_t collision_smem(const RobotDev& R, bool do_world, bool do_self, int Wcp, int Wov) {
    size_t b = sizeof(uint32_t) * (kRows * kLinks + kRows + (kRows & 1));   // wmask, smask
    b += sizeof(int2) * kRows + sizeof(int) * kRows;                  // krange, hrow
    b += sizeof(int) * (kRows & 1) + sizeof(unsigned long long) * kTile;   // touched
    b += sizeof(float) * kTile * kLinks;                              // wcost
    b += sizeof(int) * 8;                                             // counters
    b += sizeof(uint32_t) * kTile * ((R.n_pairs + 31) >> 5);          // pmask
    b += sizeof(uint16_t) * (kTile * kLinks + kTile * R.lp_gp_off[R.n_link_pairs] + kTile * 64);
    b = (b + 15) & ~(size_t)15;
    if (do_world) b += sizeof(uint32_t) * kTile * (Wcp + 1);
    if (do_self) b += sizeof(uint32_t) * kTile * (Wov + 1);
    b += sizeof(float) * (size_t)kRows * (R.cols | 1);                // ctile
    return b + 16;
}

}  // namespace

cudaError_t launch_collision(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                             const Fmt& fcp, const Fmt& fov, const CollisionArgs& a,
                             cudaStream_t s) {
    const long long P = (long long)a.B * a.H;
    if (P <= 0) return cudaSuccess;
    const int Wos = row_words_of(fos, R.cols);
    const int Wcp = a.do_world ? row_words_of(fcp, R.cols) : 0;
    const int Wov = a.do_self ? row_words_of(fov, R.cols) : 0;
    const size_t smem = collision_smem(R, a.do_world, a.do_self, Wcp, Wov);
    cudaError_t e = cudaFuncSetAttribute(collision_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (P + kTile - 1) / kTile;
    collision_kernel<<<(unsigned)grid, kThreads, smem, s>>>(R, W, fos, fcp, fov, a, Wos, Wcp,
                                                            Wov);
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
