// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients, reading packed
// out_spheres and writing packed closest_pt[_swept] / out_vec.
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// Tile = kTile consecutive poses (+1 halo pose on each side for the swept
// samples).
//  1. decode the packed rows into an FP32 shared tile (row stride 3S|1, odd);
//  2. broadphase, per (pose, link): a bounding sphere of the link's spheres;
//     per (pose, link, cuboid) and (segment, link, cuboid) a cull bit from the
//     1-Lipschitz box SDF at the bounding-sphere centre; per pose a mask of
//     the link pairs whose bounding spheres come within eta_self;
//  3. narrowphase, one lane per (sphere, pose) item, warps sphere-major (the
//     sphere's radius, link and partner list are warp-uniform, read from the
//     __grid_constant__ robot as broadcasts); each item gathers its complete
//     gradient (no scatter), encodes its 3 codes and ORs the non-zero ones into
//     shared packed rows (OR is order-independent: deterministic);
//  4. per-pose costs reduced in a fixed order; packed tiles streamed out.
//
// Culling is exact: a (link, cuboid) or (link, link) combination is skipped
// only when its bound clears the activation distance by kSlack = 1e-4 m,
// orders of magnitude above the FP32 evaluation error of the distances for
// workspace-scale coordinates (|x| < 100 m), so every skipped term would have
// evaluated to phi <= 0, i.e. exactly 0.  The surviving terms are accumulated
// in the same order as without culling, so VAPR_OPT_CULL on and off give
// bit-identical results (checked by tests/test_gpu_parity.py).
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

// Box signed distance at c (for the broadphase bound).
__device__ __forceinline__ float box_sdf(const Cub& b, float cx, float cy, float cz) {
    const float dx = cx - b.q2.y, dy = cy - b.q2.z, dz = cz - b.q2.w;
    const float px = fmaf(b.q0.x, dx, fmaf(b.q0.y, dy, b.q0.z * dz));
    const float py = fmaf(b.q0.w, dx, fmaf(b.q1.x, dy, b.q1.y * dz));
    const float pz = fmaf(b.q1.z, dx, fmaf(b.q1.w, dy, b.q2.x * dz));
    const float ux = fabsf(px) - b.q3.x, uy = fabsf(py) - b.q3.y, uz = fabsf(pz) - b.q3.z;
    const float ox = fmaxf(ux, 0.f), oy = fmaxf(uy, 0.f), oz = fmaxf(uz, 0.f);
    return sqrtf(fmaf(ox, ox, fmaf(oy, oy, oz * oz))) + fminf(fmaxf(ux, fmaxf(uy, uz)), 0.f);
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

__device__ __forceinline__ void or_code(uint32_t* row, int e, float v, const Fmt& f) {
    if (__float_as_uint(v) == 0u) return;          // +0 -> code 0 (the sparse common case)
    const uint32_t c = encode(v, f);
    const int w = e / f.pf;
    atomicOr(row + w, c << ((e - w * f.pf) * f.t));
}

__global__ void __launch_bounds__(kThreads, 2)
collision_kernel(const __grid_constant__ RobotDev R, const WorldsDev Wd, const Fmt fos,
                 const Fmt fcp, const Fmt fov, const CollisionArgs a, int Wos, int Wcp,
                 int Wov) {
    extern __shared__ float4 smem4[];
    const int S = R.n_spheres;
    const int cols = R.cols;
    const int cs = cols | 1;                       // odd fp32 row stride
    const long long P = (long long)a.B * a.H;
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    // ---- shared layout (float4 first for alignment)
    float4* lb = smem4;                                          // [kRows * 9]
    uint32_t* wmask = reinterpret_cast<uint32_t*>(lb + kRows * kLinks);   // [kRows * 9]
    uint32_t* smask = wmask + kRows * kLinks;                   // [kRows]
    int2* krange = reinterpret_cast<int2*>(smask + kRows);       // [kRows]
    float* ctile = reinterpret_cast<float*>(krange + kRows);     // [kRows * cs], row 0 = p0-1
    float* cpart = ctile + kRows * cs;                           // [S * kTile]
    uint32_t* wcp = reinterpret_cast<uint32_t*>(cpart + S * kTile);   // [kTile * (Wcp+1)]
    uint32_t* wov = wcp + (a.do_world ? kTile * (Wcp + 1) : 0);       // [kTile * (Wov+1)]
    const int WcpS = Wcp + 1, WovS = Wov + 1;

    // ---- 1. decode rows p0-1 .. p0+np into the FP32 tile; zero the outputs
    const long long r_lo = max(p0 - 1, 0LL);
    const long long r_hi = min(p0 + np + 1, P);           // exclusive
    const int row_off = int(r_lo - (p0 - 1));             // tile row of global row r_lo
    {
        const int nrows = int(r_hi - r_lo);
        const int nw = nrows * Wos;
        const uint32_t* src = a.os + r_lo * Wos;
        const int dr = kThreads / Wos, dw = kThreads % Wos;
        int r = tid / Wos, w = tid - (tid / Wos) * Wos;
        with_pf(fos.pf, [&](auto Pc) {
            constexpr int PF = decltype(Pc)::value;
            for (int i = tid; i < nw; i += kThreads) {
                float x[PF];
                decode_word_t<PF>(__ldg(src + i), x, fos);
                float* dst = ctile + (row_off + r) * cs + w * PF;
#pragma unroll
                for (int j = 0; j < PF; ++j)
                    if (w * PF + j < cols) dst[j] = x[j];
                r += dr;
                w += dw;
                if (w >= Wos) {
                    w -= Wos;
                    ++r;
                }
            }
        });
    }
    if (a.do_world)
        for (int i = tid; i < kTile * WcpS; i += kThreads) wcp[i] = 0u;
    if (a.do_self)
        for (int i = tid; i < kTile * WovS; i += kThreads) wov[i] = 0u;
    // world cuboid range of every tile row
    for (int row = tid; row < kRows; row += kThreads) {
        const long long pg = p0 - 1 + row;
        int2 kr = make_int2(0, 0);
        if (a.do_world && pg >= 0 && pg < P) {
            const int wi = __ldg(a.world_idx + pg / a.H);
            if (wi >= 0 && wi < Wd.n_worlds) kr = make_int2(__ldg(Wd.off + wi), __ldg(Wd.off + wi + 1));
        }
        krange[row] = kr;
    }
    __syncthreads();

    // ---- 2a. link bounding spheres (rows present in the tile)
    for (int task = tid; task < kRows * kLinks; task += kThreads) {
        const int row = task / kLinks, l = task - row * kLinks;
        const long long pg = p0 - 1 + row;
        if (pg < 0 || pg >= P) continue;
        const float* c = ctile + row * cs;
        const int s0 = R.link_start[l], s1 = R.link_start[l + 1];
        float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
        for (int s = s0; s < s1; ++s)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], c[3 * s + k]);
                hi[k] = fmaxf(hi[k], c[3 * s + k]);
            }
        const float mx = 0.5f * (lo[0] + hi[0]), my = 0.5f * (lo[1] + hi[1]),
                    mz = 0.5f * (lo[2] + hi[2]);
        float rad = -1.f;                  // empty link: never active
        for (int s = s0; s < s1; ++s) {
            const float dx = c[3 * s] - mx, dy = c[3 * s + 1] - my, dz = c[3 * s + 2] - mz;
            rad = fmaxf(rad, sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) + R.sr[s]);
        }
        lb[row * kLinks + l] = make_float4(mx, my, mz, rad);
    }
    __syncthreads();

    // ---- 2b. world cull masks (bits 0-15: pose, 16-31: segment row->row+1)
    //          and self link-pair masks
    const int nsub = (a.do_world && a.swept) ? a.sweep_steps : 0;
    for (int task = tid; task < kRows * kLinks + kRows; task += kThreads) {
        if (task < kRows * kLinks) {
            const int row = task / kLinks, l = task - row * kLinks;
            const long long pg = p0 - 1 + row;
            uint32_t m = 0;
            const int2 kr = krange[row];
            if (a.do_world && pg >= 0 && pg < P && kr.y > kr.x) {
                const float4 b0 = lb[row * kLinks + l];
                const bool seg = nsub > 0 && row + 1 < kRows && pg + 1 < P &&
                                 (pg + 1) % a.H != 0;
                float4 bs = b0;
                if (seg) {
                    const float4 b1 = lb[(row + 1) * kLinks + l];
                    const float dx = b1.x - b0.x, dy = b1.y - b0.y, dz = b1.z - b0.z;
                    const float half = 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    bs = make_float4(b0.x + 0.5f * dx, b0.y + 0.5f * dy, b0.z + 0.5f * dz,
                                     fmaxf(b0.w, b1.w) + half);
                }
                if (b0.w >= 0.f) {
                    for (int k = kr.x; k < kr.y; ++k) {
                        const Cub cb = load_cub(Wd.cub, k);
                        const int bit = k - kr.x;
                        if (!a.cull || box_sdf(cb, b0.x, b0.y, b0.z) - b0.w - a.eta_w <= kSlack)
                            m |= 1u << bit;
                        if (seg && (!a.cull ||
                                    box_sdf(cb, bs.x, bs.y, bs.z) - bs.w - a.eta_w <= kSlack))
                            m |= 1u << (16 + bit);
                    }
                }
            }
            wmask[task] = m;
        } else {
            const int row = task - kRows * kLinks;
            const long long pg = p0 - 1 + row;
            uint32_t m = 0;
            if (a.do_self && pg >= 0 && pg < P) {
                for (int la = 0; la < kLinks; ++la)
                    for (int lbk = la; lbk < kLinks; ++lbk) {
                        const int idx = R.lp_index[la][lbk];
                        if (idx < 0) continue;
                        const float4 A4 = lb[row * kLinks + la], B4 = lb[row * kLinks + lbk];
                        const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                        const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                        if (!a.cull || d - A4.w - B4.w - a.eta_s <= kSlack) m |= 1u << idx;
                    }
            }
            smask[row] = m;
        }
    }
    __syncthreads();

    // ---- 3. narrowphase items (sphere s, pose p), sphere-major per warp
    const int lane = tid & 31, warp = tid >> 5;
    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    constexpr int halves = kTile / 32;
    const int n_tasks = S * halves;
    const float inv_n1 = 1.f / float(nsub + 1);
    for (int task = warp; task < n_tasks; task += kWarps) {
        const int s = task / halves;
        const int p = (task - s * halves) * 32 + lane;
        if (p >= np) continue;
        const int row = p + 1;
        const long long pg = p0 + p;
        const int h = int(pg % a.H);
        const float* crow = ctile + row * cs;
        const float cx = crow[3 * s], cy = crow[3 * s + 1], cz = crow[3 * s + 2];
        const float r = R.sr[s];
        int ls = 0;
#pragma unroll
        for (int l = 1; l < kLinks; ++l) ls += (s >= R.link_start[l]) ? 1 : 0;
        float cost = 0.f;
        if (a.do_world) {
            Acc acc{0.f, 0.f, 0.f, 0.f};
            const int k0 = krange[row].x;
            const float A = r + a.eta_w;
            uint32_t own = wmask[row * kLinks + ls] & 0xffffu;
            while (own) {
                const int bit = __ffs(own) - 1;
                own &= own - 1;
                world_term(load_cub(Wd.cub, k0 + bit), cx, cy, cz, A, a.eta_w, inv_eta_w, hoe_w,
                           a.w_w, 1.f, 1.f, acc);
            }
            if (nsub > 0) {
                if (h < a.H - 1) {          // samples of segment (h, h+1): cost + (1-tau) grad
                    const uint32_t segm = wmask[row * kLinks + ls] >> 16;
                    if (segm) {
                        const float* nrow = crow + cs;
                        const float nx = nrow[3 * s], ny = nrow[3 * s + 1], nz = nrow[3 * s + 2];
                        for (int j = 1; j <= nsub; ++j) {
                            const float tau = float(j) * inv_n1, omt = 1.f - tau;
                            const float sx = fmaf(tau, nx, omt * cx), sy = fmaf(tau, ny, omt * cy),
                                        sz = fmaf(tau, nz, omt * cz);
                            uint32_t m = segm;
                            while (m) {
                                const int bit = __ffs(m) - 1;
                                m &= m - 1;
                                world_term(load_cub(Wd.cub, k0 + bit), sx, sy, sz, A, a.eta_w,
                                           inv_eta_w, hoe_w, a.w_w, 1.f, omt, acc);
                            }
                        }
                    }
                }
                if (h > 0) {                // samples of segment (h-1, h): tau grad only
                    const uint32_t segm = wmask[(row - 1) * kLinks + ls] >> 16;
                    if (segm) {
                        const float* prow = crow - cs;
                        const float qx = prow[3 * s], qy = prow[3 * s + 1], qz = prow[3 * s + 2];
                        for (int j = 1; j <= nsub; ++j) {
                            const float tau = float(j) * inv_n1, omt = 1.f - tau;
                            const float sx = fmaf(tau, cx, omt * qx), sy = fmaf(tau, cy, omt * qy),
                                        sz = fmaf(tau, cz, omt * qz);
                            uint32_t m = segm;
                            while (m) {
                                const int bit = __ffs(m) - 1;
                                m &= m - 1;
                                world_term(load_cub(Wd.cub, k0 + bit), sx, sy, sz, A, a.eta_w,
                                           inv_eta_w, hoe_w, a.w_w, 0.f, tau, acc);
                            }
                        }
                    }
                }
            }
            cost += acc.cost;
            uint32_t* orow = wcp + p * WcpS;
            or_code(orow, 3 * s + 0, acc.gx + 0.f, fcp);
            or_code(orow, 3 * s + 1, acc.gy + 0.f, fcp);
            or_code(orow, 3 * s + 2, acc.gz + 0.f, fcp);
        }
        if (a.do_self) {
            float gx = 0.f, gy = 0.f, gz = 0.f, sc = 0.f;
            const uint32_t lm = smask[row];
            for (int l2 = 0; l2 < kLinks; ++l2) {
                const int idx = R.lp_index[ls][l2];
                if (idx < 0 || !((lm >> idx) & 1u)) continue;
                const int j0 = R.adj_link_off[s][l2], j1 = R.adj_link_off[s][l2 + 1];
                for (int jj = j0; jj < j1; ++jj) {
                    const int o = R.adj[jj];
                    const float dx = cx - crow[3 * o], dy = cy - crow[3 * o + 1],
                                dz = cz - crow[3 * o + 2];
                    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    const float Rs = r + R.sr[o] + a.eta_s;
                    // sqrt(fl(Rs^2)) rounds back to Rs and sqrt is monotone, so
                    // d2 >= fl(Rs^2) implies fl(sqrt(d2)) >= Rs, i.e. phi <= 0: exact.
                    if (d2 >= Rs * Rs) continue;
                    const float d = sqrtf(d2);
                    const float phi = Rs - d;
                    if (phi <= 0.f) continue;
                    float hh, dh;
                    if (phi <= a.eta_s) {
                        hh = phi * phi * hoe_s;
                        dh = phi * inv_eta_s;
                    } else {
                        hh = phi - 0.5f * a.eta_s;
                        dh = 1.f;
                    }
                    float ux, uy, uz;
                    if (d > 0.f) {
                        const float inv = 1.f / d;
                        ux = dx * inv;
                        uy = dy * inv;
                        uz = dz * inv;
                    } else {                 // coincident centres: (1,0,0) from the lower index
                        ux = (s < o) ? 1.f : -1.f;
                        uy = uz = 0.f;
                    }
                    const float k = -a.w_s * dh;
                    gx = fmaf(k, ux, gx);
                    gy = fmaf(k, uy, gy);
                    gz = fmaf(k, uz, gz);
                    if (s < o) sc = fmaf(a.w_s, hh, sc);     // each pair's cost counted once
                }
            }
            cost += sc;
            uint32_t* orow = wov + p * WovS;
            or_code(orow, 3 * s + 0, gx + 0.f, fov);
            or_code(orow, 3 * s + 1, gy + 0.f, fov);
            or_code(orow, 3 * s + 2, gz + 0.f, fov);
        }
        cpart[s * kTile + p] = cost;
    }
    __syncthreads();

    // ---- 4. per-pose cost (fixed order) and coalesced packed stores
    if (tid < np) {
        float c = 0.f;
        for (int s = 0; s < S; ++s) c += cpart[s * kTile + tid];
        a.cost[p0 + tid] = c;
    }
    if (a.do_world) {
        const int n = np * Wcp;
        uint32_t* dst = a.cp + p0 * Wcp;
        const int dr = kThreads / Wcp, dw = kThreads % Wcp;
        int r = tid / Wcp, w = tid - (tid / Wcp) * Wcp;
        for (int i = tid; i < n; i += kThreads) {
            __stcs(dst + i, wcp[r * WcpS + w]);
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
            __stcs(dst + i, wov[r * WovS + w]);
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

}  // namespace

cudaError_t launch_collision(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                             const Fmt& fcp, const Fmt& fov, const CollisionArgs& a,
                             cudaStream_t s) {
    const long long P = (long long)a.B * a.H;
    if (P <= 0) return cudaSuccess;
    const int Wos = row_words_of(fos, R.cols);
    const int Wcp = a.do_world ? row_words_of(fcp, R.cols) : 0;
    const int Wov = a.do_self ? row_words_of(fov, R.cols) : 0;
    const int cs = R.cols | 1;
    size_t smem = sizeof(float4) * kRows * kLinks + sizeof(uint32_t) * (kRows * kLinks + kRows) +
                  sizeof(int2) * kRows +
                  sizeof(float) * ((size_t)kRows * cs + (size_t)R.n_spheres * kTile);
    if (a.do_world) smem += sizeof(uint32_t) * kTile * (Wcp + 1);
    if (a.do_self) smem += sizeof(uint32_t) * kTile * (Wov + 1);
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
