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
//  0. stage in shared memory everything that lanes index divergently: the
//     robot's pair / group tables, sphere radii, and the cuboids of the
//     tile's worlds (constant-bank reads serialise on divergent addresses);
//  1. load the packed rows with all loads in flight, decode them into an FP32
//     tile (row stride 3S|1, odd), track the largest decoded coordinate;
//  2. broadphase.  The spheres of a link (or of a half-link group) lie in a
//     ball around a reference sphere whose radius is rigid (computed once on
//     the host) plus the quantisation-error margin.  World: per (segment,
//     link, cuboid) -- or per (pose, link, cuboid) for the discrete cost -- a
//     cull bit from a lower bound of the 1-Lipschitz box SDF at the ball
//     centre.  Self: per (pose, link pair) a ball-ball test, then per live
//     link pair its (<= 4) half-link group pairs;
//  3. the live (pose, link) world tasks and live (pose, group pair) self tasks
//     are compacted into dense shared lists (one atomic per warp) and
//     processed by all threads; world tasks gather the complete gradient of
//     each sphere of the link (no scatter) and OR its codes into shared packed
//     rows (OR is order-independent); self tasks mark the active sphere pairs
//     of their pose in a per-pose bitmask over canonical pair ids;
//  4. one item per (pose, touched sphere) gathers its self gradient over the
//     active pairs in id order; one thread per pose sums its costs in a fixed
//     order; the packed tiles are streamed out with coalesced stores.
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

namespace vapr {

namespace {

constexpr int kTile = 32;           // poses per tile
constexpr int kRows = kTile + 2;    // with the two halo poses
constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr float kSlack = 1e-4f;

struct Acc {
    float cost, gx, gy, gz;
};

#ifdef VAPR_PHASES
__device__ unsigned long long g_phase_cycles[16];
#endif

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

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

// Shared-memory carve-up and derived sizes, computed once on the host and
// passed by value (kernel-parameter space): nothing of it is recomputed in
// the tile loop.
struct Geo {
    int Wos, Wcp, Wov;         // packed row words
    int Qos;                   // 16-byte groups per out_spheres row
    int cs;                    // FP32 tile row stride (floats)
    int pmw;                   // words of the per-pose active-pair mask
    int ngp;                   // half-link group pairs
    int npairs, nlp, S;
    uint32_t rc_cp, rc_ov;     // e / pf reciprocals (16-bit fixed point)
    // byte offsets into dynamic shared memory
    unsigned stage, ctile, lball, scub, kcache, wmask, hrow, krange, wcost, counters, pmask, touched, spm, sr,
        rl, ref, pij, gpid, gpoff, gpab, lpab, lpgp, l1, stask, wtask, wcp, wov, total;
};

inline int tile_stride(int cols, int Wos, int pf) {
    int cs = ((cols + 3) & ~3);
    if (cs < Wos * pf) cs = Wos * pf;
    if (cs % 32 == 0) cs += 4;           // rows of one column spread over banks
    return cs;
}

Geo make_geo(const RobotDev& R, const Fmt& fos, const Fmt& fcp, const Fmt& fov, int do_world,
             int do_self) {
    Geo g{};
    g.Wos = row_words_of(fos, R.cols);
    g.Wcp = do_world ? row_words_of(fcp, R.cols) : 0;
    g.Wov = do_self ? row_words_of(fov, R.cols) : 0;
    g.Qos = g.Wos / 4;
    g.cs = tile_stride(R.cols, g.Wos, fos.pf);
    g.pmw = (R.n_pairs + 31) >> 5;
    g.ngp = R.lp_gp_off[R.n_link_pairs];
    g.npairs = R.n_pairs;
    g.nlp = R.n_link_pairs;
    g.S = R.n_spheres;
    g.rc_cp = 65536u / fcp.pf + 1u;
    g.rc_ov = 65536u / fov.pf + 1u;
    unsigned o = 0;
    auto take = [&](unsigned bytes, unsigned align) {
        o = (o + align - 1) / align * align;
        const unsigned at = o;
        o += bytes;
        return at;
    };
    g.stage = take(4u * kRows * g.Wos + 16u * kRows, 16);      // + world ids (kRows ints)
    g.ctile = take(4u * kRows * g.cs, 16);
    g.lball = take(16u * kRows * kLinks, 16);
    g.scub = take(64u * kMaxCuboids * 2, 16);                  // 2-world cuboid cache
    g.kcache = take(4u * kRows, 4);
    g.touched = take(8u * kTile + 4u * kTile, 8);
    g.krange = take(8u * kRows, 8);
    g.wmask = take(4u * kRows * kLinks, 4);
    g.hrow = take(4u * kRows, 4);
    g.wcost = take(4u * kTile * kMaxSpheres, 4);
    g.counters = take(4u * 8, 4);
    g.pmask = take(4u * kTile * g.pmw, 4);
    g.spm = take(do_self ? 4u * g.S * g.pmw : 0u, 4);
    g.sr = take(4u * kMaxSpheres, 4);
    g.rl = take(4u * 3 * kLinks, 4);
    g.ref = take(4u * 3 * kLinks, 4);
    g.pij = take(2u * g.npairs, 2);
    g.gpid = take(2u * g.npairs, 2);
    g.gpoff = take(2u * (kMaxGroupPairs + 1), 2);
    g.gpab = take(2u * kMaxGroupPairs, 2);
    g.lpab = take(2u * 33, 2);
    g.lpgp = take(2u * 33, 2);
    g.l1 = take(2u * kTile * 64, 2);
    g.stask = take(2u * kTile * (g.ngp > 0 ? g.ngp : 1), 2);
    g.wtask = take(2u * kTile * kMaxSpheres + kMaxSpheres, 2);   // + sphere -> link table
    g.wcp = take(4u * kTile * g.Wcp, 16);
    g.wov = take(4u * kTile * g.Wov, 16);
    g.total = o + 16;
    return g;
}

__global__ void __launch_bounds__(kThreads, 4)
collision_kernel(const __grid_constant__ RobotDev R, const __grid_constant__ Geo G,
                 const WorldsDev Wd, const Fmt fos, const Fmt fcp, const Fmt fov,
                 const CollisionArgs a) {
    extern __shared__ float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    uint32_t* stage = reinterpret_cast<uint32_t*>(base + G.stage);    // packed rows of one tile
    int* swid = reinterpret_cast<int*>(stage + kRows * G.Wos);        // world index per row
    float* ctile = reinterpret_cast<float*>(base + G.ctile);
    float4* lball = reinterpret_cast<float4*>(base + G.lball);        // link ball per (row, link)
    Cub* scub = reinterpret_cast<Cub*>(base + G.scub);                // cuboids of <= 2 worlds
    int* kcache = reinterpret_cast<int*>(base + G.kcache);            // row's cache base, -1: global
    unsigned long long* touched = reinterpret_cast<unsigned long long*>(base + G.touched);
    uint32_t* pwm = reinterpret_cast<uint32_t*>(touched + kTile);   // [kTile] non-zero pmask words
    int2* krange = reinterpret_cast<int2*>(base + G.krange);
    uint32_t* wmask = reinterpret_cast<uint32_t*>(base + G.wmask);
    int* hrow = reinterpret_cast<int*>(base + G.hrow);
    float* wcost = reinterpret_cast<float*>(base + G.wcost);
    int* counters = reinterpret_cast<int*>(base + G.counters);
    uint32_t* pmask = reinterpret_cast<uint32_t*>(base + G.pmask);
    uint32_t* spm = reinterpret_cast<uint32_t*>(base + G.spm);       // pair-id mask of each sphere
    float* ssr = reinterpret_cast<float*>(base + G.sr);
    float* link_rl = reinterpret_cast<float*>(base + G.rl);
    float* grp_rl = link_rl + kLinks;
    int* link_ref = reinterpret_cast<int*>(base + G.ref);
    int* grp_ref = link_ref + kLinks;
    uint16_t* spij = reinterpret_cast<uint16_t*>(base + G.pij);     // i | j << 8
    uint16_t* sgpid = reinterpret_cast<uint16_t*>(base + G.gpid);
    uint16_t* sgpoff = reinterpret_cast<uint16_t*>(base + G.gpoff);
    uint16_t* sgpab = reinterpret_cast<uint16_t*>(base + G.gpab);   // a | b << 8
    uint16_t* slpab = reinterpret_cast<uint16_t*>(base + G.lpab);
    uint16_t* slpgp = reinterpret_cast<uint16_t*>(base + G.lpgp);
    uint16_t* l1 = reinterpret_cast<uint16_t*>(base + G.l1);
    uint16_t* stask = reinterpret_cast<uint16_t*>(base + G.stask);
    uint16_t* wtask = reinterpret_cast<uint16_t*>(base + G.wtask);
    uint8_t* slink = reinterpret_cast<uint8_t*>(wtask + kTile * kMaxSpheres);   // link of sphere
    uint32_t* wcp = reinterpret_cast<uint32_t*>(base + G.wcp);
    uint32_t* wov = reinterpret_cast<uint32_t*>(base + G.wov);

    const int cs = G.cs, PMW = G.pmw;
    const long long P = (long long)a.B * a.H;
    const long long n_tiles = (P + kTile - 1) / kTile;
    const int tid = threadIdx.x;
    const int lane = tid & 31;

    // ---- 0. stage the divergently-indexed tables (once per persistent CTA)
    for (int i = tid; i < G.S; i += kThreads) ssr[i] = R.sr[i];
    if (tid < kLinks)
        for (int s2 = R.link_start[tid]; s2 < R.link_start[tid + 1]; ++s2) slink[s2] = (uint8_t)tid;
    if (tid < kLinks) {
        link_rl[tid] = R.link_rl[tid];
        link_ref[tid] = R.link_ref[tid];
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
        // spm[s]: bit pid set iff sphere s belongs to pair pid
        for (int i = tid; i < G.S * PMW; i += kThreads) spm[i] = 0u;
    }
    __syncthreads();
    if (a.do_self)
        for (int pid = tid; pid < G.npairs; pid += kThreads) {
            atomicOr(spm + R.pair_i[pid] * PMW + (pid >> 5), 1u << (pid & 31));
            atomicOr(spm + R.pair_j[pid] * PMW + (pid >> 5), 1u << (pid & 31));
        }

    // cp.async prefetch of a tile's packed rows (p0-1 .. p0+np, clamped) and
    // of its rows' world indices into the stage buffer
    auto prefetch = [&](long long tl) {
        if (tl >= n_tiles) return;
        const long long q0 = tl * kTile;
        const long long rlo = max(q0 - 1, 0LL), rhi = min(q0 + kTile + 1, P);
        const int nq = int(rhi - rlo) * G.Qos;
        const uint4* src = reinterpret_cast<const uint4*>(a.os + rlo * G.Wos);
        uint4* dst = reinterpret_cast<uint4*>(stage);
        for (int q = tid; q < nq; q += kThreads) cp_async16(dst + q, src + q);
        if (a.do_world && tid < kRows) {
            const long long pg = q0 - 1 + tid;
            if (pg >= 0 && pg < P) cp_async4(swid + tid, a.world_idx + pg / a.H);
        }
    };
    // contiguous chunk of tiles per CTA: consecutive tiles belong to the same
    // trajectories / problems, so the problem's cuboids stay in L1
    const long long per_cta = (n_tiles + gridDim.x - 1) / gridDim.x;
    const long long t_begin = blockIdx.x * per_cta;
    const long long t_end = min(n_tiles, t_begin + per_cta);
    if (t_begin < t_end) prefetch(t_begin);
    cp_async_commit();

    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const int nsub = (a.do_world && a.swept) ? a.sweep_steps : 0;
    const float inv_n1 = 1.f / float(nsub + 1);

#ifdef VAPR_PHASES
    __shared__ unsigned long long ph_acc[16];
    if (tid < 16) ph_acc[tid] = 0ull;
    long long ph_t = clock64();
#define VAPR_PHASE(i)                                   \
    if (tid == 0) {                                     \
        const long long t_ = clock64();                 \
        ph_acc[i] += (unsigned long long)(t_ - ph_t);   \
        ph_t = t_;                                      \
    }
#else
#define VAPR_PHASE(i)
#endif

    for (long long tile = t_begin; tile < t_end; ++tile) {
    const long long p0 = tile * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const long long r_lo = max(p0 - 1, 0LL);
    const long long r_hi = min(p0 + np + 1, P);           // exclusive
    const int row_off = int(r_lo - (p0 - 1));             // tile row of global row r_lo
    cp_async_wait_all();
    if (tid < 8) counters[tid] = 0;
    __syncthreads();
    VAPR_PHASE(1);

    // ---- 1. rows' step index and cuboid range; decode; zero the outputs
    if (tid < kRows) {
        const int row = tid;
        const long long pg = p0 - 1 + row;
        int hh = -1;
        int2 kr = make_int2(0, 0);
        if (pg >= 0 && pg < P) {
            hh = int(pg % a.H);                // 64-bit division: once per row
            if (a.do_world) {
                const int wi = swid[row];
                if (wi >= 0 && wi < Wd.n_worlds)
                    kr = make_int2(__ldg(Wd.off + wi), __ldg(Wd.off + wi + 1));
            }
        }
        hrow[row] = hh;
        krange[row] = kr;
        if (kr.y > kr.x) atomicMax(counters + 6, kr.y - kr.x);
    }
    float amax = 0.f;
    {
        // one thread per 16-byte group of 4 packed words (4 PF elements
        // starting at a multiple of 4): one 16-byte shared load, 4 PF
        // decodes, PF 16-byte shared stores
        const int nq = int(r_hi - r_lo) * G.Qos;
        const uint4* sw = reinterpret_cast<const uint4*>(stage);
        int r = tid / G.Qos, g = tid - (tid / G.Qos) * G.Qos;
        const int dr = kThreads / G.Qos, dg = kThreads - dr * G.Qos;
        with_pf(fos.pf, [&](auto Pc) {
            constexpr int PF = decltype(Pc)::value;
            for (int q = tid; q < nq; q += kThreads) {
                const uint4 v = sw[q];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                float x[4 * PF];
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) decode_word_t<PF>(w4[j4], x + j4 * PF, fos);
                float4* d4 = reinterpret_cast<float4*>(ctile + (row_off + r) * cs + 4 * PF * g);
#pragma unroll
                for (int j = 0; j < PF; ++j) {
                    d4[j] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
                    amax = fmaxf(amax, fmaxf(fmaxf(fabsf(x[4 * j]), fabsf(x[4 * j + 1])),
                                             fmaxf(fabsf(x[4 * j + 2]), fabsf(x[4 * j + 3]))));
                }
                r += dr;
                g += dg;
                if (g >= G.Qos) {
                    g -= G.Qos;
                    ++r;
                }
            }
        });
    }
    {
        uint32_t ab = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));   // non-negative
        if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(counters + 2), ab);
    }
    if (a.do_world)
        for (int i = tid; i < kTile * G.Wcp / 4; i += kThreads)
            reinterpret_cast<uint4*>(wcp)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (a.do_self) {
        for (int i = tid; i < kTile * G.Wov / 4; i += kThreads)
            reinterpret_cast<uint4*>(wov)[i] = make_uint4(0u, 0u, 0u, 0u);
        for (int i = tid; i < kTile * PMW; i += kThreads) pmask[i] = 0u;
        if (tid < kTile) {
            touched[tid] = 0ull;
            pwm[tid] = 0u;
        }
    }
    if (a.do_world)
        for (int i = tid; i < kTile * G.S; i += kThreads) wcost[i] = 0.f;
    for (int i = tid; i < kRows * kLinks; i += kThreads) wmask[i] = 0u;
    __syncthreads();
    VAPR_PHASE(2);

    // the stage buffer is free: prefetch the next tile behind this one's compute
    if (tile + 1 < t_end) prefetch(tile + 1);
    cp_async_commit();

    // Quantisation margin: a decoded coordinate y of an FK value x satisfies
    // |y - x| <= 2^-(M+1) |x| + 2^-(bias+M) (half an ulp; the subnormal
    // quantum covers the bottom of the range) unless the code saturated; two
    // centres per distance and sqrt(3) per vector give the ball margin.  With
    // a saturated coordinate in the tile (|y| == max_finite) there is no bound
    // and culling is switched off for the tile.
    const float amaxf = __uint_as_float((uint32_t)counters[2]);
    bool can_cull = a.cull != 0;
    float margin = 0.f;
    if (fos.kind != KIND_IDENTITY) {
        if (amaxf >= decode(fos.maxcode, fos)) can_cull = false;
        const float rel = ldexpf(1.f, -(fos.M + 1));
        const float sub = ldexpf(1.f, -((1 << (fos.E - 1)) - 1) - fos.M);
        margin = 2.f * 1.7320509f * (rel * amaxf * 1.01f + sub);
    }
    // cuboid kk of the world of tile row `row` (global range start k0)
    auto cuboid = [&](int row, int k0, int kk) -> Cub {
        const int c = kcache[row];
        if (c >= 0) return scub[c + kk];
        const int k = k0 + kk;
        return Cub{__ldg(Wd.cub + 4 * k), __ldg(Wd.cub + 4 * k + 1), __ldg(Wd.cub + 4 * k + 2),
                   __ldg(Wd.cub + 4 * k + 3)};
    };
    // cuboid cache: the worlds of the first and last pose of the tile (a tile
    // spans one or two trajectories in practice); other rows read global memory
    if (a.do_world) {
        const int wa = (hrow[1] >= 0) ? swid[1] : -1, wb = (hrow[np] >= 0) ? swid[np] : -1;
        for (int i = tid; i < 2 * kMaxCuboids * 4; i += kThreads) {
            const int slot = i / (kMaxCuboids * 4), rest = i - slot * kMaxCuboids * 4;
            const int w = slot ? wb : wa;
            if (w < 0 || w >= Wd.n_worlds) continue;
            const int c0 = __ldg(Wd.off + w), c1 = __ldg(Wd.off + w + 1);
            if (c0 + (rest >> 2) < c1)
                reinterpret_cast<float4*>(scub)[i] = __ldg(Wd.cub + 4 * (c0 + (rest >> 2)) + (rest & 3));
        }
        if (tid < kRows) {
            const int w = swid[tid];
            kcache[tid] = (hrow[tid] < 0) ? -1 : (w == wa ? 0 : (w == wb ? kMaxCuboids : -1));
        }
    }
    // link balls of every present row
    for (int i = tid; i < kRows * kLinks; i += kThreads) {
        const int row = i / kLinks, l = i - row * kLinks;
        const float* c = ctile + row * cs + 3 * link_ref[l];
        lball[i] = make_float4(c[0], c[1], c[2], link_rl[l] + margin);
    }
    __syncthreads();
    VAPR_PHASE(3);

    // ---- 2. broadphase
    // world: one task per (cuboid, row, link) triple, cuboid-major so the
    // lanes of a warp mostly share the cuboid (an L1 broadcast); the (rare)
    // live bits are ORed into wmask: bits 0-15 pose (discrete), 16-31 segment
    // row -> row+1 (swept; a ball around both endpoint balls bounds every
    // sample on the segment)
    if (a.do_world) {
        const int kmax = counters[6];
        const int ntask = kRows * kLinks * kmax;
        // four independent triples per step so their loads and arithmetic interleave
        for (int t0 = tid; t0 < ntask; t0 += 4 * kThreads) {
            float sdf[4], lim[4];
            int wi[4], bit[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int task = t0 + u * kThreads;
                wi[u] = -1;
                sdf[u] = 0.f;
                lim[u] = 0.f;
                bit[u] = 0;
                if (task >= ntask) continue;
                const int kk = task / (kRows * kLinks);
                const int rl = task - kk * (kRows * kLinks);
                const int row = rl / kLinks, l = rl - row * kLinks;
                const int2 kr = krange[row];
                const int h = hrow[row];
                if (h < 0 || kk >= kr.y - kr.x || link_rl[l] < 0.f) continue;
                const float4 b0 = lball[rl];
                float mx = b0.x, my = b0.y, mz = b0.z, rs = b0.w;
                bit[u] = kk;
                if (nsub > 0) {
                    if (!(h + 1 < a.H && row + 1 < kRows && hrow[row + 1] >= 0)) continue;
                    const float4 b1 = lball[rl + kLinks];
                    const float dx = b1.x - b0.x, dy = b1.y - b0.y, dz = b1.z - b0.z;
                    mx += 0.5f * dx;
                    my += 0.5f * dy;
                    mz += 0.5f * dz;
                    rs = fmaxf(b0.w, b1.w) + 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    bit[u] += 16;
                }
                const Cub cb = cuboid(row, kr.x, kk);
                sdf[u] = box_sdf_lb(cb, mx, my, mz);
                lim[u] = rs + a.eta_w + kSlack;
                wi[u] = rl;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (wi[u] >= 0 && (!can_cull || sdf[u] <= lim[u])) atomicOr(wmask + wi[u], 1u << bit[u]);
        }
    }
    // self level 1: live (pose, link pair) by the link balls (l1 list)
    if (a.do_self)
        for (int b0 = tid - lane; b0 < kTile * 32; b0 += kThreads) {
            const int task = b0 + lane;
            const int p = task >> 5, lp = task & 31;
            bool live = false;
            if (p < np && lp < G.nlp) {
                const int la = slpab[lp] & 0xff, lb = slpab[lp] >> 8;
                const float4 A4 = lball[(p + 1) * kLinks + la], B4 = lball[(p + 1) * kLinks + lb];
                const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                const float lim = A4.w + B4.w + a.eta_s + kSlack;
                live = !can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim;
            }
            const int slot = warp_append(counters + 3, live, lane);
            if (live) l1[slot] = (uint16_t)task;
        }
    __syncthreads();
    VAPR_PHASE(4);

    // live (pose, sphere) world items (the sphere's link has a live cuboid);
    // self level 2: live (pose, group pair)
    if (a.do_world)
        for (int b0 = tid - lane; b0 < kTile * G.S; b0 += kThreads) {
            const int item = b0 + lane;
            const int p = item / G.S, sp = item - p * G.S;
            bool live = false;
            if (p < np) {
                const int row = p + 1, h = hrow[row], l = slink[sp];
                uint32_t m;
                if (nsub > 0)
                    m = (wmask[row * kLinks + l] >> 16) |
                        (h > 0 ? (wmask[(row - 1) * kLinks + l] >> 16) : 0u);
                else
                    m = wmask[row * kLinks + l] & 0xffffu;
                live = m != 0u;
            }
            const int slot = warp_append(counters + 0, live, lane);
            if (live) wtask[slot] = (uint16_t)item;
        }
    if (a.do_self) {
        const int n1 = counters[3];
        for (int b0 = tid - lane; b0 < n1 * 4; b0 += kThreads) {
            const int it = b0 + lane;
            bool live = false;
            int p = 0, g = 0;
            if (it < n1 * 4) {
                const int e = l1[it >> 2];
                p = e >> 5;
                const int lp = e & 31;
                g = slpgp[lp] + (it & 3);
                if (g < slpgp[lp + 1]) {
                    const int ga = sgpab[g] & 0xff, gb = sgpab[g] >> 8;
                    const float* ca = ctile + (p + 1) * cs + 3 * grp_ref[ga];
                    const float* cb = ctile + (p + 1) * cs + 3 * grp_ref[gb];
                    const float dx = ca[0] - cb[0], dy = ca[1] - cb[1], dz = ca[2] - cb[2];
                    const float lim = grp_rl[ga] + grp_rl[gb] + 2.f * margin + a.eta_s + kSlack;
                    live = !can_cull || fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= lim * lim;
                }
            }
            const int slot = warp_append(counters + 1, live, lane);
            if (live) stask[slot] = (uint16_t)(p * kMaxGroupPairs + g);
        }
    }
    __syncthreads();
    VAPR_PHASE(5);

    // ---- 3a. world tasks: all spheres of one link of one pose
    const int n_wtask = counters[0], n_stask = counters[1];
#ifdef VAPR_PHASES
    if (tid == 0) {
        ph_acc[10] += n_wtask;
        ph_acc[11] += n_stask;
        ph_acc[12] += counters[3];
        ph_acc[14] += counters[6];
    }
#endif
    for (int t = tid; t < n_wtask; t += kThreads) {
        const int item = wtask[t];
        const int p = item / G.S, sp = item - p * G.S;
        const int l = slink[sp];
        const int row = p + 1, h = hrow[row];
        const int k0 = krange[row].x;
        uint32_t m_own, m_fwd = 0, m_bwd = 0;
        if (nsub > 0) {
            m_fwd = (h < a.H - 1) ? (wmask[row * kLinks + l] >> 16) : 0u;
            m_bwd = (h > 0) ? (wmask[(row - 1) * kLinks + l] >> 16) : 0u;
            m_own = m_fwd | m_bwd;     // a segment ball contains both endpoint balls
        } else {
            m_own = wmask[row * kLinks + l] & 0xffffu;
        }
        const float* crow = ctile + row * cs;
        const float cx = crow[3 * sp], cy = crow[3 * sp + 1], cz = crow[3 * sp + 2];
        const float A = ssr[sp] + a.eta_w;
        Acc acc{0.f, 0.f, 0.f, 0.f};
        for (uint32_t m = m_own; m; m &= m - 1)
            world_term(cuboid(row, k0, __ffs(m) - 1), cx, cy, cz, A, a.eta_w, inv_eta_w, hoe_w,
                       a.w_w, 1.f, 1.f, acc);
        if (m_fwd) {                // samples of segment (h, h+1): cost + (1-tau) grad
            const float* nrow = crow + cs;
            const float nx = nrow[3 * sp], ny = nrow[3 * sp + 1], nz = nrow[3 * sp + 2];
            for (int j = 1; j <= nsub; ++j) {
                const float tau = float(j) * inv_n1, omt = 1.f - tau;
                const float sx = fmaf(tau, nx, omt * cx), sy = fmaf(tau, ny, omt * cy),
                            sz = fmaf(tau, nz, omt * cz);
                for (uint32_t m = m_fwd; m; m &= m - 1)
                    world_term(cuboid(row, k0, __ffs(m) - 1), sx, sy, sz, A, a.eta_w, inv_eta_w,
                               hoe_w, a.w_w, 1.f, omt, acc);
            }
        }
        if (m_bwd) {                // samples of segment (h-1, h): tau grad only
            const float* prow = crow - cs;
            const float qx = prow[3 * sp], qy = prow[3 * sp + 1], qz = prow[3 * sp + 2];
            for (int j = 1; j <= nsub; ++j) {
                const float tau = float(j) * inv_n1, omt = 1.f - tau;
                const float sx = fmaf(tau, cx, omt * qx), sy = fmaf(tau, cy, omt * qy),
                            sz = fmaf(tau, cz, omt * qz);
                for (uint32_t m = m_bwd; m; m &= m - 1)
                    world_term(cuboid(row, k0, __ffs(m) - 1), sx, sy, sz, A, a.eta_w, inv_eta_w,
                               hoe_w, a.w_w, 0.f, tau, acc);
            }
        }
        uint32_t* orow = wcp + p * G.Wcp;
        or_code(orow, 3 * sp + 0, acc.gx + 0.f, fcp, G.rc_cp);
        or_code(orow, 3 * sp + 1, acc.gy + 0.f, fcp, G.rc_cp);
        or_code(orow, 3 * sp + 2, acc.gz + 0.f, fcp, G.rc_cp);
        wcost[item] = acc.cost;
    }
    // ---- 3b. self tasks: the active sphere pairs of one group pair of one
    //          pose, four candidate pairs in flight per step (independent loads
    //          and arithmetic interleave)
    for (int t = tid; t < n_stask; t += kThreads) {
        const int task = stask[t];
        const int p = task / kMaxGroupPairs, g = task - p * kMaxGroupPairs;
        const float* crow = ctile + (p + 1) * cs;
        unsigned long long tb = 0ull;
        uint32_t wm = 0u;
        const int k0 = sgpoff[g], k1 = sgpoff[g + 1];
        for (int k = k0; k < k1; k += 4) {
            int pid[4], ii[4], jj[4];
            float d2[4], Rs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                pid[u] = (k + u < k1) ? sgpid[k + u] : sgpid[k];
                ii[u] = spij[pid[u]] & 0xff;
                jj[u] = spij[pid[u]] >> 8;
                const float dx = crow[3 * ii[u]] - crow[3 * jj[u]];
                const float dy = crow[3 * ii[u] + 1] - crow[3 * jj[u] + 1];
                const float dz = crow[3 * ii[u] + 2] - crow[3 * jj[u] + 2];
                d2[u] = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                Rs[u] = ssr[ii[u]] + ssr[jj[u]] + a.eta_s;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                // same exact early-out as self_pair: d2 >= fl(Rs^2) => phi <= 0
                if (k + u >= k1 || d2[u] >= Rs[u] * Rs[u]) continue;
                if (Rs[u] - sqrtf(d2[u]) <= 0.f) continue;
                atomicOr(pmask + p * PMW + (pid[u] >> 5), 1u << (pid[u] & 31));
                wm |= 1u << (pid[u] >> 5);
                tb |= (1ull << ii[u]) | (1ull << jj[u]);
            }
        }
        if (tb) {
            atomicOr(touched + p, tb);
            atomicOr(pwm + p, wm);
        }
    }
    __syncthreads();
    VAPR_PHASE(6);

    // ---- 4a. per pose: list its touched spheres; sum its cost in a fixed
    //          order (world per link, then the active self pairs by pair id)
    if (tid < np) {
        const int p = tid;
        float cost = 0.f;
        if (a.do_world)
            for (int sp = 0; sp < G.S; ++sp) cost += wcost[p * G.S + sp];
        if (a.do_self) {
            unsigned long long tb = touched[p];
            if (tb) {
                int slot = atomicAdd(counters + 4, __popcll(tb));
                for (; tb; tb &= tb - 1) l1[slot++] = (uint16_t)(p * 64 + __ffsll((long long)tb) - 1);
                const float* crow = ctile + (p + 1) * cs;
                const uint32_t* pm = pmask + p * PMW;
                float scost = 0.f;
                for (uint32_t wmk = pwm[p]; wmk; wmk &= wmk - 1) {
                    const int wd = __ffs(wmk) - 1;
                    for (uint32_t m = pm[wd]; m; m &= m - 1) {
                        const int pid = (wd << 5) + __ffs(m) - 1;
                        float vx, vy, vz, c;
                        self_pair(crow, spij[pid] & 0xff, spij[pid] >> 8, ssr, a.eta_s,
                                  inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c);
                        scost += c;
                    }
                }
                cost += scost;
            }
        }
        a.cost[p0 + p] = cost;
    }
    __syncthreads();
    VAPR_PHASE(7);

    // ---- 4b. self gradients: one item per (pose, touched sphere), gathered
    //          over its active pairs in canonical id order -- for a fixed
    //          sphere that is its partners in ascending order, independent of
    //          culling and of the task order
    if (a.do_self) {
        const int nt = counters[4];
#ifdef VAPR_PHASES
        if (tid == 0) ph_acc[13] += nt;
#endif
        for (int t = tid; t < nt; t += kThreads) {
            const int it = l1[t];
            const int p = it >> 6, s = it & 63;
            const float* crow = ctile + (p + 1) * cs;
            const uint32_t* pm = pmask + p * PMW;
            const uint32_t* sm_ = spm + s * PMW;
            float gx = 0.f, gy = 0.f, gz = 0.f;
            for (uint32_t wmk = pwm[p]; wmk; wmk &= wmk - 1) {
                const int wd = __ffs(wmk) - 1;
                for (uint32_t m = pm[wd] & sm_[wd]; m; m &= m - 1) {
                    const int pid = (wd << 5) + __ffs(m) - 1;
                    const int i = spij[pid] & 0xff, j = spij[pid] >> 8;
                    float vx, vy, vz, c;
                    self_pair(crow, i, j, ssr, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c);
                    const float sg = (i == s) ? -1.f : 1.f;
                    gx = fmaf(sg, vx, gx);
                    gy = fmaf(sg, vy, gy);
                    gz = fmaf(sg, vz, gz);
                }
            }
            uint32_t* orow = wov + p * G.Wov;
            or_code(orow, 3 * s + 0, gx + 0.f, fov, G.rc_ov);
            or_code(orow, 3 * s + 1, gy + 0.f, fov, G.rc_ov);
            or_code(orow, 3 * s + 2, gz + 0.f, fov, G.rc_ov);
        }
    }
    __syncthreads();
    VAPR_PHASE(8);

    // ---- 5. coalesced 16-byte packed stores (tile rows are contiguous in HBM)
    if (a.do_world) {
        uint4* dst = reinterpret_cast<uint4*>(a.cp + p0 * G.Wcp);
        for (int i = tid; i < np * G.Wcp / 4; i += kThreads)
            __stcs(dst + i, reinterpret_cast<const uint4*>(wcp)[i]);
    }
    if (a.do_self) {
        uint4* dst = reinterpret_cast<uint4*>(a.ov + p0 * G.Wov);
        for (int i = tid; i < np * G.Wov / 4; i += kThreads)
            __stcs(dst + i, reinterpret_cast<const uint4*>(wov)[i]);
    }
    __syncthreads();
    VAPR_PHASE(9);
    }  // tile loop
    cp_async_wait_all();
#ifdef VAPR_PHASES
    if (tid < 16) atomicAdd(&g_phase_cycles[tid], ph_acc[tid]);
#endif
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

#ifdef VAPR_PHASES
extern "C" int vapr_debug_phase_cycles(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif

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
    // persistent CTAs: as many as fit on the device (the robot tables are
    // staged once per CTA), each looping over tiles
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, collision_kernel, kThreads, smem);
    const long long tiles = (P + kTile - 1) / kTile;
    const long long grid = std::min<long long>(tiles, (long long)sms * std::max(per_sm, 1));
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
