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

// Shared-memory carve-up (sizes depend on the robot and the formats).
struct Layout {
    int pmw, ngp, npairs;
    unsigned stage, swid, touched, krange, wmask, hrow, wslot, wcost, counters, pmask, sr, rl, ref, pij,
        gpid, gpoff, gpab, lpab, lpgp, wtask, stask, l1, wcp, wov, ctile, total;
};

// FP32 tile row stride: a multiple of 4 floats (16-byte vector stores), at
// least one packed row's worth of decoded elements, and not a multiple of 32
// (rows of one column spread over several banks).
__host__ __device__ inline int tile_stride(int cols, int Wos, int pf) {
    int cs = ((cols + 3) & ~3);
    if (cs < Wos * pf) cs = Wos * pf;
    if (cs % 32 == 0) cs += 4;
    return cs;
}

__host__ __device__ inline Layout make_layout(const RobotDev& R, int do_world, int do_self,
                                              int Wos, int Wcp, int Wov, int pfos) {
    Layout L{};
    L.pmw = (R.n_pairs + 31) >> 5;
    L.ngp = R.lp_gp_off[R.n_link_pairs];
    L.npairs = R.n_pairs;
    unsigned o = 0;
    auto take = [&](unsigned bytes, unsigned align) {
        o = (o + align - 1) / align * align;
        const unsigned at = o;
        o += bytes;
        return at;
    };
    L.stage = take(sizeof(uint32_t) * 2 * kRows * Wos, 16);
    L.swid = take(sizeof(int) * 2 * kRows, 4);
    L.touched = take(sizeof(unsigned long long) * kTile, 8);
    L.krange = take(sizeof(int2) * kRows, 8);
    L.wmask = take(sizeof(uint32_t) * kRows * kLinks, 4);
    L.hrow = take(sizeof(int) * kRows, 4);
    L.wslot = take(sizeof(int) * kRows, 4);
    L.wcost = take(sizeof(float) * kTile * kLinks, 4);
    L.counters = take(sizeof(int) * 8, 4);
    L.pmask = take(sizeof(uint32_t) * kTile * L.pmw, 4);
    L.sr = take(sizeof(float) * kMaxSpheres, 4);
    L.rl = take(sizeof(float) * 3 * kLinks, 4);          // link radii [9], group radii [18]
    L.ref = take(sizeof(int) * 3 * kLinks, 4);           // link refs [9], group refs [18]
    L.pij = take(sizeof(uint16_t) * L.npairs, 2);
    L.gpid = take(sizeof(uint16_t) * L.npairs, 2);
    L.gpoff = take(sizeof(uint16_t) * (kMaxGroupPairs + 1), 2);
    L.gpab = take(sizeof(uint16_t) * kMaxGroupPairs, 2);
    L.lpab = take(sizeof(uint16_t) * 33, 2);
    L.lpgp = take(sizeof(uint16_t) * 33, 2);
    L.wtask = take(sizeof(uint16_t) * kTile * kLinks, 2);
    L.stask = take(sizeof(uint16_t) * kTile * (L.ngp > 0 ? L.ngp : 1), 2);
    L.l1 = take(sizeof(uint16_t) * kTile * 64, 2);
    L.wcp = take(do_world ? sizeof(uint32_t) * kTile * Wcp : 0u, 16);
    L.wov = take(do_self ? sizeof(uint32_t) * kTile * Wov : 0u, 16);
    L.ctile = take(sizeof(float) * kRows * tile_stride(R.cols, Wos, pfos), 16);
    L.total = o + 16;
    return L;
}

__global__ void __launch_bounds__(kThreads, 6)
collision_kernel(const __grid_constant__ RobotDev R, const WorldsDev Wd, const Fmt fos,
                 const Fmt fcp, const Fmt fov, const CollisionArgs a, int Wos, int Wcp,
                 int Wov) {
    extern __shared__ float4 smem4[];
    char* base = reinterpret_cast<char*>(smem4);
    const Layout L = make_layout(R, a.do_world, a.do_self, Wos, Wcp, Wov, fos.pf);
    uint32_t* stage = reinterpret_cast<uint32_t*>(base + L.stage);   // [2][kRows * Wos] packed rows
    int* swid = reinterpret_cast<int*>(base + L.swid);              // [2][kRows] world index
    unsigned long long* touched = reinterpret_cast<unsigned long long*>(base + L.touched);
    int2* krange = reinterpret_cast<int2*>(base + L.krange);     // cuboid range of each row
    uint32_t* wmask = reinterpret_cast<uint32_t*>(base + L.wmask);
    int* hrow = reinterpret_cast<int*>(base + L.hrow);           // step index h, -1 if absent
    int* wslot = reinterpret_cast<int*>(base + L.wslot);         // world of each row
    float* wcost = reinterpret_cast<float*>(base + L.wcost);
    int* counters = reinterpret_cast<int*>(base + L.counters);
    uint32_t* pmask = reinterpret_cast<uint32_t*>(base + L.pmask);
    float* ssr = reinterpret_cast<float*>(base + L.sr);
    float* link_rl = reinterpret_cast<float*>(base + L.rl);
    float* grp_rl = link_rl + kLinks;
    int* link_ref = reinterpret_cast<int*>(base + L.ref);
    int* grp_ref = link_ref + kLinks;
    uint16_t* spij = reinterpret_cast<uint16_t*>(base + L.pij);  // i | j << 8
    uint16_t* sgpid = reinterpret_cast<uint16_t*>(base + L.gpid);
    uint16_t* sgpoff = reinterpret_cast<uint16_t*>(base + L.gpoff);
    uint16_t* sgpab = reinterpret_cast<uint16_t*>(base + L.gpab);  // a | b << 8
    uint16_t* slpab = reinterpret_cast<uint16_t*>(base + L.lpab);
    uint16_t* slpgp = reinterpret_cast<uint16_t*>(base + L.lpgp);
    uint16_t* wtask = reinterpret_cast<uint16_t*>(base + L.wtask);
    uint16_t* stask = reinterpret_cast<uint16_t*>(base + L.stask);
    uint16_t* l1 = reinterpret_cast<uint16_t*>(base + L.l1);
    uint32_t* wcp = reinterpret_cast<uint32_t*>(base + L.wcp);
    uint32_t* wov = reinterpret_cast<uint32_t*>(base + L.wov);
    float* ctile = reinterpret_cast<float*>(base + L.ctile);

    const int cols = R.cols;
    const int cs = tile_stride(cols, Wos, fos.pf);  // fp32 tile row stride
    const long long P = (long long)a.B * a.H;
    const long long n_tiles = (P + kTile - 1) / kTile;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int WcpS = Wcp, WovS = Wov;              // packed output row strides (16 B multiples)
    const int PMW = L.pmw;

    // ---- 0. stage the divergently-indexed tables (once per persistent CTA)
    for (int i = tid; i < R.n_spheres; i += kThreads) ssr[i] = R.sr[i];
    if (tid < kLinks) {
        link_rl[tid] = R.link_rl[tid];
        link_ref[tid] = R.link_ref[tid];
    }
    if (tid < 2 * kLinks) {
        grp_rl[tid] = R.grp_rl[tid];
        grp_ref[tid] = R.grp_ref[tid];
    }
    if (a.do_self) {
        for (int i = tid; i < L.npairs; i += kThreads) {
            spij[i] = (uint16_t)(R.pair_i[i] | (R.pair_j[i] << 8));
            sgpid[i] = R.gp_pid[i];
        }
        for (int i = tid; i <= L.ngp; i += kThreads) sgpoff[i] = R.gp_off[i];
        for (int i = tid; i < L.ngp; i += kThreads)
            sgpab[i] = (uint16_t)(R.gp_a[i] | (R.gp_b[i] << 8));
        for (int i = tid; i < R.n_link_pairs; i += kThreads)
            slpab[i] = (uint16_t)(R.lp_a[i] | (R.lp_b[i] << 8));
        for (int i = tid; i <= R.n_link_pairs; i += kThreads) slpgp[i] = R.lp_gp_off[i];
    }
    __syncthreads();

    // ---- cp.async prefetch of a tile's packed rows (p0-1 .. p0+np, clamped)
    //      and of its rows' world indices into stage buffer `buf`, so the
    //      global-memory latency of tile t+1 overlaps the compute of tile t.
    const int stage_words = kRows * Wos;
    auto prefetch = [&](long long tl, int buf) {
        if (tl >= n_tiles) return;
        const long long q0 = tl * kTile;
        const int nq_ = (int)min((long long)kTile, P - q0);
        const long long rlo = max(q0 - 1, 0LL), rhi = min(q0 + nq_ + 1, P);
        const int nq = int(rhi - rlo) * (Wos / 4);
        const uint4* src = reinterpret_cast<const uint4*>(a.os + rlo * Wos);
        uint4* dst = reinterpret_cast<uint4*>(stage + buf * stage_words);
        for (int q = tid; q < nq; q += kThreads) cp_async16(dst + q, src + q);
        if (a.do_world)
            for (int row = tid; row < kRows; row += kThreads) {
                const long long pg = q0 - 1 + row;
                if (pg >= 0 && pg < P) cp_async4(swid + buf * kRows + row, a.world_idx + pg / a.H);
            }
    };
    prefetch(blockIdx.x, 0);
    cp_async_commit();
    int buf = 0;

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
    for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const long long p0 = tile * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    prefetch(tile + gridDim.x, buf ^ 1);
    cp_async_commit();
    cp_async_wait_1();                 // this thread's copies of the current tile
    if (tid < 8) counters[tid] = 0;
    __syncthreads();                   // ... and everyone else's
    VAPR_PHASE(1);
    // rows' step index h and cuboid range
    for (int row = tid; row < kRows; row += kThreads) {
        const long long pg = p0 - 1 + row;
        int hh = -1;
        int2 kr = make_int2(0, 0);
        if (pg >= 0 && pg < P) {
            hh = int(pg % a.H);                // 64-bit division: once per row
            if (a.do_world) {
                const int wi = swid[buf * kRows + row];
                if (wi >= 0 && wi < Wd.n_worlds) kr = make_int2(__ldg(Wd.off + wi), __ldg(Wd.off + wi + 1));
            }
        }
        hrow[row] = hh;
        krange[row] = kr;
        if (kr.y > kr.x) atomicMax(counters + 6, kr.y - kr.x);
    }

    // ---- 1. decode the staged packed rows into the FP32 tile
    const long long r_lo = max(p0 - 1, 0LL);
    const long long r_hi = min(p0 + np + 1, P);           // exclusive
    const int row_off = int(r_lo - (p0 - 1));             // tile row of global row r_lo
    float amax = 0.f;
    {
        // one thread per 16-byte group of 4 packed words (4 PF elements,
        // starting at a multiple of 4): one 16-byte shared load, 4 PF decodes,
        // PF 16-byte shared stores
        const int Q = Wos / 4;
        const int nq = int(r_hi - r_lo) * Q;
        const uint4* sw = reinterpret_cast<const uint4*>(stage + buf * stage_words);
        with_pf(fos.pf, [&](auto Pc) {
            constexpr int PF = decltype(Pc)::value;
            for (int q = tid; q < nq; q += kThreads) {
                const int r = q / Q, g = q - r * Q;
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
            }
        });
    }
    {
        uint32_t ab = __float_as_uint(amax);            // non-negative: bits are monotone
        ab = __reduce_max_sync(0xffffffffu, ab);
        if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(counters + 2), ab);
    }
    if (a.do_world)
        for (int i = tid; i < kTile * WcpS / 4; i += kThreads)
            reinterpret_cast<uint4*>(wcp)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (a.do_self) {
        for (int i = tid; i < kTile * WovS / 4; i += kThreads)
            reinterpret_cast<uint4*>(wov)[i] = make_uint4(0u, 0u, 0u, 0u);
        for (int i = tid; i < kTile * PMW; i += kThreads) pmask[i] = 0u;
        if (tid < kTile) touched[tid] = 0ull;
    }
    for (int i = tid; i < kTile * kLinks; i += kThreads) wcost[i] = 0.f;
    for (int i = tid; i < kRows * kLinks; i += kThreads) wmask[i] = 0u;
    __syncthreads();
    VAPR_PHASE(2);

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
    // ball of link / group with reference sphere `ref` in tile row `row`
    auto ball = [&](int row, int ref, float rl) {
        const float* c = ctile + row * cs + 3 * ref;
        return make_float4(c[0], c[1], c[2], rl + margin);
    };
    // cuboids are read through L1 (a problem's world is shared by all its
    // seeds' tiles, so the lines stay resident)
    auto cuboid = [&](int k) -> Cub {
        return Cub{__ldg(Wd.cub + 4 * k), __ldg(Wd.cub + 4 * k + 1), __ldg(Wd.cub + 4 * k + 2),
                   __ldg(Wd.cub + 4 * k + 3)};
    };

    // ---- 2. world cull masks per (row, link): bits 0-15 pose (discrete),
    //         bits 16-31 segment row -> row+1 (swept)
    const int nsub = (a.do_world && a.swept) ? a.sweep_steps : 0;
    // One task per (row, cuboid, link) triple, cuboid-major so the lanes of
    // a warp mostly share the cuboid (an L1 broadcast); the (rare) live bits
    // are ORed into wmask.
    if (a.do_world) {
        const int kmax = counters[6];
        const int ntask = kRows * kLinks * kmax;
        for (int task = tid; task < ntask; task += kThreads) {
            const int kk = task / (kRows * kLinks);
            const int rl = task - kk * (kRows * kLinks);
            const int row = rl / kLinks, l = rl - row * kLinks;
            const int2 kr = krange[row];
            const int h = hrow[row];
            if (h < 0 || kk >= kr.y - kr.x || link_rl[l] < 0.f) continue;
            const Cub cb = cuboid(kr.x + kk);
            const float4 b0 = ball(row, link_ref[l], link_rl[l]);
            if (nsub > 0) {
                if (!(h + 1 < a.H && row + 1 < kRows && hrow[row + 1] >= 0)) continue;
                // segment row -> row+1 of the same trajectory: one ball
                // around both endpoint balls bounds every sample
                const float4 b1 = ball(row + 1, link_ref[l], link_rl[l]);
                const float dx = b1.x - b0.x, dy = b1.y - b0.y, dz = b1.z - b0.z;
                const float half = 0.5f * sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                const bool live =
                    !can_cull || box_sdf_lb(cb, b0.x + 0.5f * dx, b0.y + 0.5f * dy, b0.z + 0.5f * dz) -
                                         fmaxf(b0.w, b1.w) - half - a.eta_w <= kSlack;
                if (live) atomicOr(wmask + row * kLinks + l, 1u << (16 + kk));
            } else {
                const bool live =
                    !can_cull || box_sdf_lb(cb, b0.x, b0.y, b0.z) - b0.w - a.eta_w <= kSlack;
                if (live) atomicOr(wmask + row * kLinks + l, 1u << kk);
            }
        }
    }
    __syncthreads();
    VAPR_PHASE(3);
    // self level 1: live (pose, link pair) by the link balls (l1 list)
    if (a.do_self)
        for (int b0 = tid - lane; b0 < kTile * R.n_link_pairs; b0 += kThreads) {
            const int task = b0 + lane;
            const int p = task / R.n_link_pairs, lp = task - p * R.n_link_pairs;
            bool live = false;
            if (p < np) {
                const int la = slpab[lp] & 0xff, lb = slpab[lp] >> 8;
                const float4 A4 = ball(p + 1, link_ref[la], link_rl[la]);
                const float4 B4 = ball(p + 1, link_ref[lb], link_rl[lb]);
                const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                live = !can_cull ||
                       sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - A4.w - B4.w - a.eta_s <= kSlack;
            }
            const int slot = warp_append(counters + 3, live, lane);
            if (live) l1[slot] = (uint16_t)(p * 32 + lp);
        }
    // live (pose, link) world tasks
    if (a.do_world)
        for (int b0 = tid - lane; b0 < kTile * kLinks; b0 += kThreads) {
            const int task = b0 + lane;
            const int p = task / kLinks, l = task - p * kLinks;
            bool live = false;
            if (p < np) {
                const int row = p + 1, h = hrow[row];
                uint32_t m;
                if (nsub > 0)
                    m = (wmask[row * kLinks + l] >> 16) |
                        (h > 0 ? (wmask[(row - 1) * kLinks + l] >> 16) : 0u);
                else
                    m = wmask[row * kLinks + l] & 0xffffu;
                live = m != 0u;
            }
            const int slot = warp_append(counters + 0, live, lane);
            if (live) wtask[slot] = (uint16_t)task;
        }
    __syncthreads();
    VAPR_PHASE(4);
    // self level 2: live (pose, group pair) among the (<= 4) of each live link pair
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
                    const float4 A4 = ball(p + 1, grp_ref[ga], grp_rl[ga]);
                    const float4 B4 = ball(p + 1, grp_ref[gb], grp_rl[gb]);
                    const float dx = A4.x - B4.x, dy = A4.y - B4.y, dz = A4.z - B4.z;
                    live = !can_cull ||
                           sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - A4.w - B4.w - a.eta_s <= kSlack;
                }
            }
            const int slot = warp_append(counters + 1, live, lane);
            if (live) stask[slot] = (uint16_t)(p * kMaxGroupPairs + g);
        }
    }
    __syncthreads();
    VAPR_PHASE(5);

    // ---- 3a. world tasks: all spheres of one link of one pose
    const uint32_t rc_cp = 65536u / fcp.pf + 1u, rc_ov = 65536u / fov.pf + 1u;
    const float inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const float inv_n1 = 1.f / float(nsub + 1);
    const int n_wtask = counters[0], n_stask = counters[1];
    for (int t = tid; t < n_wtask; t += kThreads) {
        const int task = wtask[t];
        const int p = task / kLinks, l = task - p * kLinks;
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
        uint32_t* orow = wcp + p * WcpS;
        float lcost = 0.f;
        for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
            const float cx = crow[3 * s], cy = crow[3 * s + 1], cz = crow[3 * s + 2];
            const float A = ssr[s] + a.eta_w;
            Acc acc{0.f, 0.f, 0.f, 0.f};
            for (uint32_t m = m_own; m; m &= m - 1)
                world_term(cuboid(k0 + __ffs(m) - 1), cx, cy, cz, A, a.eta_w, inv_eta_w, hoe_w,
                           a.w_w, 1.f, 1.f, acc);
            if (m_fwd) {                // samples of segment (h, h+1): cost + (1-tau) grad
                const float* nrow = crow + cs;
                const float nx = nrow[3 * s], ny = nrow[3 * s + 1], nz = nrow[3 * s + 2];
                for (int j = 1; j <= nsub; ++j) {
                    const float tau = float(j) * inv_n1, omt = 1.f - tau;
                    const float sx = fmaf(tau, nx, omt * cx), sy = fmaf(tau, ny, omt * cy),
                                sz = fmaf(tau, nz, omt * cz);
                    for (uint32_t m = m_fwd; m; m &= m - 1)
                        world_term(cuboid(k0 + __ffs(m) - 1), sx, sy, sz, A, a.eta_w, inv_eta_w,
                                   hoe_w, a.w_w, 1.f, omt, acc);
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
                        world_term(cuboid(k0 + __ffs(m) - 1), sx, sy, sz, A, a.eta_w, inv_eta_w,
                                   hoe_w, a.w_w, 0.f, tau, acc);
                }
            }
            lcost += acc.cost;
            or_code(orow, 3 * s + 0, acc.gx + 0.f, fcp, rc_cp);
            or_code(orow, 3 * s + 1, acc.gy + 0.f, fcp, rc_cp);
            or_code(orow, 3 * s + 2, acc.gz + 0.f, fcp, rc_cp);
        }
        wcost[task] = lcost;
    }
    // ---- 3b. self tasks: the active sphere pairs of one group pair of one pose
    for (int t = tid; t < n_stask; t += kThreads) {
        const int task = stask[t];
        const int p = task / kMaxGroupPairs, g = task - p * kMaxGroupPairs;
        const float* crow = ctile + (p + 1) * cs;
        for (int k = sgpoff[g]; k < sgpoff[g + 1]; ++k) {
            const int pid = sgpid[k];
            const int i = spij[pid] & 0xff, j = spij[pid] >> 8;
            float vx, vy, vz, c;
            if (self_pair(crow, i, j, ssr, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c)) {
                atomicOr(pmask + p * PMW + (pid >> 5), 1u << (pid & 31));
                atomicOr(touched + p, (1ull << i) | (1ull << j));
            }
        }
    }
    __syncthreads();
    VAPR_PHASE(6);

    // ---- 4a. self gradients: one item per (pose, touched sphere), gathered
    //          over the pose's active pairs in canonical id order, which for a
    //          fixed sphere s is its partners in ascending order (independent
    //          of culling and of the task order).
    if (a.do_self) {
        for (int b0 = tid - lane; b0 < np * 64; b0 += kThreads) {
            const int it = b0 + lane;
            const int p = it >> 6, s = it & 63;
            const bool live = it < np * 64 && ((touched[p] >> s) & 1ull);
            const int slot = warp_append(counters + 4, live, lane);
            if (live) l1[slot] = (uint16_t)it;        // l1 is free again
        }
        __syncthreads();
    VAPR_PHASE(7);
        const int nt = counters[4];
        for (int t = tid; t < nt; t += kThreads) {
            const int it = l1[t];
            const int p = it >> 6, s = it & 63;
            const float* crow = ctile + (p + 1) * cs;
            const uint32_t* pm = pmask + p * PMW;
            float gx = 0.f, gy = 0.f, gz = 0.f;
            for (int wd = 0; wd < PMW; ++wd)
                for (uint32_t m = pm[wd]; m; m &= m - 1) {
                    const int pid = (wd << 5) + __ffs(m) - 1;
                    const int i = spij[pid] & 0xff, j = spij[pid] >> 8;
                    if (i != s && j != s) continue;
                    float vx, vy, vz, c;
                    self_pair(crow, i, j, ssr, a.eta_s, inv_eta_s, hoe_s, a.w_s, vx, vy, vz, c);
                    const float sg = (i == s) ? -1.f : 1.f;
                    gx = fmaf(sg, vx, gx);
                    gy = fmaf(sg, vy, gy);
                    gz = fmaf(sg, vz, gz);
                }
            uint32_t* orow = wov + p * WovS;
            or_code(orow, 3 * s + 0, gx + 0.f, fov, rc_ov);
            or_code(orow, 3 * s + 1, gy + 0.f, fov, rc_ov);
            or_code(orow, 3 * s + 2, gz + 0.f, fov, rc_ov);
        }
    }
    // ---- 4b. per-pose cost: world per link, then the active self pairs in id order
    if (tid < np) {
        const int p = tid;
        float cost = 0.f;
        for (int l = 0; l < kLinks; ++l) cost += wcost[p * kLinks + l];
        if (a.do_self && touched[p]) {
            const float* crow = ctile + (p + 1) * cs;
            const uint32_t* pm = pmask + p * PMW;
            float scost = 0.f;
            for (int wd = 0; wd < PMW; ++wd)
                for (uint32_t m = pm[wd]; m; m &= m - 1) {
                    const int pid = (wd << 5) + __ffs(m) - 1;
                    float vx, vy, vz, c;
                    self_pair(crow, spij[pid] & 0xff, spij[pid] >> 8, ssr, a.eta_s, inv_eta_s,
                              hoe_s, a.w_s, vx, vy, vz, c);
                    scost += c;
                }
            cost += scost;
        }
        a.cost[p0 + p] = cost;
    }
    __syncthreads();
    VAPR_PHASE(8);

    // ---- 5. coalesced 16-byte packed stores (tile rows are contiguous in HBM)
    if (a.do_world) {
        uint4* dst = reinterpret_cast<uint4*>(a.cp + p0 * Wcp);
        for (int i = tid; i < np * Wcp / 4; i += kThreads) __stcs(dst + i, reinterpret_cast<const uint4*>(wcp)[i]);
    }
    if (a.do_self) {
        uint4* dst = reinterpret_cast<uint4*>(a.ov + p0 * Wov);
        for (int i = tid; i < np * Wov / 4; i += kThreads) __stcs(dst + i, reinterpret_cast<const uint4*>(wov)[i]);
    }
    __syncthreads();
    VAPR_PHASE(9);
    buf ^= 1;
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
    const int Wos = row_words_of(fos, R.cols);
    const int Wcp = a.do_world ? row_words_of(fcp, R.cols) : 0;
    const int Wov = a.do_self ? row_words_of(fov, R.cols) : 0;
    const size_t smem = make_layout(R, a.do_world, a.do_self, Wos, Wcp, Wov, fos.pf).total;
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
