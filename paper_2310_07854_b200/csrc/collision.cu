// collision.cu -- a3 + a4: world (sphere-vs-cuboid, discrete or swept) and
// self (sphere-pair) collision costs and their gradients, reading packed
// out_spheres and writing packed closest_pt[_swept] / out_vec.
// P:86 ("Robot-environment and robot-self distance queries are utilized in the
// cost function"), P:189 (tensor roles).  Cost form: DESIGN.md readings
// c13-c17 (box SDF, smooth hinge, summed over cuboids / listed pairs; swept =
// linear sub-samples with the exact gradient to both endpoints).
//
// Tile = kTile consecutive poses (+1 halo pose on each side for the swept
// samples).  Phase 1 decodes the packed rows into an FP32 shared tile (row
// stride 157 words, odd).  Phase 2 runs one lane per (sphere, pose) item with
// warps assigned sphere-major, so the 32 lanes of a warp share the sphere s:
// its radius, link and self-collision partner list are warp-uniform
// (__grid_constant__ broadcast) and only the pose varies.  Each item gathers
// its complete gradient (no scatter), encodes its 3 codes and ORs non-zero
// codes into shared packed rows (OR is order-independent, so the result is
// deterministic).  Per-pose costs are reduced in a fixed order.  Phase 3
// streams the packed tiles out with coalesced stores.
//
// Culling is exact: a term is skipped only when the FP32 evaluation of the
// full formula is provably 0 (see the comments at each test), so results are
// bit-identical with VAPR_OPT_CULL on or off.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kTile = 64;           // poses per CTA
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;

struct Acc {
    float cost, gx, gy, gz;
};

// f(c) and grad f(c) summed over the cuboids of one world; adds into acc with
// weight `gw` on the gradient and `cw` on the cost.
__device__ __forceinline__ void world_point(float cx, float cy, float cz, float A, float eta,
                                            float inv_eta, float half_over_eta, float w,
                                            const float4* __restrict__ cub, int k0, int k1,
                                            float cw, float gw, Acc& acc) {
    for (int k = k0; k < k1; ++k) {
        const float4 q0 = __ldg(cub + 4 * k + 0);   // rt00 rt01 rt02 rt10
        const float4 q1 = __ldg(cub + 4 * k + 1);   // rt11 rt12 rt20 rt21
        const float4 q2 = __ldg(cub + 4 * k + 2);   // rt22 tx ty tz
        const float4 q3 = __ldg(cub + 4 * k + 3);   // hx hy hz pad
        const float dx = cx - q2.y, dy = cy - q2.z, dz = cz - q2.w;
        const float px = fmaf(q0.x, dx, fmaf(q0.y, dy, q0.z * dz));
        const float py = fmaf(q0.w, dx, fmaf(q1.x, dy, q1.y * dz));
        const float pz = fmaf(q1.z, dx, fmaf(q1.w, dy, q2.x * dz));
        const float ux = fabsf(px) - q3.x, uy = fabsf(py) - q3.y, uz = fabsf(pz) - q3.z;
        const float umax = fmaxf(ux, fmaxf(uy, uz));
        // sdf >= umax in FP32 (sqrt(fl(a^2)) rounds back to a; adding terms
        // only grows it), so A - umax <= 0 implies phi = A - sdf <= 0: exact.
        if (A - umax <= 0.f) continue;
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
            glx = copysignf(ox * inv, px >= 0.f ? 1.f : -1.f);
            gly = copysignf(oy * inv, py >= 0.f ? 1.f : -1.f);
            glz = copysignf(oz * inv, pz >= 0.f ? 1.f : -1.f);
        }
        const float phi = A - sdf;
        if (phi <= 0.f) continue;
        float h, dh;
        if (phi <= eta) {
            h = phi * phi * half_over_eta;
            dh = phi * inv_eta;
        } else {
            h = phi - 0.5f * eta;
            dh = 1.f;
        }
        acc.cost = fmaf(cw * w, h, acc.cost);
        // world gradient = R g_local; R = (R^T)^T
        const float gxw = fmaf(q0.x, glx, fmaf(q0.w, gly, q1.z * glz));
        const float gyw = fmaf(q0.y, glx, fmaf(q1.x, gly, q1.w * glz));
        const float gzw = fmaf(q0.z, glx, fmaf(q1.y, gly, q2.x * glz));
        const float sc = -w * dh * gw;
        acc.gx = fmaf(sc, gxw, acc.gx);
        acc.gy = fmaf(sc, gyw, acc.gy);
        acc.gz = fmaf(sc, gzw, acc.gz);
    }
}

__device__ __forceinline__ void or_code(uint32_t* row, int e, float v, const Fmt& f) {
    const uint32_t c = encode(v, f);
    if (c != 0u) {
        const int w = e / f.pf;
        atomicOr(row + w, c << ((e - w * f.pf) * f.t));
    }
}

__global__ void __launch_bounds__(kThreads)
collision_kernel(const __grid_constant__ RobotDev R, const WorldsDev Wd, const Fmt fos,
                 const Fmt fcp, const Fmt fov, const CollisionArgs a, int Wos, int Wcp,
                 int Wov) {
    extern __shared__ float smem[];
    const int S = R.n_spheres;
    const int cols = R.cols;
    const int cs = cols | 1;                       // odd fp32 row stride
    const long long P = (long long)a.B * a.H;
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    // shared layout
    float* ctile = smem;                                   // [(kTile+2) * cs], row 0 = pose p0-1
    float* cpart = ctile + (kTile + 2) * cs;               // [S * kTile]
    uint32_t* wcp = reinterpret_cast<uint32_t*>(cpart + S * kTile);   // [kTile * (Wcp+1)]
    uint32_t* wov = wcp + (a.do_world ? kTile * (Wcp + 1) : 0);       // [kTile * (Wov+1)]
    const int WcpS = Wcp + 1, WovS = Wov + 1;

    // ---- phase 1: decode rows p0-1 .. p0+np into the FP32 tile; zero outputs
    const long long r_lo = max(p0 - 1, 0LL);
    const long long r_hi = min(p0 + np + 1, P);           // exclusive
    const long long nwords = (r_hi - r_lo) * Wos;
    const uint32_t* src = a.os + r_lo * Wos;
    for (long long i = tid; i < nwords; i += kThreads) {
        const int r = int(i / Wos), w = int(i - (long long)r * Wos);
        const uint32_t word = __ldg(src + i);
        float* dst = ctile + (int(r_lo - (p0 - 1)) + r) * cs;
        for (int j = 0; j < fos.pf; ++j) {
            const int e = w * fos.pf + j;
            if (e < cols) dst[e] = decode(code_at(word, j, fos), fos);
        }
    }
    if (a.do_world)
        for (int i = tid; i < kTile * WcpS; i += kThreads) wcp[i] = 0u;
    if (a.do_self)
        for (int i = tid; i < kTile * WovS; i += kThreads) wov[i] = 0u;
    __syncthreads();

    // ---- phase 2: items (sphere s, pose p), sphere-major per warp
    const int lane = tid & 31, warp = tid >> 5;
    const float Aw_eta = a.eta_w, inv_eta_w = 1.f / a.eta_w, hoe_w = 0.5f / a.eta_w;
    const float inv_eta_s = 1.f / a.eta_s, hoe_s = 0.5f / a.eta_s;
    const int halves = kTile / 32;
    const int n_tasks = S * halves;
    const int nsub = a.swept ? a.sweep_steps : 0;
    const float inv_n1 = 1.f / float(nsub + 1);
    for (int task = warp; task < n_tasks; task += kWarps) {
        const int s = task / halves;
        const int p = (task - s * halves) * 32 + lane;
        if (p >= np) continue;
        const long long pg = p0 + p;
        const int b = int(pg / a.H);
        const int h = int(pg - (long long)b * a.H);
        const float* crow = ctile + (p + 1) * cs;
        const float cx = crow[3 * s], cy = crow[3 * s + 1], cz = crow[3 * s + 2];
        const float r = R.sr[s];
        float cost = 0.f;
        if (a.do_world) {
            Acc acc{0.f, 0.f, 0.f, 0.f};
            const int wi = __ldg(a.world_idx + b);
            int k0 = 0, k1 = 0;
            if (wi >= 0 && wi < Wd.n_worlds) {
                k0 = __ldg(Wd.off + wi);
                k1 = __ldg(Wd.off + wi + 1);
            }
            const float A = r + Aw_eta;
            world_point(cx, cy, cz, A, a.eta_w, inv_eta_w, hoe_w, a.w_w, Wd.cub, k0, k1, 1.f,
                        1.f, acc);
            if (nsub > 0) {
                if (h < a.H - 1) {          // samples of segment (h, h+1): cost + (1-tau) grad
                    const float* nrow = crow + cs;
                    const float nx = nrow[3 * s], ny = nrow[3 * s + 1], nz = nrow[3 * s + 2];
                    for (int j = 1; j <= nsub; ++j) {
                        const float tau = float(j) * inv_n1, omt = 1.f - tau;
                        world_point(fmaf(tau, nx, omt * cx), fmaf(tau, ny, omt * cy),
                                    fmaf(tau, nz, omt * cz), A, a.eta_w, inv_eta_w, hoe_w,
                                    a.w_w, Wd.cub, k0, k1, 1.f, omt, acc);
                    }
                }
                if (h > 0) {                // samples of segment (h-1, h): tau grad only
                    const float* prow = crow - cs;
                    const float qx = prow[3 * s], qy = prow[3 * s + 1], qz = prow[3 * s + 2];
                    for (int j = 1; j <= nsub; ++j) {
                        const float tau = float(j) * inv_n1, omt = 1.f - tau;
                        world_point(fmaf(tau, cx, omt * qx), fmaf(tau, cy, omt * qy),
                                    fmaf(tau, cz, omt * qz), A, a.eta_w, inv_eta_w, hoe_w,
                                    a.w_w, Wd.cub, k0, k1, 0.f, tau, acc);
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
            const int j0 = R.adj_off[s], j1 = R.adj_off[s + 1];
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
                } else {                     // coincident centres: (1,0,0) from the lower index
                    ux = (s < o) ? 1.f : -1.f;
                    uy = uz = 0.f;
                }
                const float k = -a.w_s * dh;
                gx = fmaf(k, ux, gx);
                gy = fmaf(k, uy, gy);
                gz = fmaf(k, uz, gz);
                if (s < o) sc = fmaf(a.w_s, hh, sc);     // each pair's cost counted once
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

    // ---- phase 3: per-pose cost (fixed order) and coalesced packed stores
    if (tid < np) {
        float c = 0.f;
        for (int s = 0; s < S; ++s) c += cpart[s * kTile + tid];
        a.cost[p0 + tid] = c;
    }
    if (a.do_world) {
        const long long n = (long long)np * Wcp;
        uint32_t* dst = a.cp + p0 * Wcp;
        for (long long i = tid; i < n; i += kThreads) {
            const int r = int(i / Wcp), c = int(i - (long long)r * Wcp);
            __stcs(dst + i, wcp[r * WcpS + c]);
        }
    }
    if (a.do_self) {
        const long long n = (long long)np * Wov;
        uint32_t* dst = a.ov + p0 * Wov;
        for (long long i = tid; i < n; i += kThreads) {
            const int r = int(i / Wov), c = int(i - (long long)r * Wov);
            __stcs(dst + i, wov[r * WovS + c]);
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
    size_t smem = sizeof(float) * ((size_t)(kTile + 2) * cs + (size_t)R.n_spheres * kTile);
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
