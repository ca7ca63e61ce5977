// bk.cu -- a6: backward kinematics, packed grad_out_spheres -> grad_q.
// P:162 step (5) "Compute backward for the above steps in the reverse
// sequence"; P:189 ("the input of backward kinematics: grad_out_spheres");
// P:196 ("sparsity-aware computation by skipping zero computations").
//
//   grad_q_j = z_j . (M_{>=j} - o_j x F_{>=j}),
//   F_l = sum_{s in link l} g_s,  M_l = sum_{s in link l} c_s x g_s,
// with the frames and the sphere centres c_s recomputed in FP32 from q
// (reading c20: the Jacobian of the true FK, not of the quantised spheres).
//
// One thread per pose.  The CTA first streams its tile of packed gradient
// rows into shared memory (coalesced) and flags the rows that hold any
// non-zero word; a pose whose row is all zero writes grad_q = 0 without
// touching the kinematics.  Active poses run the forward chain once, keeping
// the 8 frames in per-thread shared storage (lane-interleaved: conflict
// free), then sweep the links from the hand down accumulating the suffix sums
// F, M -- no prefix/total differences, so no cancellation -- and skipping
// zero spheres.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kTile = 64;                 // poses (= threads) per CTA
constexpr int kFrameFloats = 12;
constexpr int kFrames = kLinks - 1;       // frames 1..7 and the hand

__global__ void __launch_bounds__(kTile)
bk_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
          long long P, int W, const uint32_t* __restrict__ gos, float* __restrict__ grad_q) {
    extern __shared__ uint32_t smem[];
    const int WS = W + 1;
    uint32_t* sw = smem;                                              // [kTile * WS]
    float* frames = reinterpret_cast<float*>(sw + kTile * WS);        // [kFrames*12][kTile]
    float* sq = frames + kFrames * kFrameFloats * kTile;              // [kTile * 7]
    int* active = reinterpret_cast<int*>(sq + kTile * kJoints);       // [kTile]
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    active[tid] = 0;
    for (int i = tid; i < np * kJoints; i += kTile) sq[i] = __ldcs(q + p0 * kJoints + i);
    __syncthreads();
    const long long nw = (long long)np * W;
    const uint32_t* src = gos + p0 * W;
    for (long long i = tid; i < nw; i += kTile) {
        const int r = int(i / W), c = int(i - (long long)r * W);
        const uint32_t v = __ldcs(src + i);
        sw[r * WS + c] = v;
        if (v) active[r] = 1;                 // benign race: every writer stores 1
    }
    __syncthreads();

    float g7[kJoints];
#pragma unroll
    for (int j = 0; j < kJoints; ++j) g7[j] = 0.f;

    if (tid < np && active[tid]) {
        const uint32_t* row = sw + tid * WS;
        // forward chain, frames 1..7 and hand into lane-interleaved smem
        Xf X;
        xf_identity(X);
        for (int l = 1; l < kLinks; ++l) {
            if (l <= kJoints) fk_step(X, R, l - 1, sq[tid * kJoints + l - 1]);
            else fk_hand(X, R);
            float* fr = frames + (l - 1) * kFrameFloats * kTile + tid;
#pragma unroll
            for (int i = 0; i < 9; ++i) fr[i * kTile] = X.r[i];
#pragma unroll
            for (int i = 0; i < 3; ++i) fr[(9 + i) * kTile] = X.p[i];
        }
        // reverse sweep: suffix sums over links l = 8 .. 1
        float Fx = 0.f, Fy = 0.f, Fz = 0.f, Mx = 0.f, My = 0.f, Mz = 0.f;
        for (int l = kLinks - 1; l >= 1; --l) {
            const float* fr = frames + (l - 1) * kFrameFloats * kTile + tid;
            Xf L;
#pragma unroll
            for (int i = 0; i < 9; ++i) L.r[i] = fr[i * kTile];
#pragma unroll
            for (int i = 0; i < 3; ++i) L.p[i] = fr[(9 + i) * kTile];
            for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
                float g[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int e = 3 * s + k;
                    const int wi = e / f.pf;
                    g[k] = decode(code_at(row[wi], e - wi * f.pf, f), f);
                }
                if (g[0] == 0.f && g[1] == 0.f && g[2] == 0.f) continue;   // zero skipping
                float cx, cy, cz;
                xf_apply(L, R.sx[s], R.sy[s], R.sz[s], cx, cy, cz);
                Fx += g[0];
                Fy += g[1];
                Fz += g[2];
                Mx += cy * g[2] - cz * g[1];
                My += cz * g[0] - cx * g[2];
                Mz += cx * g[1] - cy * g[0];
            }
            if (l <= kJoints) {
                // z_l . (M - o_l x F)
                const float ox = L.p[0], oy = L.p[1], oz = L.p[2];
                const float tx = Mx - (oy * Fz - oz * Fy);
                const float ty = My - (oz * Fx - ox * Fz);
                const float tz = Mz - (ox * Fy - oy * Fx);
                g7[l - 1] = L.r[2] * tx + L.r[5] * ty + L.r[8] * tz;
            }
        }
    }
    __syncthreads();
    // stage grad_q through smem (reuse sq) for a coalesced store
    if (tid < np) {
#pragma unroll
        for (int j = 0; j < kJoints; ++j) sq[tid * kJoints + j] = g7[j];
    }
    __syncthreads();
    for (int i = tid; i < np * kJoints; i += kTile) __stcs(grad_q + p0 * kJoints + i, sq[i]);
}

}  // namespace

cudaError_t launch_bk(const RobotDev& R, const Fmt& fgos, const float* q, long long P,
                      const uint32_t* gos, float* grad_q, cudaStream_t s) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fgos, R.cols);
    const size_t smem = sizeof(uint32_t) * kTile * (W + 1) +
                        sizeof(float) * (kFrames * kFrameFloats * kTile + kTile * kJoints) +
                        sizeof(int) * kTile;
    cudaError_t e = cudaFuncSetAttribute(bk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (P + kTile - 1) / kTile;
    bk_kernel<<<(unsigned)grid, kTile, smem, s>>>(R, fgos, q, P, W, gos, grad_q);
    return cudaGetLastError();
}

}  // namespace vapr
