// bk.cu -- a6: backward kinematics, packed grad_out_spheres -> grad_q.
// P:162 step (5) "Compute backward for the above steps in the reverse
// sequence"; P:189 ("the input of backward kinematics: grad_out_spheres");
// P:196 ("sparsity-aware computation by skipping zero computations").
//
//   grad_q_j = sum_{l >= j} z_j . (M_l - o_j x F_l),
//   F_l = sum_{s in link l} g_s,  M_l = sum_{s in link l} c_s x g_s,
// with the frames and the sphere centres c_s recomputed in FP32 from q
// (reading c20: the Jacobian of the true FK, not of the quantised spheres).
//
// The CTA streams its tile of packed gradient rows into shared memory with
// coalesced loads and, for the rare non-zero words, marks the spheres they
// touch in a per-pose 64-bit mask.  One thread per pose then runs the chain
// only if its mask is non-zero; each link's (F_l, M_l) is folded into the
// joint accumulators j <= l as soon as the link's frame is known, so no frame
// is stored and no prefix/total difference (cancellation) is formed.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kTile = 128;                 // poses (= threads) per CTA

__global__ void __launch_bounds__(kTile)
bk_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
          long long P, int W, const uint32_t* __restrict__ gos, float* __restrict__ grad_q,
          uint32_t rc) {
    extern __shared__ unsigned long long smem8[];
    const int WS = W + 1;
    unsigned long long* smask = smem8;                                // [kTile]
    float4* so = reinterpret_cast<float4*>(smask + kTile);            // [kMaxSpheres] sphere offsets
    float* sq = reinterpret_cast<float*>(so + kMaxSpheres);           // [kTile * 7]
    uint32_t* sw = reinterpret_cast<uint32_t*>(sq + kTile * kJoints); // [kTile * WS]
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    smask[tid] = 0ull;
    // sphere offsets are indexed per lane (by each pose's non-zero spheres):
    // stage them in shared memory instead of the serialising constant bank
    for (int i = tid; i < R.n_spheres; i += kTile) so[i] = make_float4(R.sx[i], R.sy[i], R.sz[i], 0.f);
    for (int i = tid; i < np * kJoints; i += kTile) sq[i] = __ldcs(q + p0 * kJoints + i);
    __syncthreads();
    {
        const int nw = np * W;
        const uint32_t* src = gos + p0 * W;
        const int dr = kTile / W, dw = kTile % W;
        int r = tid / W, w = tid - (tid / W) * W;
        for (int i = tid; i < nw; i += kTile) {
            const uint32_t v = __ldcs(src + i);
            sw[r * WS + w] = v;
            if (v) {
                unsigned long long m = 0;
                for (int j = 0; j < f.pf; ++j)
                    if (code_at(v, j, f)) {
                        const int e = w * f.pf + j;
                        if (e < R.cols) m |= 1ull << (e / 3);
                    }
                atomicOr(smask + r, m);
            }
            r += dr;
            w += dw;
            if (w >= W) {
                w -= W;
                ++r;
            }
        }
    }
    __syncthreads();

    float gq[kJoints];
#pragma unroll
    for (int j = 0; j < kJoints; ++j) gq[j] = 0.f;

    const unsigned long long mask = (tid < np) ? smask[tid] : 0ull;
    if (mask) {
        const uint32_t* row = sw + tid * WS;
        float zx[kJoints], zy[kJoints], zz[kJoints], ox[kJoints], oy[kJoints], oz[kJoints];
        Xf X;
        xf_identity(X);
#pragma unroll
        for (int l = 1; l < kLinks; ++l) {
            if (l <= kJoints) {
                fk_step(X, R, l - 1, sq[tid * kJoints + l - 1]);
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
            while (lm) {
                const int s = s0 + __ffsll((long long)lm) - 1;
                lm &= lm - 1;
                float g[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int e = 3 * s + k;
                    const int wi = int((e * rc) >> 16);
                    g[k] = decode(code_at(row[wi], e - wi * f.pf, f), f);
                }
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
            // fold link l into every joint j <= l: z_j . (M_l - o_j x F_l)
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
    __syncthreads();
    // stage grad_q through smem (reuse sq) for a coalesced store
    if (tid < np) {
#pragma unroll
        for (int j = 0; j < kJoints; ++j) sq[tid * kJoints + j] = gq[j];
    }
    __syncthreads();
    for (int i = tid; i < np * kJoints; i += kTile) __stcs(grad_q + p0 * kJoints + i, sq[i]);
}

}  // namespace

cudaError_t launch_bk(const RobotDev& R, const Fmt& fgos, const float* q, long long P,
                      const uint32_t* gos, float* grad_q, cudaStream_t s) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fgos, R.cols);
    const size_t smem = sizeof(unsigned long long) * kTile + sizeof(float4) * kMaxSpheres +
                        sizeof(float) * kTile * kJoints +
                        sizeof(uint32_t) * kTile * (W + 1);
    cudaError_t e = cudaFuncSetAttribute(bk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t rc = 65536u / fgos.pf + 1u;
    const long long grid = (P + kTile - 1) / kTile;
    bk_kernel<<<(unsigned)grid, kTile, smem, s>>>(R, fgos, q, P, W, gos, grad_q, rc);
    return cudaGetLastError();
}

}  // namespace vapr
