// fk.cu -- a2: forward kinematics -> packed out_spheres.
// P:86 (forward kinematics), P:189 ("The output of forward kinematics:
// out_spheres"); quantised at the store (reading c19).
//
// Phase A: one thread per pose walks the 8-row modified-DH chain in FP32
// (full-precision sincosf) and places the spheres of each link as soon as its
// frame is known, writing the 3S centre coordinates into an FP32 shared tile
// (row stride 3S|1 words, odd: the 32 lanes -- 32 poses writing the same
// element -- hit 32 distinct banks).
// Phase B: the CTA packs the tile word by word (PF compile-time via with_pf,
// hardware cvt fast path for E5M10 / E8M7 / FP8 / FP6 / FP4) and streams the
// packed rows to HBM with coalesced stores.
// Link frames are NOT written to memory: backward kinematics recomputes them
// (DESIGN.md §6), so HBM sees q (28 B/pose) in and out_spheres out.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kTile = 128;   // poses (= threads) per CTA

__global__ void __launch_bounds__(kTile)
fk_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
          long long P, int W, uint32_t* __restrict__ os) {
    extern __shared__ float smem[];
    const int cols = R.cols;
    const int cs = cols | 1;
    float* sq = smem;                       // [kTile * 7]
    float* tile = smem + kTile * kJoints;   // [kTile * cs]
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    for (int i = tid; i < np * kJoints; i += kTile) sq[i] = __ldcs(q + p0 * kJoints + i);
    __syncthreads();

    if (tid < np) {
        float* row = tile + tid * cs;
        Xf X;
        xf_identity(X);
        for (int l = 0; l < kLinks; ++l) {
            if (l >= 1 && l <= kJoints) fk_step(X, R, l - 1, sq[tid * kJoints + l - 1]);
            if (l == kLinks - 1) fk_hand(X, R);
            for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
                float cx, cy, cz;
                xf_apply(X, R.sx[s], R.sy[s], R.sz[s], cx, cy, cz);
                row[3 * s + 0] = cx;
                row[3 * s + 1] = cy;
                row[3 * s + 2] = cz;
            }
        }
    }
    __syncthreads();

    // Phase B: word w of row r <- elements [w*PF, w*PF + PF) of tile row r
    const int nw = np * W;
    const int dr = kTile / W, dw = kTile % W;
    int r = tid / W, w = tid - (tid / W) * W;
    uint32_t* dst = os + p0 * W;
    with_pf(f.pf, [&](auto Pc) {
        constexpr int PF = decltype(Pc)::value;
        for (int i = tid; i < nw; i += kTile) {
            const float* src = tile + r * cs + w * PF;
            float x[PF];
#pragma unroll
            for (int j = 0; j < PF; ++j) x[j] = (w * PF + j < cols) ? src[j] : 0.f;
            __stcs(dst + i, encode_word_t<PF>(x, f));
            r += dr;
            w += dw;
            if (w >= W) {
                w -= W;
                ++r;
            }
        }
    });
}

}  // namespace

cudaError_t launch_fk(const RobotDev& R, const Fmt& fos, const float* q, long long P,
                      uint32_t* os, cudaStream_t s) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fos, R.cols);
    const size_t smem = sizeof(float) * kTile * (kJoints + (R.cols | 1));
    cudaError_t e = cudaFuncSetAttribute(fk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (P + kTile - 1) / kTile;
    fk_kernel<<<(unsigned)grid, kTile, smem, s>>>(R, fos, q, P, W, os);
    return cudaGetLastError();
}

}  // namespace vapr
