// fk.cu -- a2: forward kinematics -> packed out_spheres.
// P:86 (forward kinematics), P:189 ("The output of forward kinematics:
// out_spheres"); quantised at the store (reading c19).
//
// One thread per pose walks the 8-row modified-DH chain in FP32 (full
// precision sincosf), places the spheres of each link as soon as its frame is
// known, and encodes the 3S centre coordinates straight into packed words in a
// bank-padded shared-memory row (row stride W+1 words, odd, so the 32 lanes of
// a warp -- 32 poses writing the same word index -- hit 32 distinct banks).
// The CTA then streams its tile of packed rows to HBM with coalesced stores.
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
    extern __shared__ uint32_t smem[];
    const int WS = W + 1;                          // padded smem row stride (odd)
    float* sq = reinterpret_cast<float*>(smem);    // [kTile * 7]
    uint32_t* sw = smem + kTile * kJoints;         // [kTile * WS]
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x;

    for (int i = tid; i < np * kJoints; i += kTile) sq[i] = __ldcs(q + p0 * kJoints + i);
    __syncthreads();

    if (tid < np) {
        uint32_t* row = sw + tid * WS;
        uint32_t acc = 0;
        int slot = 0, word = 0;
        auto emit = [&](float v) {
            acc |= encode(v, f) << (slot * f.t);
            if (++slot == f.pf) {
                row[word++] = acc;
                acc = 0;
                slot = 0;
            }
        };
        Xf X;
        xf_identity(X);
        for (int l = 0; l < kLinks; ++l) {
            if (l >= 1 && l <= kJoints) fk_step(X, R, l - 1, sq[tid * kJoints + l - 1]);
            if (l == kLinks - 1) fk_hand(X, R);
            for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
                float cx, cy, cz;
                xf_apply(X, R.sx[s], R.sy[s], R.sz[s], cx, cy, cz);
                emit(cx);
                emit(cy);
                emit(cz);
            }
        }
        if (slot != 0) row[word++] = acc;
        for (; word < W; ++word) row[word] = 0u;   // 16-byte row padding
    }
    __syncthreads();

    // coalesced tile store: consecutive threads write consecutive words
    const long long nw = (long long)np * W;
    uint32_t* dst = os + p0 * W;
    for (long long i = tid; i < nw; i += kTile) {
        const int r = int(i / W), c = int(i - (long long)r * W);
        __stcs(dst + i, sw[r * WS + c]);
    }
}

}  // namespace

cudaError_t launch_fk(const RobotDev& R, const Fmt& fos, const float* q, long long P,
                      uint32_t* os, cudaStream_t s) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fos, R.cols);
    const size_t smem = sizeof(float) * kTile * kJoints + sizeof(uint32_t) * kTile * (W + 1);
    cudaError_t e = cudaFuncSetAttribute(fk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (P + kTile - 1) / kTile;
    fk_kernel<<<(unsigned)grid, kTile, smem, s>>>(R, fos, q, P, W, os);
    return cudaGetLastError();
}

}  // namespace vapr
