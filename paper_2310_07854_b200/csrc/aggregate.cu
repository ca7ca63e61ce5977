// aggregate.cu -- a5: grad_out_spheres = Q_gos(dequant(closest_pt[_swept]) +
// dequant(out_vec)), elementwise over pose rows.  P:162 step (4)
// "Aggregating the costs"; P:189 ("the input of backward kinematics:
// grad_out_spheres").  The two inputs and the output may each have a
// different format and hence a different packing factor.
//
// One thread per output word (coalesced stores; neighbouring threads share
// the L1-cached input words).  The inputs are >99 % zero in the paper's
// workloads ("sparsity-aware computation by skipping zero
// computations"): when every input word overlapping the output word's
// elements is zero the output word is zero (+0 + +0 = +0 -> code 0) and no
// element is decoded.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

// e / pf for e < 4096 and pf in 1..8 via a 16-bit reciprocal (exact there).
__device__ __forceinline__ int div_pf(int e, uint32_t recip) { return int((e * recip) >> 16); }

__global__ void __launch_bounds__(256)
aggregate_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int cols, int Wc, int Wo, int Wg,
                 const uint32_t* __restrict__ cp, const uint32_t* __restrict__ ov,
                 long long rows, uint32_t* __restrict__ gos, uint32_t rc_cp, uint32_t rc_ov) {
    const long long n = rows * Wg;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long step = (long long)gridDim.x * blockDim.x;
    const long long dr = step / Wg;
    const int dw = int(step - dr * Wg);
    long long r = i0 / Wg;
    int w = int(i0 - r * Wg);
    with_pf(fg.pf, [&](auto Pc) {
        constexpr int PF = decltype(Pc)::value;
        for (long long i = i0; i < n; i += step) {
            const int e0 = w * PF;
            uint32_t out = 0;
            if (e0 < cols) {
                const int e1 = min(e0 + PF, cols) - 1;
                const uint32_t* crow = cp + r * Wc;
                const uint32_t* orow = ov + r * Wo;
                const int c0 = div_pf(e0, rc_cp), c1 = div_pf(e1, rc_cp);
                const int o0 = div_pf(e0, rc_ov), o1 = div_pf(e1, rc_ov);
                uint32_t any = 0;
                for (int k = c0; k <= c1; ++k) any |= __ldg(crow + k);
                for (int k = o0; k <= o1; ++k) any |= __ldg(orow + k);
                if (any) {
                    float x[PF];
#pragma unroll
                    for (int j = 0; j < PF; ++j) {
                        const int e = e0 + j;
                        x[j] = 0.f;
                        if (e < cols) {
                            const int ic = div_pf(e, rc_cp), io = div_pf(e, rc_ov);
                            const uint32_t cc = code_at(__ldg(crow + ic), e - ic * fcp.pf, fcp);
                            const uint32_t co = code_at(__ldg(orow + io), e - io * fov.pf, fov);
                            if (cc | co) x[j] = decode(cc, fcp) + decode(co, fov);
                        }
                    }
                    out = encode_word_t<PF>(x, fg);
                }
            }
            __stcs(gos + i, out);
            r += dr;
            w += dw;
            if (w >= Wg) {
                w -= Wg;
                ++r;
            }
        }
    });
}

}  // namespace

cudaError_t launch_aggregate(const Fmt& fcp, const Fmt& fov, const Fmt& fgos, int cols,
                             const uint32_t* cp, const uint32_t* ov, long long rows,
                             uint32_t* gos, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const int Wc = row_words_of(fcp, cols), Wo = row_words_of(fov, cols),
              Wg = row_words_of(fgos, cols);
    const uint32_t rc_cp = 65536u / fcp.pf + 1u, rc_ov = 65536u / fov.pf + 1u;
    const long long n = rows * Wg;
    long long grid = (n + 255) / 256;
    if (grid > 148LL * 16) grid = 148LL * 16;
    aggregate_kernel<<<(unsigned)grid, 256, 0, s>>>(fcp, fov, fgos, cols, Wc, Wo, Wg, cp, ov,
                                                    rows, gos, rc_cp, rc_ov);
    return cudaGetLastError();
}

}  // namespace vapr
