// aggregate.cu -- a5: grad_out_spheres = Q_gos(dequant(closest_pt[_swept]) +
// dequant(out_vec)), elementwise over pose rows.  P:162 step (4)
// "Aggregating the costs"; P:189 ("the input of backward kinematics:
// grad_out_spheres").  The two inputs and the output may each have a
// different format and hence a different packing factor.
//
// One thread per output word; consecutive threads produce consecutive words of
// the same row, so the stores are coalesced and the (L1-cached) input words
// are shared by neighbouring threads.  The inputs are >99 % zero in the
// paper's workloads: a zero input word decodes to +0 and is skipped.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

// e / pf for e < 4096 and pf in 1..8 via a 16-bit reciprocal (exact in that
// range; checked on the host in make_fmt's unit test of the API).
__device__ __forceinline__ int div_pf(int e, uint32_t recip) { return int((e * recip) >> 16); }

__global__ void __launch_bounds__(256)
aggregate_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int cols, int Wc, int Wo, int Wg,
                 const uint32_t* __restrict__ cp, const uint32_t* __restrict__ ov,
                 long long rows, uint32_t* __restrict__ gos, uint32_t rc_cp, uint32_t rc_ov) {
    const long long n = rows * Wg;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / Wg;
        const int w = int(i - r * Wg);
        const uint32_t* crow = cp + r * Wc;
        const uint32_t* orow = ov + r * Wo;
        uint32_t acc = 0;
        int lc = -1, lo = -1;
        uint32_t wc = 0, wo = 0;
        for (int j = 0; j < fg.pf; ++j) {
            const int e = w * fg.pf + j;
            if (e >= cols) break;
            const int ic = div_pf(e, rc_cp), io = div_pf(e, rc_ov);
            if (ic != lc) { wc = __ldg(crow + ic); lc = ic; }
            if (io != lo) { wo = __ldg(orow + io); lo = io; }
            const uint32_t cc = code_at(wc, e - ic * fcp.pf, fcp);
            const uint32_t co = code_at(wo, e - io * fov.pf, fov);
            if ((cc | co) == 0u) continue;                 // +0 + +0 = +0 -> code 0
            const float g = decode(cc, fcp) + decode(co, fov);
            acc |= encode(g, fg) << (j * fg.t);
        }
        __stcs(gos + i, acc);
    }
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
