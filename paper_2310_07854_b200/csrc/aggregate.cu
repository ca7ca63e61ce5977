// aggregate.cu -- a5: grad_out_spheres = Q_gos(dequant(closest_pt[_swept]) +
// dequant(out_vec)), elementwise over pose rows.  P:162 step (4)
// "Aggregating the costs"; P:189 ("the input of backward kinematics:
// grad_out_spheres").  The two inputs and the output may each have a
// different format and hence a different packing factor.
//
// One CTA per tile of kRows pose rows.  Both input tiles are streamed into
// shared memory with 16-byte coalesced loads; rows whose input words are all
// zero are flagged on the way.  The inputs are >99 % zero in the paper's
// workloads ("sparsity-aware computation by skipping zero
// computations"): a flagged-zero row produces zero output words without any
// decoding (+0 + +0 = +0 -> code 0), and inside a non-zero row an output word
// whose overlapping input words are zero is zero as well.  Each thread emits
// one 16-byte group of 4 output words (coalesced 16-byte stores).
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kRows = 64;
constexpr int kThreads = 256;

// e / pf for e < 4096 and pf in 1..8 via a 16-bit reciprocal (exact there).
__device__ __forceinline__ int div_pf(int e, uint32_t recip) { return int((e * recip) >> 16); }

__global__ void __launch_bounds__(kThreads)
aggregate_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int cols, int Wc, int Wo, int Wg,
                 const uint32_t* __restrict__ cp, const uint32_t* __restrict__ ov,
                 long long rows, uint32_t* __restrict__ gos, uint32_t rc_cp, uint32_t rc_ov) {
    extern __shared__ uint4 smem_a[];
    uint32_t* sc = reinterpret_cast<uint32_t*>(smem_a);     // [kRows * Wc]
    uint32_t* so = sc + kRows * Wc;                         // [kRows * Wo]
    int* nz = reinterpret_cast<int*>(so + kRows * Wo);      // [kRows]
    const long long r0 = (long long)blockIdx.x * kRows;
    const int nr = (int)min((long long)kRows, rows - r0);
    const int tid = threadIdx.x;
    if (tid < kRows) nz[tid] = 0;
    __syncthreads();
    {
        const uint4* gc = reinterpret_cast<const uint4*>(cp + r0 * Wc);
        const uint4* go = reinterpret_cast<const uint4*>(ov + r0 * Wo);
        const int qc = Wc / 4, qo = Wo / 4;
        for (int i = tid; i < nr * qc; i += kThreads) {
            const uint4 v = __ldcs(gc + i);
            reinterpret_cast<uint4*>(sc)[i] = v;
            if (v.x | v.y | v.z | v.w) nz[i / qc] = 1;
        }
        for (int i = tid; i < nr * qo; i += kThreads) {
            const uint4 v = __ldcs(go + i);
            reinterpret_cast<uint4*>(so)[i] = v;
            if (v.x | v.y | v.z | v.w) nz[i / qo] = 1;
        }
    }
    __syncthreads();
    const int qg = Wg / 4;
    uint4* dst = reinterpret_cast<uint4*>(gos + r0 * Wg);
    with_pf(fg.pf, [&](auto Pc) {
        constexpr int PF = decltype(Pc)::value;
        for (int i = tid; i < nr * qg; i += kThreads) {
            const int r = i / qg, g = i - r * qg;
            uint32_t out[4] = {0u, 0u, 0u, 0u};
            if (nz[r]) {
                const uint32_t* crow = sc + r * Wc;
                const uint32_t* orow = so + r * Wo;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e0 = (4 * g + k) * PF;
                    if (e0 >= cols) continue;
                    const int e1 = min(e0 + PF, cols) - 1;
                    uint32_t any = 0;
                    for (int m = div_pf(e0, rc_cp); m <= div_pf(e1, rc_cp); ++m) any |= crow[m];
                    for (int m = div_pf(e0, rc_ov); m <= div_pf(e1, rc_ov); ++m) any |= orow[m];
                    if (!any) continue;
                    float x[PF];
#pragma unroll
                    for (int j = 0; j < PF; ++j) {
                        const int e = e0 + j;
                        x[j] = 0.f;
                        if (e < cols) {
                            const int ic = div_pf(e, rc_cp), io = div_pf(e, rc_ov);
                            const uint32_t cc = code_at(crow[ic], e - ic * fcp.pf, fcp);
                            const uint32_t co = code_at(orow[io], e - io * fov.pf, fov);
                            if (cc | co) x[j] = decode(cc, fcp) + decode(co, fov);
                        }
                    }
                    out[k] = encode_word_t<PF>(x, fg);
                }
            }
            __stcs(dst + i, make_uint4(out[0], out[1], out[2], out[3]));
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
    const size_t smem = sizeof(uint32_t) * kRows * (Wc + Wo) + sizeof(int) * kRows;
    cudaError_t e = cudaFuncSetAttribute(aggregate_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long grid = (rows + kRows - 1) / kRows;
    aggregate_kernel<<<(unsigned)grid, kThreads, smem, s>>>(fcp, fov, fgos, cols, Wc, Wo, Wg, cp,
                                                            ov, rows, gos, rc_cp, rc_ov);
    return cudaGetLastError();
}

}  // namespace vapr
