// codec.cu -- a1: standalone packed ExMy quantise / dequantise kernels
// (vapr_quantize / vapr_dequantize).  P:227 "quantizing the tensors from FP32
// to the specified data format and dequantizing them back to FP32"; layout per
// P:218 (floor(32/t) codes per 32-bit word), rows padded to 16 B.
//
// HBM-bound streaming kernels.  Unit of work = one 16-byte group of 4 packed
// words of one row (4*pf elements).  A warp owns 32 consecutive groups; their
// FP32 inputs form ONE contiguous span of the [rows, cols] array (rows are
// contiguous and a group never straddles rows), which the warp moves with
// coalesced loads/stores through a bank-padded shared-memory staging buffer.
// Packed words are moved as one 16-byte vector per lane: a warp touches 512
// contiguous bytes per instruction.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kMaxPf = 8;
constexpr int kSpan = 32 * 4 * kMaxPf;            // floats per warp span (max)
constexpr int kSpanPad = kSpan + kSpan / 32;      // +1 word per 32 (bank padding)

__device__ __forceinline__ int padi(int i) { return i + (i >> 5); }

struct GroupGeom {
    long long groups;       // rows * gpr
    int gpr;                // groups per row = row_words / 4
    int cols;
    int epg;                // elements per group = 4 * pf
};

// flat FP32 index of the first element of group g, and its valid element count
__device__ __forceinline__ void group_span(const GroupGeom& G, long long g, long long& flat,
                                           int& n) {
    const long long r = g / G.gpr;
    const int gw = int(g - r * G.gpr);
    const int e0 = gw * G.epg;
    flat = r * (long long)G.cols + e0;
    n = max(0, min(G.epg, G.cols - e0));
}

__global__ void __launch_bounds__(32 * kWarpsPerCta)
quantize_kernel(const float* __restrict__ x, uint4* __restrict__ out, GroupGeom G, Fmt f) {
    __shared__ float stage[kWarpsPerCta][kSpanPad];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sm = stage[warp];
    const long long nwarps = (long long)gridDim.x * kWarpsPerCta;
    for (long long g0 = ((long long)blockIdx.x * kWarpsPerCta + warp) * 32; g0 < G.groups;
         g0 += nwarps * 32) {
        const long long g = g0 + lane;
        long long flat0, flat_last;
        int n0, nl;
        group_span(G, g0, flat0, n0);
        const long long glast = min(g0 + 31, G.groups - 1);
        group_span(G, glast, flat_last, nl);
        const int span = int(flat_last + nl - flat0);
        for (int i = lane; i < span; i += 32) sm[padi(i)] = __ldcs(x + flat0 + i);
        __syncwarp();
        if (g < G.groups) {
            long long flat;
            int n;
            group_span(G, g, flat, n);
            const int base = int(flat - flat0);
            uint32_t w[4];
            with_pf(f.pf, [&](auto P) {
                constexpr int PF = decltype(P)::value;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float x[PF];
#pragma unroll
                    for (int j = 0; j < PF; ++j) {
                        const int e = k * PF + j;
                        x[j] = (e < n) ? sm[padi(base + e)] : 0.f;
                    }
                    w[k] = encode_word_t<PF>(x, f);
                }
            });
            __stcs(out + g, make_uint4(w[0], w[1], w[2], w[3]));
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(32 * kWarpsPerCta)
dequantize_kernel(const uint4* __restrict__ in, float* __restrict__ y, GroupGeom G, Fmt f) {
    __shared__ float stage[kWarpsPerCta][kSpanPad];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sm = stage[warp];
    const long long nwarps = (long long)gridDim.x * kWarpsPerCta;
    for (long long g0 = ((long long)blockIdx.x * kWarpsPerCta + warp) * 32; g0 < G.groups;
         g0 += nwarps * 32) {
        const long long g = g0 + lane;
        long long flat0, flat_last;
        int n0, nl;
        group_span(G, g0, flat0, n0);
        const long long glast = min(g0 + 31, G.groups - 1);
        group_span(G, glast, flat_last, nl);
        const int span = int(flat_last + nl - flat0);
        if (g < G.groups) {
            long long flat;
            int n;
            group_span(G, g, flat, n);
            const int base = int(flat - flat0);
            const uint4 v = __ldcs(in + g);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            with_pf(f.pf, [&](auto P) {
                constexpr int PF = decltype(P)::value;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float x[PF];
                    decode_word_t<PF>(w[k], x, f);
#pragma unroll
                    for (int j = 0; j < PF; ++j) {
                        const int e = k * PF + j;
                        if (e < n) sm[padi(base + e)] = x[j];
                    }
                }
            });
        }
        __syncwarp();
        for (int i = lane; i < span; i += 32) __stcs(y + flat0 + i, sm[padi(i)]);
        __syncwarp();
    }
}

int grid_for(long long groups, int sms) {
    const long long per_cta = 32LL * kWarpsPerCta;
    long long ctas = (groups + per_cta - 1) / per_cta;
    const long long cap = (long long)sms * 8;   // persistent-ish: 8 CTAs per SM
    if (ctas > cap) ctas = cap;
    return int(ctas < 1 ? 1 : ctas);
}

}  // namespace

cudaError_t launch_quantize(const Fmt& f, const float* x, size_t rows, size_t cols,
                            size_t row_words, uint32_t* packed, int sms, cudaStream_t s) {
    GroupGeom G{(long long)rows * (long long)(row_words / 4), int(row_words / 4), int(cols),
                4 * f.pf};
    if (G.groups == 0) return cudaSuccess;
    quantize_kernel<<<grid_for(G.groups, sms), 32 * kWarpsPerCta, 0, s>>>(
        x, reinterpret_cast<uint4*>(packed), G, f);
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const Fmt& f, const uint32_t* packed, size_t rows, size_t cols,
                              size_t row_words, float* y, int sms, cudaStream_t s) {
    GroupGeom G{(long long)rows * (long long)(row_words / 4), int(row_words / 4), int(cols),
                4 * f.pf};
    if (G.groups == 0) return cudaSuccess;
    dequantize_kernel<<<grid_for(G.groups, sms), 32 * kWarpsPerCta, 0, s>>>(
        reinterpret_cast<const uint4*>(packed), y, G, f);
    return cudaGetLastError();
}

}  // namespace vapr
