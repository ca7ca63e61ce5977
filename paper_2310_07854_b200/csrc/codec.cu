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
//
// Fast path (cols % 4 == 0, 16-byte aligned arrays -- every group then starts
// on a 16-byte boundary of the FP32 array): no staging, a thread per group
// moves its 4*pf FP32 values with pf 16-byte loads / stores of its own, and
// E8M23 is a plain 16-byte copy.
#include <algorithm>

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

// ---- fast path: cols % 4 == 0 ------------------------------------------------
// group -> (first element, count) with a 32-bit row division when the group
// count fits (the usual case), 64-bit otherwise
__device__ __forceinline__ void group_span_fast(const GroupGeom& G, long long g, long long& flat,
                                                int& n) {
    if (G.groups < (1ll << 32)) {
        const uint32_t r = uint32_t(g) / uint32_t(G.gpr);
        const int e0 = int(uint32_t(g) - r * uint32_t(G.gpr)) * G.epg;
        flat = (long long)r * G.cols + e0;
        n = max(0, min(G.epg, G.cols - e0));
    } else {
        group_span(G, g, flat, n);
    }
}

// A warp's 32 consecutive groups cover one contiguous, 16-byte aligned span
// of the FP32 array (rows are contiguous, a partial group ends a row and has a
// multiple of 4 elements).  The span moves between HBM and a per-warp shared
// buffer as coalesced 16-byte accesses (lane i takes float4 i, i + 32, ...);
// a lane reads / writes its group's float4s in the buffer, which inserts one
// float4 of padding per 8 so that both access patterns are conflict-free.
constexpr int kAWarps = 8;
constexpr int kAF4 = 32 * kMaxPf;                      // float4 per span (max: 32 groups x pf)
__device__ __forceinline__ int pad4(int i) { return i + (i >> 3); }

__global__ void __launch_bounds__(32 * kAWarps)
dequantize_aligned_kernel(const uint4* __restrict__ in, float4* __restrict__ y, GroupGeom G, Fmt f) {
    __shared__ float4 stage[kAWarps][kAF4 + kAF4 / 8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4* sm = stage[warp];
    const long long nw = (long long)gridDim.x * kAWarps;
    with_pf(f.pf, [&](auto P) {
        constexpr int PF = decltype(P)::value;
        // the next span's packed group is loaded one iteration ahead (its
        // latency overlaps this span's decode and stores)
        long long g0 = ((long long)blockIdx.x * kAWarps + warp) * 32;
        uint4 qn = (g0 + lane < G.groups) ? __ldcs(in + g0 + lane) : make_uint4(0u, 0u, 0u, 0u);
        for (; g0 < G.groups; g0 += nw * 32) {
            const uint4 q = qn;
            {
                const long long gn = g0 + nw * 32 + lane;
                if (gn < G.groups) qn = __ldcs(in + gn);
            }
            long long flat0, flat_last, flat;
            int n0, nl, n;
            group_span_fast(G, g0, flat0, n0);
            const long long glast = min(g0 + 31, G.groups - 1);
            group_span_fast(G, glast, flat_last, nl);
            const int span4 = int(flat_last + nl - flat0) >> 2;
            const long long g = g0 + lane;
            if (g < G.groups) {
                group_span_fast(G, g, flat, n);
                float v[4 * PF];
                if constexpr (PF == 2) {
                    decode_group_t<2>(q, v, f);
                } else {
                    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) decode_word_t<PF>(w[k], v + k * PF, f);
                }
                const int b4 = int(flat - flat0) >> 2;
#pragma unroll
                for (int k = 0; k < PF; ++k)
                    if (4 * k < n) sm[pad4(b4 + k)] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            }
            __syncwarp();
            float4* dst = y + (flat0 >> 2);
            for (int i = lane; i < span4; i += 32) __stcs(dst + i, sm[pad4(i)]);
            __syncwarp();
        }
    });
}

// Direct variants (no staging): a thread moves its group's pf float4s with
// its own 16-byte accesses -- faster for the wide formats (pf <= 3), whose
// groups are short; quantize's loads go through L1 (each 32-byte sector is
// read by consecutive lanes' loads).
__global__ void __launch_bounds__(256)
quantize_direct_kernel(const float4* __restrict__ x, uint4* __restrict__ out, GroupGeom G, Fmt f) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    with_pf(f.pf, [&](auto P) {
        constexpr int PF = decltype(P)::value;
        for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < G.groups; g += stride) {
            long long flat;
            int n;
            group_span_fast(G, g, flat, n);
            const float4* src = x + (flat >> 2);
            float v[4 * PF];
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const float4 q = (4 * k < n) ? __ldg(src + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = encode_word_t<PF>(v + k * PF, f);
            __stcs(out + g, make_uint4(w[0], w[1], w[2], w[3]));
        }
    });
}

#ifndef VAPR_DQ_DIRECT_MAXPF      // dequantise: formats with pf up to this use the direct kernel
#define VAPR_DQ_DIRECT_MAXPF 2
#endif
#ifndef VAPR_DQ_U2
#define VAPR_DQ_U2 2                // 16-bit formats: groups per thread per iteration
#endif                              // (E8M7 0.75 -> 0.87 of the copy peak; pf 3: 1 is faster)
__global__ void __launch_bounds__(256)
dequantize_direct_kernel(const uint4* __restrict__ in, float4* __restrict__ y, GroupGeom G, Fmt f) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    with_pf(f.pf, [&](auto P) {
        constexpr int PF = decltype(P)::value;
        constexpr int VAPR_DQ_U = (PF == 2) ? VAPR_DQ_U2 : 1;
        for (long long g0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; g0 < G.groups;
             g0 += stride * VAPR_DQ_U) {
            uint4 q[VAPR_DQ_U];
#pragma unroll
            for (int u = 0; u < VAPR_DQ_U; ++u) {
                const long long g = g0 + u * stride;
                q[u] = (g < G.groups) ? __ldcs(in + g) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < VAPR_DQ_U; ++u) {
                const long long g = g0 + u * stride;
                if (g >= G.groups) break;
                long long flat;
                int n;
                group_span_fast(G, g, flat, n);
                float v[4 * PF];
                if constexpr (PF == 2) {
                    decode_group_t<2>(q[u], v, f);
                } else {
                    const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) decode_word_t<PF>(w[k], v + k * PF, f);
                }
                float4* dst = y + (flat >> 2);
#pragma unroll
                for (int k = 0; k < PF; ++k)
                    if (4 * k < n) __stcs(dst + k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
            }
        }
    });
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
    if (cols % 4 == 0) {
        if (f.kind == KIND_IDENTITY)              // E8M23: the packed rows are the FP32 rows
            return cudaMemcpyAsync(packed, x, sizeof(float) * rows * cols, cudaMemcpyDeviceToDevice, s);
        const long long blocks = std::min<long long>((G.groups + 255) / 256, (long long)sms * 16);
        quantize_direct_kernel<<<(unsigned)std::max(1LL, blocks), 256, 0, s>>>(
            reinterpret_cast<const float4*>(x), reinterpret_cast<uint4*>(packed), G, f);
        return cudaGetLastError();
    }
    quantize_kernel<<<grid_for(G.groups, sms), 32 * kWarpsPerCta, 0, s>>>(
        x, reinterpret_cast<uint4*>(packed), G, f);
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const Fmt& f, const uint32_t* packed, size_t rows, size_t cols,
                              size_t row_words, float* y, int sms, cudaStream_t s) {
    GroupGeom G{(long long)rows * (long long)(row_words / 4), int(row_words / 4), int(cols),
                4 * f.pf};
    if (G.groups == 0) return cudaSuccess;
    if (cols % 4 == 0) {
        if (f.kind == KIND_IDENTITY)
            return cudaMemcpyAsync(y, packed, sizeof(float) * rows * cols, cudaMemcpyDeviceToDevice, s);
        if (f.pf <= VAPR_DQ_DIRECT_MAXPF) {
            const long long blocks = std::min<long long>((G.groups + 255) / 256, (long long)sms * 16);
            dequantize_direct_kernel<<<(unsigned)std::max(1LL, blocks), 256, 0, s>>>(
                reinterpret_cast<const uint4*>(packed), reinterpret_cast<float4*>(y), G, f);
        } else {
            const long long blocks = std::min<long long>((G.groups + 32 * kAWarps - 1) / (32 * kAWarps),
                                                         (long long)sms * 6);
            dequantize_aligned_kernel<<<(unsigned)std::max(1LL, blocks), 32 * kAWarps, 0, s>>>(
                reinterpret_cast<const uint4*>(packed), reinterpret_cast<float4*>(y), G, f);
        }
        return cudaGetLastError();
    }
    dequantize_kernel<<<grid_for(G.groups, sms), 32 * kWarpsPerCta, 0, s>>>(
        reinterpret_cast<const uint4*>(packed), y, G, f);
    return cudaGetLastError();
}

}  // namespace vapr
