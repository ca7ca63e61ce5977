// aggregate.cu -- a5: grad_out_spheres = Q_gos(dequant(closest_pt[_swept]) +
// dequant(out_vec)), elementwise over pose rows.  P:162 step (4)
// "Aggregating the costs"; P:189 ("the input of backward kinematics:
// grad_out_spheres").  The two inputs and the output may each have a
// different format and hence a different packing factor.
//
// One CTA per tile of kRows pose rows.  Both input tiles are streamed into
// shared memory with 16-byte coalesced loads, then three word-parallel passes
// (each templated on its own packing factor): decode closest_pt into an FP32
// tile, decode out_vec and add (all-zero words skipped: "sparsity-aware
// computation by skipping zero computations"), encode the sums into packed
// grad_out_spheres words (hardware cvt where exact) with coalesced stores.
// The sum is the same single FP32 addition per element as before, so the
// result is bit-identical to decode(cp) + decode(ov) -> encode.
//
// SPARSE (N3, VAPR_OPT_SPARSE): the third pass is emit_sparse_rows (a warp
// per row, a lane per sphere: encode3 -- the same codes as encode_word_t --
// then bitmap, rank and packing) writing the tile in the sparse form.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "sparse.cuh"
#include "tap.cuh"

namespace vapr {

namespace {

#ifndef VAPR_AGG_ROWS
#define VAPR_AGG_ROWS 16
#endif
constexpr int kRows = VAPR_AGG_ROWS;
#ifndef VAPR_AGG_THREADS
#define VAPR_AGG_THREADS 128
#endif
constexpr int kThreads = VAPR_AGG_THREADS;
#ifndef VAPR_AGG_SW                // sparse aggregation: per-thread staged words per input
#define VAPR_AGG_SW 16
#endif
constexpr int kSW = VAPR_AGG_SW;
#ifndef VAPR_AGG_ROWS_BELOW       // vapr_cost_grad sparse aggregation: warp-per-row form below
#define VAPR_AGG_ROWS_BELOW 65536
#endif

// Decode the packed tile `src` (rows of W words, pf values per word) into the
// FP32 tile x (stride xs): x = value (ADD = false) or x += value (ADD = true).
// One thread per word.  Pass 1 (ADD = false) raises *negz when it decodes a
// -0.  Pass 2 skips an all-zero word (x + +0 = x) unless the tile holds a -0
// (x = -0 needs the add: -0 + +0 = +0).
template <int PF, bool ADD>
__device__ __forceinline__ void decode_tile(const uint32_t* src, int W, int nr, int cols,
                                            uint32_t rw, float* x, int xs, const Fmt& f,
                                            int* negz) {
    const bool skip_zero = ADD ? (*negz == 0) : true;
    for (int i = threadIdx.x; i < nr * W; i += kThreads) {
        const int r = int((uint32_t(i) * rw) >> 24), w = i - r * W;
        const uint32_t v = src[i];
        const int e0 = w * PF;
        float* xr = x + r * xs + e0;
        if (v == 0u && skip_zero) {
            if (!ADD) {
#pragma unroll
                for (int j = 0; j < PF; ++j) xr[j] = 0.f;
            }
            continue;
        }
        float d[PF];
        decode_word_t<PF>(v, d, f);
        bool nz = false;
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            if (!ADD) nz |= __float_as_uint(d[j]) == 0x80000000u;
            xr[j] = ADD ? xr[j] + d[j] : d[j];
        }
        if (!ADD && nz) *negz = 1;
    }
}

template <bool SPARSE>
__global__ void __launch_bounds__(kThreads)
aggregate_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int cols, int Wc, int Wo, int Wg,
                 const uint32_t* __restrict__ cp, const uint32_t* __restrict__ ov,
                 long long rows, uint32_t* __restrict__ gos, uint32_t rw_c, uint32_t rw_o,
                 uint32_t rw_g, int xs, const SparseOut sp) {
    pdl_wait();         // vapr_cost_grad: the collision passes / cost reduction are complete
    extern __shared__ uint4 smem_a[];
    uint32_t* sc = reinterpret_cast<uint32_t*>(smem_a);     // [kRows * Wc]
    uint32_t* so = sc + kRows * Wc;                         // [kRows * Wo]
    float* x = reinterpret_cast<float*>(so + kRows * Wo);   // [kRows * xs] FP32 sums
    __shared__ int negz;
    const long long r0 = (long long)blockIdx.x * kRows;
    const int nr = (int)min((long long)kRows, rows - r0);
    const int tid = threadIdx.x;
    if (tid == 0) negz = 0;
    {
        const uint4* gc = reinterpret_cast<const uint4*>(cp + r0 * Wc);
        const uint4* go = reinterpret_cast<const uint4*>(ov + r0 * Wo);
        const int qc = Wc / 4, qo = Wo / 4;
#pragma unroll 4
        for (int i = tid; i < nr * qc; i += kThreads) reinterpret_cast<uint4*>(sc)[i] = __ldcs(gc + i);
#pragma unroll 4
        for (int i = tid; i < nr * qo; i += kThreads) reinterpret_cast<uint4*>(so)[i] = __ldcs(go + i);
    }
    __syncthreads();
    with_pf(fcp.pf, [&](auto Pc) {
        decode_tile<decltype(Pc)::value, false>(sc, Wc, nr, cols, rw_c, x, xs, fcp, &negz);
    });
    __syncthreads();
    with_pf(fov.pf, [&](auto Pc) {
        decode_tile<decltype(Pc)::value, true>(so, Wo, nr, cols, rw_o, x, xs, fov, &negz);
    });
    __syncthreads();
#ifdef VAPR_DEBUG_TAP
    for (int i = tid; i < nr * cols; i += kThreads) {
        const int r = i / cols, e = i - r * cols;
        VAPR_TAP(1, (r0 + r) * cols + e, x[r * xs + e]);
    }
#endif
    if constexpr (SPARSE) {
        __shared__ SparseTileSmem<kRows> sm;
        uint32_t* wbuf = reinterpret_cast<uint32_t*>(x + kRows * xs);   // [kWarps * cols]
        emit_sparse_rows<kRows, kThreads / 32>(nr, cols / 3, fg, sp.rcp, sm, wbuf, cols, r0,
                                               sp.seg0 + (uint32_t)blockIdx.x * kRows * sp.wmax, sp.mask,
                                               sp.off, sp.pool, sp.used,
                                               [&](int r, int s, uint32_t* c) {
                                                   const float* xr = x + r * xs + 3 * s;
                                                   encode3(xr[0], xr[1], xr[2], fg, c);
                                               });
        return;
    }
    // slots past the last element that the encode pass reads: +0, whatever
    // the inputs' padding held
    const int tail = Wg * fg.pf - cols;
    for (int i = tid; i < nr * tail; i += kThreads) {
        const int r = i / tail;
        x[r * xs + cols + (i - r * tail)] = 0.f;
    }
    __syncthreads();
    uint32_t* dst = gos + r0 * Wg;
    with_pf(fg.pf, [&](auto Pc) {
        constexpr int PF = decltype(Pc)::value;
        for (int i = tid; i < nr * Wg; i += kThreads) {
            const int r = int((uint32_t(i) * rw_g) >> 24), w = i - r * Wg;
            const int e0 = w * PF;
            float v[PF];
#pragma unroll
            for (int j = 0; j < PF; ++j) v[j] = x[r * xs + e0 + j];
            __stcs(dst + i, encode_word_t<PF>(v, fg));
        }
    });
}

// N3 (VAPR_OPT_SPARSE): closest_pt[_swept] and out_vec in the sparse form
// (per-row sphere bitmap, the non-zero spheres' codes packed in ascending
// sphere order at pool + row * ceil(cols / pf)) -> grad_out_spheres in the
// sparse form.  A thread per row: a row with both bitmaps empty (most rows)
// costs two 8-byte loads; otherwise the union of the two bitmaps in ascending
// order, each element dec(cp) + dec(ov) in FP32 (+0 for a sphere absent from
// one side: its dense value), encode3, and the codes of the spheres with a
// non-zero code packed as they come.
__global__ void __launch_bounds__(128)
aggregate_sparse_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int wc, int wo,
                        const uint32_t* __restrict__ cp, const unsigned long long* __restrict__ cpm,
                        const uint32_t* __restrict__ ov, const unsigned long long* __restrict__ ovm,
                        long long rows, uint32_t rcp_c, uint32_t rcp_o, const SparseOut sp) {
    pdl_wait();         // vapr_cost_grad: the collision passes / cost reduction are complete
    // the row's pool words (both inputs) staged in a per-thread shared row
    // first -- independent loads, all in flight -- instead of a global load
    // per code inside the sphere loop (rows longer than kSW words: direct)
    __shared__ uint32_t sbuf[128 * (2 * kSW + 1)];
    uint32_t* mine = sbuf + threadIdx.x * (2 * kSW + 1);        // odd stride: conflict-free
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nw = 0u;
    if (p < rows) {
        const unsigned long long mc = __ldcs(cpm + p), mo = __ldcs(ovm + p);
        unsigned long long m = mc | mo, mg = 0ull;
        const uint32_t o = sp.seg0 + (uint32_t)p * sp.wmax;
        if (m) {
            const uint32_t ncw = ((uint32_t)(3 * __popcll(mc) + fcp.pf - 1) * rcp_c) >> 16;
            const uint32_t now = ((uint32_t)(3 * __popcll(mo) + fov.pf - 1) * rcp_o) >> 16;
            const uint32_t* rc = cp + p * wc;
            const uint32_t* ro = ov + p * wo;
            if (ncw <= kSW && now <= kSW) {
#pragma unroll 4
                for (uint32_t w = 0; w < ncw; ++w) mine[w] = __ldcs(rc + w);
#pragma unroll 4
                for (uint32_t w = 0; w < now; ++w) mine[kSW + w] = __ldcs(ro + w);
                rc = mine;
                ro = mine + kSW;
            }
            uint32_t word = 0u;
            int q = 0;
            int kc = 0, ko = 0;                       // codes consumed from each side
            while (m) {
                const int s = __ffsll((long long)m) - 1;
                m &= m - 1;
                const bool inc = (mc >> s) & 1ull, ino = (mo >> s) & 1ull;
                float x[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float a = 0.f, b = 0.f;
                    if (inc) {
                        const uint32_t e = kc + c, w = (e * rcp_c) >> 16;      // e / pf
                        a = decode_sp(code_at(rc[w], int(e - w * fcp.pf), fcp), fcp);
                    }
                    if (ino) {
                        const uint32_t e = ko + c, w = (e * rcp_o) >> 16;
                        b = decode_sp(code_at(ro[w], int(e - w * fov.pf), fov), fov);
                    }
                    x[c] = a + b;
                }
                kc += inc ? 3 : 0;
                ko += ino ? 3 : 0;
                uint32_t c3[3];
                encode3(x[0], x[1], x[2], fg, c3);
                if (!(c3[0] | c3[1] | c3[2])) continue;
                mg |= 1ull << s;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    word |= (fg.t == 32) ? c3[c] : (c3[c] << (q * fg.t));
                    if (++q == fg.pf) {
                        sp.pool[o + nw++] = word;
                        word = 0u;
                        q = 0;
                    }
                }
            }
            if (q) sp.pool[o + nw++] = word;
        }
        sp.mask[p] = mg;
        sp.off[p] = nw ? o : 0u;
    }
    // the words in use: one reduction per warp
#pragma unroll
    for (int d = 16; d; d >>= 1) nw += __shfl_xor_sync(0xffffffffu, nw, d);
    if ((threadIdx.x & 31) == 0 && nw) atomicAdd(sp.used, nw);
}

// The same sums, a warp per row and a lane per sphere (emit_sparse_rows):
// every code load of a row is in flight at once -- the latency form for
// small batches, where the thread-per-row kernel's serial sphere loop (a
// dependent global load per sphere) is the critical path.  Bit-identical
// (the same a + b and encode3); pool layout: the tile segments of
// emit_sparse_rows (readers go through off[]).
constexpr int kSmRows = 16, kSmWarps = 4;
__global__ void __launch_bounds__(32 * kSmWarps)
aggregate_sparse_rows_kernel(const Fmt fcp, const Fmt fov, const Fmt fg, int cols, int wc, int wo,
                             const uint32_t* __restrict__ cp, const unsigned long long* __restrict__ cpm,
                             const uint32_t* __restrict__ ov, const unsigned long long* __restrict__ ovm,
                             long long rows, uint32_t rcp_c, uint32_t rcp_o, const SparseOut sp) {
    pdl_wait();         // vapr_cost_grad: the collision passes / cost reduction are complete
    __shared__ SparseTileSmem<kSmRows> sm;
    __shared__ uint32_t wbuf[kSmWarps * 3 * 64];
    __shared__ unsigned long long smc[kSmRows], smo[kSmRows];
    const long long r0 = (long long)blockIdx.x * kSmRows;
    const int nr = (int)min((long long)kSmRows, rows - r0);
    if ((int)threadIdx.x < nr) {
        smc[threadIdx.x] = __ldcs(cpm + r0 + threadIdx.x);
        smo[threadIdx.x] = __ldcs(ovm + r0 + threadIdx.x);
    }
    __syncthreads();
    const uint32_t seg = sp.seg0 + (uint32_t)r0 * sp.wmax;
    emit_sparse_rows<kSmRows, kSmWarps>(
        nr, cols / 3, fg, sp.rcp, sm, wbuf, 3 * 64, r0, seg, sp.mask + 0, sp.off + 0, sp.pool,
        sp.used, [&](int r, int s, uint32_t* c) {
            const unsigned long long mc = smc[r], mo = smo[r], bit = 1ull << s;
            if (!((mc | mo) & bit)) return;
            const long long p = r0 + r;
            float x[3];
            const int kc = 3 * __popcll(mc & (bit - 1ull)), ko = 3 * __popcll(mo & (bit - 1ull));
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                float a = 0.f, b = 0.f;
                if (mc & bit) {
                    const uint32_t e = kc + q, w = (e * rcp_c) >> 16;
                    a = decode_sp(code_at(__ldcs(cp + p * wc + w), int(e - w * fcp.pf), fcp), fcp);
                }
                if (mo & bit) {
                    const uint32_t e = ko + q, w = (e * rcp_o) >> 16;
                    b = decode_sp(code_at(__ldcs(ov + p * wo + w), int(e - w * fov.pf), fov), fov);
                }
                x[q] = a + b;
            }
            encode3(x[0], x[1], x[2], fg, c);
        });
}

}  // namespace

cudaError_t launch_aggregate_sparse(const Fmt& fcp, const Fmt& fov, const Fmt& fgos, int cols,
                                    const uint32_t* cp_pool, const unsigned long long* cpm,
                                    const uint32_t* ov_pool, const unsigned long long* ovm,
                                    long long rows, const SparseOut& sparse, cudaStream_t s,
                                    bool pdl) {
    if (rows <= 0) return cudaSuccess;
    SparseOut spo = sparse;
    spo.wmax = (uint32_t)((cols + fgos.pf - 1) / fgos.pf);
    spo.rcp = 65536u / fgos.pf + 1u;
    const int wc = (cols + fcp.pf - 1) / fcp.pf, wo = (cols + fov.pf - 1) / fov.pf;
    if (rows < VAPR_AGG_ROWS_BELOW) {       // small batch: latency form
        const long long g = (rows + kSmRows - 1) / kSmRows;
        return launch_k(aggregate_sparse_rows_kernel, dim3((unsigned)g), dim3(32 * kSmWarps), 0, s,
                        pdl, fcp, fov, fgos, cols, wc, wo, cp_pool, cpm, ov_pool, ovm, rows,
                        65536u / fcp.pf + 1u, 65536u / fov.pf + 1u, spo);
    }
    const long long grid = (rows + 127) / 128;
    return launch_k(aggregate_sparse_kernel, dim3((unsigned)grid), dim3(128), 0, s, pdl, fcp, fov,
                    fgos, wc, wo, cp_pool, cpm, ov_pool, ovm, rows, 65536u / fcp.pf + 1u,
                    65536u / fov.pf + 1u, spo);
}

cudaError_t launch_aggregate(const Fmt& fcp, const Fmt& fov, const Fmt& fgos, int cols,
                             const uint32_t* cp, const uint32_t* ov, long long rows,
                             uint32_t* gos, cudaStream_t s, const SparseOut* sparse, bool pdl) {
    if (rows <= 0) return cudaSuccess;
    const int Wc = row_words_of(fcp, cols), Wo = row_words_of(fov, cols),
              Wg = row_words_of(fgos, cols);
    // i / W for i < kRows * W via 24-bit reciprocals: exact while
    // kRows W^2 < 2^24, and i * rw fits 32 bits
    const uint32_t rw_c = (1u << 24) / Wc + 1u, rw_o = (1u << 24) / Wo + 1u,
                   rw_g = (1u << 24) / Wg + 1u;
    for (int Wx : {Wc, Wo, Wg})
        if ((long long)kRows * Wx * Wx >= (1 << 24) ||
            (long long)kRows * Wx * ((1u << 24) / Wx + 1u) >= (1ll << 32))
            return cudaErrorInvalidValue;
    // FP32 tile wide enough for every word of all three rows (the padding
    // slots hold +0), odd stride: the word-parallel passes spread over banks
    const int xs = std::max(Wc * fcp.pf, std::max(Wo * fov.pf, Wg * fgos.pf)) | 1;
    size_t smem = sizeof(uint32_t) * kRows * (Wc + Wo) + sizeof(float) * kRows * xs;
    if (sparse) smem += sizeof(uint32_t) * (kThreads / 32) * cols;  // per-warp code buffers
    auto kern = sparse ? aggregate_kernel<true> : aggregate_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    SparseOut spo{};
    if (sparse) {
        spo = *sparse;
        spo.wmax = (uint32_t)((cols + fgos.pf - 1) / fgos.pf);
        spo.rcp = 65536u / fgos.pf + 1u;
    }
    const long long grid = (rows + kRows - 1) / kRows;
#ifdef VAPR_DEBUG_TAP
    const bool tapped = tap_arm(1, rows, cols, s) != nullptr;
#endif
    e = launch_k(kern, dim3((unsigned)grid), dim3(kThreads), smem, s, pdl, fcp, fov, fgos, cols, Wc,
                 Wo, Wg, cp, ov, rows, gos, rw_c, rw_o, rw_g, xs, spo);
    if (e != cudaSuccess) return e;
#ifdef VAPR_DEBUG_TAP
    if (tapped) tap_disarm(1, s);
#endif
    return cudaGetLastError();
}

}  // namespace vapr
