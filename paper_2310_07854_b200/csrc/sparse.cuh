// sparse.cuh -- N3: emit a tile of rows in the sparse sphere-tensor form
// (include/vapr.h "N3"; reading c42).
//
// One warp per row (rows warp, warp + kWarps, ...), a lane owns spheres lane
// and lane + 32 and holds their three codes in registers (fetched by the
// caller's get(r, s, c[3]): encoded from FP32 sums in the aggregation,
// extracted from dense words in vapr_sparsify).
//   A. bitmap = two ballots; words = ceil(3 popc / pf) (reciprocal multiply);
//   B. warp 0: prefix of the rows' word counts (shuffles); the tile's rows
//      go back to back from its own segment of the pool, word seg0 + tile *
//      kMaxRows * wmax (wmax = ceil(3S / pf), the worst case) -- no
//      allocation atomics, a deterministic layout -- and *used is counted
//      with one fire-and-forget reduction per tile;
//   C. per row: rank k = popc of the set spheres below; codes 3k + c are
//      staged in rank order in a per-warp shared buffer (plain stores), then
//      lane w builds word w from its pf codes and stores it (coalesced).
#pragma once
#include "common.cuh"

namespace vapr {

// A sphere's three values -> codes (one kind switch; hardware pair
// conversions where exact for all three, as encode_word_t; else generic).
__device__ __forceinline__ void encode3(float x0, float x1, float x2, const Fmt& f, uint32_t* c) {
    if ((__float_as_uint(x0) | __float_as_uint(x1) | __float_as_uint(x2)) == 0u) {
        c[0] = c[1] = c[2] = 0u;                      // +0 -> code 0 in every format
        return;
    }
    if (f.kind == KIND_IDENTITY) {
        c[0] = __float_as_uint(x0);
        c[1] = __float_as_uint(x1);
        c[2] = __float_as_uint(x2);
        return;
    }
    const uint32_t amax = max(__float_as_uint(x0) & 0x7fffffffu,
                              max(__float_as_uint(x1) & 0x7fffffffu, __float_as_uint(x2) & 0x7fffffffu));
    if (amax < f.hw_limit) {
        uint32_t p, q;
        switch (f.kind) {
            case KIND_F16: p = cvt_f16x2(x0, x1); q = cvt_f16x2(x2, 0.f);
                c[0] = p & 0xffffu; c[1] = p >> 16; c[2] = q & 0xffffu; return;
            case KIND_BF16: p = cvt_bf16x2(x0, x1); q = cvt_bf16x2(x2, 0.f);
                c[0] = p & 0xffffu; c[1] = p >> 16; c[2] = q & 0xffffu; return;
            case KIND_E4M3: p = cvt_e4m3x2(x0, x1); q = cvt_e4m3x2(x2, 0.f);
                c[0] = p & 0xffu; c[1] = (p >> 8) & 0xffu; c[2] = q & 0xffu; return;
            case KIND_E5M2: p = cvt_e5m2x2(x0, x1); q = cvt_e5m2x2(x2, 0.f);
                c[0] = p & 0xffu; c[1] = (p >> 8) & 0xffu; c[2] = q & 0xffu; return;
            case KIND_E2M1: p = cvt_e2m1x2(x0, x1); q = cvt_e2m1x2(x2, 0.f);
                c[0] = p & 0xfu; c[1] = (p >> 4) & 0xfu; c[2] = q & 0xfu; return;
            case KIND_E2M3: p = cvt_e2m3x2(x0, x1); q = cvt_e2m3x2(x2, 0.f);
                c[0] = p & 0x3fu; c[1] = (p >> 8) & 0x3fu; c[2] = q & 0x3fu; return;
            case KIND_E3M2: p = cvt_e3m2x2(x0, x1); q = cvt_e3m2x2(x2, 0.f);
                c[0] = p & 0x3fu; c[1] = (p >> 8) & 0x3fu; c[2] = q & 0x3fu; return;
            default: break;
        }
    }
    c[0] = encode_generic(x0, f);
    c[1] = encode_generic(x1, f);
    c[2] = encode_generic(x2, f);
}

template <int kMaxRows>
struct SparseTileSmem {
    unsigned long long m[kMaxRows];
    uint32_t words[kMaxRows];
    uint32_t off[kMaxRows];
};

// wbuf: shared, kWarps x wstride words (wstride >= 3S: one code each).  rcp =
// 65536 / pf + 1 (exact i / pf for i < 4096).  seg = the tile's first pool
// word (seg0 + tile * kMaxRows * wmax).  All threads of the CTA call this (it
// synchronises).  Rows r0 .. r0 + nr of mask / off are written.
template <int kMaxRows, int kWarps, class Get>
__device__ __forceinline__ void emit_sparse_rows(int nr, int S, const Fmt& f, uint32_t rcp,
                                                 SparseTileSmem<kMaxRows>& sm, uint32_t* wbuf,
                                                 int wstride, long long r0, uint32_t seg,
                                                 unsigned long long* __restrict__ mask,
                                                 uint32_t* __restrict__ off,
                                                 uint32_t* __restrict__ pool,
                                                 uint32_t* __restrict__ used, Get get) {
    constexpr int kRowsPerWarp = (kMaxRows + kWarps - 1) / kWarps;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t code[kRowsPerWarp][2][3];
    uint32_t bal[kRowsPerWarp][2];
    // A. codes, bitmaps, word counts
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; ++j) {
        const int r = warp + j * kWarps;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = lane + 32 * h;
            code[j][h][0] = code[j][h][1] = code[j][h][2] = 0u;
            if (r < nr && s < S) get(r, s, code[j][h]);
            bal[j][h] = __ballot_sync(0xffffffffu, (code[j][h][0] | code[j][h][1] | code[j][h][2]) != 0u);
        }
        if (r < nr && lane == 0) {
            const int n3 = 3 * (__popc(bal[j][0]) + __popc(bal[j][1]));
            sm.m[r] = (unsigned long long)bal[j][0] | ((unsigned long long)bal[j][1] << 32);
            sm.words[r] = (uint32_t)(((uint32_t)(n3 + f.pf - 1) * rcp) >> 16);
        }
    }
    __syncthreads();
    // B. the tile's pool range and the rows' offsets
    if (warp == 0) {
        const uint32_t w = lane < nr ? sm.words[lane] : 0u;
        uint32_t inc = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0 && total) atomicAdd(used, total);     // result unused: a reduction
        if (lane < nr) {
            sm.off[lane] = w ? seg + inc - w : 0u;
            mask[r0 + lane] = sm.m[lane];
            off[r0 + lane] = w ? seg + inc - w : 0u;
        }
    }
    __syncthreads();
    // C. pack and store
    uint32_t* wb = wbuf + warp * wstride;
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; ++j) {
        const int r = warp + j * kWarps;
        if (r >= nr) break;                           // warp-uniform
        const int n = (int)sm.words[r];
        if (n == 0) continue;
        const int ncode = 3 * (__popc(bal[j][0]) + __popc(bal[j][1]));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!((bal[j][h] >> lane) & 1u)) continue;
            const int k = (h ? __popc(bal[j][0]) : 0) + __popc(bal[j][h] & below);
            wb[3 * k] = code[j][h][0];
            wb[3 * k + 1] = code[j][h][1];
            wb[3 * k + 2] = code[j][h][2];
        }
        __syncwarp();
        uint32_t* dst = pool + sm.off[r];
        for (int w = lane; w < n; w += 32) {
            const int i0 = w * f.pf;
            uint32_t word = 0u;
            for (int q = 0; q < f.pf && i0 + q < ncode; ++q) word |= wb[i0 + q] << (q * f.t);
            dst[w] = word;
        }
        __syncwarp();
    }
}

}  // namespace vapr
