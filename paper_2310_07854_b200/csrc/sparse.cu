// sparse.cu -- N3: dense packed sphere tensor <-> sparse form (include/vapr.h
// "N3"; reading c42).
//
// sparsify: one CTA per tile of kRows rows; the dense rows are copied to
// shared memory (16-byte coalesced loads) and emit_sparse_rows (sparse.cuh)
// extracts each sphere's codes and writes the bitmaps, offsets and the
// tile's pool segment.
// densify: one thread per dense output word; each slot's sphere is looked up
// in the row's bitmap, its rank gives the code index in the row's pool range.
#include "common.cuh"
#include "kernels.cuh"
#include "sparse.cuh"

namespace vapr {

namespace {

constexpr int kRows = 16;
constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads)
sparsify_kernel(const Fmt f, const uint32_t* __restrict__ packed, long long rows, int cols, int W,
                uint32_t rcp, uint32_t wmax, unsigned long long* __restrict__ mask,
                uint32_t* __restrict__ off, uint32_t* __restrict__ pool,
                uint32_t* __restrict__ used) {
    extern __shared__ uint4 smem_s4[];
    uint32_t* rw = reinterpret_cast<uint32_t*>(smem_s4);    // [kRows * W] dense rows
    uint32_t* wbuf = rw + kRows * W;                         // [kWarps * cols] code buffers
    __shared__ SparseTileSmem<kRows> sm;
    const long long r0 = (long long)blockIdx.x * kRows;
    const int nr = (int)min((long long)kRows, rows - r0);
    const uint4* src = reinterpret_cast<const uint4*>(packed + r0 * W);
    for (int i = threadIdx.x; i < nr * W / 4; i += kThreads) smem_s4[i] = __ldcs(src + i);
    __syncthreads();
    emit_sparse_rows<kRows, kWarps>(nr, cols / 3, f, rcp, sm, wbuf, cols, r0,
                                    (uint32_t)blockIdx.x * kRows * wmax, mask, off, pool, used,
                                    [&](int r, int s, uint32_t* c) {
                                        const uint32_t* row = rw + r * W;
#pragma unroll
                                        for (int k = 0; k < 3; ++k) {
                                            const uint32_t e = 3u * s + k;
                                            const uint32_t w = (e * rcp) >> 16;
                                            c[k] = code_at(row[w], (int)(e - w * f.pf), f);
                                        }
                                    });
}

__global__ void __launch_bounds__(256)
densify_kernel(const Fmt f, const unsigned long long* __restrict__ mask,
               const uint32_t* __restrict__ off, const uint32_t* __restrict__ pool, long long rows,
               int cols, int W, uint32_t* __restrict__ packed) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * W) return;
    const long long r = i / W;
    const int w = (int)(i - r * W);
    const unsigned long long m = mask[r];
    uint32_t word = 0u;
    if (m) {
        const uint32_t o = off[r];
        for (int j = 0; j < f.pf; ++j) {
            const int e = w * f.pf + j;
            if (e >= cols) break;
            const int s = e / 3, c = e - 3 * s;
            if (!((m >> s) & 1ull)) continue;
            const int ci = 3 * __popcll(m & ((1ull << s) - 1ull)) + c;
            const uint32_t src = pool[o + ci / f.pf];
            word |= code_at(src, ci % f.pf, f) << (j * f.t);
        }
    }
    packed[i] = word;
}

}  // namespace

cudaError_t launch_sparsify(const Fmt& f, const uint32_t* packed, long long rows, int cols,
                            const SparseOut& o, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(o.used, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || rows <= 0) return e;
    const int W = row_words_of(f, cols);
    const size_t smem = sizeof(uint32_t) * (kRows * W + kWarps * cols);
    e = cudaFuncSetAttribute(sparsify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t rcp = 65536u / f.pf + 1u;
    const long long grid = (rows + kRows - 1) / kRows;
    const uint32_t wmax = (uint32_t)((cols + f.pf - 1) / f.pf);
    sparsify_kernel<<<(unsigned)grid, kThreads, smem, s>>>(f, packed, rows, cols, W, rcp, wmax,
                                                           o.mask, o.off, o.pool, o.used);
    return cudaGetLastError();
}

cudaError_t launch_densify(const Fmt& f, const SparseIn& in, long long rows, int cols,
                           uint32_t* packed, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const int W = row_words_of(f, cols);
    const long long n = rows * W;
    densify_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(f, in.mask, in.off, in.pool, rows,
                                                               cols, W, packed);
    return cudaGetLastError();
}

}  // namespace vapr
