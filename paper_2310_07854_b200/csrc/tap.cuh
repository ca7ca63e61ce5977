// tap.cuh -- TEST-ONLY debug tap (SURVEY.md §8(b) "Test-only export", §8(c)
// parity contract (i)): with -DVAPR_DEBUG_TAP, vapr_debug_tap(ctx, slot, dst)
// makes the next launch that produces `slot` also write that slot's FP32
// pre-quantisation values to dst [rows, cols] (zero where the kernel encodes
// nothing), so the oracle codec of those values can be checked against the
// packed words bit for bit.  Release builds compile none of this (no symbol,
// no branch on the hot path).
#pragma once
#ifdef VAPR_DEBUG_TAP
#include <cuda_runtime.h>

namespace vapr {

// armed host pointers, one per slot (api.cu); a launcher consumes its slot's
extern float* g_tap_host[5];

}  // namespace vapr

// each translation unit gets its own device table (no -rdc): the launchers in
// that unit set it around their launch
static __device__ float* d_tap[5];

namespace vapr {
namespace {

// arm: move the host pointer of `slot` into this unit's device table (zeroing
// the destination first); returns the pointer (nullptr when not armed)
inline float* tap_arm(int slot, long long rows, int cols, cudaStream_t s) {
    float* p = g_tap_host[slot];
    g_tap_host[slot] = nullptr;
    if (p) cudaMemsetAsync(p, 0, sizeof(float) * (size_t)rows * cols, s);
    cudaMemcpyToSymbolAsync(d_tap, &p, sizeof(p), sizeof(float*) * slot, cudaMemcpyHostToDevice, s);
    return p;
}

inline void tap_disarm(int slot, cudaStream_t s) {
    float* z = nullptr;
    cudaMemcpyToSymbolAsync(d_tap, &z, sizeof(z), sizeof(float*) * slot, cudaMemcpyHostToDevice, s);
}

}  // namespace
}  // namespace vapr

#define VAPR_TAP(slot, idx, value)                        \
    do {                                                  \
        if (d_tap[slot]) d_tap[slot][idx] = (value);      \
    } while (0)
#else
#define VAPR_TAP(slot, idx, value) \
    do {                           \
    } while (0)
#endif
