// lbfgs.cu -- N1: the optimiser steps around the rollout.
// "(1) Given N, step scales of step direction ... (6) Use line search to pick
// one from N. (7) Lastly, compute step direction (L-BFGS) and buffer
// updates"; PAPER.md:86 (the L-BFGS step-direction kernel).  Readings c29-c33
// (DESIGN.md §3): FIFO history of (s, y) pairs kept when s.y > eps, two-loop
// recursion with gamma = s.y / y.y of the newest pair, argmin line search
// with ties to the smaller scale and a strict-improvement guard, history
// cleared (or the rejected direction shrunk tenfold) after a failed search.
//
// candidates_kernel: the N x B line-search batch, x + s_n d, one rounding per
//   operation (fl(x + fl(s d))), float4-vectorised, HBM-bound.
// lbfgs_step_kernel: LPI lanes per batch item (the smallest power of two >= D,
//   at most 32: IKO's D = 7 packs four items per warp); the item's D-vectors
//   live in registers, every dot product is a sub-group reduction, the history
//   is streamed twice (two-loop recursion) with coalesced loads.
#include "common.cuh"
#include "kernels.cuh"

namespace vapr {

namespace {

constexpr int kMaxPerLane = 16;        // D <= 512
constexpr int kStepWarps = 4;

// grid.y = the scale index n: cand[n] = fl(x + fl(s_n d)), no index division
__global__ void candidates_kernel(const float* __restrict__ x, const float* __restrict__ d,
                                  long long BD, const __grid_constant__ LbfgsScales sc,
                                  float* __restrict__ cand) {
    const int n = blockIdx.y;
    const float s = sc.s[n];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if ((BD & 3) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* d4 = reinterpret_cast<const float4*>(d);
        float4* c4 = reinterpret_cast<float4*>(cand + n * BD);
        for (long long i = i0; i < (BD >> 2); i += stride) {
            const float4 xv = __ldg(x4 + i), dv = __ldg(d4 + i);
            __stcs(c4 + i, make_float4(__fadd_rn(xv.x, __fmul_rn(s, dv.x)),
                                       __fadd_rn(xv.y, __fmul_rn(s, dv.y)),
                                       __fadd_rn(xv.z, __fmul_rn(s, dv.z)),
                                       __fadd_rn(xv.w, __fmul_rn(s, dv.w))));
        }
    } else {
        float* c = cand + n * BD;
        for (long long i = i0; i < BD; i += stride)
            c[i] = __fadd_rn(__ldg(x + i), __fmul_rn(s, __ldg(d + i)));
    }
}

// sum / max over the LPI lanes of a sub-group (xor shuffles stay inside it)
template <int LPI>
__device__ __forceinline__ float grp_sum(float v) {
#pragma unroll
    for (int o = LPI / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, LPI);
    return v;
}
template <int LPI>
__device__ __forceinline__ int grp_max(int v) {
#pragma unroll
    for (int o = LPI / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o, LPI));
    return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One sub-group of LPI lanes per batch item (32 / LPI items per warp; LPI =
// the smallest power of two >= D, at most 32), its D-vectors in registers
// (element i = sub-lane + LPI k).  Every shuffle is executed by the whole
// warp: branches between the items of a warp are predicated, loop bounds are
// warp maxima.
template <int LPI>
__global__ void __launch_bounds__(32 * kStepWarps)
lbfgs_step_kernel(int B, int D, int N, const __grid_constant__ LbfgsScales sc,
                  const float* __restrict__ cand_cost,
                  const float* __restrict__ cand_grad, float* __restrict__ x,
                  float* __restrict__ g, float* __restrict__ cost, float* __restrict__ d,
                  float* __restrict__ hs, float* __restrict__ hy, float* __restrict__ hrho,
                  int32_t* __restrict__ hcount, int32_t* __restrict__ hhead,
                  int32_t* __restrict__ chosen, int m, float eps,
                  const uint8_t* __restrict__ fixed) {
    constexpr int G = 32 / LPI;                    // items per warp
    constexpr int KPL = (LPI == 32) ? kMaxPerLane : 1;   // LPI < 32 only when D <= LPI
    __shared__ float s_alpha[kStepWarps][G][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int sub = lane / LPI, sl = lane % LPI;
    const int b = (blockIdx.x * kStepWarps + wib) * G + sub;
    const bool valid = b < B;
    if (__all_sync(0xffffffffu, !valid)) return;
    const long long o = (long long)(valid ? b : 0) * D;
    auto each = [&](auto&& f) {
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
            const int i = sl + LPI * k;
            if (valid && i < D) f(k, i);
        }
    };

    // (6) line search: argmin over the candidates, ties to the smaller scale,
    // strict improvement on the current cost required (NaN never improves)
    float best = valid ? cost[b] : 0.f;
    int nb = -1;
    for (int n0 = 0; n0 < N; n0 += LPI) {
        const int n = n0 + sl;
        const float c = (valid && n < N) ? cand_cost[(long long)n * B + b] : 0.f;
        const bool ok = valid && n < N && c < best;
        float cm = ok ? c : __int_as_float(0x7f800000);
        int im = ok ? n : 0x7fffffff;
#pragma unroll
        for (int off = LPI / 2; off > 0; off >>= 1) {
            const float c2 = __shfl_xor_sync(0xffffffffu, cm, off, LPI);
            const int i2 = __shfl_xor_sync(0xffffffffu, im, off, LPI);
            if (c2 < cm || (c2 == cm && i2 < im)) {
                cm = c2;
                im = i2;
            }
        }
        if (im != 0x7fffffff) {
            best = cm;
            nb = im;
        }
    }
    if (valid && sl == 0 && chosen) chosen[b] = nb;

    int count = valid ? hcount[b] : 0, head = valid ? hhead[b] : 0;
    const bool acc = valid && nb >= 0;
    if (valid && nb < 0) {
        // c32: no improvement -> clear a non-empty history (next d = -g), or
        // shrink an already steepest-descent direction tenfold
        if (count > 0) {
            each([&](int, int i) { d[o + i] = (fixed && fixed[i]) ? 0.f : -g[o + i]; });
            if (sl == 0) {
                hcount[b] = 0;
                hhead[b] = 0;
            }
        } else {
            each([&](int, int i) { d[o + i] = (fixed && fixed[i]) ? 0.f : 0.1f * d[o + i]; });
        }
    }

    // accept candidate nb: x' = fl(x + fl(s d)) (the evaluated point), g' its
    // gradient; the pair (s, y) = (x' - x, g' - g) joins the history iff s.y > eps
    float gv[KPL], q[KPL], sv[KPL], yv[KPL];
    float sy = 0.f;
    if (acc) {
        const float s = sc.s[nb];
        const float* gn = cand_grad + ((long long)nb * B + b) * D;
        each([&](int k, int i) {
            const float xo = x[o + i];
            const float xn = __fadd_rn(xo, __fmul_rn(s, d[o + i]));
            const bool fz = fixed && fixed[i];
            const float gnew = fz ? 0.f : gn[i];
            sv[k] = xn - xo;
            yv[k] = gnew - (fz ? 0.f : g[o + i]);
            sy = fmaf(sv[k], yv[k], sy);
            x[o + i] = xn;
            g[o + i] = gnew;
            gv[k] = gnew;
        });
    }
    sy = grp_sum<LPI>(sy);
    if (acc) {
        if (sl == 0) cost[b] = best;
        if (sy > eps) {
            const long long so = ((long long)b * m + head) * D;
            each([&](int k, int i) {
                hs[so + i] = sv[k];
                hy[so + i] = yv[k];
            });
            if (sl == 0) hrho[(long long)b * m + head] = 1.f / sy;
            head = (head + 1 == m) ? 0 : head + 1;
            count = min(count + 1, m);
            if (sl == 0) {
                hhead[b] = head;
                hcount[b] = count;
            }
        }
    }
    __syncwarp();

    // (7) two-loop recursion over the history, newest to oldest and back
    // (accepted items; the loop bound is the warp's largest history)
    const int cnt = acc ? count : 0;
    const int tmax = warp_max(cnt);
#pragma unroll
    for (int k = 0; k < KPL; ++k) q[k] = acc ? gv[k] : 0.f;
    float* alpha = s_alpha[wib][sub];
    for (int t = 0; t < tmax; ++t) {
        const bool on = t < cnt;
        int slot = head - 1 - t;
        if (slot < 0) slot += m;
        const float* si = hs + ((long long)(valid ? b : 0) * m + slot) * D;
        const float* yi = hy + ((long long)(valid ? b : 0) * m + slot) * D;
        float dot = 0.f;
        if (on) each([&](int k, int i) { dot = fmaf(si[i], q[k], dot); });
        dot = grp_sum<LPI>(dot);
        if (on) {
            const float a = hrho[(long long)b * m + slot] * dot;
            if (sl == 0) alpha[t] = a;
            each([&](int k, int i) { q[k] = fmaf(-a, yi[i], q[k]); });
        }
    }
    __syncwarp();
    // gamma from the newest pair
    float gamma = 1.f;
    {
        float a = 0.f, c = 0.f;
        const int newest = (head == 0) ? m - 1 : head - 1;
        if (cnt > 0) {
            const float* si = hs + ((long long)b * m + newest) * D;
            const float* yi = hy + ((long long)b * m + newest) * D;
            each([&](int, int i) {
                a = fmaf(si[i], yi[i], a);
                c = fmaf(yi[i], yi[i], c);
            });
        }
        a = grp_sum<LPI>(a);
        c = grp_sum<LPI>(c);
        if (cnt > 0) gamma = a / c;
    }
#pragma unroll
    for (int k = 0; k < KPL; ++k) q[k] *= gamma;
    for (int t = tmax - 1; t >= 0; --t) {            // oldest to newest
        const bool on = t < cnt;
        int slot = head - 1 - t;
        if (slot < 0) slot += m;
        const float* si = hs + ((long long)(valid ? b : 0) * m + slot) * D;
        const float* yi = hy + ((long long)(valid ? b : 0) * m + slot) * D;
        float dot = 0.f;
        if (on) each([&](int k, int i) { dot = fmaf(yi[i], q[k], dot); });
        dot = grp_sum<LPI>(dot);
        if (on) {
            const float beta = hrho[(long long)b * m + slot] * dot;
            const float coef = alpha[t] - beta;
            each([&](int k, int i) { q[k] = fmaf(si[i], coef, q[k]); });
        }
    }
    if (acc) each([&](int k, int i) { d[o + i] = -q[k]; });
}

}  // namespace

cudaError_t launch_lbfgs_candidates(const float* x, const float* d, long long B, int D, int N,
                                    const LbfgsScales& sc, float* cand, cudaStream_t s) {
    const long long BD = B * (long long)D;
    if (BD <= 0 || N <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long work = (BD & 3) == 0 ? (BD >> 2) : BD;
    const long long gx = std::max<long long>(1, std::min<long long>((work + 255) / 256,
                                                                   (long long)sms * 8 / N + 1));
    candidates_kernel<<<dim3((unsigned)gx, (unsigned)N), 256, 0, s>>>(x, d, BD, sc, cand);
    return cudaGetLastError();
}

cudaError_t launch_lbfgs_step(int B, int D, int N, const LbfgsScales& sc, const float* cand_cost,
                              const float* cand_grad, float* x, float* g, float* cost, float* d,
                              float* hs, float* hy, float* hrho, int32_t* hcount, int32_t* hhead,
                              int32_t* chosen, int m, float eps, const uint8_t* fixed,
                              cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    // lanes per item: the smallest power of two >= D, at most 32
    const int lpi = D <= 4 ? 4 : D <= 8 ? 8 : D <= 16 ? 16 : 32;
    const int per_block = kStepWarps * (32 / lpi);
    const int grid = (B + per_block - 1) / per_block;
#define VAPR_LBFGS_LAUNCH(L)                                                                      \
    lbfgs_step_kernel<L><<<grid, 32 * kStepWarps, 0, s>>>(B, D, N, sc, cand_cost, cand_grad, x, \
                                                          g, cost, d, hs, hy, hrho, hcount,       \
                                                          hhead, chosen, m, eps, fixed)
    switch (lpi) {
        case 4: VAPR_LBFGS_LAUNCH(4); break;
        case 8: VAPR_LBFGS_LAUNCH(8); break;
        case 16: VAPR_LBFGS_LAUNCH(16); break;
        default: VAPR_LBFGS_LAUNCH(32); break;
    }
#undef VAPR_LBFGS_LAUNCH
    return cudaGetLastError();
}

}  // namespace vapr
