// bk.cu -- a6: backward kinematics, packed grad_out_spheres -> grad_q.
// P:162 step (5) "Compute backward for the above steps in the reverse
// sequence"; P:189 ("the input of backward kinematics: grad_out_spheres");
// P:196 ("sparsity-aware computation by skipping zero computations").
//
//   grad_q_j = sum_{l >= j} z_j . (M_l - o_j x F_l),
//   F_l = sum_{s in link l} g_s,  M_l = sum_{s in link l} c_s x g_s,
// with the frames and the sphere centres c_s recomputed in FP32 from q
// (reading c20: the Jacobian of the true FK, not of the quantised spheres).
//
// The CTA streams its tile of packed gradient rows into shared memory with
// coalesced 16-byte loads; each thread then finds its pose's non-zero spheres
// (a 64-bit mask, SWAR test per word) and runs the chain only if the mask is
// non-zero; each link's (F_l, M_l) is folded into the
// joint accumulators j <= l as soon as the link's frame is known, so no frame
// is stored and no prefix/total difference (cancellation) is formed.
//
// SPR (N3, VAPR_OPT_SPARSE): grad_out_spheres in the sparse form -- the mask
// is the row's bitmap, the row's pool words (L2: the aggregation pass just
// wrote them) are copied to the pose's shared row, and the k-th set sphere's
// codes are 3k + c of it; no dense tile copy, no SWAR scan.
#include "common.cuh"
#include "kernels.cuh"
#include "sparse.cuh"

namespace vapr {

namespace {

#ifndef VAPR_BK_TILE
#define VAPR_BK_TILE 128
#endif
constexpr int kTile = VAPR_BK_TILE;         // threads per CTA
constexpr int kMaxTP = 4 * kTile;           // poses per CTA at most
constexpr int kAggRows = 16;                // AGG: poses per CTA (the aggregation tile)

// IKO: the N2 pose / bound terms; SP: the gradient slot is IEEE E5M10 (its
// exponent-31 codes decode to inf / NaN, reading c41) -- a separate
// instantiation so the common ones carry no fixup.
// VAPR_BK_MINB (tuning knob): minimum resident CTAs per SM; unset = the plain
// bound (an explicit 1 lets ptxas use ~150 registers and is slower)
#ifndef VAPR_BK_PPT               // poses per thread (CTA tile = VAPR_BK_PPT x threads, at most 4)
#define VAPR_BK_PPT 2
#endif
#ifdef VAPR_BK_MINB
#define VAPR_BK_BOUNDS __launch_bounds__(kTile, VAPR_BK_MINB)
#else
#define VAPR_BK_BOUNDS __launch_bounds__(kTile)
#endif
template <bool IKO, bool SP, bool SPR, bool AGG>
__global__ void VAPR_BK_BOUNDS
bk_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
          long long P, int W, const uint32_t* __restrict__ gos, float* __restrict__ grad_q,
          uint32_t rc, uint32_t rq, uint32_t f_lo, uint32_t f_hi, uint32_t rt, const IkArgs ik,
          const SparseIn spi, int tp, const AggArgs ag) {
    // tp poses per CTA (a multiple of kTile): with about half of the poses
    // carrying a gradient, two poses per thread keep the compacted chains
    // on every warp instead of leaving half the CTA at the barrier
    extern __shared__ unsigned long long smem8[];
    const int WS = W + 4;                 // 16-byte aligned rows
    float4* so = reinterpret_cast<float4*>(smem8);                    // [kMaxSpheres] sphere offsets
    float* sq = reinterpret_cast<float*>(so + kMaxSpheres);           // [tp * 7]
    uint32_t* sw = reinterpret_cast<uint32_t*>(sq + tp * kJoints);    // [tp * WS]
    float* sg = reinterpret_cast<float*>(sw + tp * WS);               // [tp * 7] grad_q
    __shared__ unsigned long long s_mask[kMaxTP];
    __shared__ int16_t s_act[kMaxTP];
    __shared__ int s_nact;
    pdl_wait();         // vapr_cost_grad: the aggregation's output is complete
    const long long p0 = (long long)blockIdx.x * tp;
    const int np = (int)min((long long)tp, P - p0);
    if constexpr (AGG) {
        // the CTA's rows of grad_out_spheres from closest_pt + out_vec (tp <=
        // kAggRows): aggregate_sparse_rows_kernel's sums, codes and layout
        __shared__ SparseTileSmem<kAggRows> asm_;
        __shared__ uint32_t awbuf[(kTile / 32) * 3 * kMaxSpheres];
        __shared__ unsigned long long amc[kAggRows], amo[kAggRows];
        if ((int)threadIdx.x < np) {
            amc[threadIdx.x] = __ldcs(ag.cpm + p0 + threadIdx.x);
            amo[threadIdx.x] = __ldcs(ag.ovm + p0 + threadIdx.x);
        }
        __syncthreads();
        const uint32_t rcp_c = 65536u / ag.fcp.pf + 1u, rcp_o = 65536u / ag.fov.pf + 1u;
        emit_sparse_rows<kAggRows, kTile / 32>(
            np, ag.cols / 3, f, ag.sp.rcp, asm_, awbuf, 3 * kMaxSpheres, p0,
            ag.sp.seg0 + (uint32_t)p0 * ag.sp.wmax, ag.sp.mask, ag.sp.off, ag.sp.pool, ag.sp.used,
            [&](int r, int s, uint32_t* c) {
                const unsigned long long mc = amc[r], mo = amo[r], bit = 1ull << s;
                if (!((mc | mo) & bit)) return;
                const long long p = p0 + r;
                float x[3];
                const int kc = 3 * __popcll(mc & (bit - 1ull)), ko = 3 * __popcll(mo & (bit - 1ull));
#pragma unroll
                for (int q3 = 0; q3 < 3; ++q3) {
                    float a = 0.f, b = 0.f;
                    if (mc & bit) {
                        const uint32_t e = kc + q3, w = (e * rcp_c) >> 16;
                        a = decode_sp(code_at(__ldcs(ag.cp + p * ag.wc + w), int(e - w * ag.fcp.pf), ag.fcp),
                                      ag.fcp);
                    }
                    if (mo & bit) {
                        const uint32_t e = ko + q3, w = (e * rcp_o) >> 16;
                        b = decode_sp(code_at(__ldcs(ag.ov + p * ag.wo + w), int(e - w * ag.fov.pf), ag.fov),
                                      ag.fov);
                    }
                    x[q3] = a + b;
                }
                encode3(x[0], x[1], x[2], f, c);
            });
        __syncthreads();          // the rows above are read below (global, same CTA)
    }
    const int tid = threadIdx.x;
    if (tid == 0) s_nact = 0;

    // sphere offsets are indexed per lane (by each pose's non-zero spheres):
    // stage them in shared memory instead of the serialising constant bank
    for (int i = tid; i < R.n_spheres; i += kTile) so[i] = make_float4(R.sx[i], R.sy[i], R.sz[i], 0.f);
#pragma unroll 4
    for (int i = tid; i < np * kJoints; i += kTile) sq[i] = __ldcs(q + p0 * kJoints + i);
    __syncthreads();
    if (!SPR) {
        // plain 16-byte copy of the tile (rows are 16-byte multiples), several
        // loads in flight
        const int Q = W / 4, nq = np * Q;
        const uint4* src = reinterpret_cast<const uint4*>(gos + p0 * W);
#pragma unroll 4
        for (int i = tid; i < nq; i += kTile) {
            const uint4 v = __ldcs(src + i);
            const int r = int((uint32_t(i) * rq) >> 20), g = i - r * Q;
            *reinterpret_cast<uint4*>(sw + r * WS + 4 * g) = v;
        }
    }
    __syncthreads();

    // the pose's non-zero spheres, from its own row (16-byte reads, stride
    // W + 4 words: conflict-free per quarter warp); a word's non-zero fields
    // come from one SWAR test, the rare non-zero words are then walked
    // compact the poses with a non-zero gradient so the chains below run in
    // full warps (each pose's result is independent of the order)
    // with the IKO pose cost every pose is active (its hand frame carries a
    // force and a torque whatever its sphere gradients)
    const bool pose_on = IKO && (ik.w_pos != 0.f || ik.w_rot != 0.f);
    for (int pt = tid; pt < np; pt += kTile) {
    unsigned long long mask = 0ull;
    if (SPR) {
        // the row's pool words (ceil(3 popc / pf), contiguous) into the
        // pose's shared row: independent loads, all in flight, instead of a
        // global load per sphere inside the chain
        mask = __ldcs(spi.mask + p0 + pt);
        if (mask) {
            const uint32_t n = ((uint32_t)(3 * __popcll(mask) + f.pf - 1) * rc) >> 16;
            const uint32_t* src = spi.pool + __ldcs(spi.off + p0 + pt);
            uint32_t* dst = sw + pt * WS;
            // four loads in flight at a time
            for (uint32_t w = 0; w < n; w += 4) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = (w + u < n) ? __ldcs(src + w + u) : 0u;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (w + u < n) dst[w + u] = v[u];
            }
        }
    } else {
        const uint4* r4 = reinterpret_cast<const uint4*>(sw + pt * WS);
        for (int g = 0; g < W / 4; ++g) {
            const uint4 v = r4[g];
            if (!(v.x | v.y | v.z | v.w)) continue;
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // top bit of each t-bit field set iff the field is non-zero
                uint32_t nzf = (((w4[k] & f_lo) + f_lo) | w4[k]) & f_hi;
                const int ebase = (4 * g + k) * f.pf;
                while (nzf) {
                    const int b = __ffs(nzf) - 1;
                    nzf &= nzf - 1;
                    const int e = ebase + int(((uint32_t)(b + 1) * rt) >> 16) - 1;
                    if (e < R.cols) mask |= 1ull << (e / 3);
                }
            }
        }
    }

    if (mask || pose_on) {
        const int k = atomicAdd(&s_nact, 1);
        s_act[k] = (int16_t)pt;
        s_mask[k] = mask;
    }
    }
    for (int i = tid; i < np * kJoints; i += kTile) sg[i] = 0.f;
    __syncthreads();
    const int nact = s_nact;
    for (int k = tid; k < nact; k += kTile) {
        const int pp = s_act[k];
        const unsigned long long pmask = s_mask[k];
        float gq[kJoints];
#pragma unroll
        for (int j = 0; j < kJoints; ++j) gq[j] = 0.f;
        const uint32_t* row = sw + pp * WS;
        // SPR: rank of the next set sphere (spheres of link 0 carry no joint)
        int kr = SPR ? __popcll(pmask & ((1ull << R.link_start[1]) - 1ull)) : 0;
        float zx[kJoints], zy[kJoints], zz[kJoints], ox[kJoints], oy[kJoints], oz[kJoints];
        Xf X;
        xf_identity(X);
#pragma unroll
        for (int l = 1; l < kLinks; ++l) {
            if (l <= kJoints) {
                fk_step(X, R, l - 1, sq[pp * kJoints + l - 1]);
                zx[l - 1] = X.r[2];
                zy[l - 1] = X.r[5];
                zz[l - 1] = X.r[8];
                ox[l - 1] = X.p[0];
                oy[l - 1] = X.p[1];
                oz[l - 1] = X.p[2];
            } else {
                fk_hand(X, R);
            }
            const int s0 = R.link_start[l], s1 = R.link_start[l + 1];
            unsigned long long lm = (pmask >> s0) & ((s1 - s0 >= 64) ? ~0ull : ((1ull << (s1 - s0)) - 1ull));
            const bool hand_ik = pose_on && l == kLinks - 1;
            if (!lm && !hand_ik) continue;
            float Fx = 0.f, Fy = 0.f, Fz = 0.f, Mx = 0.f, My = 0.f, Mz = 0.f;
            if (hand_ik) {
                // N2: the pose cost's force F at the hand origin p and torque tau
                // act on the hand link: F_l += F, M_l += p x F + tau
                const long long pg = p0 + pp;
                const int wi = ik.world_idx[pg / ik.H];
                if (wi >= 0 && wi < ik.n_goals) {
                    float F[3], tau[3];
                    ik_pose_cost(X, ik.goals + 12 * wi, ik.w_pos, ik.w_rot, F, tau);
                    Fx = F[0];
                    Fy = F[1];
                    Fz = F[2];
                    Mx = X.p[1] * F[2] - X.p[2] * F[1] + tau[0];
                    My = X.p[2] * F[0] - X.p[0] * F[2] + tau[1];
                    Mz = X.p[0] * F[1] - X.p[1] * F[0] + tau[2];
                }
            }
            while (lm) {
                const int s = s0 + __ffsll((long long)lm) - 1;
                lm &= lm - 1;
                float g[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int e = SPR ? 3 * kr + c : 3 * s + c;
                    const int wi = int((e * rc) >> 16);
                    const uint32_t code = code_at(row[wi], e - wi * f.pf, f);
                    g[c] = SP ? decode_sp(code, f) : decode(code, f);
                }
                if (SPR) ++kr;
                float cx, cy, cz;
                const float4 o4 = so[s];
                xf_apply(X, o4.x, o4.y, o4.z, cx, cy, cz);
                Fx += g[0];
                Fy += g[1];
                Fz += g[2];
                Mx += cy * g[2] - cz * g[1];
                My += cz * g[0] - cx * g[2];
                Mz += cx * g[1] - cy * g[0];
            }
            // fold link l into every joint j <= l: z_j . (M_l - o_j x F_l)
#pragma unroll
            for (int j = 0; j < kJoints; ++j) {
                if (j < l) {
                    const float tx = Mx - (oy[j] * Fz - oz[j] * Fy);
                    const float ty = My - (oz[j] * Fx - ox[j] * Fz);
                    const float tz = Mz - (ox[j] * Fy - oy[j] * Fx);
                    gq[j] += zx[j] * tx + zy[j] * ty + zz[j] * tz;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kJoints; ++j) sg[pp * kJoints + j] = gq[j];
    }
    __syncthreads();
    // N2 bound cost: its gradient is per joint, for every pose
    if (IKO && ik.w_bound != 0.f)
        for (int pt = tid; pt < np; pt += kTile)
            for (int j = 0; j < kJoints; ++j) {
                float dq;
                ik_bound(sq[pt * kJoints + j], R.q_lo[j], R.q_hi[j], ik.w_bound, dq);
                sg[pt * kJoints + j] += dq;
            }
    __syncthreads();
    // coalesced grad_q store (zero for poses without a gradient)
    for (int i = tid; i < np * kJoints; i += kTile) __stcs(grad_q + p0 * kJoints + i, sg[i]);
}

}  // namespace

cudaError_t launch_bk(const RobotDev& R, const Fmt& fgos, const float* q, long long P,
                      const uint32_t* gos, float* grad_q, cudaStream_t s, const IkArgs* ik,
                      const SparseIn* sparse, bool pdl, const AggArgs* agg) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fgos, R.cols);
    // poses per CTA: the most (up to 4 per thread) whose tile keeps 4 CTAs
    // per SM (the register bound) in shared memory
    auto smem_of = [&](int t) {
        return sizeof(float4) * kMaxSpheres + sizeof(float) * t * kJoints +
               sizeof(uint32_t) * t * (W + 4) + sizeof(float) * t * kJoints;
    };
    const uint32_t rq = (1u << 20) / (W / 4) + 1u;      // i / (W/4) for i < tp * W / 4
    // (i rq) >> 20 = i / Q while i (rq Q - 2^20) < 2^20 (the excess stays below
    // one quotient step)
    auto rq_exact = [&](int t) {
        const long long Q = W / 4, e = (long long)rq * Q - (1ll << 20);
        return e >= 0 && (long long)t * Q * e < (1ll << 20);
    };
    // (small batches keep one pose per thread: more CTAs, shorter latency;
    // with the aggregation in front, kAggRows poses per CTA)
    int tp = (agg && sparse) ? kAggRows : kTile;
    for (int t = VAPR_BK_PPT * kTile; !agg && t > kTile && P >= (long long)t * 4 * 148; t /= 2)
        if (smem_of(t) <= 56 * 1024 && rq_exact(t)) {
            tp = t;
            break;
        }
    if (!rq_exact(tp)) return cudaErrorInvalidValue;
    const size_t smem = smem_of(tp);
    cudaError_t e = cudaSuccess;
    const uint32_t rc = 65536u / fgos.pf + 1u;
    // SWAR masks of the format's fields: top bits, low t-1 bits; slot = (b+1)/t - 1
    uint32_t f_lo = 0u, f_hi = 0u;
    for (int j = 0; j < fgos.pf; ++j) {
        const int at = j * fgos.t;
        f_hi |= 1u << (at + fgos.t - 1);
        f_lo |= (uint32_t)(((1ull << (fgos.t - 1)) - 1ull) << at);
    }
    const uint32_t rt = 65536u / fgos.t + 1u;
    const long long grid = (P + tp - 1) / tp;
    const bool iko = ik && ik_on(*ik);
    const bool sp = fgos.kind == KIND_F16_IEEE;
    auto pick = [&](auto spr) {
        constexpr bool S = decltype(spr)::value;
        return iko ? (sp ? bk_kernel<true, true, S, false> : bk_kernel<true, false, S, false>)
                   : (sp ? bk_kernel<false, true, S, false> : bk_kernel<false, false, S, false>);
    };
    auto kern = sparse ? pick(IC<1>{}) : pick(IC<0>{});
    AggArgs ag{};
    if (agg && sparse && !iko) {
        kern = sp ? bk_kernel<false, true, true, true> : bk_kernel<false, false, true, true>;
        ag = *agg;
        ag.sp.wmax = (uint32_t)((R.cols + fgos.pf - 1) / fgos.pf);
        ag.sp.rcp = 65536u / fgos.pf + 1u;
    } else if (agg) {
        return cudaErrorInvalidValue;
    }
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    IkArgs none{};
    const SparseIn dense{};
    return launch_k(kern, dim3((unsigned)grid), dim3(kTile), smem, s, pdl, R, fgos, q, P, W, gos,
                    grad_q, rc, rq, f_lo, f_hi, rt, iko ? *ik : none, sparse ? *sparse : dense, tp,
                    ag);
}

}  // namespace vapr
