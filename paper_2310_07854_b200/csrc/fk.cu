// fk.cu -- a2: forward kinematics -> packed out_spheres.
// P:86 (forward kinematics), P:189 ("The output of forward kinematics:
// out_spheres"); quantised at the store (reading c19).
//
// One thread per pose walks the 8-row modified-DH chain in FP32 (sincos_joint:
// ~1 ulp, bounded argument) and places the spheres of each link as soon as its frame
// is known.  The 3S coordinates stream through a PF-deep register shift
// buffer (PF = codes per word, a compile-time constant via with_pf; the
// element count is warp-uniform, so there is no divergence) and every full
// buffer is encoded into one packed word (hardware cvt fast path for
// E5M10 / E8M7 / FP8 / FP6 / FP4).  Each warp stages its 32 rows 32 words
// at a time in a small shared chunk (stride 33 words, odd, so the 32 lanes --
// 32 poses writing the same word index -- hit 32 distinct banks); every full
// chunk is streamed to HBM at once, eight lanes per pose writing its 128
// contiguous bytes (one whole line) with 16-byte stores.  Shared memory per
// warp is a fixed 4.2 KB whatever the row width, so occupancy is set by
// registers (9 CTAs, 36 warps per SM), not by a staged row tile.  Link frames are NOT written to
// memory: backward kinematics recomputes them, so HBM sees q
// (28 B/pose) in and out_spheres out.
#include "common.cuh"
#include "kernels.cuh"
#include "tap.cuh"

namespace vapr {

namespace {

constexpr int kTile = 128;   // poses (= threads) per CTA
#ifndef VAPR_FK_MINB             // resident CTAs per SM the register budget targets
#define VAPR_FK_MINB 9
#endif

#ifndef VAPR_FK_CHUNK            // words per pose per warp flush (a multiple of 4)
#define VAPR_FK_CHUNK 32
#endif
constexpr int kChunk = VAPR_FK_CHUNK;
constexpr int kLPR = kChunk / 4;     // lanes per pose row segment in a drain
constexpr int kCS = kChunk + 1;      // chunk row stride (odd: conflict-free lane writes)

// A warp's rows, kChunk words at a time: put() is warp-uniform (every pose
// has the same word sequence), a full chunk goes to HBM as 128-byte segments
// per pose (lane = kLPR pose + part), poses >= np are computed but not stored.
struct RowStore {
    uint32_t* buf;                   // this warp's [32][kCS] chunk
    uint32_t* os;                    // the warp's first row in HBM
    int W, np, lane;
    int n = 0, chunk = 0;
    __device__ __forceinline__ void put(uint32_t v) {
        buf[lane * kCS + n] = v;
        if (++n == kChunk) drain();
    }
    __device__ __forceinline__ void drain() {
        __syncwarp();
        const int parts = n >> 2;    // n is a multiple of 4 (rows are 16-byte multiples)
#pragma unroll
        for (int k = 0; k < kLPR; ++k) {
            const int i = k * 32 + lane, p = i / kLPR, part = i % kLPR;
            if (p < np && part < parts) {
                const uint32_t* src = buf + p * kCS + 4 * part;
                __stcs(reinterpret_cast<uint4*>(os + (long long)p * W + chunk * kChunk + 4 * part),
                       make_uint4(src[0], src[1], src[2], src[3]));
            }
        }
        __syncwarp();
        n = 0;
        ++chunk;
    }
};

template <int PF>
struct Emitter {
    float buf[PF];
    int count = 0;
    int word = 0;
    __device__ __forceinline__ void push(float v, RowStore& row, const Fmt& f) {
#pragma unroll
        for (int j = 0; j < PF - 1; ++j) buf[j] = buf[j + 1];
        buf[PF - 1] = v;
        if (++count == PF) {
            row.put(encode_word_t<PF>(buf, f));
            ++word;
            count = 0;
        }
    }
    __device__ __forceinline__ void flush(RowStore& row, int W, const Fmt& f) {
        if (count) {                                // the tail of the last word is +0
            const int pad = PF - count;
            for (int k = 0; k < pad; ++k) push(0.f, row, f);
        }
        for (; word < W; ++word) row.put(0u);      // 16-byte row padding
        if (row.n) row.drain();
    }
};

// E5M10 (two codes per word, the 43-bit set's out_spheres format): a sphere's
// three values per call with a phase bit (uniform across the CTA: every pose
// has the same sphere sequence) and the hardware f16x2 conversion where it is
// exact (|x| < 65520), the generic word encoder otherwise.
struct EmitterF16 {
    float buf = 0.f;
    bool odd = false;
    int word = 0;
    __device__ __forceinline__ static uint32_t enc2(float a, float b, const Fmt& f) {
        const uint32_t amax = max(__float_as_uint(a) & 0x7fffffffu, __float_as_uint(b) & 0x7fffffffu);
        if (amax < f.hw_limit) return cvt_f16x2(a, b);
        const float x[2] = {a, b};
        return encode_word_t<2>(x, f);
    }
    __device__ __forceinline__ void sphere(float x, float y, float z, RowStore& row, const Fmt& f) {
        if (!odd) {
            row.put(enc2(x, y, f));
            ++word;
            buf = z;
        } else {
            row.put(enc2(buf, x, f));
            row.put(enc2(y, z, f));
            word += 2;
        }
        odd = !odd;
    }
    __device__ __forceinline__ void flush(RowStore& row, int W, const Fmt& f) {
        if (odd) {
            row.put(enc2(buf, 0.f, f));
            ++word;
        }
        for (; word < W; ++word) row.put(0u);
        if (row.n) row.drain();
    }
};

// ee_pose (reading c43): the hand frame as position +
// unit quaternion (w, x, y, z) with w >= 0, Shepperd's method (the largest of
// 1 + tr, 1 + 2 R_ii - tr picks the well-conditioned component).  X.r is
// row-major.
__device__ __forceinline__ void hand_ee_pose(const Xf& X, float* e) {
    const float* m = X.r;
    const float tr = m[0] + m[4] + m[8];
    float w, x, y, z;
    if (tr > 0.f) {
        const float s = 2.f * sqrtf(1.f + tr);
        w = 0.25f * s; x = (m[7] - m[5]) / s; y = (m[2] - m[6]) / s; z = (m[3] - m[1]) / s;
    } else if (m[0] > m[4] && m[0] > m[8]) {
        const float s = 2.f * sqrtf(1.f + m[0] - m[4] - m[8]);
        w = (m[7] - m[5]) / s; x = 0.25f * s; y = (m[1] + m[3]) / s; z = (m[2] + m[6]) / s;
    } else if (m[4] > m[8]) {
        const float s = 2.f * sqrtf(1.f + m[4] - m[0] - m[8]);
        w = (m[2] - m[6]) / s; x = (m[1] + m[3]) / s; y = 0.25f * s; z = (m[5] + m[7]) / s;
    } else {
        const float s = 2.f * sqrtf(1.f + m[8] - m[0] - m[4]);
        w = (m[3] - m[1]) / s; x = (m[2] + m[6]) / s; y = (m[5] + m[7]) / s; z = 0.25f * s;
    }
    const float sg = (w < 0.f) ? -1.f : 1.f;
    e[0] = X.p[0]; e[1] = X.p[1]; e[2] = X.p[2];
    e[3] = sg * w; e[4] = sg * x; e[5] = sg * y; e[6] = sg * z;
}

// EE: also write ee_pose -- its own instantiation (the common one keeps its registers)
template <bool IKO, bool EE>
__global__ void __launch_bounds__(kTile, VAPR_FK_MINB)
fk_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
          long long P, int W, uint32_t* __restrict__ os, const IkArgs ik,
          float* __restrict__ ee) {
    __shared__ float sq[kTile * kJoints];
    __shared__ uint32_t sw[kTile * kCS];
    // vapr_cost_grad: the self collision pass (a programmatic dependent) may
    // launch and stage its tables while FK drains; it waits for FK's output
    pdl_trigger();
    const long long p0 = (long long)blockIdx.x * kTile;
    const int np = (int)min((long long)kTile, P - p0);
    const int tid = threadIdx.x, lane = tid & 31, w0 = tid & ~31;
    const bool valid = tid < np;

    // poses past the end walk q = 0 (every lane takes part in the chunk drains)
    for (int i = tid; i < kTile * kJoints; i += kTile)
        sq[i] = (i < np * kJoints) ? __ldcs(q + p0 * kJoints + i) : 0.f;
    __syncthreads();

    if (w0 < np) {
        RowStore row{sw + w0 * kCS, os + (p0 + w0) * W, W, np - w0, lane};
        // the chain, the IKO terms at the hand, and every sphere centre handed
        // to `emit(x, y, z)` in sphere order
        auto walk = [&](auto&& emit) {
            Xf X;
            xf_identity(X);
            for (int l = 0; l < kLinks; ++l) {
                if (l >= 1 && l <= kJoints) fk_step(X, R, l - 1, sq[tid * kJoints + l - 1]);
                if (l == kLinks - 1) {
                    fk_hand(X, R);
                    if constexpr (EE) {
                        if (valid) hand_ee_pose(X, ee + (p0 + tid) * 7);
                    }
                    if constexpr (IKO) {   // N2: pose + bound cost of this pose -> cost_pose
                        float c = 0.f, F[3], tau[3];
                        const long long pg = p0 + tid;
                        const int wi = valid ? ik.world_idx[pg / ik.H] : -1;
                        if ((ik.w_pos != 0.f || ik.w_rot != 0.f) && wi >= 0 && wi < ik.n_goals)
                            c = ik_pose_cost(X, ik.goals + 12 * wi, ik.w_pos, ik.w_rot, F, tau);
                        if (ik.w_bound != 0.f)
                            for (int j = 0; j < kJoints; ++j) {
                                float dq;
                                c += ik_bound(sq[tid * kJoints + j], R.q_lo[j], R.q_hi[j],
                                              ik.w_bound, dq);
                            }
                        if (valid) ik.cost[pg] = c;
                    }
                }
                for (int s = R.link_start[l]; s < R.link_start[l + 1]; ++s) {
                    float cx, cy, cz;
                    xf_apply(X, R.sx[s], R.sy[s], R.sz[s], cx, cy, cz);
                    if (valid) {
                        VAPR_TAP(0, (p0 + tid) * R.cols + 3 * s, cx);
                        VAPR_TAP(0, (p0 + tid) * R.cols + 3 * s + 1, cy);
                        VAPR_TAP(0, (p0 + tid) * R.cols + 3 * s + 2, cz);
                    }
                    emit(cx, cy, cz);
                }
            }
        };
        if (f.kind == KIND_F16) {
            EmitterF16 em;
            walk([&](float x, float y, float z) { em.sphere(x, y, z, row, f); });
            em.flush(row, W, f);
        } else {
            with_pf(f.pf, [&](auto Pc) {
                constexpr int PF = decltype(Pc)::value;
                Emitter<PF> em;
                walk([&](float x, float y, float z) {
                    em.push(x, row, f);
                    em.push(y, row, f);
                    em.push(z, row, f);
                });
                em.flush(row, W, f);
            });
        }
    }
}

// Small batches (latency): kSL lanes per pose, each walking the whole chain
// (it is short) but placing only the spheres s = sub, sub + kSL, ... into a
// shared FP32 row tile; the CTA then encodes the tile word-parallel and
// stores its rows as one contiguous, coalesced range.  The same chain
// arithmetic and exact codes as fk_kernel, so the output is bit-identical;
// the serial work per thread drops from the whole row to ~1/kSL of it.
constexpr int kSL = 8;                       // lanes per pose
constexpr int kSRows = 128 / kSL;            // poses per CTA
__global__ void __launch_bounds__(128)
fk_small_kernel(const __grid_constant__ RobotDev R, const Fmt f, const float* __restrict__ q,
                long long P, int W, uint32_t* __restrict__ os) {
    extern __shared__ float st[];            // [kSRows][xs] FP32 rows (+0 beyond cols)
    pdl_trigger();
    const int xs = W * f.pf;
    const long long p0 = (long long)blockIdx.x * kSRows;
    const int np = (int)min((long long)kSRows, P - p0);
    const int r = threadIdx.x / kSL, sub = threadIdx.x % kSL;
    for (int i = threadIdx.x; i < kSRows * xs; i += 128) st[i] = 0.f;
    __syncthreads();
    if (r < np) {
        float qv[kJoints];
#pragma unroll
        for (int j = 0; j < kJoints; ++j) qv[j] = __ldg(q + (p0 + r) * kJoints + j);
        float* row = st + r * xs;
        Xf X;
        xf_identity(X);
        for (int l = 0; l < kLinks; ++l) {
            if (l >= 1 && l <= kJoints) fk_step(X, R, l - 1, qv[l - 1]);
            if (l == kLinks - 1) fk_hand(X, R);
            const int s0 = R.link_start[l], s1 = R.link_start[l + 1];
            // this lane's spheres of the link: s = sub (mod kSL)
            for (int s = s0 + ((sub - s0) % kSL + kSL) % kSL; s < s1; s += kSL) {
                float cx, cy, cz;
                xf_apply(X, R.sx[s], R.sy[s], R.sz[s], cx, cy, cz);
                row[3 * s] = cx;
                row[3 * s + 1] = cy;
                row[3 * s + 2] = cz;
                VAPR_TAP(0, (p0 + r) * R.cols + 3 * s, cx);
                VAPR_TAP(0, (p0 + r) * R.cols + 3 * s + 1, cy);
                VAPR_TAP(0, (p0 + r) * R.cols + 3 * s + 2, cz);
            }
        }
    }
    __syncthreads();
    uint32_t* dst = os + p0 * W;
    with_pf(f.pf, [&](auto Pc) {
        constexpr int PF = decltype(Pc)::value;
        for (int i = threadIdx.x; i < np * W; i += 128) {
            const int rr = i / W, w = i - rr * W;
            float x[PF];
#pragma unroll
            for (int j = 0; j < PF; ++j) x[j] = st[rr * xs + w * PF + j];
            __stcs(dst + i, encode_word_t<PF>(x, f));
        }
    });
}

}  // namespace

cudaError_t launch_fk(const RobotDev& R, const Fmt& fos, const float* q, long long P,
                      uint32_t* os, cudaStream_t s, const IkArgs* ik, float* ee) {
    if (P <= 0) return cudaSuccess;
    const int W = row_words_of(fos, R.cols);
    const bool iko = ik && ik_on(*ik);
    auto kern = iko ? (ee ? fk_kernel<true, true> : fk_kernel<true, false>)
                    : (ee ? fk_kernel<false, true> : fk_kernel<false, false>);
#ifndef VAPR_FK_SMALL_BELOW
#define VAPR_FK_SMALL_BELOW 8192
#endif
    if (!iko && !ee && P < VAPR_FK_SMALL_BELOW) {
        const size_t smem = sizeof(float) * kSRows * W * fos.pf;
        if (smem <= 48 * 1024) {
#ifdef VAPR_DEBUG_TAP
            const bool tapped_s = tap_arm(0, P, R.cols, s) != nullptr;
#endif
            fk_small_kernel<<<(unsigned)((P + kSRows - 1) / kSRows), 128, smem, s>>>(R, fos, q, P, W, os);
#ifdef VAPR_DEBUG_TAP
            if (tapped_s) tap_disarm(0, s);
#endif
            return cudaGetLastError();
        }
    }
    const long long grid = (P + kTile - 1) / kTile;
    IkArgs none{};
#ifdef VAPR_DEBUG_TAP
    const bool tapped = tap_arm(0, P, R.cols, s) != nullptr;
#endif
    kern<<<(unsigned)grid, kTile, 0, s>>>(R, fos, q, P, W, os, iko ? *ik : none, ee);
#ifdef VAPR_DEBUG_TAP
    if (tapped) tap_disarm(0, s);
#endif
    return cudaGetLastError();
}

}  // namespace vapr
