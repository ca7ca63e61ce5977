// kernels.cuh -- host-side launch helpers for the libvapr kernels.
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "common.cuh"

namespace vapr {

// Launch `kern` normally, or (pdl) as a programmatic dependent of the previous
// kernel on the stream -- the kernel must pdl_wait() before touching its
// predecessor's outputs.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, bool pdl, Args&&... args) {
    if (!pdl) {
        kern<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// World table on the device: per cuboid 16 floats = R^T (row-major 3x3), t,
// half extents, pad; offsets [n_worlds + 1].
struct WorldsDev {
    const float4* cub;
    const int32_t* off;
    int32_t n_worlds;
};

struct CollisionArgs {
    const uint32_t* os;       // packed out_spheres
    const int32_t* world_idx;
    int32_t B, H;
    int32_t do_world, do_self;
    int32_t swept, sweep_steps;
    float eta_w, w_w, eta_s, w_s;
    int32_t cull;
    float* cost;              // [B*H] (world + self of the enabled parts)
    uint32_t* cp;             // world gradient: dense rows, or (cp_mask) the sparse pool
    uint32_t* ov;             // self gradient: dense rows, or (ov_mask) the sparse pool
    // N3 (VAPR_OPT_SPARSE; nullable = dense rows): per-pose sphere bitmaps.
    // With them a pose's non-zero codes are packed in ascending sphere order
    // at pool + pose * ceil(cols / pf) (reading c42)
    unsigned long long* cp_mask;
    unsigned long long* ov_mask;
    // vapr_cost_grad (nullable): the self pass writes its cost here and
    // traj_reduce adds it, so the self pass may overlap the world pass's tail
    // (programmatic dependent launch); the order of the sums is unchanged
    float* self_cost;
    // N4 fused rollout (VAPR_OPT_FUSED; fused = 1, world and self in one
    // pass): the tile rows come from FK of q in the kernel (os unused), each
    // out_spheres coordinate quantise->dequantised in registers; the world /
    // self gradients likewise (cp / ov unused), summed on chip, quantised with
    // fgos and folded by BK into grad_q -- no tensor makes an HBM round trip
    int32_t fused;
    const float* q;           // [B*H, 7]
    float* grad_q;            // [B*H, 7]
    Fmt fgos;
    // the robot's CTA tables as a device image (collision_table_image; the
    // eta-dependent distances without eta): staged with 16-byte loads instead
    // of divergent parameter-space reads
    const uint4* tab_img;
    int32_t tab_img_bytes;
    int32_t tile_poses;       // internal: poses per warp tile (<= 15; fewer for small batches)
    long long n_tiles;        // internal: ceil(B H / tile_poses)
    int32_t pdl;              // internal: 1 = PDL dependent of FK (wait, then trigger the
                              // second pass), 2 = trigger at start, wait for pass 1 at exit
    int32_t cost_accumulate;  // internal: cost += (this pass) instead of cost =
    unsigned int* sched;      // internal: tile-scheduler slot {next grab, finished CTAs}, zero
};

cudaError_t launch_quantize(const Fmt& f, const float* x, size_t rows, size_t cols,
                            size_t row_words, uint32_t* packed, int sms, cudaStream_t s);
cudaError_t launch_dequantize(const Fmt& f, const uint32_t* packed, size_t rows, size_t cols,
                              size_t row_words, float* y, int sms, cudaStream_t s);
// IKO terms of vapr_cost_grad (N2): pose cost of the hand frame against
// goals[world_idx[pose / H]] and the joint-bound cost; disabled when all
// weights are 0 (then the pointers may be null)
struct IkArgs {
    const float* goals;        // [n_goals][12] R row-major, p
    int32_t n_goals;
    const int32_t* world_idx;  // [B] (the chunk's)
    int32_t H;
    float w_pos, w_rot, w_bound;
    float* cost;               // FK: cost_pose [P] = pose + bound (the collision passes add)
};
inline bool ik_on(const IkArgs& k) { return k.w_pos != 0.f || k.w_rot != 0.f || k.w_bound != 0.f; }

// ee (nullable): [P, 7] hand position + unit quaternion (w >= 0)
cudaError_t launch_fk(const RobotDev& R, const Fmt& fos, const float* q, long long P,
                      uint32_t* os, cudaStream_t s, const IkArgs* ik = nullptr,
                      float* ee = nullptr);
cudaError_t launch_collision(const RobotDev& R, const WorldsDev& W, const Fmt& fos,
                             const Fmt& fcp, const Fmt& fov, const CollisionArgs& a,
                             unsigned int* sched_ring, unsigned int* sched_next, cudaStream_t s);
// The byte image of the collision kernel's shared robot tables (layout of
// its Geo; the activation distances without eta_s), built once per robot.
std::vector<uint8_t> collision_table_image(const RobotDev& R);
constexpr int kSchedSlots = 256;   // scheduler slots per context (in-flight collision passes)
// add (nullable): cost_pose += add first (the self pass's separate cost);
// cost_traj (nullable): the per-trajectory sums
cudaError_t launch_traj_reduce(float* cost_pose, int32_t B, int32_t H, float* cost_traj,
                               cudaStream_t s, const float* add = nullptr, bool pdl = false);
// N3 sparse form of a sphere tensor (include/vapr.h "N3"; sparse.cuh)
struct SparseOut {
    unsigned long long* mask;  // [rows] (the caller offsets it to the first row)
    uint32_t* off;             // [rows]
    uint32_t* pool;            // shared by all rows / chunks
    uint32_t* used;            // pool words in use (a counter)
    uint32_t seg0;             // pool word of the launch's row 0 segment: row0 * ceil(cols / pf)
    uint32_t wmax;             // ceil(cols / pf) (set by the launcher)
    uint32_t rcp;              // 65536 / pf + 1 (set by the launcher)
};
struct SparseIn {
    const unsigned long long* mask;
    const uint32_t* off;
    const uint32_t* pool;
};
cudaError_t launch_sparsify(const Fmt& f, const uint32_t* packed, long long rows, int cols,
                            const SparseOut& o, cudaStream_t s);
cudaError_t launch_densify(const Fmt& f, const SparseIn& in, long long rows, int cols,
                           uint32_t* packed, cudaStream_t s);
// sparse (nullable): write grad_out_spheres in the sparse form instead of gos
cudaError_t launch_aggregate(const Fmt& fcp, const Fmt& fov, const Fmt& fgos, int cols,
                             const uint32_t* cp, const uint32_t* ov, long long rows,
                             uint32_t* gos, cudaStream_t s, const SparseOut* sparse = nullptr,
                             bool pdl = false);
// N3 sparse inputs (cp / ov: sphere bitmaps + packed non-zero codes at
// pool + row * ceil(cols / pf)) -> the sparse form of grad_out_spheres
cudaError_t launch_aggregate_sparse(const Fmt& fcp, const Fmt& fov, const Fmt& fgos, int cols,
                                    const uint32_t* cp_pool, const unsigned long long* cpm,
                                    const uint32_t* ov_pool, const unsigned long long* ovm,
                                    long long rows, const SparseOut& sparse, cudaStream_t s,
                                    bool pdl = false);
// Small batches (sparse storage): the aggregation done by BK's own CTAs for
// their poses first (aggregate_sparse_rows_kernel's arithmetic and layout),
// then BK on the rows just written -- one launch fewer
struct AggArgs {
    Fmt fcp, fov;
    const uint32_t* cp;        // closest_pt[_swept] pool (rows at p * wc)
    const unsigned long long* cpm;
    const uint32_t* ov;        // out_vec pool (rows at p * wo)
    const unsigned long long* ovm;
    int32_t cols, wc, wo;
    SparseOut sp;              // grad_out_spheres (seg0 / mask / off of the launch's rows)
};
// sparse (nullable): read grad_out_spheres from the sparse form instead of gos
// agg (nullable, with sparse): aggregate first (AggArgs)
cudaError_t launch_bk(const RobotDev& R, const Fmt& fgos, const float* q, long long P,
                      const uint32_t* gos, float* grad_q, cudaStream_t s,
                      const IkArgs* ik = nullptr, const SparseIn* sparse = nullptr,
                      bool pdl = false, const AggArgs* agg = nullptr);
// N1 optimiser (lbfgs.cu)
struct LbfgsScales {
    float s[32];
};
cudaError_t launch_lbfgs_candidates(const float* x, const float* d, long long B, int D, int N,
                                    const LbfgsScales& sc, float* cand, cudaStream_t s);
cudaError_t launch_lbfgs_step(int B, int D, int N, const LbfgsScales& sc, const float* cand_cost,
                              const float* cand_grad, float* x, float* g, float* cost, float* d,
                              float* hs, float* hy, float* hrho, int32_t* hcount, int32_t* hhead,
                              int32_t* chosen, int m, float eps, const uint8_t* fixed,
                              cudaStream_t s);
cudaError_t launch_best_per_problem(const float* cost_traj, int32_t n_problems, int32_t seeds,
                                    float* best_cost, int32_t* best_seed, cudaStream_t s);

// words per packed row (multiple of 4)
inline int row_words_of(const Fmt& f, int cols) {
    const int w = (cols + f.pf - 1) / f.pf;
    return (w + 3) & ~3;
}

}  // namespace vapr
