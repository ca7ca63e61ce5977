/*
 * vapr.h -- C ABI of libvapr: the B200 (sm_100a) data-parallel hot path of
 * VaPr (arXiv 2310.07854, "VaPr: Variable-Precision Tensors to Accelerate
 * Robot Motion Planning"): the batched trajectory-optimisation rollout
 *   forward kinematics -> world (sphere-vs-cuboid) and self collision costs
 *   -> gradient aggregation -> backward kinematics,
 * with the paper's five large intermediate tensors stored in HBM in
 * per-tensor, packed, round-to-nearest-even ExMy formats.
 *
 * Citations are PAPER.md line numbers ("P:n") and DESIGN.md sections.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Memory.  Every pointer argument that names a tensor is DEVICE memory
 *    owned by the caller (allocated with PyTorch, cudaMalloc, ...), unless the
 *    comment says "host".  The library never allocates, frees or synchronises
 *    on the hot path; all work is enqueued on the caller's `stream`
 *    (a cudaStream_t passed as void*, NULL = legacy default stream).
 *  - Errors.  Arguments are validated synchronously before anything is
 *    enqueued; on any error nothing is launched and no output is touched.
 *    A failed launch or an earlier asynchronous fault on the device is
 *    reported as VAPR_ERR_CUDA.  No C++ exception crosses the ABI.
 *  - Alignment.  Device pointers must be 16-byte aligned
 *    (VAPR_ERR_INVALID_ARG otherwise).
 *  - Layouts (row-major, contiguous):
 *      q, grad_q            float32 [B, H, 7]   (radians / cost per radian)
 *      world_idx            int32   [B]         world of each trajectory
 *      cost_pose            float32 [B, H]
 *      cost_traj            float32 [B]
 *      packed tensor        uint32  [B*H rows, vapr_packed_row_words(fmt, 3S)]
 *    A packed row holds the 3S = 156 elements of one pose, sphere-major
 *    (x0 y0 z0 x1 y1 z1 ...).  Element i of a row lives in word i / pf at bit
 *    offset (i % pf) * t, LSB first, where t = 1 + E + M and pf = floor(32/t)
 *    codes per 32-bit word ("A 32-bit GPU register can store one FP32,
 *    two FP16, three FP10, four FP8, five FP6, six FP5, or eight FP4").
 *    Unused high bits of a word are zero; rows are padded with zero words to
 *    a multiple of 4 words (16 B).  A code is sign | exponent(E) | mantissa(M)
 *    with the sign at bit t-1 ("E3M1 as a FP data type of 3-bit
 *    exponent, 1-bit mantissa, and 1 sign bit").
 *  - Threading.  A context may be used from several host threads and streams
 *    concurrently for launches; vapr_set_* calls must not race with launches
 *    that use the same context.
 */
#ifndef VAPR_H
#define VAPR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    VAPR_OK = 0,
    VAPR_ERR_INVALID_FORMAT = 1,   /* E not in [2,8], M < 1, M > 23 or 1+E+M > 32 */
    VAPR_ERR_INVALID_ARG = 2,      /* NULL / misaligned pointer, bad value, small workspace */
    VAPR_ERR_SHAPE = 3,            /* B < 1, H < 1, swept with H < 2, too many spheres ... */
    VAPR_ERR_CUDA = 4,             /* launch failure or pending asynchronous device fault */
    VAPR_ERR_NOT_INITIALIZED = 5,  /* robot, worlds or formats not set on the context */
    VAPR_ERR_UNSUPPORTED = 6       /* valid request this build does not implement */
} vapr_status;

/* An ExMy floating-point format: 1 sign bit, E exponent bits (bias
 * 2^(E-1)-1), M mantissa bits, subnormals, no inf/NaN codes for t < 32,
 * round to nearest even with saturation to +-max_finite, NaN -> +max_finite,
 * E8M23 = FP32 bit identity (readings c1-c9 of
 * DESIGN.md §3).  Valid: E in [2,8], M in [1,23], 1+E+M <= 32. */
typedef struct { int32_t exp_bits, man_bits; } vapr_format;

/* IEEE special-value mode: OR'd into man_bits of E5M10
 * or E8M7 only.  Encoding is IEEE round-to-nearest-even -- the library's
 * generic integer encoder with the inf code as its clamp (overflow -> +-inf)
 * and 0x7FFF for NaN, which is what PAPER.md:259's __floats2half2_rn path
 * produces -- and the top exponent decodes to inf / NaN, instead of the
 * all-finite reading (c3-c7).  Identical to the reading for every finite |x|
 * below the format's overflow threshold. */
#define VAPR_FMT_IEEE 0x100

/* Tensor slots, in Table II column order (names from P:189). */
enum {
    VAPR_OUT_SPHERES = 0,       /* FK output: sphere centres            */
    VAPR_GRAD_OUT_SPHERES = 1,  /* BK input: aggregated sphere gradients */
    VAPR_OUT_VEC = 2,           /* self-collision gradient buffer        */
    VAPR_CLOSEST_PT = 3,        /* world-collision gradient, discrete    */
    VAPR_CLOSEST_PT_SWEPT = 4,  /* world-collision gradient, swept       */
    VAPR_NUM_SLOTS = 5
};

#define VAPR_MAX_SPHERES 64
#define VAPR_MAX_PAIRS 1024
#define VAPR_MAX_CUBOIDS_PER_WORLD 16

typedef struct vapr_ctx vapr_ctx;   /* opaque; one per device */

/* Robot model (host memory; copied by vapr_set_robot).  Modified DH (Craig):
 * row i = 0..7 gives T_i = RotX(dh_alpha[i]) TransX(dh_a[i]) RotZ(theta_i)
 * TransZ(dh_d[i]), theta_i = q_i for i < 7 and 0 for the fixed flange row 7;
 * the hand frame is flange . RotZ(hand_rz).  Sphere s is attached to frame
 * sphere_link[s] in 0..8 (0 = base, 1..7 = joint frames, 8 = hand) at local
 * offset sphere_xyzr[s][0..2] with radius sphere_xyzr[s][3] (metres; the radius
 * is never quantised).  Spheres must be sorted by link.  pairs[k] = (i, j) are
 * the self-collision pairs (reading c18). */
typedef struct {
    int32_t n_spheres;                 /* 1..VAPR_MAX_SPHERES */
    int32_t n_pairs;                   /* 0..VAPR_MAX_PAIRS   */
    double dh_a[8], dh_d[8], dh_alpha[8];
    double hand_rz;
    const int32_t *sphere_link;        /* host [n_spheres]    */
    const float *sphere_xyzr;          /* host [n_spheres][4] */
    const uint16_t *pairs;             /* host [n_pairs][2]   */
    double q_lo[7], q_hi[7];           /* joint limits (rad), for the bound cost (N2, c36) */
} vapr_robot;

/* One oriented box (64 B): R = world-from-box rotation (row-major 3x3),
 * t = box centre (world), half = half extents (metres). */
typedef struct { float R[9]; float t[3]; float half[3]; float pad; } vapr_cuboid;

/* Cost parameters (readings c14, c17): smooth-hinge activation
 * distances eta_* (m), weights w_*, swept = 1 for the TO swept world cost with
 * sweep_steps >= 0 linear sub-samples per segment, 0 for the discrete cost.
 * The IKO terms of vapr_cost_grad (N2, PAPER.md:162 step (3) "pose ... and
 * bound position"; readings c34-c36): pose cost w_pose_pos |p - p_g|^2 +
 * w_pose_rot |R - R_g|_F^2 of the hand frame against the goal of the
 * trajectory's problem (vapr_set_goals, indexed like world_idx), bound cost
 * w_bound sum_j max(0, q_j - q_hi)^2 + max(0, q_lo - q_j)^2.  All three 0
 * (the TO default): no IKO terms. */
typedef struct {
    float eta_world, eta_self, w_world, w_self;
    int32_t swept, sweep_steps;
    float w_pose_pos, w_pose_rot, w_bound;
} vapr_cost_params;

/* Options (vapr_set_option). */
enum {
    VAPR_OPT_CULL = 0,     /* 1 (default): exact broadphase culling; 0: brute force */
    VAPR_OPT_STREAMS = 1,  /* vapr_cost_grad: trajectory chunks on this many context-owned
                              streams (1..8, default 1), forked from and joined back to the
                              caller's stream; results are bit-identical for any value */
    VAPR_OPT_SPARSE = 2,   /* N3: 1 = vapr_cost_grad stores the three gradient tensors
                              (closest_pt[_swept], out_vec, grad_out_spheres) in the sparse
                              form (the collision passes write the first two, aggregation
                              reads them and writes the third, BK reads it; the workspace
                              holds the sparse regions instead of the dense slots, see
                              vapr_cost_grad_sparse_layout); 0 (default) = dense.  cost and
                              grad_q are bit-identical either way.  Changes the workspace
                              size: query vapr_cost_grad_workspace_bytes after setting it. */
    VAPR_OPT_FUSED = 3     /* N4: 1 = vapr_cost_grad runs the whole rollout
                              -- FK, world + self collision, aggregation, BK -- in ONE kernel
                              (plus the per-trajectory cost sum): every tensor of the five
                              slots is quantise->dequantised in registers / shared memory
                              (its format's exact RNE codes, decoded at once: the error a
                              stored tensor injects, "quantizing the tensors from FP32
                              to the specified data format and dequantizing them back to
                              FP32") and never written to HBM.  cost_pose, cost_traj and
                              grad_q are bit-identical to the materialised path.  The
                              workspace shrinks to the cost scratch (query
                              vapr_cost_grad_workspace_bytes after setting it); IKO weights
                              and VAPR_OPT_SPARSE = 1 are VAPR_ERR_UNSUPPORTED with it.
                              0 (default) = materialised. */
};

/* ---- context and tables ------------------------------------------------ */
vapr_status vapr_create(int device, vapr_ctx **out);
vapr_status vapr_destroy(vapr_ctx *ctx);
const char *vapr_status_string(vapr_status s);
const char *vapr_version(void);
/* The CUDA runtime's error string behind the most recent VAPR_ERR_CUDA
 * returned on the calling host thread ("no error" if none); a static string
 * owned by the CUDA runtime, never freed by the caller.  Diagnostics only. */
const char *vapr_last_cuda_error(void);

/* IKO pose goals (N2): goals[w] = the hand-frame goal of problem / world w,
 * 12 floats (R row-major 3x3, then p), host memory, copied; n_goals >= 0.
 * vapr_cost_grad reads goal world_idx[b] for trajectory b when a pose weight
 * is non-zero (VAPR_ERR_NOT_INITIALIZED if no goals were set; an index
 * outside [0, n_goals) contributes no pose cost). */
vapr_status vapr_set_goals(vapr_ctx *ctx, const float *goals, int32_t n_goals);

/* "E<e>M<m>", case-insensitive. */
vapr_status vapr_format_parse(const char *s, vapr_format *out);
vapr_status vapr_format_check(vapr_format f);
/* Words per packed row of `cols` elements: roundup4(ceil(cols / floor(32/t)));
 * 0 for an invalid format. */
size_t vapr_packed_row_words(vapr_format f, size_t cols);

/* Formats of the five slots, indexed by VAPR_OUT_SPHERES.. ("provide
 * reduced-precision FP data types for the tensors"). */
vapr_status vapr_set_formats(vapr_ctx *ctx, const vapr_format fmts[VAPR_NUM_SLOTS]);
vapr_status vapr_set_robot(vapr_ctx *ctx, const vapr_robot *robot);
/* n_worlds worlds; world w owns cuboids[offsets[w] .. offsets[w+1]) (host
 * arrays, copied to the device; at most VAPR_MAX_CUBOIDS_PER_WORLD each). */
vapr_status vapr_set_worlds(vapr_ctx *ctx, int32_t n_worlds, const vapr_cuboid *cuboids,
                            const int32_t *offsets);
vapr_status vapr_set_option(vapr_ctx *ctx, int32_t option, int32_t value);
/* Stage timing hook (measurement): with n = 6 caller-owned
 * cudaEvent_t handles, every later vapr_cost_grad on one stream
 * (VAPR_OPT_STREAMS = 1) records events[0] before FK and events[i] after
 * stage i: 1 FK, 2 collision (both passes), 3 cost reduction, 4 aggregation,
 * 5 BK -- the per-kernel durations of the launches the call makes, on its own
 * stream.  n = 0 clears it.  The events stay owned by the caller (destroying
 * one while set is undefined).  VAPR_ERR_INVALID_ARG for other n. */
vapr_status vapr_set_stage_events(vapr_ctx *ctx, void *const *events, int32_t n);

/* ---- a1: codec (context free) ------------------------------------------ */
/* Quantise x [rows, cols] float32 to packed [rows, row_words] (P:227
 * "quantizing the tensors from FP32 to the specified data format"). */
vapr_status vapr_quantize(vapr_format f, const float *x, size_t rows, size_t cols,
                          uint32_t *packed, void *stream);
/* Dequantise packed [rows, row_words] to y [rows, cols] float32 (P:227
 * "dequantizing them back to FP32").  Exact. */
vapr_status vapr_dequantize(vapr_format f, const uint32_t *packed, size_t rows, size_t cols,
                            float *y, void *stream);

/* ---- a2: forward kinematics -> packed out_spheres ----------------------- */
/* P:86 (forward kinematics), P:189 ("The output of forward kinematics:
 * out_spheres").  out_spheres [B*H, row_words(fmt[OUT_SPHERES], 3S)].
 * ee_pose (nullable, 16-byte aligned): [B*H, 7] FP32 hand frame (reading c34)
 * as (p_x, p_y, p_z, q_w, q_x, q_y, q_z), the unit quaternion with q_w >= 0
 * (reading c43). */
vapr_status vapr_fk_spheres(vapr_ctx *ctx, const float *q, int32_t B, int32_t H,
                            uint32_t *out_spheres, float *ee_pose, void *stream);

/* ---- a3: world collision ----------------------------------------------- */
/* P:86, P:189 ("the output of collision cost: closest_pt for IKO and
 * closest_pt_swept for TO").  Reads packed out_spheres; writes cost [B, H]
 * (weighted smooth-hinge world cost per pose; swept: plus the samples of
 * segment (h, h+1)) and grad = the weighted d(world cost)/d(sphere centre),
 * packed at fmt[CLOSEST_PT] (swept = 0) or fmt[CLOSEST_PT_SWEPT] (swept = 1). */
vapr_status vapr_world_collision(vapr_ctx *ctx, const uint32_t *out_spheres,
                                 const int32_t *world_idx, int32_t B, int32_t H,
                                 int32_t swept, int32_t sweep_steps, float eta, float weight,
                                 float *cost, uint32_t *grad, void *stream);

/* ---- a4: self collision ------------------------------------------------ */
/* P:86, P:189 ("the input of self-collision cost: out_vec").  cost [B, H];
 * out_vec = weighted d(self cost)/d(sphere centre), packed at fmt[OUT_VEC]. */
vapr_status vapr_self_collision(vapr_ctx *ctx, const uint32_t *out_spheres, int32_t B,
                                int32_t H, float eta, float weight, float *cost,
                                uint32_t *out_vec, void *stream);

/* ---- a3+a4 fused: one pass over out_spheres (the vapr_cost_grad stage) --- */
/* cost_pose [B, H] = world + self cost; cost_traj [B] (nullable) = sum over h.
 * cp_grad at fmt[CLOSEST_PT(_SWEPT)] and out_vec at fmt[OUT_VEC]. */
vapr_status vapr_collision(vapr_ctx *ctx, const uint32_t *out_spheres, const int32_t *world_idx,
                           int32_t B, int32_t H, const vapr_cost_params *params,
                           float *cost_pose, float *cost_traj, uint32_t *cp_grad,
                           uint32_t *out_vec, void *stream);

/* ---- a5: aggregation -> packed grad_out_spheres ------------------------- */
/* P:162 step (4) "Aggregating the costs", P:189 ("the input of backward
 * kinematics: grad_out_spheres"): gos = Q(dequant(cp_grad) + dequant(out_vec))
 * elementwise over n_rows pose rows.  cp_grad is read at fmt[CLOSEST_PT_SWEPT]
 * if swept else fmt[CLOSEST_PT]. */
vapr_status vapr_aggregate(vapr_ctx *ctx, const uint32_t *cp_grad, int32_t swept,
                           const uint32_t *out_vec, int64_t n_rows,
                           uint32_t *grad_out_spheres, void *stream);

/* ---- a6: backward kinematics -> grad_q ----------------------------------- */
/* P:162 step (5) "Compute backward".  grad_q_j = sum over spheres on
 * links >= j of z_j . ((c_s - o_j) x g_s), c_s the FK centre recomputed in
 * FP32 from q (reading c20), g = dequant(grad_out_spheres); zero rows and
 * zero spheres are skipped ("sparsity-aware computation"). */
vapr_status vapr_backward_kinematics(vapr_ctx *ctx, const float *q, int32_t B, int32_t H,
                                     const uint32_t *grad_out_spheres, float *grad_q,
                                     void *stream);

/* ---- a7: the composed rollout cost + gradient --------------------------- */
/* FK -> fused collision (swept per params) -> aggregate -> BK on `stream`;
 * every live tensor (out_spheres, closest_pt[_swept], out_vec,
 * grad_out_spheres) is written once to HBM, packed, inside `workspace`
 * (P:162).  cost_pose and cost_traj are nullable. */
size_t vapr_cost_grad_workspace_bytes(const vapr_ctx *ctx, int32_t B, int32_t H);
/* Byte offsets of the packed tensors inside the workspace (slot-indexed;
 * SIZE_MAX for a slot that is not live) -- lets callers inspect them. */
vapr_status vapr_cost_grad_workspace_layout(const vapr_ctx *ctx, int32_t B, int32_t H,
                                            int32_t swept, size_t offsets[VAPR_NUM_SLOTS]);
vapr_status vapr_cost_grad(vapr_ctx *ctx, const float *q, const int32_t *world_idx,
                           int32_t B, int32_t H, const vapr_cost_params *params,
                           void *workspace, size_t workspace_bytes,
                           float *cost_pose, float *cost_traj, float *grad_q, void *stream);

/* The same computation from HOST buffers: q_host [B, H, 7] in, grad_q_host
 * [B, H, 7] and cost_traj_host [B] (nullable) out, with the host<->device
 * copies pipelined against the compute.  The batch is split into n_chunks
 * contiguous trajectory ranges (0 = automatic: up to ~700k poses per chunk;
 * the first and last chunks are a quarter of the others, so the exposed
 * copies are short); chunk i's H2D copy, chunk i-1's compute and chunk i-2's
 * D2H copies run concurrently on two context-owned copy streams and `stream`.  Every output
 * is bit-identical to vapr_cost_grad's (the kernels see the same rows).
 * Device buffers (caller-owned): q_dev [B*H*7], workspace (as for
 * vapr_cost_grad), cost_pose_dev [B*H] (nullable: workspace scratch),
 * cost_traj_dev [B], grad_q_dev [B*H*7].  Host buffers should be pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to overlap; pageable
 * memory works but serialises.  The call is stream-ordered: it returns after
 * enqueueing, and everything (including the D2H copies) is complete when
 * `stream` is.  Errors: as vapr_cost_grad; VAPR_ERR_INVALID_ARG for null or
 * misaligned device buffers or n_chunks < 0. */
vapr_status vapr_cost_grad_host(vapr_ctx *ctx, const float *q_host, const int32_t *world_idx,
                                int32_t B, int32_t H, const vapr_cost_params *params,
                                void *workspace, size_t workspace_bytes, float *q_dev,
                                float *cost_pose_dev, float *cost_traj_dev, float *grad_q_dev,
                                float *cost_traj_host, float *grad_q_host, int32_t n_chunks,
                                void *stream);

/* ---- N1: the optimiser steps around vapr_cost_grad ----- */
/* PAPER.md:162 "(1) Given N, step scales of step direction ... (6) Use line
 * search to pick one from N. (7) Lastly, compute step direction (L-BFGS) and
 * buffer updates".  Readings c29-c33.  A batch
 * item b owns the D-vector x[b] (for trajectory optimisation D = 7 H: the
 * trajectory's joint values, layout [B, H, 7] = [B, D]).  All pointers are
 * device pointers, row-major, 4-byte aligned, caller-owned; scales is a HOST
 * array of N strictly increasing positive floats, 1 <= N <= 32. */
#define VAPR_LBFGS_MAX_M 32
#define VAPR_LBFGS_MAX_D 512

/* Step (1): the N x B line-search batch cand[n, b, :] = fl(x[b] + fl(s_n d[b]))
 * ([N, B, D], i.e. N*B trajectories in vapr_cost_grad's layout). */
vapr_status vapr_lbfgs_candidates(const float *x, const float *d, int32_t B, int32_t D,
                                  const float *scales, int32_t N, float *cand, void *stream);

/* Steps (6) and (7) for every batch item, given the costs cand_cost [N, B]
 * and gradients cand_grad [N, B, D] of the candidates (vapr_cost_grad on
 * the batch above): chosen[b] = the argmin candidate if its cost is strictly
 * below cost[b] (ties to the smaller scale), else -1.  Accepted: x, g, cost
 * take the candidate's values, (x' - x, g' - g) joins the history when
 * s.y > curvature_eps (FIFO of m, slot head[b], count[b]).  Rejected: a
 * non-empty history is cleared, else d is shrunk tenfold (c32).  Finally d
 * (in: the direction the candidates used) becomes the two-loop direction
 * -H g.  History buffers: hist_s, hist_y [B, m, D], hist_rho [B, m],
 * hist_count, hist_head [B] (zero-initialised by the caller for an empty
 * history).  chosen is nullable.  Errors: VAPR_ERR_SHAPE for B < 0, D < 1,
 * D > VAPR_LBFGS_MAX_D, N outside [1, 32], m outside [1, VAPR_LBFGS_MAX_M];
 * VAPR_ERR_INVALID_ARG for null buffers or non-positive / non-increasing
 * scales.  fixed (nullable, device, [D] bytes, shared by all items): a
 * non-zero entry freezes that coordinate -- its gradient (as stored and as
 * used) and direction are 0, so the optimisation runs over the free
 * coordinates only (N4: trajectory endpoints held at start and goal). */
vapr_status vapr_lbfgs_step(int32_t B, int32_t D, const float *scales, int32_t N,
                            const float *cand_cost, const float *cand_grad, float *x, float *g,
                            float *cost, float *d, float *hist_s, float *hist_y, float *hist_rho,
                            int32_t *hist_count, int32_t *hist_head, int32_t *chosen, int32_t m,
                            float curvature_eps, const uint8_t *fixed, void *stream);

/* ---- N3: sparsity-aware storage of a sphere tensor ----- */
/* "grad_out_spheres, out_vec, closest_pt, and closest_pt_swept
 * have more than 99% of sparsity".  Reading c42 (definition in
 * oracle/sparse.py).  A packed sphere tensor of `rows` rows of cols = 3S codes
 * (S <= 64 spheres, codes c = x, y, z of sphere s at 3s + c) in sparse form:
 *   mask[rows]  uint64: bit s set iff one of sphere s's three codes is
 *               non-zero as a t-bit integer (a -0 code counts);
 *   off[rows]   uint32: the row's first word in pool (0 for an empty row);
 *   pool        uint32: a row's codes are those of its set spheres in
 *               ascending order, code index i = 3k + c for the k-th set
 *               sphere, in word off + i / pf at bits (i % pf) t (LSB-first,
 *               pf = floor(32 / t), as in dense rows); n = ceil(3 popc(mask)
 *               / pf) words, unused high slots 0;
 *   used        uint32 (device): pool words in use, = the sum of n.
 * Rows occupy disjoint word ranges inside the pool capacity; their placement
 * is the writer's (this library: each tile of 16 consecutive rows packs its
 * rows back to back from word 16 wmax tile, wmax = ceil(cols / pf), so the
 * layout is deterministic); everything else is determined.  Row offsets are
 * 32-bit: the capacity must stay below 2^32 words (VAPR_ERR_SHAPE).  Stored
 * data: 12 bytes per row + 4 used bytes. */

/* Pool capacity that always suffices: rows * ceil(cols / pf) words. */
size_t vapr_sparse_pool_words(vapr_format f, size_t cols, size_t rows);
/* Dense packed [rows, row_words] -> sparse form.  mask, off, pool, used:
 * device, caller-owned, 8 / 4 / 4 / 4-byte aligned; pool_words >=
 * vapr_sparse_pool_words (else VAPR_ERR_SHAPE); *used is reset by the call
 * (stream-ordered).  cols % 3 == 0 and cols / 3 <= 64, else VAPR_ERR_SHAPE. */
vapr_status vapr_sparsify(vapr_format f, const uint32_t *packed, size_t rows, size_t cols,
                          uint64_t *mask, uint32_t *off, uint32_t *pool, size_t pool_words,
                          uint32_t *used, void *stream);
/* Sparse form -> dense packed [rows, row_words] (padding words 0). */
vapr_status vapr_densify(vapr_format f, const uint64_t *mask, const uint32_t *off,
                         const uint32_t *pool, size_t rows, size_t cols, uint32_t *packed,
                         void *stream);
/* With VAPR_OPT_SPARSE = 1: byte offsets inside vapr_cost_grad's workspace
 * of (0) grad_out_spheres' mask [B*H], (1) its off [B*H], (2) used [1], (3)
 * its pool [pool_words]; (4) closest_pt[_swept]'s and (5) out_vec's mask
 * [B*H] uint64; (6) closest_pt[_swept]'s and (7) out_vec's pool.  The two
 * collision outputs use implicit row offsets: row p's codes start at word
 * p * ceil(cols / pf) of their pool (capacity B*H*ceil(cols / pf) words);
 * *pool_words = grad_out_spheres' pool capacity.  The dense entries of
 * vapr_cost_grad_workspace_layout for the three gradient slots are SIZE_MAX.
 * VAPR_ERR_INVALID_ARG when the option is off. */
vapr_status vapr_cost_grad_sparse_layout(const vapr_ctx *ctx, int32_t B, int32_t H,
                                         size_t offsets[8], size_t *pool_words);

/* ---- test-only export (libvapr_tap.so, built with -DVAPR_DEBUG_TAP) ----- */
/* SURVEY.md §8(b) "Test-only export", §8(c) parity contract (i): the next
 * launch that produces `slot` also writes that slot's FP32 pre-quantisation
 * values to dst (device, [rows, 3S] float32, caller-owned; zero-filled by the
 * launch first, so elements the kernel never encodes read +0).  One-shot;
 * dst = NULL disarms.  Not thread-safe (one process-wide table).  The
 * aggregation taps the dense form only.  Release builds (libvapr.so) do not
 * export the symbol and carry no tap code. */
#ifdef VAPR_DEBUG_TAP
vapr_status vapr_debug_tap(vapr_ctx *ctx, int32_t slot, float *dst);
#endif

/* ---- e: per-problem reduction (multi-GPU sharding) ---------------------- */
/* best_cost[p] = min over the seeds of problem p of cost_traj, best_seed[p] =
 * its lowest argmin; problem p owns trajectories [p*seeds, (p+1)*seeds). */
vapr_status vapr_best_per_problem(const float *cost_traj, int32_t n_problems, int32_t seeds,
                                  float *best_cost, int32_t *best_seed, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* VAPR_H */
