"""Thin ctypes binding of libvapr (include/vapr.h).

Argument marshalling only: torch tensors are passed as raw device pointers,
the current torch CUDA stream as the `stream` argument, host numpy arrays for
the table setters.  Every function has the C name; a non-OK status raises
VaprError.  There is no CPU fallback: if libvapr.so is missing or fails to
load, importing this module raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libvapr.so")
# development hook: A/B timing of kernel variants built with
# `python -m paper_2310_07854_b200.build --variant NAME -DMACRO=...`
if os.environ.get("VAPR_SO"):
    SO_PATH = os.path.abspath(os.environ["VAPR_SO"])

VAPR_OUT_SPHERES, VAPR_GRAD_OUT_SPHERES, VAPR_OUT_VEC, VAPR_CLOSEST_PT, VAPR_CLOSEST_PT_SWEPT = range(5)
VAPR_NUM_SLOTS = 5
VAPR_OPT_CULL = 0
VAPR_OPT_STREAMS = 1
VAPR_OPT_SPARSE = 2
VAPR_OPT_FUSED = 3
STATUS = {0: "VAPR_OK", 1: "VAPR_ERR_INVALID_FORMAT", 2: "VAPR_ERR_INVALID_ARG",
          3: "VAPR_ERR_SHAPE", 4: "VAPR_ERR_CUDA", 5: "VAPR_ERR_NOT_INITIALIZED",
          6: "VAPR_ERR_UNSUPPORTED"}

# every symbol include/vapr.h declares (checked by tests/test_abi.py)
EXPORTS = ("vapr_create", "vapr_destroy", "vapr_status_string", "vapr_version",
           "vapr_last_cuda_error",
           "vapr_format_parse", "vapr_format_check", "vapr_packed_row_words",
           "vapr_set_formats", "vapr_set_robot", "vapr_set_worlds", "vapr_set_goals",
           "vapr_set_option", "vapr_set_stage_events",
           "vapr_quantize", "vapr_dequantize", "vapr_fk_spheres", "vapr_world_collision",
           "vapr_self_collision", "vapr_collision", "vapr_aggregate",
           "vapr_backward_kinematics", "vapr_cost_grad_workspace_bytes",
           "vapr_cost_grad_workspace_layout", "vapr_cost_grad", "vapr_cost_grad_host",
           "vapr_lbfgs_candidates", "vapr_lbfgs_step", "vapr_best_per_problem",
           "vapr_sparse_pool_words", "vapr_sparsify", "vapr_densify",
           "vapr_cost_grad_sparse_layout")


class VaprError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


class vapr_format(ctypes.Structure):
    _fields_ = [("exp_bits", ctypes.c_int32), ("man_bits", ctypes.c_int32)]


class vapr_robot(ctypes.Structure):
    _fields_ = [("n_spheres", ctypes.c_int32), ("n_pairs", ctypes.c_int32),
                ("dh_a", ctypes.c_double * 8), ("dh_d", ctypes.c_double * 8),
                ("dh_alpha", ctypes.c_double * 8), ("hand_rz", ctypes.c_double),
                ("sphere_link", ctypes.c_void_p), ("sphere_xyzr", ctypes.c_void_p),
                ("pairs", ctypes.c_void_p),
                ("q_lo", ctypes.c_double * 7), ("q_hi", ctypes.c_double * 7)]


class vapr_cost_params(ctypes.Structure):
    _fields_ = [("eta_world", ctypes.c_float), ("eta_self", ctypes.c_float),
                ("w_world", ctypes.c_float), ("w_self", ctypes.c_float),
                ("swept", ctypes.c_int32), ("sweep_steps", ctypes.c_int32),
                ("w_pose_pos", ctypes.c_float), ("w_pose_rot", ctypes.c_float),
                ("w_bound", ctypes.c_float)]


def _load():
    if not os.path.exists(SO_PATH):
        raise ImportError(f"libvapr.so not built ({SO_PATH}); run "
                          "`python -m paper_2310_07854_b200.build`")
    lib = ctypes.CDLL(SO_PATH)
    P, I32, I64, SZ, F = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                          ctypes.c_float)
    sig = {
        "vapr_create": ([ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], I32),
        "vapr_destroy": ([P], I32),
        "vapr_status_string": ([I32], ctypes.c_char_p),
        "vapr_version": ([], ctypes.c_char_p),
        "vapr_last_cuda_error": ([], ctypes.c_char_p),
        "vapr_format_parse": ([ctypes.c_char_p, ctypes.POINTER(vapr_format)], I32),
        "vapr_format_check": ([vapr_format], I32),
        "vapr_packed_row_words": ([vapr_format, SZ], SZ),
        "vapr_set_formats": ([P, P], I32),
        "vapr_set_robot": ([P, ctypes.POINTER(vapr_robot)], I32),
        "vapr_set_worlds": ([P, I32, P, P], I32),
        "vapr_set_goals": ([P, P, I32], I32),
        "vapr_set_option": ([P, I32, I32], I32),
        "vapr_set_stage_events": ([P, P, I32], I32),
        "vapr_quantize": ([vapr_format, P, SZ, SZ, P, P], I32),
        "vapr_dequantize": ([vapr_format, P, SZ, SZ, P, P], I32),
        "vapr_fk_spheres": ([P, P, I32, I32, P, P, P], I32),
        "vapr_world_collision": ([P, P, P, I32, I32, I32, I32, F, F, P, P, P], I32),
        "vapr_self_collision": ([P, P, I32, I32, F, F, P, P, P], I32),
        "vapr_collision": ([P, P, P, I32, I32, ctypes.POINTER(vapr_cost_params), P, P, P, P, P], I32),
        "vapr_aggregate": ([P, P, I32, P, I64, P, P], I32),
        "vapr_backward_kinematics": ([P, P, I32, I32, P, P, P], I32),
        "vapr_cost_grad_workspace_bytes": ([P, I32, I32], SZ),
        "vapr_cost_grad_workspace_layout": ([P, I32, I32, I32, ctypes.POINTER(SZ * 5)], I32),
        "vapr_cost_grad": ([P, P, P, I32, I32, ctypes.POINTER(vapr_cost_params), P, SZ, P, P, P, P], I32),
        "vapr_cost_grad_host": ([P, P, P, I32, I32, ctypes.POINTER(vapr_cost_params), P, SZ, P, P, P,
                                 P, P, P, I32, P], I32),
        "vapr_lbfgs_candidates": ([P, P, I32, I32, P, I32, P, P], I32),
        "vapr_lbfgs_step": ([I32, I32, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, I32,
                             ctypes.c_float, P, P], I32),
        "vapr_best_per_problem": ([P, I32, I32, P, P, P], I32),
        "vapr_sparse_pool_words": ([vapr_format, SZ, SZ], SZ),
        "vapr_sparsify": ([vapr_format, P, SZ, SZ, P, P, P, SZ, P, P], I32),
        "vapr_densify": ([vapr_format, P, P, P, SZ, SZ, P, P], I32),
        "vapr_cost_grad_sparse_layout": ([P, I32, I32, ctypes.POINTER(SZ * 8), ctypes.POINTER(SZ)],
                                         I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if hasattr(lib, "vapr_debug_tap"):        # the test-only tap build (VAPR_SO=libvapr_tap.so)
        lib.vapr_debug_tap.argtypes = [P, I32, P]
        lib.vapr_debug_tap.restype = I32
    return lib


lib = _load()


def _check(st, where):
    if st != 0:
        if STATUS.get(st) == "VAPR_ERR_CUDA":
            where = f"{where} [{lib.vapr_last_cuda_error().decode()}]"
        raise VaprError(st, where)


def _ptr(t):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(t):
    """Host pointer of a contiguous CPU tensor (None -> NULL)."""
    if t is None:
        return None
    if t.is_cuda:
        raise ValueError("expected a host (CPU) tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(int(stream))


def fmt(f):
    if isinstance(f, vapr_format):
        return f
    if isinstance(f, str):
        out = vapr_format()
        _check(lib.vapr_format_parse(f.encode(), ctypes.byref(out)), "vapr_format_parse")
        return out
    E, M = f
    return vapr_format(int(E), int(M))


# ------------------------------------------------------------ context-free
def vapr_format_parse(s):
    f = fmt(s)
    return (f.exp_bits, f.man_bits)


def vapr_format_check(f):
    return lib.vapr_format_check(fmt(f)) == 0


def vapr_packed_row_words(f, cols):
    return int(lib.vapr_packed_row_words(fmt(f), cols))


def vapr_quantize(f, x, rows, cols, packed, stream=None):
    _check(lib.vapr_quantize(fmt(f), _ptr(x), rows, cols, _ptr(packed), _stream(stream)),
           "vapr_quantize")


def vapr_dequantize(f, packed, rows, cols, y, stream=None):
    _check(lib.vapr_dequantize(fmt(f), _ptr(packed), rows, cols, _ptr(y), _stream(stream)),
           "vapr_dequantize")


def vapr_sparse_pool_words(f, cols, rows):
    return int(lib.vapr_sparse_pool_words(fmt(f), cols, rows))


def vapr_sparsify(f, packed, rows, cols, mask, off, pool, used, stream=None):
    """Dense packed rows -> sparse form (N3); pool capacity from pool.numel()."""
    _check(lib.vapr_sparsify(fmt(f), _ptr(packed), rows, cols, _ptr(mask), _ptr(off), _ptr(pool),
                             pool.numel(), _ptr(used), _stream(stream)), "vapr_sparsify")


def vapr_densify(f, mask, off, pool, rows, cols, packed, stream=None):
    _check(lib.vapr_densify(fmt(f), _ptr(mask), _ptr(off), _ptr(pool), rows, cols, _ptr(packed),
                            _stream(stream)), "vapr_densify")


def vapr_best_per_problem(cost_traj, n_problems, seeds, best_cost, best_seed, stream=None):
    _check(lib.vapr_best_per_problem(_ptr(cost_traj), n_problems, seeds, _ptr(best_cost),
                                     _ptr(best_seed), _stream(stream)), "vapr_best_per_problem")


# ------------------------------------------------------------ context
def vapr_create(device=0):
    h = ctypes.c_void_p()
    _check(lib.vapr_create(int(device), ctypes.byref(h)), "vapr_create")
    return h


def vapr_destroy(ctx):
    _check(lib.vapr_destroy(ctx), "vapr_destroy")


def vapr_set_formats(ctx, formats):
    arr = (vapr_format * 5)(*[fmt(f) for f in formats])
    _check(lib.vapr_set_formats(ctx, ctypes.cast(arr, ctypes.c_void_p)), "vapr_set_formats")


def vapr_set_robot(ctx, robot):
    link = np.ascontiguousarray(robot["sphere_link"], np.int32)
    xyzr = np.ascontiguousarray(robot["sphere_xyzr"], np.float32)
    pairs = np.ascontiguousarray(robot["pairs"], np.uint16)
    r = vapr_robot()
    r.n_spheres = len(link)
    r.n_pairs = pairs.shape[0]
    for i in range(8):
        r.dh_a[i] = float(robot["dh_a"][i])
        r.dh_d[i] = float(robot["dh_d"][i])
        r.dh_alpha[i] = float(robot["dh_alpha"][i])
    r.hand_rz = float(robot["hand_rz"])
    for j in range(7):
        r.q_lo[j] = float(robot["q_lo"][j])
        r.q_hi[j] = float(robot["q_hi"][j])
    r.sphere_link = link.ctypes.data
    r.sphere_xyzr = xyzr.ctypes.data
    r.pairs = pairs.ctypes.data if pairs.size else None
    _check(lib.vapr_set_robot(ctx, ctypes.byref(r)), "vapr_set_robot")


def vapr_set_worlds(ctx, cuboids, offsets):
    cub = np.ascontiguousarray(cuboids, np.float32).reshape(-1, 16)
    off = np.ascontiguousarray(offsets, np.int32)
    _check(lib.vapr_set_worlds(ctx, len(off) - 1, cub.ctypes.data if cub.size else None,
                               off.ctypes.data), "vapr_set_worlds")


def vapr_set_goals(ctx, goals):
    "IKO hand-frame goals, one per problem / world: [n, 12] (R row-major, p)."
    g = np.ascontiguousarray(goals, np.float32).reshape(-1, 12)
    _check(lib.vapr_set_goals(ctx, g.ctypes.data if g.size else None, g.shape[0]),
           "vapr_set_goals")


def vapr_set_option(ctx, option, value):
    _check(lib.vapr_set_option(ctx, option, int(value)), "vapr_set_option")


def vapr_set_stage_events(ctx, events):
    """events: 6 torch.cuda.Event (or None to clear) -- vapr_cost_grad then
    records them between its stages on its stream (include/vapr.h)."""
    if not events:
        _check(lib.vapr_set_stage_events(ctx, None, 0), "vapr_set_stage_events")
        return
    for e in events:            # torch creates the CUDA event lazily
        e.record()
    arr = (ctypes.c_void_p * 6)(*[ctypes.c_void_p(e.cuda_event) for e in events])
    _check(lib.vapr_set_stage_events(ctx, arr, 6), "vapr_set_stage_events")


def cost_params(p):
    return vapr_cost_params(float(p["eta_world"]), float(p["eta_self"]), float(p["w_world"]),
                            float(p["w_self"]), int(p["swept"]), int(p["sweep_steps"]),
                            float(p.get("w_pose_pos", 0.0)), float(p.get("w_pose_rot", 0.0)),
                            float(p.get("w_bound", 0.0)))


def vapr_fk_spheres(ctx, q, B, H, out_spheres, stream=None, ee_pose=None):
    """ee_pose (optional): [B*H, 7] float32 hand position + unit quaternion (w >= 0)."""
    _check(lib.vapr_fk_spheres(ctx, _ptr(q), B, H, _ptr(out_spheres),
                               _ptr(ee_pose) if ee_pose is not None else None, _stream(stream)),
           "vapr_fk_spheres")


def vapr_world_collision(ctx, out_spheres, world_idx, B, H, swept, sweep_steps, eta, weight,
                         cost, grad, stream=None):
    _check(lib.vapr_world_collision(ctx, _ptr(out_spheres), _ptr(world_idx), B, H, int(swept),
                                    int(sweep_steps), float(eta), float(weight), _ptr(cost),
                                    _ptr(grad), _stream(stream)), "vapr_world_collision")


def vapr_self_collision(ctx, out_spheres, B, H, eta, weight, cost, out_vec, stream=None):
    _check(lib.vapr_self_collision(ctx, _ptr(out_spheres), B, H, float(eta), float(weight),
                                   _ptr(cost), _ptr(out_vec), _stream(stream)),
           "vapr_self_collision")


def vapr_collision(ctx, out_spheres, world_idx, B, H, params, cost_pose, cost_traj, cp_grad,
                   out_vec, stream=None):
    p = cost_params(params)
    _check(lib.vapr_collision(ctx, _ptr(out_spheres), _ptr(world_idx), B, H, ctypes.byref(p),
                              _ptr(cost_pose), _ptr(cost_traj), _ptr(cp_grad), _ptr(out_vec),
                              _stream(stream)), "vapr_collision")


def vapr_aggregate(ctx, cp_grad, swept, out_vec, n_rows, grad_out_spheres, stream=None):
    _check(lib.vapr_aggregate(ctx, _ptr(cp_grad), int(swept), _ptr(out_vec), int(n_rows),
                              _ptr(grad_out_spheres), _stream(stream)), "vapr_aggregate")


def vapr_backward_kinematics(ctx, q, B, H, grad_out_spheres, grad_q, stream=None):
    _check(lib.vapr_backward_kinematics(ctx, _ptr(q), B, H, _ptr(grad_out_spheres),
                                        _ptr(grad_q), _stream(stream)),
           "vapr_backward_kinematics")


def vapr_cost_grad_workspace_bytes(ctx, B, H):
    return int(lib.vapr_cost_grad_workspace_bytes(ctx, B, H))


def vapr_cost_grad_workspace_layout(ctx, B, H, swept):
    arr = (ctypes.c_size_t * 5)()
    _check(lib.vapr_cost_grad_workspace_layout(ctx, B, H, int(swept), ctypes.byref(arr)),
           "vapr_cost_grad_workspace_layout")
    return [None if v == ctypes.c_size_t(-1).value else int(v) for v in arr]


def vapr_cost_grad_sparse_layout(ctx, B, H):
    """(byte offsets of gos mask, off, used, pool, cp bitmaps, ov bitmaps, cp
    pool, ov pool; gos pool capacity in words) with VAPR_OPT_SPARSE."""
    arr = (ctypes.c_size_t * 8)()
    pw = ctypes.c_size_t()
    _check(lib.vapr_cost_grad_sparse_layout(ctx, B, H, ctypes.byref(arr), ctypes.byref(pw)),
           "vapr_cost_grad_sparse_layout")
    return [int(v) for v in arr], int(pw.value)


def vapr_cost_grad(ctx, q, world_idx, B, H, params, workspace, cost_pose, cost_traj, grad_q,
                   stream=None, _p=None):
    p = _p if _p is not None else cost_params(params)
    nbytes = workspace.numel() * workspace.element_size()
    _check(lib.vapr_cost_grad(ctx, _ptr(q), _ptr(world_idx), B, H, ctypes.byref(p),
                              _ptr(workspace), nbytes, _ptr(cost_pose), _ptr(cost_traj),
                              _ptr(grad_q), _stream(stream)), "vapr_cost_grad")


def vapr_cost_grad_host(ctx, q_host, world_idx, B, H, params, workspace, q_dev, cost_pose_dev,
                        cost_traj_dev, grad_q_dev, cost_traj_host, grad_q_host, n_chunks=0,
                        stream=None, _p=None):
    """Host-buffer variant with pipelined copies (include/vapr.h)."""
    p = _p if _p is not None else cost_params(params)
    nbytes = workspace.numel() * workspace.element_size()
    _check(lib.vapr_cost_grad_host(ctx, _hptr(q_host), _ptr(world_idx), B, H, ctypes.byref(p),
                                   _ptr(workspace), nbytes, _ptr(q_dev), _ptr(cost_pose_dev),
                                   _ptr(cost_traj_dev), _ptr(grad_q_dev), _hptr(cost_traj_host),
                                   _hptr(grad_q_host), int(n_chunks), _stream(stream)),
           "vapr_cost_grad_host")


def _scales(scales):
    arr = (ctypes.c_float * len(scales))(*[float(v) for v in scales])
    return arr, len(scales)


def vapr_lbfgs_candidates(x, d, B, D, scales, cand, stream=None):
    """cand [N, B, D] = fl(x + fl(s_n d)) (include/vapr.h, N1 step (1))."""
    arr, n = _scales(scales)
    _check(lib.vapr_lbfgs_candidates(_ptr(x), _ptr(d), B, D, arr, n, _ptr(cand), _stream(stream)),
           "vapr_lbfgs_candidates")


def vapr_lbfgs_step(B, D, scales, cand_cost, cand_grad, x, g, cost, d, hist_s, hist_y, hist_rho,
                    hist_count, hist_head, chosen=None, m=10, curvature_eps=1e-10, fixed=None,
                    stream=None):
    """Line-search selection, history update and two-loop direction (N1 steps (6), (7))."""
    arr, n = _scales(scales)
    _check(lib.vapr_lbfgs_step(B, D, arr, n, _ptr(cand_cost), _ptr(cand_grad), _ptr(x), _ptr(g),
                               _ptr(cost), _ptr(d), _ptr(hist_s), _ptr(hist_y), _ptr(hist_rho),
                               _ptr(hist_count), _ptr(hist_head), _ptr(chosen), int(m),
                               float(curvature_eps), _ptr(fixed), _stream(stream)),
           "vapr_lbfgs_step")
