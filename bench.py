"""bench.py -- rollout cost+grad throughput of the VaPr hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--formats 43bit] [--impl vapr|reference]

A step = one vapr_cost_grad over the whole resident batch (FK -> fused world
(swept) + self collision -> aggregate -> BK, every live tensor packed in HBM)
plus the per-problem best-seed reduction (and, for N > 1, one NCCL all-gather
of the per-problem results).  Workload = BASELINE.json config 4 per GPU:
800 problems (100 per MotionBenchMaker-like environment) x 100 TO seeds x 32
steps = 2.56M poses, 52 spheres (weak scaling: every rank owns its own 800
problems).  The working set (~1.5 GB of packed tensors at 43 bits) is >10x
the 126 MB L2, so no flush is needed between steps.  One JSON line on rank 0.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rollout cost+grad evals/sec (B*H*spheres) and HBM GB/s vs peak, per format set"
UNIT = "sphere-evals/s"
# libvapr launches per step: fk, collision world pass, collision self pass,
# traj_reduce, aggregate, bk (vapr_cost_grad) + best_per_problem
LAUNCHES_PER_STEP = 7
S = 52


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="vapr", choices=["vapr", "reference"])
    ap.add_argument("--formats", default="43bit")
    ap.add_argument("--problems-per-env", type=int, default=100)
    ap.add_argument("--seeds", type=int, default=100)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=0,
                    help="e2e: trajectory chunks of the pipelined host call (0 = automatic)")
    ap.add_argument("--storage", default="sparse", choices=["sparse", "dense"],
                    help="grad_out_spheres / collision-output storage inside vapr_cost_grad "
                         "(VAPR_OPT_SPARSE, N3; results bit-identical)")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32 comparison run")
    ap.add_argument("--no-iko", action="store_true",
                    help="skip the IKO leg (N2: H = 1, 1000 seeds x 800 problems, pose + bound costs)")
    ap.add_argument("--no-to", action="store_true",
                    help="skip the TO-iteration leg (N1: L-BFGS + N-scale line search)")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the end-to-end leg (profiling runs: keeps the launch list to the device step)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph legs")
    ap.add_argument("--cpu-sample-poses", type=int, default=20480)
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
def packing_factor(E, M):
    return 32 // (1 + E + M)


def v_alg(fmt):
    """Algorithmic bytes of one packed pose row: 4 * 3S / pf (the paper's
    register-packing model)."""
    return 4.0 * 3 * S / packing_factor(*fmt)


def stage_bytes(fm, swept=True):
    """Algorithmic HBM bytes per pose of each kernel."""
    os_, gos, ov, cp, cps = (v_alg(f) for f in fm)
    c = cps if swept else cp
    return {"fk": 28 + os_, "collision": os_ + c + ov + 4, "aggregate": c + ov + gos,
            "bk": 28 + gos + 28}


class Clocks:
    """Samples nvidia-smi clocks / throttle reasons in a background thread."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- cpu / oracle
def oracle_sample(fm, n_poses, H, key_offset=0):
    """A bounded sample of the config-4 workload (same generator, same
    formats) for the oracle: n_poses // H trajectories spread over the 8
    environments."""
    from workloads import config4
    from workloads.scenes import ENVIRONMENTS
    n_traj = max(8, n_poses // H)
    seeds = max(1, n_traj // len(ENVIRONMENTS))
    return config4(problems_per_env=1, seeds=seeds, H=H, formats=fm,
                   problem_offset=key_offset, n_problems=len(ENVIRONMENTS))


def run_oracle(wl):
    from oracle.rollout import rollout_workload
    t0 = time.perf_counter()
    rollout_workload(wl)
    return time.perf_counter() - t0


def cpu_baseline(fm, H, n_poses):
    wl = oracle_sample(fm, n_poses, H)
    dt = run_oracle(wl)
    return {"value": wl.poses * S / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{wl.poses} poses ({wl.B} trajectories x {H} steps, 8 envs) of the same "
                      f"workload generator, float64 numpy + C codec, single thread, {dt:.1f} s"}


# ----------------------------------------------------------------- reference arm
def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads.configs import FORMAT_SETS
    fm = FORMAT_SETS[args.formats]
    n_poses = max(args.H * 8, args.cpu_sample_poses // 4)
    wl = oracle_sample(fm, n_poses, args.H)
    for _ in range(args.warmup):
        run_oracle(wl)
    times = [run_oracle(wl) for _ in range(args.steps)]
    t = float(np.sum(times))
    value = wl.poses * S * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config4 sample: {wl.poses} poses/step ({wl.B} traj x "
                                   f"{args.H} steps, 8 envs), formats {args.formats}",
                       "formats": args.formats},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{wl.poses} poses per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2310_07854_b200 import binding as vb
    from paper_2310_07854_b200.rollout import Rollout
    from paper_2310_07854_b200.dist import shard_problems, gather_best, max_over_ranks
    from workloads import config4
    from workloads.configs import FORMAT_SETS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("VAPR_DIST_BACKEND", "nccl") != "nccl":
        local = 0                     # functional multi-rank check on one GPU
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink; VAPR_DIST_BACKEND=gloo is a functional check of the
        # multi-rank logic on one GPU (never a measurement)
        backend = os.environ.get("VAPR_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    fm = FORMAT_SETS[args.formats]
    n_prob = args.problems_per_env * 8
    # weak scaling: rank r owns global problems [r*n_prob, (r+1)*n_prob)
    ids = shard_problems(rank, world, per_rank=n_prob)
    wl = config4(problems_per_env=args.problems_per_env, seeds=args.seeds, H=args.H,
                 formats=fm, problem_offset=ids[0], n_problems=len(ids))
    P = wl.poses
    sparse = args.storage == "sparse"
    r = Rollout(wl, device=local, sparse=sparse)
    stream = torch.cuda.current_stream(dev)
    best_c = torch.empty(n_prob, dtype=torch.float32, device=dev)
    best_s = torch.empty(n_prob, dtype=torch.int32, device=dev)

    def step():
        r.run()
        vb.vapr_best_per_problem(r.cost_traj, n_prob, args.seeds, best_c, best_s)
        gather_best(best_c, best_s, world)       # the path's only collective

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, k, w):
        for _ in range(w):
            fn()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1), dev) / k

    with Clocks(local) as clk:
        ms = timed(step, args.steps, args.warmup)
    clocks = clk.summary()
    value = world * P * S / (ms * 1e-3)

    # measured sparsity of the gradient tensors ("report the
    # measured nonzero fraction per run"; PAPER.md:196 >99 % zeros), from the
    # sparse mode's per-pose sphere bitmaps of the last step
    sparsity = None
    if sparse:
        offs, _ = vb.vapr_cost_grad_sparse_layout(r.ctx.h, wl.B, wl.H)
        names_m = {"grad_out_spheres": offs[0], "closest_pt_swept": offs[4], "out_vec": offs[5]}
        sparsity = {}
        for nm, o in names_m.items():
            m = r.workspace[o:o + 8 * P].view(torch.int64)
            bits = torch.zeros(P, dtype=torch.int64, device=dev)
            for k in range(S):
                bits += (m >> k) & 1
            sparsity[nm] = {"nonzero_sphere_frac": round(float(bits.sum()) / (P * S), 5),
                            "nonzero_pose_frac": round(float((bits > 0).sum()) / P, 4)}

    # ---- per-kernel durations (the stage entry points, launched stage by
    # stage on the same stream with events between them; dense storage: the
    # standalone calls take dense tensors) for the roofline of the dominant one
    p = wl.params
    swept = p["swept"]
    rd = Rollout(wl, device=local) if sparse else r
    lay = vb.vapr_cost_grad_workspace_layout(rd.ctx.h, wl.B, wl.H, swept)
    W = {i: vb.vapr_packed_row_words(fm[i], 3 * S) for i in range(5)}
    cps = 4 if swept else 3
    ws = rd.workspace

    def slot(i):
        return ws[lay[i]:lay[i] + 4 * W[i] * P]

    names = ["fk", "collision", "aggregate", "bk"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    acc = {n: 0.0 for n in names}

    def staged():
        ev[0].record(stream)
        vb.vapr_fk_spheres(rd.ctx.h, rd.q, wl.B, wl.H, slot(0))
        ev[1].record(stream)
        vb.vapr_collision(rd.ctx.h, slot(0), rd.world_idx, wl.B, wl.H, p, rd.cost_pose,
                          rd.cost_traj, slot(cps), slot(2))
        ev[2].record(stream)
        vb.vapr_aggregate(rd.ctx.h, slot(cps), swept, slot(2), P, slot(1))
        ev[3].record(stream)
        vb.vapr_backward_kinematics(rd.ctx.h, rd.q, wl.B, wl.H, slot(1), rd.grad_q)
        ev[4].record(stream)

    for _ in range(2):
        staged()
    torch.cuda.synchronize(dev)
    for _ in range(args.steps):
        staged()
        torch.cuda.synchronize(dev)
        for i, n in enumerate(names):
            acc[n] += ev[i].elapsed_time(ev[i + 1])
    kms = {n: acc[n] / args.steps for n in names}
    sb = stage_bytes(fm, bool(swept))
    a_min = sum(sb.values())
    dom = max(kms, key=kms.get)
    hbm, peak_kind = peaks()
    achieved = sb[dom] * P / (kms[dom] * 1e-3) / 1e9
    traffic = None
    try:        # DRAM bytes per launch from the committed ncu capture of this workload
        tj = json.load(open(os.path.join(ROOT, "profiles", "r1", "traffic.json")))
        if tj["formats"] == args.formats and tj["poses"] == P:
            traffic = tj["bytes_per_launch"].get(dom)
    except Exception:
        pass
    if rd is not r:
        del rd, ws
        torch.cuda.empty_cache()
    issue = None
    try:        # the dominant kernel is issue-bound: its ncu issue utilisation
        ij = json.load(open(os.path.join(ROOT, "profiles", "r1", "issue.json")))
        issue = ij.get(dom)
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "stage_calls": "dense standalone entry points", "achieved": achieved, "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "bytes_per_launch_alg": sb[dom] * P, "bytes_per_pose": sb[dom],
                "limiter": ("instruction issue (ncu, profiles/r1/issue.json); HBM frac is low "
                            "because the collision passes spend ~10x more issue slots than bytes"),
                "issue": issue,
                "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
                "kernel_frac": {n: round(sb[n] * P / (kms[n] * 1e-3) / 1e9 / hbm, 4) for n in names}}

    # ---- the step as a CUDA graph (SURVEY.md §8(d) timing protocol), on the
    # bench workload and on the launch-bound config 2 (eager vs graph)
    graph = None
    if not args.no_graph:
        from workloads import config2
        g = r.capture_graph()
        graph = {"ms_per_step": timed(g.replay, args.steps, args.warmup)}
        del g
        r2 = Rollout(config2(), device=local, sparse=sparse)
        g2 = r2.capture_graph()
        graph["config2_eager_us"] = 1e3 * timed(r2.run, 50, 10)
        graph["config2_graph_us"] = 1e3 * timed(g2.replay, 50, 10)
        del g2, r2
        torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers
    q_host = torch.from_numpy(np.ascontiguousarray(wl.q)).pin_memory()
    gq_host = torch.empty(P * 7, dtype=torch.float32).pin_memory()
    ct_host = torch.empty(wl.B, dtype=torch.float32).pin_memory()

    def e2e_step():
        # vapr_cost_grad_host: H2D of q, compute and D2H of grad_q / cost_traj
        # pipelined over trajectory chunks (the public host-buffer call)
        r.run_host(q_host, gq_host, ct_host, n_chunks=args.chunks)
        vb.vapr_best_per_problem(r.cost_traj, n_prob, args.seeds, best_c, best_s)
        gather_best(best_c, best_s, world)

    e2e = None
    if not args.no_e2e:
        e2e_ms = timed(e2e_step, max(3, args.steps // 2), 2)
        e2e = {"value": world * P * S / (e2e_ms * 1e-3), "unit": UNIT, "chunks": args.chunks,
               "h2d_bytes_per_step": q_host.numel() * 4,
               "d2h_bytes_per_step": gq_host.numel() * 4 + ct_host.numel() * 4,
               "ms_per_step": e2e_ms}

    # ---- a full TO iteration: candidates for N step
    # scales, vapr_cost_grad over the N x B batch, line search + L-BFGS
    to_iter = None
    if not args.no_to:
        from paper_2310_07854_b200.optimize import TrajOpt
        opt = TrajOpt(wl, device=local, sparse=sparse)
        opt.reset()
        to_ms = timed(opt.step, max(3, args.steps // 4), 2)
        to_iter = {"ms_per_iteration": to_ms, "line_search_scales": list(opt.scales),
                   "trajectories": opt.B * world, "poses_evaluated_per_iteration": opt.N * P * world,
                   "trajectory_iterations_per_s": opt.B * world / (to_ms * 1e-3),
                   "history_m": opt.m}
        del opt
        torch.cuda.empty_cache()

    # ---- the IKO workload: H = 1, pose + bound + discrete
    # world + self costs; one vapr_cost_grad and one full L-BFGS iteration
    iko = None
    if not args.no_iko:
        from paper_2310_07854_b200.optimize import TrajOpt
        from workloads import config_iko
        wli = config_iko(problems_per_env=args.problems_per_env, seeds=1000, formats=fm,
                         problem_offset=ids[0], n_problems=len(ids))
        opt = TrajOpt(wli, device=local, sparse=sparse)
        opt.reset()
        ev_ms = timed(opt.base.run, max(3, args.steps // 2), 2)
        it_ms = timed(opt.step, max(3, args.steps // 4), 2)
        iko = {"poses": wli.poses * world, "seeds_per_problem": 1000,
               "cost_grad_ms": ev_ms, "cost_grad_pose_evals_per_s": wli.poses * world / (ev_ms * 1e-3),
               "iteration_ms": it_ms, "line_search_scales": list(opt.scales),
               "seed_iterations_per_s": wli.B * world / (it_ms * 1e-3)}
        del opt
        torch.cuda.empty_cache()

    # ---- FP32 comparison (the >= 2x target of BASELINE.json) on the same batch
    fp32 = None
    if not args.no_fp32 and args.formats != "fp32":
        r.set_formats(FORMAT_SETS["fp32"])
        ms32 = timed(step, max(3, args.steps // 2), 2)
        fp32 = {"value": world * P * S / (ms32 * 1e-3), "ms_per_step": ms32,
                "speedup_of_formats": ms32 / ms, "storage": args.storage}
        r.set_formats(fm)
        if sparse:
            # the paper's baseline layout: FP32 in dense storage (its sparsity is
            # compute skipping only)
            r32 = Rollout(wl, device=local, formats=FORMAT_SETS["fp32"])

            def step32():
                r32.run()
                vb.vapr_best_per_problem(r32.cost_traj, n_prob, args.seeds, best_c, best_s)
                gather_best(best_c, best_s, world)

            ms32d = timed(step32, max(3, args.steps // 2), 2)
            fp32["dense_ms_per_step"] = ms32d
            fp32["speedup_vs_dense_fp32"] = ms32d / ms
            del r32
            torch.cuda.empty_cache()

    if rank == 0:
        # the oracle leg runs on rank 0 of a 1-GPU run only (the contract)
        cpu = None if (args.no_cpu or world > 1) else cpu_baseline(fm, args.H, args.cpu_sample_poses)
        bits = sum(1 + e + m for e, m in fm)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32+packed-ExMy", "data": "synthetic",
            "config": {"workload": f"config4: {n_prob} problems ({args.problems_per_env} per "
                                   f"MBM-like env) x {args.seeds} TO seeds x {args.H} steps per GPU, "
                                   "52 spheres, swept n=1",
                       "formats": args.formats, "format_bits": bits,
                       "storage": args.storage + (" (VAPR_OPT_SPARSE: collision outputs as masked "
                                                   "rows, grad_out_spheres as bitmap + packed codes)"
                                                   if sparse else ""),
                       "formats_exmy": ["E%dM%d" % f for f in fm],
                       "poses_per_gpu": P, "problems_per_gpu": n_prob,
                       "l2": "inputs > L2 (packed working set >> 126 MB), no flush",
                       "parallelism": f"problem-sharded x{world}"},
            "hbm_alg_gbs": a_min * P * world / (ms * 1e-3) / 1e9,
            "hbm_frac_step": a_min * P / (ms * 1e-3) / 1e9 / hbm,
            "bytes_per_pose_alg": a_min,
            "roofline": roofline,
            "e2e": e2e,
            "graph": graph,
            "sparsity": sparsity,
            "fp32": fp32,
            "to_iteration": to_iter,
            "iko": iko,
            "cpu_baseline": cpu,
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
