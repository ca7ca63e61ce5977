"""bench.py -- rollout cost+grad throughput of the VaPr hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--formats 43bit] [--impl vapr|reference]
                    [--scaling strong|weak] [--storage sparse|dense]

A step = one vapr_cost_grad over the whole resident batch (FK -> world (swept)
and self collision -> aggregate -> BK, every live tensor packed in HBM) plus
the per-problem best-seed reduction (and, for N > 1, one NCCL all-gather of
the per-problem results).  Workload = BASELINE.json config 4: 800 problems
(100 per MotionBenchMaker-like environment) x 100 TO seeds x 32 steps, 52
spheres; `--scaling strong` (default, the configured split)
shards the 800 problems round-robin (problem p on rank p mod N, so every rank
keeps the environment mix); `--scaling weak` gives every rank its own 800.
At N = 1 both are the 2.56M-pose batch.  The working set (~1.5 GB of packed
tensors at 43 bits) is >10x the 126 MB L2, so no flush is needed between
steps.  One JSON line on rank 0.
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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: config 4's 800 problems sharded round-robin over the ranks; "
                         "weak: 800 problems per rank")
    ap.add_argument("--problems-per-env", type=int, default=100)
    ap.add_argument("--seeds", type=int, default=100)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=0,
                    help="e2e: trajectory chunks of the pipelined host call (0 = automatic)")
    ap.add_argument("--storage", default="sparse", choices=["sparse", "dense"],
                    help="grad_out_spheres / collision-output storage inside vapr_cost_grad "
                         "(VAPR_OPT_SPARSE, N3; results bit-identical)")
    ap.add_argument("--no-formats", action="store_true",
                    help="skip the format-set legs (FP32, FP16, per-environment Table II, dense)")
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
    return {"fk": 28 + os_, "collision": os_ + c + ov + 4, "reduce": 4 + 4.0 / 32,
            "aggregate": c + ov + gos, "bk": 28 + gos + 28}


def a_min(fm, swept=True):
    """A_min: the path's algorithmic bytes per pose: q read
    twice, grad_q written, one FP32 cost, every live packed tensor written
    once and read once."""
    os_, gos, ov, cp, cps = (v_alg(f) for f in fm)
    c = cps if swept else cp
    return 28 + 28 + 28 + 4 + 2 * (os_ + c + ov + gos)


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


def shard_ids(scaling, rank, world, problems_per_env):
    from paper_2310_07854_b200.dist import shard_problems
    n = problems_per_env * 8
    if scaling == "weak":
        return shard_problems(rank, world, per_rank=n)
    return shard_problems(rank, world, n_global=n, mode="strong")


# ----------------------------------------------------------------- cpu / oracle
# The oracle (test infrastructure, oracle/) timed on the host cores: a bounded
# sample of the config-4 workload (same generator, same formats), on one core
# and on all of them (a process pool over trajectory chunks).
def oracle_sample(fm, n_poses, H):
    """n_poses // H trajectories spread over the 8 environments."""
    from workloads import config4
    from workloads.scenes import ENVIRONMENTS
    n_traj = max(8, n_poses // H)
    seeds = max(1, n_traj // len(ENVIRONMENTS))
    return config4(problems_per_env=1, seeds=seeds, H=H, formats=fm,
                   problem_offset=0, n_problems=len(ENVIRONMENTS))


def _oracle_chunk(args):
    """Worker: the oracle rollout of trajectories [b0, b1) of the sample."""
    import dataclasses
    from oracle.rollout import rollout_workload
    wl, b0, b1 = args
    sub = dataclasses.replace(wl, q=wl.q[b0:b1], world_idx=wl.world_idx[b0:b1])
    t0 = time.perf_counter()
    rollout_workload(sub)
    return time.perf_counter() - t0


def _pool(cores):
    import multiprocessing as mp
    env = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}
    os.environ.update(env)
    ctx = mp.get_context("spawn")          # no CUDA state crosses into the workers
    pool = ctx.Pool(cores)
    pool.map(_oracle_chunk, [(oracle_sample(((8, 23),) * 5, 64, 32), 0, 1)] * cores)   # warm up
    return pool


def oracle_time(wl, cores, pool=None):
    """Wall seconds of the oracle over the sample: 1 core in-process, or
    `cores` workers over equal trajectory chunks."""
    if cores == 1:
        return _oracle_chunk((wl, 0, wl.B))
    cuts = np.linspace(0, wl.B, cores + 1).astype(int)
    t0 = time.perf_counter()
    pool.map(_oracle_chunk, [(wl, int(cuts[i]), int(cuts[i + 1])) for i in range(cores)])
    return time.perf_counter() - t0


def cpu_baseline(fm, H, n_poses):
    wl = oracle_sample(fm, n_poses, H)
    cores = os.cpu_count() or 1
    t1 = oracle_time(wl, 1)
    out = {"value": None, "unit": UNIT, "cores": cores, "kind": "oracle",
           "value_1core": wl.poses * S / t1,
           "sample": f"{wl.poses} poses ({wl.B} trajectories x {H} steps, 8 envs) of the same "
                     f"workload generator, float64 numpy + C codec; 1 core {t1:.1f} s"}
    if cores > 1:
        pool = _pool(cores)
        try:
            tn = oracle_time(wl, cores, pool)
        finally:
            pool.close()
            pool.join()
        out["value"] = wl.poses * S / tn
        out["sample"] += f", {cores} cores (process pool over trajectory chunks) {tn:.2f} s"
    else:
        out["value"] = out["value_1core"]
    return out


# ----------------------------------------------------------------- reference arm
def reference_arm(args):
    """The base contract's reference arm for this tier: the oracle as it
    stands, on the box's host cores (a process pool), on the same metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads.configs import FORMAT_SETS
    fm = FORMAT_SETS[args.formats]
    cores = os.cpu_count() or 1
    n_poses = max(args.H * 8 * cores, args.cpu_sample_poses)
    wl = oracle_sample(fm, n_poses, args.H)
    pool = _pool(cores) if cores > 1 else None
    try:
        for _ in range(args.warmup):
            oracle_time(wl, cores, pool)
        times = [oracle_time(wl, cores, pool) for _ in range(args.steps)]
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    t = float(np.sum(times))
    value = wl.poses * S * args.steps / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config4 sample: {wl.poses} poses/step ({wl.B} traj x "
                                   f"{args.H} steps, 8 envs), formats {args.formats}",
                       "formats": args.formats},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{wl.poses} poses per step, {cores} worker processes"},
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
    from paper_2310_07854_b200.dist import gather_best, max_over_ranks
    from workloads import config4
    from workloads.configs import FORMAT_SETS
    from workloads.scenes import ENVIRONMENTS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("VAPR_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = 0                     # functional multi-rank check on one GPU
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink, its init log on (the driver checks nranks);
        # VAPR_DIST_BACKEND=gloo is a functional check of the multi-rank logic
        # on one GPU (never a measurement)
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    fm = FORMAT_SETS[args.formats]
    ids = shard_ids(args.scaling, rank, world, args.problems_per_env)
    n_prob = len(ids)
    wl = config4(problems_per_env=args.problems_per_env, seeds=args.seeds, H=args.H,
                 formats=fm, problem_ids=ids)
    P = wl.poses
    sparse = args.storage == "sparse"
    r = Rollout(wl, device=local, sparse=sparse)
    stream = torch.cuda.current_stream(dev)
    best_c = torch.empty(n_prob, dtype=torch.float32, device=dev)
    best_s = torch.empty(n_prob, dtype=torch.int32, device=dev)

    def step_of(rr, n_p=n_prob, seeds=args.seeds, bc=best_c, bs=best_s):
        def f():
            rr.run()
            vb.vapr_best_per_problem(rr.cost_traj, n_p, seeds, bc, bs)
            gather_best(bc, bs, world)       # the path's only collective
        return f

    step = step_of(r)

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

    # poses processed by all ranks per step
    poses_total = (P * world if args.scaling == "weak"
                   else args.problems_per_env * 8 * args.seeds * args.H)
    with Clocks(local) as clk:
        ms = timed(step, args.steps, args.warmup)
    clocks = clk.summary()
    value = poses_total * S / (ms * 1e-3)

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

    # ---- per-kernel durations of the timed step itself: vapr_cost_grad
    # records caller-owned CUDA events between its launches on its stream
    # (vapr_set_stage_events), so the roofline is taken on exactly the kernels
    # the step runs (sparse storage included)
    names = ["fk", "collision", "reduce", "aggregate", "bk"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    vb.vapr_set_stage_events(r.ctx.h, ev)
    acc = {n: 0.0 for n in names}
    for _ in range(2):
        r.run()
    torch.cuda.synchronize(dev)
    for _ in range(args.steps):
        r.run()
        torch.cuda.synchronize(dev)
        for i, n in enumerate(names):
            acc[n] += ev[i].elapsed_time(ev[i + 1])
    vb.vapr_set_stage_events(r.ctx.h, None)
    kms = {n: acc[n] / args.steps for n in names}
    swept = bool(wl.params["swept"])
    sb = stage_bytes(fm, swept)
    dom = max(kms, key=kms.get)
    hbm, peak_kind = peaks()
    achieved = sb[dom] * P / (kms[dom] * 1e-3) / 1e9
    prof = {}
    try:        # DRAM bytes per launch and the limiter, from the committed ncu capture
        prof = json.load(open(os.path.join(ROOT, "profiles", "r2", "roofline_ncu.json")))
    except Exception:
        pass
    kp = prof.get("kernels", {}).get(dom, {}) if prof.get("formats") == args.formats and \
        prof.get("poses") == P else {}
    # "bound" names the roofline the fraction is taken against (the path is
    # HBM-shaped: bytes per pose, no dense contraction); "regime" what ncu
    # measured the dominant kernel to be limited by (profiles/r2)
    roofline = {"bound": "hbm", "kernel": dom,
                "regime": ("instruction issue (both passes ~75 % issue-active at 22-24 warps/SM, 16-bit tile rows)"
                           if dom == "collision" else "see limiter"),
                "stage_calls": "the timed step's own launches (vapr_set_stage_events, "
                               f"{args.storage} storage)",
                "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": kp.get("dram_bytes"),
                "bytes_per_launch_alg": sb[dom] * P, "bytes_per_pose": sb[dom],
                "limiter": kp.get("limiter", "see profiles/r2 (ncu)"),
                "issue": kp.get("issue"),
                "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
                "kernel_frac": {n: round(sb[n] * P / (kms[n] * 1e-3) / 1e9 / hbm, 4) for n in names}}

    # ---- the step as a CUDA graph (SURVEY.md §8(d) timing protocol), on the
    # bench workload and on the launch-bound configs 1 and 2 (eager vs graph)
    graph = None
    if not args.no_graph:
        from workloads import config1, config2
        g = r.capture_graph()
        graph = {"ms_per_step": timed(g.replay, args.steps, args.warmup)}
        del g
        for nm, wsmall in (("config1", config1()), ("config2", config2())):
            r2 = Rollout(wsmall, device=local, sparse=sparse)
            g2 = r2.capture_graph()
            graph[f"{nm}_eager_us"] = 1e3 * timed(r2.run, 50, 10)
            graph[f"{nm}_graph_us"] = 1e3 * timed(g2.replay, 50, 10)
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
        e2e = {"value": poses_total * S / (e2e_ms * 1e-3), "unit": UNIT, "chunks": args.chunks,
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
                   "trajectories": opt.B, "poses_evaluated_per_iteration": opt.N * P,
                   "trajectory_iterations_per_s": opt.B / (to_ms * 1e-3),
                   "history_m": opt.m, "per_rank": True}
        del opt
        torch.cuda.empty_cache()

    # ---- the IKO workload: H = 1, pose + bound + discrete
    # world + self costs; one vapr_cost_grad and one full L-BFGS iteration
    iko = None
    if not args.no_iko:
        from paper_2310_07854_b200.optimize import TrajOpt
        from workloads import config_iko
        wli = config_iko(problems_per_env=args.problems_per_env, seeds=1000, formats=fm,
                         problem_ids=ids)
        opt = TrajOpt(wli, device=local, sparse=sparse)
        opt.reset()
        ev_ms = timed(opt.base.run, max(3, args.steps // 2), 2)
        it_ms = timed(opt.step, max(3, args.steps // 4), 2)
        iko = {"poses": wli.poses, "seeds_per_problem": 1000,
               "cost_grad_ms": ev_ms, "cost_grad_pose_evals_per_s": wli.poses / (ev_ms * 1e-3),
               "iteration_ms": it_ms, "line_search_scales": list(opt.scales),
               "seed_iterations_per_s": wli.B / (it_ms * 1e-3), "per_rank": True}
        del opt
        torch.cuda.empty_cache()

    # ---- format sets on the same batch (FP32,
    # FP16-all, each environment's own Table II row, and the 43-bit set in
    # dense storage -- the method's materialised layout)
    formats = None
    if not args.no_formats:
        formats = {}

        def leg(name, fmt_set, storage):
            rr = r if (storage == args.storage and fmt_set == fm) else \
                Rollout(wl, device=local, formats=fmt_set, sparse=(storage == "sparse"),
                        fused=(storage == "fused"))
            t = timed(step_of(rr), max(3, args.steps // 2), 2)
            bits = sum(1 + e + m for e, m in fmt_set)
            formats[name] = {"ms_per_step": t, "value": poses_total * S / (t * 1e-3),
                             "storage": storage, "bits": bits,
                             # fused (N4): no tensor touches HBM -- q in, grad_q / cost out
                             "hbm_frac_step": (a_min(fmt_set, swept) if storage != "fused" else 60)
                             * P / (t * 1e-3) / 1e9 / hbm}
            if rr is not r:
                del rr
                torch.cuda.empty_cache()

        for st in ("sparse", "dense", "fused"):
            leg(f"fp32_{st}", FORMAT_SETS["fp32"], st)
            leg(f"fp16_{st}", FORMAT_SETS["fp16"], st)
            leg(f"{args.formats}_{st}", fm, st)
        # every environment with its own Table II row: the
        # rank's problems of environment e as one sub-batch with e's formats,
        # the eight sub-batches back to back as one step
        subs = []
        for e, env in enumerate(ENVIRONMENTS):
            eids = [p for p in ids if p % 8 == e]
            if not eids:
                continue
            we = config4(problems_per_env=args.problems_per_env, seeds=args.seeds, H=args.H,
                         formats=FORMAT_SETS[env], problem_ids=eids)
            re_ = Rollout(we, device=local, sparse=sparse)
            bc = torch.empty(len(eids), dtype=torch.float32, device=dev)
            bs = torch.empty(len(eids), dtype=torch.int32, device=dev)
            subs.append((re_, len(eids), bc, bs))

        def env_step():
            for re_, ne, bc, bs in subs:
                re_.run()
                vb.vapr_best_per_problem(re_.cost_traj, ne, args.seeds, bc, bs)
            gather_best(best_c, best_s, world)

        t = timed(env_step, max(3, args.steps // 2), 2)
        formats["per_env_table2"] = {
            "ms_per_step": t, "value": poses_total * S / (t * 1e-3), "storage": args.storage,
            "bits": {env: sum(1 + e + m for e, m in FORMAT_SETS[env]) for env in ENVIRONMENTS}}
        del subs
        torch.cuda.empty_cache()
        for st in ("sparse", "dense", "fused"):
            f32 = formats[f"fp32_{st}"]["ms_per_step"]
            for k in list(formats):
                if k.endswith(st) or (k == "per_env_table2" and st == args.storage):
                    formats[k][f"speedup_vs_fp32_{st}"] = f32 / formats[k]["ms_per_step"]

    if rank == 0:
        # the oracle leg runs on rank 0 of a 1-GPU run only (the contract)
        cpu = None if (args.no_cpu or world > 1) else cpu_baseline(fm, args.H, args.cpu_sample_poses)
        bits = sum(1 + e + m for e, m in fm)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32+packed-ExMy", "data": "synthetic",
            "config": {"workload": f"config4: {args.problems_per_env * 8} problems "
                                   f"({args.problems_per_env} per MBM-like env) x {args.seeds} TO "
                                   f"seeds x {args.H} steps, 52 spheres, swept n=1, "
                                   + ("sharded round-robin over the ranks (problem p on rank p mod N)"
                                      if args.scaling == "strong" else "per rank"),
                       "formats": args.formats, "format_bits": bits,
                       "storage": args.storage + (" (VAPR_OPT_SPARSE: collision outputs as masked "
                                                   "rows, grad_out_spheres as bitmap + packed codes)"
                                                   if sparse else ""),
                       "formats_exmy": ["E%dM%d" % f for f in fm],
                       "poses_per_gpu": P, "problems_per_gpu": n_prob,
                       "l2": "inputs > L2 (packed working set >> 126 MB), no flush",
                       "parallelism": f"problem-sharded x{world} ({args.scaling})"},
            "nccl_ranks": world,
            "hbm_alg_gbs": a_min(fm, swept) * poses_total / (ms * 1e-3) / 1e9,
            "hbm_frac_step": a_min(fm, swept) * P / (ms * 1e-3) / 1e9 / hbm,
            "bytes_per_pose_alg": a_min(fm, swept),
            "roofline": roofline,
            "e2e": e2e,
            "graph": graph,
            "sparsity": sparsity,
            "format_sets": formats,
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
