"""BASELINE.json's five configs as concrete seeded synthetic inputs
("Configs").

A Workload carries host numpy arrays only; the oracle and the CUDA binding
each consume them.  Sizes can be scaled down (problems per environment,
seeds, horizon) for parity tests while keeping the structure.
"""
from dataclasses import dataclass, field

import numpy as np

from .robot import panda_robot
from .scenes import ENVIRONMENTS, make_worlds, _key
from .trajectories import make_trajectories

# Slot order: out_spheres, grad_out_spheres, out_vec, closest_pt,
# closest_pt_swept (Table II column order).
FP32 = ((8, 23),) * 5
FP16 = ((5, 10),) * 5
FORMAT_SETS = {
    "fp32": FP32,
    "fp16": FP16,
    # Table II combinatorial rows
    "bookshelf_small": ((5, 10), (4, 3), (2, 1), (2, 2), (4, 3)),
    "bookshelf_tall": ((5, 10), (3, 1), (2, 1), (2, 1), (3, 1)),
    "bookshelf_thin": ((5, 10), (2, 3), (3, 1), (3, 2), (2, 2)),
    "box": ((5, 10), (3, 2), (2, 2), (3, 2), (3, 1)),
    "box_flipped": ((5, 10), (2, 1), (3, 2), (2, 2), (3, 1)),
    "cage": ((5, 10), (5, 2), (2, 1), (2, 1), (2, 3)),
    "table_pick": ((8, 7), (3, 1), (3, 1), (2, 2), (3, 2)),
    "table_under_pick": ((5, 10), (3, 2), (2, 2), (4, 3), (4, 3)),
    # config 1's reduced set: out_spheres E4M3, rest FP32
    "config1_e4m3": ((4, 3),) + ((8, 23),) * 4,
    # per-slot maxima of Table II quoted in the appendix
    "maxima46": ((5, 10), (4, 3), (3, 2), (4, 3), (4, 3)),
    # packing-factor coverage for the parity tests: pf 5 and 8 leave a
    # partial last word in a 156-element row; pf 3 (t = 10); E8M7 (bf16 cvt)
    "pf5_pf8": ((2, 3), (2, 1), (3, 2), (2, 1), (4, 1)),
    "pf3": ((5, 4), (3, 6), (6, 3), (2, 7), (4, 5)),
    "bf16": ((8, 7),) * 5,
}
FORMAT_SETS["43bit"] = FORMAT_SETS["table_under_pick"]

DEFAULT_PARAMS = dict(eta_world=0.025, eta_self=0.01, w_world=1.0,
                      w_self=1.0, swept=1, sweep_steps=1,
                      w_pose_pos=0.0, w_pose_rot=0.0, w_bound=0.0)


@dataclass
class Workload:
    name: str
    q: np.ndarray                 # [B, H, 7] float32
    world_idx: np.ndarray         # [B] int32
    cuboids: np.ndarray           # [n_cuboids, 16] float32
    world_offsets: np.ndarray     # [n_worlds + 1] int32
    robot: dict
    params: dict = field(default_factory=lambda: dict(DEFAULT_PARAMS))
    envs: tuple = ()              # environment of each world
    formats: tuple = FP32
    goals: np.ndarray = None      # [n_worlds, 12] float32 (R row-major, p): IKO pose goals (N2)

    @property
    def B(self):
        return self.q.shape[0]

    @property
    def H(self):
        return self.q.shape[1]

    @property
    def poses(self):
        return self.q.shape[0] * self.q.shape[1]


def make_workload(name, envs_per_problem, problem_ids, seeds, H,
                  formats=FP32, params=None, cuboids=None, offsets=None,
                  salt=0):
    """Generic builder: problem i uses environment envs_per_problem[i], world
    key (salt, problem_ids[i]) and `seeds` trajectories keyed the same way."""
    robot = panda_robot()
    keys = [(salt, int(p)) for p in problem_ids]
    if cuboids is None:
        cuboids, offsets = make_worlds(envs_per_problem, keys)
    qs = [make_trajectories(k, seeds, H, robot["q_lo"], robot["q_hi"])
          for k in keys]
    q = np.concatenate(qs, 0) if qs else np.zeros((0, H, 7), np.float32)
    world_idx = np.repeat(np.arange(len(keys), dtype=np.int32), seeds)
    p = dict(DEFAULT_PARAMS)
    if params:
        p.update(params)
    return Workload(name, q, world_idx, cuboids, offsets, robot, p,
                    tuple(envs_per_problem), tuple(formats))


def config1(reduced=True):
    """1 problem, 4 seeds x 32 steps, 1 cuboid, FP32 vs E4M3 out_spheres."""
    cub = np.zeros((1, 16), np.float32)
    cub[0, 0:9] = np.eye(3).reshape(-1)
    cub[0, 9:12] = (0.45, 0.0, 0.30)
    cub[0, 12:15] = (0.15, 0.30, 0.02)
    off = np.array([0, 1], np.int32)
    fm = FORMAT_SETS["config1_e4m3"] if reduced else FP32
    return make_workload("config1", ["single_cuboid"], [0], 4, 32, fm,
                         cuboids=cub, offsets=off, salt=1)


def config2():
    """table_under_pick, 12 seeds x 32 steps, the 43-bit Table II set."""
    return make_workload("config2", ["table_under_pick"], [0], 12, 32,
                         FORMAT_SETS["43bit"], salt=2)


def config4(problems_per_env=100, seeds=100, H=32, formats="43bit",
            problem_offset=0, n_problems=None, problem_ids=None):
    """800 problems (100 per environment) x 100 TO seeds x 32 steps.

    Problem p (global id) uses environment ENVIRONMENTS[p % 8] so that any
    contiguous or strided shard keeps the environment mix.  `problem_offset`
    / `n_problems` select a contiguous shard of the global problem ids,
    `problem_ids` any list of them (the strong-scaling round-robin shard)."""
    total = problems_per_env * len(ENVIRONMENTS)
    if n_problems is None:
        n_problems = total
    ids = (list(problem_ids) if problem_ids is not None
           else list(range(problem_offset, problem_offset + n_problems)))
    envs = [ENVIRONMENTS[p % len(ENVIRONMENTS)] for p in ids]
    fm = FORMAT_SETS[formats] if isinstance(formats, str) else formats
    return make_workload("config4", envs, ids, seeds, H, fm, salt=4)


def config3(n_problems=400, seeds=80, H=32, formats=FP32):
    """BASELINE config 3's cost path: the three bookshelf
    environments, 400 problems x 80 TO seeds (top of the paper's TO sweep,
    P:191) x 32 steps = 1.024M poses; problem p uses bookshelf_{small, tall,
    thin}[p % 3]."""
    shelves = ("bookshelf_small", "bookshelf_tall", "bookshelf_thin")
    ids = list(range(n_problems))
    envs = [shelves[p % 3] for p in ids]
    fm = FORMAT_SETS[formats] if isinstance(formats, str) else formats
    return make_workload("config3", envs, ids, seeds, H, fm, salt=3)


def config5(problems_per_env=10, seeds=20, H=32):
    """NSGA-II proxy batch: 8 envs x 10 problems x 20 seeds x 32 steps."""
    ids = list(range(problems_per_env * len(ENVIRONMENTS)))
    envs = [ENVIRONMENTS[p % len(ENVIRONMENTS)] for p in ids]
    return make_workload("config5", envs, ids, seeds, H, FP32, salt=5)


def make_goals(keys):
    """One end-effector goal pose per problem (N2, reading c37): position
    uniform in a box in front of the robot, orientation a uniform random
    rotation (unit quaternion from 4 normals).  Pure sampling -- no robot
    arithmetic (reachability is not required of a cost-function workload)."""
    out = np.zeros((len(keys), 12), np.float32)
    for i, k in enumerate(keys):
        rng = np.random.Generator(np.random.Philox(key=_key(k, 0x60A1)))
        w, x, y, z = rng.normal(size=4)
        n = np.sqrt(w * w + x * x + y * y + z * z)
        w, x, y, z = w / n, x / n, y / n, z / n
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                      [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                      [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        out[i, :9] = R.reshape(-1)
        out[i, 9:] = rng.uniform([0.3, -0.4, 0.2], [0.7, 0.4, 0.7])
    return out


IKO_PARAMS = dict(swept=0, sweep_steps=0, w_pose_pos=1.0, w_pose_rot=0.5, w_bound=1.0)


def config_iko(problems_per_env=10, seeds=400, formats="43bit", problem_offset=0,
               n_problems=None, problem_ids=None):
    """N2 IKO workload: H = 1, `seeds` random joint configurations per problem
    (100-2000 IKO seeds), discrete world collision (closest_pt,
    slot 3), self collision, pose cost to the problem's goal and joint-bound
    cost (PAPER.md:162 step (3)); problems cycle through the 8 environments."""
    total = problems_per_env * len(ENVIRONMENTS)
    if n_problems is None:
        n_problems = total
    ids = (list(problem_ids) if problem_ids is not None
           else list(range(problem_offset, problem_offset + n_problems)))
    envs = [ENVIRONMENTS[p % len(ENVIRONMENTS)] for p in ids]
    fm = FORMAT_SETS[formats] if isinstance(formats, str) else formats
    wl = make_workload("iko", envs, ids, seeds, 1, fm, params=IKO_PARAMS, salt=7)
    wl.goals = make_goals([(7, int(p)) for p in ids])
    return wl


def codec_sweep_inputs(n, kind, key=0):
    """Codec inputs with the value distributions of the real tensors
    (SURVEY.md §8(d) config 3): 'position' ~ U(-1, 1.2) m; 'gradient' 98 %
    zeros, the rest log-uniform in [1e-4, 1e2] with random sign; 'bits' =
    uniformly random FP32 bit patterns (every class: subnormal, inf, NaN)."""
    rng = np.random.Generator(np.random.Philox(key=_key((key, n), 0xC0DE)))
    if kind == "position":
        return rng.uniform(-1.0, 1.2, n).astype(np.float32)
    if kind == "gradient":
        x = np.zeros(n, np.float64)
        nz = rng.random(n) >= 0.98
        k = int(nz.sum())
        mag = 10.0 ** rng.uniform(-4.0, 2.0, k)
        sgn = np.where(rng.random(k) < 0.5, -1.0, 1.0)
        x[nz] = sgn * mag
        return x.astype(np.float32)
    if kind == "bits":
        return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    raise ValueError(kind)


def edge_values():
    """Generic FP32 edge cases (format independent): signed zeros, FP32
    subnormals, normals at binade edges, max, inf, NaN."""
    bits = [0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x007FFFFF,
            0x807FFFFF, 0x00400000, 0x00800000, 0x80800000, 0x3F800000,
            0xBF800000, 0x7F7FFFFF, 0xFF7FFFFF, 0x7F800000, 0xFF800000,
            0x7FC00000, 0xFFC00000, 0x7F800001, 0xFFFFFFFF]
    return np.asarray(bits, np.uint32).view(np.float32)
