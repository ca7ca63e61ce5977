"""vapr_cost_grad inside a CUDA graph (SURVEY.md §8(d) timing protocol): a
replay gives bit-identical cost / grad_q to the eager call, also after the
trajectories are updated in place, in dense and sparse storage."""
import numpy as np
import pytest
import torch

from workloads import config2, config4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


@pytest.mark.parametrize("sparse", [False, True])
@pytest.mark.parametrize("which", ["config2", "config4_small"])
def test_graph_replay_bit_identical(vb, sparse, which):
    from paper_2310_07854_b200.rollout import Rollout
    wl = config2() if which == "config2" else config4(problems_per_env=1, seeds=6, H=32)
    eager = Rollout(wl, sparse=sparse)
    r = Rollout(wl, sparse=sparse)
    g = r.capture_graph()
    rng = np.random.default_rng(1)
    for it in range(3):
        q = (wl.q + (rng.normal(0, 0.05, wl.q.shape) if it else 0)).astype(np.float32)
        eager.q.copy_(torch.from_numpy(q))
        r.q.copy_(torch.from_numpy(q))
        eager.run()
        g.replay()
        a, b = eager.results(), r.results()
        for k in ("cost_pose", "cost_traj", "grad_q"):
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), (it, k)
