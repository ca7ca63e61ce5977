"""Collision tiling is invisible in the results: the poses per
warp tile (VAPR_TILE_POSES; the launcher picks fewer than 15 for small
batches, and one-pose tiles spread the broadphase over the warp) change
nothing -- cost, grad_q and every stored tensor are bit-identical for 1, 2,
7, 15 and 16 poses per tile (16: the passes without a halo pose -- self, and
discrete world), dense, sparse and fused, swept and discrete."""
import dataclasses
import os

import numpy as np
import pytest
import torch

from workloads import config1, config4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def _run(wl, tp, sparse, fused=False):
    from paper_2310_07854_b200.rollout import Rollout
    os.environ["VAPR_TILE_POSES"] = str(tp)
    try:
        r = Rollout(wl, sparse=sparse, fused=fused)
        r.run()
        out = r.results()
        if not sparse and not fused:
            slot = 4 if wl.params["swept"] else 3
            out["cp"] = r.packed(slot)
            out["ov"] = r.packed(2)
            out["gos"] = r.packed(1)
        return out
    finally:
        del os.environ["VAPR_TILE_POSES"]


def _discrete(wl):
    p = dict(wl.params)
    p["swept"] = 0
    return dataclasses.replace(wl, params=p)


@pytest.mark.parametrize("mode", ["dense", "sparse", "fused"])
@pytest.mark.parametrize("name", ["mixed", "discrete", "config1"])
def test_tile_poses_invisible(vb, name, mode):
    wl = {"mixed": lambda: config4(problems_per_env=1, seeds=3, H=32),
          "discrete": lambda: _discrete(config4(problems_per_env=1, seeds=2, H=16)),
          "config1": config1}[name]()
    ref = _run(wl, 15, mode == "sparse", mode == "fused")
    for tp in (1, 2, 7, 16):
        got = _run(wl, tp, mode == "sparse", mode == "fused")
        for k, v in ref.items():
            a, b = np.asarray(v), np.asarray(got[k])
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (name, mode, tp, k)
