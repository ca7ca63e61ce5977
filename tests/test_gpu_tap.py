"""Parity contract (i) of SURVEY.md §8(c) through the test-only tap build:
tests/tap_check.py runs vapr_cost_grad from libvapr_tap.so (a subprocess, so
the release library of the other tests stays the one loaded here) and checks
oracle_codec(the kernels' FP32 pre-quantisation values) == packed words, bit
for bit, for every packed tensor and several format sets."""
import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_packed_words_equal_oracle_codec_of_tapped_values():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200.build import TAP_SO
    assert os.path.exists(TAP_SO), "libvapr_tap.so not built (python -m paper_2310_07854_b200.build)"
    env = dict(os.environ, VAPR_SO=TAP_SO)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "tap_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    assert len(lines) == 24
    assert all(l["bit_exact"] for l in lines)
    # every slot actually carried non-zero values somewhere
    for sl in (0, 1, 2):
        assert any(l["slot"] == sl and l["nonzero_values"] > 0 for l in lines), sl
