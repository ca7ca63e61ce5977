import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (exhaustive) test")


def golden(name):
    """Rows of a whitespace-separated fixture under tests/golden/."""
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def pytest_sessionfinish(session, exitstatus):
    """With VAPR_PARITY_REPORT=<path>: write the largest err / limit of every
    FP32 comparison and the largest code distance of every packed comparison
    (tests/parity_utils.py records them) -- how tight the tolerances are."""
    path = os.environ.get("VAPR_PARITY_REPORT")
    if not path:
        return
    import json
    import parity_utils
    with open(path, "w") as f:
        json.dump(parity_utils.REPORT, f, indent=1, sort_keys=True)
