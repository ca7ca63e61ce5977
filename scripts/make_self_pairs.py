"""Write workloads/data/panda_self_pairs.json (reading c18 of DESIGN.md §3).

Self-collision pairs = all sphere pairs on links whose index differs by >= 2,
minus the pairs already active (phi = r_i + r_j + eta_self - d > 0) at the
Panda ready pose (0, -pi/4, 0, -3pi/4, 0, pi/2, pi/4).  Calls only oracle/
and workloads/ (a stored value is written by a committed script that calls only
the oracle).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from workloads.robot import panda_robot, candidate_pairs, READY_POSE  # noqa: E402
from oracle.kinematics import sphere_centers  # noqa: E402

ETA_SELF = 0.01


def main():
    robot = panda_robot(pairs=np.zeros((0, 2), np.uint16))
    cand = candidate_pairs(robot["sphere_link"])
    c = sphere_centers(np.array([READY_POSE]), robot)[0]
    r = robot["sphere_xyzr"][:, 3].astype(np.float64)
    keep = []
    for i, j in cand:
        d = np.linalg.norm(c[i] - c[j])
        if r[i] + r[j] + ETA_SELF - d <= 0.0:
            keep.append([int(i), int(j)])
    out = {"candidates": int(len(cand)), "eta_self": ETA_SELF,
           "ready_pose": list(READY_POSE), "n_pairs": len(keep), "pairs": keep}
    path = os.path.join(os.path.dirname(__file__), "..", "workloads", "data",
                        "panda_self_pairs.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"{len(cand)} candidates, {len(keep)} kept -> {path}")


if __name__ == "__main__":
    main()
