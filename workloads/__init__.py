"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This package holds *data and random numbers only* -- none of the method's
arithmetic (no kinematics, no SDF, no codec).  Both `oracle/` and the CUDA
path (through `paper_2310_07854_b200`) read the arrays produced here; neither
imports the other.  Every generator is keyed by an explicit integer seed tuple
and uses numpy's counter-based Philox bit generator, so the same (config,
problem, seed) key yields the same numbers on any machine and under any
sharding of the problems across ranks ("Synthetic inputs").
"""
from .robot import panda_robot, READY_POSE, ROBOT_FRAMES
from .scenes import ENVIRONMENTS, make_world, make_worlds
from .trajectories import make_trajectories
from .configs import (FORMAT_SETS, Workload, config1, config2, config3, config4,
                      config5, config_iko, make_workload, make_goals,
                      codec_sweep_inputs, edge_values)

__all__ = ["panda_robot", "READY_POSE", "ROBOT_FRAMES", "ENVIRONMENTS",
           "make_world", "make_worlds", "make_trajectories", "FORMAT_SETS",
           "Workload", "config1", "config2", "config3", "config4", "config5",
           "config_iko", "make_workload", "make_goals", "codec_sweep_inputs",
           "edge_values"]
