"""Probe the SSCG_NCCL_SELF path step by step (debugging aid)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from gpu_cases import Problem  # noqa: E402

slabs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
graph = sys.argv[2] if len(sys.argv) > 2 else "1"
if graph == "0":
    os.environ["SSCG_NO_GRAPH"] = "1"
os.environ["SSCG_NCCL_SELF"] = "1"
P = Problem("7pt", 40, 36, 33, 10, 20)
t = time.time()
with P.gpu_solver(slabs=slabs) as S:
    print("setup", time.time() - t, flush=True)
    x = S.solve(P.b_gpu(), rtol=0.0, max_outer=0)
    print("solve0", time.time() - t, flush=True)
    x = S.solve(P.b_gpu(), rtol=0.0, max_outer=2).cpu().numpy()
    print("solve2", time.time() - t, S.stats().allreduces, flush=True)
