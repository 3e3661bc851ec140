"""Config-1 tracking: GPU vs oracle iteration count and cost trace (dev tool)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle")]

import torch  # noqa: E402

import pmxgen  # noqa: E402
import pyoracle  # noqa: E402
from paper_2412_12392_b200 import Context, MatchSet, Pointmap, abi, sim3  # noqa: E402

H, W = 384, 512
dev = torch.device("cuda")
c = pmxgen.config1(seed=1)
rng = np.random.default_rng(0)
pa = np.arange(H * W, dtype=np.int32)
v = c["valid_k"].copy()
pa, v = pmxgen.inject_outliers(pa, v, 0.1, 1, H * W)
q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
Tt = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
ctx = Context(0)
p = abi.default_solve_pose_params()
p.max_iterations = 10
p.weights.distance_weight = 0.1
r = ctx.track_given_matches(Pointmap(Tt(c["canonical"]), Tt(c["canonical_valid"]), H, W),
                            Pointmap(Tt(c["X_f_f"]), Tt(c["valid_f"]), H, W), MatchSet(Tt(pa), Tt(q), Tt(v)), sim3(),
                            params=p)
om = pyoracle.MatchSet(pa, np.arange(H * W), q.astype(np.float64), v)
ro = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], H, W, om, sim3(),
                                  params=p)
print("gpu iterations", r.iterations, "oracle", ro.iterations)
print("gpu trace", list(r.cost_trace))
print("orc trace", list(ro.cost_trace))
print("t gpu", list(r.T_kf.t[:]), "orc", list(ro.T_kf.t[:]))
