"""Time config-1 tracking (10 GN iterations over 196,608 matches) with the
library named by PMX_LIB: k_track_gn ms and the whole call (dev tool)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, MatchSet, Pointmap, abi, sim3  # noqa: E402

H, W = 384, 512
dev = torch.device("cuda")
ctx = Context(0)
c = pmxgen.config1(seed=1)
Tt = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
gt = c["gt_pixel_a"] if "gt_pixel_a" in c else None
pa = np.arange(H * W, dtype=np.int32)
v = c["valid_k"].astype(np.uint8)
pa, v = pmxgen.inject_outliers(pa, v, 0.1, 1, H * W)
q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
M = MatchSet(Tt(pa), Tt(q), Tt(v))
can = Pointmap(Tt(c["canonical"]), Tt(c["canonical_valid"]), H, W)
src = Pointmap(Tt(c["X_f_f"]), Tt(c["valid_f"]), H, W)
p = abi.default_solve_pose_params()
p.max_iterations = 10
p.weights.distance_weight = 0.1
for _ in range(3):
    r = ctx.track_given_matches(can, src, M, sim3(), params=p)
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.track_given_matches(can, src, M, sim3(), params=p)
    ts.append((time.perf_counter() - t0) * 1e3)
ctx.profile_enable(True)
ctx.profile_reset()
for _ in range(10):
    r = ctx.track_given_matches(can, src, M, sim3(), params=p)
k = ctx.profile_get("k_track_gn")
print(json.dumps({"lib": os.environ.get("PMX_LIB", "default"), "call_ms": round(min(ts), 4),
                  "k_track_gn_ms": round(k[0] / max(k[1], 1), 4), "iterations": r.iterations,
                  "cost_trace": list(r.cost_trace)[:3], "t": list(r.T_kf.t[:])}), flush=True)
