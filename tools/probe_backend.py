"""Timing probe of the backend (config 3/4 shapes) and tracking (config 1).

python tools/probe_backend.py [--kf 100] [--reach 4] [--iters 10]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, Graph, MatchSet, Pointmap, abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kf", type=int, default=100)
ap.add_argument("--reach", type=int, default=4)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--loops", type=int, default=1)
ap.add_argument("--no-graphs", action="store_true")
a = ap.parse_args()
H, W = 384, 512
t0 = time.time()
g = pmxgen.backend_graph(a.kf, a.reach, 3, loops=a.loops)
print(f"gen {time.time() - t0:.1f}s: {len(g['edges'])} edges, overlap {np.mean([m['valid'].mean() for m in g['matches']]):.3f}")
dev = torch.device("cuda")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
ms = [MatchSet(T(m["pixel_a"]), T(m["confidence"]), T(m["valid"])) for m in g["matches"]]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s)
if a.no_graphs:
    ctx.set_device_graphs(False)
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
p.max_iterations = a.iters
init = [P.to_struct(abi.pmx_sim3) for P in g["init"]]
for rep in range(2):
    G = Graph(cans, list(init), g["edges"], ms)
    ctx.profile_enable(True)
    ctx.profile_reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.global_optimize(G, p)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    et, en = ctx.profile_get("k_edge_terms")
    lt, ln = ctx.profile_get("k_ldlt")
    gl, _ = ctx.profile_get("gn_loop")
    ctx.profile_enable(False)
    err0 = max(np.abs(P.t - Q.t).max() for P, Q in zip(g["init"], g["gt"]))
    err = max(np.abs(np.array(P.t[:]) - Q.t).max() for P, Q in zip(G.poses, g["gt"]))
    nm = sum(m["valid"].size for m in g["matches"])
    print(f"rep {rep}: {r.iterations} it, {dt * 1e3:.1f} ms total, {dt * 1e3 / max(1, r.iterations):.2f} ms/it; "
          f"k_edge_terms {et / max(1, en):.3f} ms x{en} ({32 * nm / (et / max(1, en) * 1e-3) / 1e9:.0f} GB/s alg), "
          f"k_ldlt {lt / max(1, r.iterations):.3f} ms/it; loop {gl:.2f} ms = {gl / max(1, r.iterations):.3f} ms/it; "
          f"|dt| {err0:.3f} -> {err:.4f}; converged {r.converged}")
