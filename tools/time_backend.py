"""Time the backend GN loop (config 3, or config 4 with 'c4') with the library
named by PMX_LIB: ms per iteration and the per-kernel split (dev tool)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, Graph, Pointmap, abi  # noqa: E402

c4 = len(sys.argv) > 1 and sys.argv[1] == "c4"
ctx = Context(0)
dev = torch.device("cuda")
g = pmxgen.backend_graph_matched(ctx, 1000 if c4 else 100, 5 if c4 else 4, 3, loops=3 if c4 else 1)
H, W = g["height"], g["width"]
cans = [Pointmap(torch.from_numpy(x).to(dev), torch.from_numpy(v).to(dev), H, W) for x, v in g["canonicals"]]
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
p.max_iterations = 5 if c4 else 10
init = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
best = None
for _ in range(3):
    ctx.profile_enable(True)
    ctx.profile_reset()
    r = ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
    loop_ms, _ = ctx.profile_get("gn_loop")
    ctx.profile_enable(False)
    best = min(best or 1e9, loop_ms / r.iterations)
ctx.set_device_graphs(False)
ctx.profile_enable(True)
ctx.profile_reset()
r = ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
split = {k: round(ctx.profile_get(k)[0], 3) for k in ("k_edge_terms", "k_ldlt", "k_cost64")}
print(json.dumps({"lib": os.environ.get("PMX_LIB", "default"), "config": "c4" if c4 else "c3",
                  "ms_per_iteration": round(best, 4), "iterations": r.iterations, "split_ms_total": split}))
