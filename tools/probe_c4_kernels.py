"""Config-4 GN loop enqueued kernel by kernel (device graphs off), for an ncu
launch list of the backend kernels (dev tool):

ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:k_(edge|sky|ldlt|bcr|gn|cost64|rel64|terms|band|blocks|retract|check|accept|apply)' \
    --csv --log-file gpurun_out/c4_launches.csv python tools/probe_c4_kernels.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, Graph, Pointmap, abi  # noqa: E402

ctx = Context(0)
dev = torch.device("cuda")
g = pmxgen.backend_graph_matched(ctx, 1000, 5, 3, loops=3)
H, W = g["height"], g["width"]
cans = [Pointmap(torch.from_numpy(x).to(dev), torch.from_numpy(v).to(dev), H, W) for x, v in g["canonicals"]]
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
p.max_iterations = 5
init = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
ctx.set_device_graphs(False)
r = ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
torch.cuda.synchronize()
print("iterations", r.iterations, "converged", r.converged, flush=True)
ct = list(r.cost_trace)
print("cost trace", ct, flush=True)
print("relative changes", [(ct[i] - ct[i + 1]) / ct[i] for i in range(len(ct) - 1)], flush=True)
ctx.profile_enable(True)
ctx.profile_reset()
r = ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
print("fp64 decisions", ctx.profile_get("backend_fp64_decisions")[1], "k_cost64", ctx.profile_get("k_cost64"), flush=True)
