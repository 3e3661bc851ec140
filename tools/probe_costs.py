"""Cost traces of the device GN loop vs the FP64 oracle-driven loop at the
config-3 size (matcher-built matches): the fp32-accumulated cost's actual
relative error, which sizes kCostBand (dev tool)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
import pyoracle  # noqa: E402
from helpers import numpy_solve  # noqa: E402
from paper_2412_12392_b200 import Context, Graph, Pointmap, abi  # noqa: E402
from paper_2412_12392_b200.distributed import global_optimize_sharded  # noqa: E402

ctx = Context(0)
n_kf = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = pmxgen.backend_graph_matched(ctx, n_kf, 4, 3, keep_host=True)
H, W = g["height"], g["width"]
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
p.max_iterations = 10
p.update_tol = 0.0  # run the end game
init = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
dev = torch.device("cuda")
cans = [Pointmap(torch.from_numpy(x).to(dev), torch.from_numpy(v).to(dev), H, W) for x, v in g["canonicals"]]
ctx.profile_enable(True)
r = ctx.global_optimize(Graph(cans, list(init), g["edges"], g["matches"]), p)
print("gpu iterations", r.iterations, "fp64 decisions", ctx.profile_get("backend_fp64_decisions")[1])
O = pyoracle.Graph(g["canonicals"], list(init), g["edges"],
                   [pyoracle.MatchSet(m["pixel_a"], np.arange(H * W), m["confidence"].astype(np.float64), m["valid"])
                    for m in g["matches_host"]], H, W)
# oracle terms at the GPU's poses of each iteration would be exact; here: the oracle-driven loop
terms_fn = lambda e0, e1, P: (setattr(O, "poses", list(P)), pyoracle.backend_edge_terms(O, p, e0, e1, threads=os.cpu_count()))[1]  # noqa: E731
cost_fn = lambda t: float(np.sum(np.asarray(t)[:, 35]) + np.sum(np.asarray(t)[:, 71]))  # noqa: E731
ro = global_optimize_sharded(list(init), len(g["edges"]), 0, p, terms_fn, numpy_solve(O, p), cost_fn)
print("oracle iterations", ro.iterations)
for k, (a, b) in enumerate(zip(r.cost_trace, ro.cost_trace)):
    print(k, f"{a:.17g} {b:.17g} rel {abs(a - b) / b:.3e}", "step rel" if k == 0 else
          f"{(ro.cost_trace[k - 1] - b) / b:.3e}")
