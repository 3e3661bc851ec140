"""Kernel timeline of one config-3 global_optimize call (torch.profiler /
CUPTI): per-kernel device time and the idle gaps of the device loop (dev tool)."""
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, Graph, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
kf = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reach = int(sys.argv[2]) if len(sys.argv) > 2 else 4
loops = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = pmxgen.backend_graph(kf, reach, 3, loops=loops)
dev = torch.device("cuda")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
ms = [MatchSet(T(m["pixel_a"]), T(m["confidence"]), T(m["valid"])) for m in g["matches"]]
ctx = Context(0)
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
p.max_iterations = int(sys.argv[4]) if len(sys.argv) > 4 else 10
init = [P.to_struct(abi.pmx_sim3) for P in g["init"]]
for _ in range(2):
    ctx.global_optimize(Graph(cans, list(init), g["edges"], ms), p)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = ctx.global_optimize(Graph(cans, list(init), g["edges"], ms), p)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "backend_trace.json")
prof.export_chrome_trace(path)
ev = sorted([e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
            key=lambda e: e["ts"])
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    a = agg[e["name"].split("(")[0][:40]]
    a[0] += 1
    a[1] += e["dur"]
print(f"iterations {r.iterations}; {len(ev)} device ops, busy {sum(e['dur'] for e in ev) / 1e3:.3f} ms, "
      f"span {(ev[-1]['ts'] + ev[-1]['dur'] - ev[0]['ts']) / 1e3:.3f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{k:42s} {n:5d} {t / 1e3:8.3f} ms")
gaps = sorted(((b["ts"] - a["ts"] - a["dur"], a["name"][:30], b["name"][:30]) for a, b in zip(ev, ev[1:])), reverse=True)
print("total gap ms", sum(x[0] for x in gaps) / 1e3)
for x in gaps[:8]:
    print(f"gap {x[0]:8.1f} us after {x[1]} before {x[2]}")
