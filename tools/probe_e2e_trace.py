"""Timeline of one e2e match_batch call with pinned host buffers (dev tool)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc, poses, edges, mk = pmxgen.config2(seed=2)


def pin(a):
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).pin_memory()
    return t.numpy().view(a.dtype)


hb = []
for e in range(n):
    p = mk(e)
    hb.append((Pointmap(pin(p["X_a"]), pin(p["valid_a"]), H, W), Pointmap(pin(p["X_b"]), pin(p["valid_b"]), H, W),
               FeatureMap(pin(p["D_a"]), pin(p["Q_a"]), H, W), FeatureMap(pin(p["D_b"]), pin(p["Q_b"]), H, W)))
outs = [MatchSet(torch.empty(H * W, dtype=torch.int32).pin_memory().numpy(),
                 torch.empty(H * W, dtype=torch.float32).pin_memory().numpy(),
                 torch.empty(H * W, dtype=torch.uint8).pin_memory().numpy()) for _ in range(n)]
ctx = Context(0)
mp = abi.default_match_params()
mp.projection.lambda_init = 1e-8
mp.projection.angle_tol = 1e-6
rp = abi.refine_params([(1, 3), (1, 3)])
for _ in range(2):
    ctx.match_batch(hb, params=mp, refine=rp, outs=outs)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.match_batch(hb, params=mp, refine=rp, outs=outs)
    ts.append((time.perf_counter() - t0) * 1e3)
print("e2e ms", [round(t, 2) for t in ts])
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ctx.match_batch(hb, params=mp, refine=rp, outs=outs)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "e2e_trace.json")
prof.export_chrome_trace(path)
ev = sorted([e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
            key=lambda e: e["ts"])
t0 = ev[0]["ts"]
h2d = [e for e in ev if "HtoD" in e["name"]]
print("device span ms", (ev[-1]["ts"] + ev[-1]["dur"] - t0) / 1e3, "H2D busy ms", sum(e["dur"] for e in h2d) / 1e3,
      "H2D count", len(h2d), "first H2D at", (h2d[0]["ts"] - t0) / 1e3, "last H2D end", (h2d[-1]["ts"] + h2d[-1]["dur"] - t0) / 1e3)
big = sorted(h2d, key=lambda e: -e["dur"])[:3]
for e in big:
    print("H2D", e["dur"], "us", e.get("args", {}).get("bytes"))
gaps = [(b["ts"] - (a["ts"] + a["dur"]), a["name"][:30]) for a, b in zip(h2d, h2d[1:])]
print("sum of gaps between H2D copies ms", sum(g for g, _ in gaps if g > 0) / 1e3, "max gap us", max(g for g, _ in gaps))
k = [e for e in ev if e.get("cat") == "kernel"]
print("kernels", len(k), "first kernel at ms", (k[0]["ts"] - t0) / 1e3, "last kernel end", (k[-1]["ts"] + k[-1]["dur"] - t0) / 1e3)
