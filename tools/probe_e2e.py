"""Where the config-2 e2e step's time goes (dev tool): pinned H2D of the
step's bytes as one copy, as the per-array copies the host path issues, and
the e2e call itself, all timed on the device."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
n = 64
sc, poses, edges, mk = pmxgen.config2(seed=2)
host = []
for e in range(n):
    p = mk(e)
    t = {}
    for k in ("X_a", "valid_a", "X_b", "valid_b", "D_a", "Q_a", "D_b", "Q_b"):
        a = np.ascontiguousarray(p[k])
        a = a.view(np.int16) if a.dtype == np.uint16 else a
        t[k] = torch.from_numpy(a).pin_memory()
    host.append(t)
arrays = [v for t in host for v in t.values()]
total = sum(v.numel() * v.element_size() for v in arrays)
dev = [torch.empty_like(v, device="cuda") for v in arrays]
big_h = torch.empty(total, dtype=torch.uint8).pin_memory()
big_d = torch.empty(total, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
out = {"bytes": total}
for name, fn in (("one_copy", lambda: big_d.copy_(big_h, non_blocking=True)),
                 ("per_array", lambda: [d.copy_(h, non_blocking=True) for d, h in zip(dev, arrays)])):
    with torch.cuda.stream(s):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out[name] = {"ms": round(ms, 3), "gbs": round(total / ms / 1e6, 2)}
ctx = Context(0)
mp = abi.default_match_params()
mp.projection.lambda_init = 1e-8
mp.projection.angle_tol = 1e-6
rp = abi.refine_params([(1, 3), (1, 3)])
houts = [MatchSet(torch.empty(H * W, dtype=torch.int32).pin_memory().numpy(),
                  torch.empty(H * W, dtype=torch.float32).pin_memory().numpy(),
                  torch.empty(H * W, dtype=torch.uint8).pin_memory().numpy()) for _ in range(n)]
hb = [(Pointmap(t["X_a"].numpy(), t["valid_a"].numpy(), H, W), Pointmap(t["X_b"].numpy(), t["valid_b"].numpy(), H, W),
       FeatureMap(t["D_a"].numpy().view(np.uint16), t["Q_a"].numpy(), H, W),
       FeatureMap(t["D_b"].numpy().view(np.uint16), t["Q_b"].numpy(), H, W)) for t in host]
ctx.match_batch(hb, params=mp, refine=rp, outs=houts)
wall = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.match_batch(hb, params=mp, refine=rp, outs=houts)
    wall.append(1e3 * (time.perf_counter() - t0))
out["e2e_ms"] = [round(x, 3) for x in wall]
print(json.dumps(out), flush=True)
