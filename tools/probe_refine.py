"""Whole-batch timing of config-2 matching with / without refinement (dev tool)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
dev = torch.device("cuda")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64


def T(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)


sc, poses, edges, mk = pmxgen.config2(seed=2)
pairs = []
for e in range(n):
    p = mk(e)
    pairs.append((Pointmap(T(p["X_a"]), T(p["valid_a"]), H, W), Pointmap(T(p["X_b"]), T(p["valid_b"]), H, W),
                  FeatureMap(T(p["D_a"]), T(p["Q_a"]), H, W), FeatureMap(T(p["D_b"]), T(p["Q_b"]), H, W)))
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s)
mp = abi.default_match_params()
mp.projection.lambda_init = 1e-8
mp.projection.angle_tol = 1e-6
outs = [MatchSet.empty(H * W, dev) for _ in range(n)]
batch = ctx.prepare_match_batch(pairs, outs)
for label, rp in (("lm only", None), ("lm+refine", abi.refine_params([(1, 3), (1, 3)])),
                  ("lm+refine 1 level", abi.refine_params([(1, 3)]))):
    for _ in range(3):
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{label:20s} {e0.elapsed_time(e1) / 10:.3f} ms per batch of {n}")
