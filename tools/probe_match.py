"""Timing probe of the matching kernels on config-2 edges (dev tool).

python tools/probe_match.py [--edges 8] [--reps 5]
Prints the k_match time per edge with and without refinement.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap, abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--edges", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--modes", default="lm,refine")
a = ap.parse_args()
H, W = 384, 512
sc, poses, edges, mk = pmxgen.config2(seed=2)
dev = torch.device("cuda")


def t(x):
    x = np.ascontiguousarray(x)
    return torch.from_numpy(x.view(np.int16) if x.dtype == np.uint16 else x).to(dev)


pairs = []
for e in range(a.edges):
    p = mk(e)
    pairs.append((Pointmap(t(p["X_a"]), t(p["valid_a"]), H, W), Pointmap(t(p["X_b"]), t(p["valid_b"]), H, W),
                  FeatureMap(t(p["D_a"]), t(p["Q_a"]), H, W), FeatureMap(t(p["D_b"]), t(p["Q_b"]), H, W)))
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s)
mp = abi.default_match_params()
mp.projection.lambda_init = 1e-8
mp.projection.angle_tol = 1e-6
rp = abi.refine_params([(1, 3), (1, 3)])
outs = [MatchSet.empty(H * W, dev) for _ in pairs]
variants = {"refine": rp, "r0": abi.refine_params([(1, 0)]), "r1": abi.refine_params([(1, 1)]),
            "r3x1": abi.refine_params([(1, 3)]), "lm": None}
for mode in a.modes.split(","):
    ref = variants[mode]
    ctx.match_batch(pairs, params=mp, refine=ref, outs=outs)
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile_reset()
    for _ in range(a.reps):
        ctx.match_batch(pairs, params=mp, refine=ref, outs=outs)
    torch.cuda.synchronize()
    ms, n = ctx.profile_get("k_match")
    rms, rn = ctx.profile_get("k_refine")
    hms, hn = ctx.profile_get("k_refine_hard")
    _, hard_px = ctx.profile_get("refine_hard_px")
    ctx.profile_enable(False)
    print(f"{mode}: k_match {ms / a.reps / a.edges * 1e3:.1f} us/edge ({n} launches), k_refine "
          f"{rms / a.reps / a.edges * 1e3:.1f} us/edge ({rn}), hard {hms / a.reps / a.edges * 1e3:.1f} us/edge "
          f"({hard_px / a.reps / a.edges:.0f} px/edge)  "
          f"valid {np.mean([o.valid.float().mean().item() for o in outs]):.4f}")
