"""Time the config-2 matcher (64 edges, device-resident) with the library
named by PMX_LIB (default build): per-kernel ms per step (dev tool)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]
import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda")


def T(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)


sc, poses, edges, mk = pmxgen.config2(seed=2)
pairs = []
for e in range(n):
    p = mk(e)
    pairs.append((Pointmap(T(p["X_a"]), T(p["valid_a"]), H, W), Pointmap(T(p["X_b"]), T(p["valid_b"]), H, W),
                  FeatureMap(T(p["D_a"]), T(p["Q_a"]), H, W), FeatureMap(T(p["D_b"]), T(p["Q_b"]), H, W)))
ctx = Context(0)
mp = abi.default_match_params()
mp.projection.lambda_init = 1e-8
mp.projection.angle_tol = 1e-6
rp = abi.refine_params([(1, 3), (1, 3)])
outs = [MatchSet.empty(H * W, dev) for _ in range(n)]
batch = ctx.prepare_match_batch(pairs, outs)
for _ in range(3):
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(10):
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
ev1.record()
torch.cuda.synchronize()
step = ev0.elapsed_time(ev1) / 10
ctx.profile_enable(True)
ctx.profile_reset()
for _ in range(10):
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
torch.cuda.synchronize()
k = {name: round(ctx.profile_get(name)[0] / 10, 4) for name in ("k_select", "k_prep", "k_match_refine")}
k["exact_path_px_per_step"] = ctx.profile_get("refine_exact_px")[1] / 10
pa = np.concatenate([o.pixel_a.cpu().numpy() for o in outs])
va = np.concatenate([o.valid.cpu().numpy() for o in outs])
qa = np.concatenate([o.confidence.cpu().numpy() for o in outs])
if os.environ.get("PMX_SAVE"):  # outputs for a variant-vs-default comparison
    np.savez(os.environ["PMX_SAVE"], pa=pa, valid=va, q=qa)
print(json.dumps({"lib": os.environ.get("PMX_LIB", "default"), "ms_per_step": round(step, 4),
                  "gpx_s": round(n * H * W / step / 1e6, 3), "kernels": k,
                  "checksum": int(pa.astype(np.int64).sum())}), flush=True)
