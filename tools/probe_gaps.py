"""Timeline of one config-2 match_batch step (torch.profiler/CUPTI): kernel
busy time vs step wall time, largest idle gaps, host time per call."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import torch
import pmxgen
import bench
from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap

H, W = 384, 512
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc, poses, edges, make_pair = pmxgen.config2(seed=2)
dev = torch.device("cuda", 0)
def T(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)
pairs = []
for e in range(n):
    p = make_pair(e)
    pairs.append((Pointmap(T(p["X_a"]), T(p["valid_a"]), H, W), Pointmap(T(p["X_b"]), T(p["valid_b"]), H, W),
                  FeatureMap(T(p["D_a"]), T(p["Q_a"]), H, W), FeatureMap(T(p["D_b"]), T(p["Q_b"]), H, W)))
ctx = Context(0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx.set_stream(stream)
mp, rp = bench.match_params()
outs = [MatchSet.empty(H * W, dev) for _ in range(n)]
batch = ctx.prepare_match_batch(pairs, outs)
for _ in range(3):
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
torch.cuda.synchronize()
hs = []
for _ in range(5):
    t0 = time.perf_counter()
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    hs.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("host ms per match_batch call (no sync):", [round(1e3 * x, 3) for x in hs])
ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev[0].record(stream)
for _ in range(5):
    ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
ev[1].record(stream)
torch.cuda.synchronize()
print("device ms per step:", ev[0].elapsed_time(ev[1]) / 5)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    torch.cuda.synchronize()
prof.export_chrome_trace(os.path.join(ROOT, "gpurun_out", "gaps_trace.json"))
import json
tr = json.load(open(os.path.join(ROOT, "gpurun_out", "gaps_trace.json")))
ks = sorted([e for e in tr["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
busy = sum(e["dur"] for e in ks)
span = ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]
print(f"2 steps: {len(ks)} device ops, busy {busy/1e3:.3f} ms, span {span/1e3:.3f} ms")
gaps = []
for a, b in zip(ks, ks[1:]):
    gaps.append((b["ts"] - (a["ts"] + a["dur"]), a["name"][:40], b["name"][:40]))
gaps.sort(reverse=True)
for g in gaps[:15]:
    print(f"gap {g[0]:9.1f} us after {g[1]} before {g[2]}")
rt = sorted([e for e in tr["traceEvents"] if e.get("cat") == "cuda_runtime"], key=lambda e: -e["dur"])
for e in rt[:10]:
    print(f"runtime {e['name']} {e['dur']:.1f} us")
