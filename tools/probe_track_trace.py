import os, sys, json, collections, time
sys.path[:0] = ['.', 'gen', 'oracle']
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import pmxgen
from paper_2412_12392_b200 import Context, MatchSet, Pointmap, abi, sim3
H, W = 384, 512
dev = torch.device('cuda')
c = pmxgen.config1(seed=1)
pa = np.arange(H * W, dtype=np.int32)
pa, v = pmxgen.inject_outliers(pa, c['valid_k'].copy(), 0.1, 1, H * W)
q = np.sqrt(c['C_f'][np.clip(pa, 0, None)].astype(np.float64) * c['C_k'].astype(np.float64)).astype(np.float32)
Tt = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
ctx = Context(0)
p = abi.default_solve_pose_params(); p.max_iterations = 10; p.weights.distance_weight = 0.1
args = (Pointmap(Tt(c['canonical']), Tt(c['canonical_valid']), H, W), Pointmap(Tt(c['X_f_f']), Tt(c['valid_f']), H, W), MatchSet(Tt(pa), Tt(q), Tt(v)), sim3())
for _ in range(3): ctx.track_given_matches(*args, params=p)
torch.cuda.synchronize()
ts=[]
for _ in range(5):
    t0=time.perf_counter(); r=ctx.track_given_matches(*args, params=p); ts.append((time.perf_counter()-t0)*1e3)
print("host-timed ms", min(ts), "iterations", r.iterations)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ctx.track_given_matches(*args, params=p); torch.cuda.synchronize()
prof.export_chrome_trace('gpurun_out/tt.json')
ev = sorted([e for e in json.load(open('gpurun_out/tt.json'))['traceEvents'] if e.get('cat') in ('kernel','gpu_memcpy','gpu_memset')], key=lambda e: e['ts'])
for e in ev: print(f"{e['name'][:50]:52s} {e['dur']:8.1f} us  at {e['ts']-ev[0]['ts']:8.1f}")
