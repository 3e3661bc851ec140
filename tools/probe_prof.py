import json, os, sys
sys.argv = [sys.argv[0], "64"]
ROOT = "/root/repo"
exec(open(os.path.join(ROOT, "tools/time_match.py")).read().split("ev0, ev1 =")[0])
def timed(k=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / k
def prof(k=10):
    ctx.profile_enable(True); ctx.profile_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    e1.record(); torch.cuda.synchronize(); ctx.profile_enable(False)
    return e0.elapsed_time(e1) / k, {n: round(ctx.profile_get(n)[0] / k, 4) for n in ("k_select", "k_prep", "k_match_refine")}
for r in range(3):
    print("timed", round(timed(), 4), "prof", prof(), "timed", round(timed(30), 4), flush=True)
