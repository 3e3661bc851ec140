#!/usr/bin/env python
"""Benchmark of the B200 hot paths against BASELINE.json's metric.

Headline (BASELINE.json metric, config 2): batched iterative projective
matching + descriptor refinement over 64 directed edges of 512x384
pointmaps -> matched pixels/s, whole job over N GPUs (the fixed 64-edge
batch sharded by edge, no collective: scaling "strong").  One "step" = one pass of the
hot path over the rank's edges.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pmx|reference]

N > 1 runs one process per GPU: under torchrun as launched by the driver,
or, when WORLD_SIZE is unset, bench.py re-executes itself under
``torch.distributed.run --nproc-per-node N`` (and fails loudly when fewer
than N GPUs are visible).  NCCL carries only the barrier / max-over-ranks
timing for matching, and the reduce + broadcast of the edge-sharded
backend line (config 4), which runs by default at N > 1.  ``--impl reference`` times the reference
algorithm on the host cores (the FP64 C++ oracle restatement of
src/camera.cpp, all threads, bounded sample) on the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

METRIC = "matched pixels/s (batched edges)"
UNIT = "px/s"
H, W = 384, 512
N_EDGES = 64
ALG_BYTES_PER_PX = 133  # X_b 12 + X_a 12 + Q_a 4 + Q_b 4 + D_a 48 + D_b 48 + idx 4 + valid 1
# Algorithmic bytes per b-pixel of each matching kernel:
#  k_select 3 radix-select rounds over the 4-B norm keys                  = 12
#  k_prep   X_a 12 + valid_a 1 + D_a 48 (rays, int8 image, norm keys)   = 61
#  k_match_refine  X_b 12 + valid_b 1 + X_a (one ray per pixel) 12 + D_b 48 + Q_a 4 + Q_b 4
#                  + pa/valid/q out 9                                  = 90
KERNEL_BYTES_PER_PX = {"k_select": 12, "k_prep": 61, "k_match_refine": 90}
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r01_dram_traffic.json")


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "20", "-i", str(gpu)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.skip = 0

    def _rows(self):
        self.f.flush()
        with open(self.f.name) as g:
            return [r for r in g.read().splitlines() if r.strip()]

    def arm(self, timeout=5.0):
        """Wait until nvidia-smi is producing samples; rows before this point
        (process start-up, warm-up) are excluded from the statistics."""
        t0 = time.time()
        while self.p is not None and time.time() - t0 < timeout and not self._rows():
            time.sleep(0.01)
        self.skip = len(self._rows()) if self.p is not None else 0

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.strip().split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        rows = rows[self.skip:] or rows[-1:]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def edge_shard(rank, world):
    per = (N_EDGES + world - 1) // world
    return list(range(rank * per, min(N_EDGES, (rank + 1) * per)))


def match_params():
    from paper_2412_12392_b200 import abi
    p = abi.default_match_params()
    p.projection.lambda_init = 1e-8   # BASELINE config 0 schedule
    p.projection.angle_tol = 1e-6
    p.projection.max_iterations = 10
    return p, abi.refine_params([(1, 3), (1, 3)])


def cpu_sample(pairs, threads):
    """Oracle (FP64 C++ restatement of src/camera.cpp) match+refine of `pairs`."""
    import pyoracle
    mp, rp = match_params()
    t = time.perf_counter()
    pyoracle.match_batch(pairs, mp, rp, threads=threads)
    return time.perf_counter() - t


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    import pmxgen
    threads = os.cpu_count() or 1
    sample_edges = max(1, min(N_EDGES, threads))
    sc, poses, edges, make_pair = pmxgen.config2(seed=2)
    pairs = [make_pair(e) for e in range(sample_edges)]
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(pairs[:1], 1)
    times = [cpu_sample(pairs, threads) for _ in range(args.steps)]
    px = sample_edges * H * W
    value = px / statistics.mean(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen/pmx_gen.cpp, seed 2)",
            "config": {"workload": "config2: batched match+refine, 64 directed edges, 512x384, 24-d fp16",
                       "sample": f"{sample_edges} of 64 edges per step"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample_edges} edges x {H}x{W} px per step, {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_backend(ctx, dev, cpu: bool, n_kf=100, reach=4, loops=1, iters=10, config="config3"):
    """BASELINE configs 3 / 4: global Gauss-Newton on a loop trajectory, ray
    mode, lambda_d 0.1 -> ms per GN iteration (lower is better), split into
    accumulation (K7) / communication (none on 1 GPU) / solve (K9) / rest.

    value: device time of the GN loop (events around the enqueued loop) per
    iteration; the whole global_optimize call (staging, match compaction,
    solver planning: once per call) is reported beside it."""
    import torch
    import pmxgen
    from paper_2412_12392_b200 import Graph, MatchSet, Pointmap, abi
    g = pmxgen.backend_graph(n_kf, reach, 3, loops=loops)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
    ms = [MatchSet(T(m["pixel_a"]), T(m["confidence"]), T(m["valid"])) for m in g["matches"]]
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = iters
    init = [P.to_struct(abi.pmx_sim3) for P in g["init"]]
    nmatch = sum(int(np.count_nonzero(m["valid"])) for m in g["matches"])  # valid matches (what a pass reads)
    ctx.global_optimize(Graph(cans, list(init), g["edges"], ms), p)  # warm-up
    runs = []
    for _ in range(3):
        G = Graph(cans, list(init), g["edges"], ms)
        ctx.profile_enable(True)
        ctx.profile_reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.global_optimize(G, p)
        torch.cuda.synchronize()
        call_ms = (time.perf_counter() - t0) * 1e3
        loop_ms, _ = ctx.profile_get("gn_loop")
        et, _ = ctx.profile_get("k_edge_terms")
        lt, _ = ctx.profile_get("k_ldlt")
        ctx.profile_enable(False)
        runs.append((loop_ms / max(1, r.iterations), call_ms, loop_ms, et, lt, r, G))
    ms_it, call_ms, loop_ms, et, lt, r, G = min(runs, key=lambda x: x[0])
    # per-kernel breakdown: the same call enqueued kernel by kernel (the graph's
    # nodes carry no event brackets); the headline stays the graph run's loop
    ctx.set_device_graphs(False)
    ctx.profile_enable(True)
    ctx.profile_reset()
    r_e = ctx.global_optimize(Graph(cans, list(init), g["edges"], ms), p)
    eager_loop_ms, _ = ctx.profile_get("gn_loop")
    et, _ = ctx.profile_get("k_edge_terms")
    lt, _ = ctx.profile_get("k_ldlt")
    ctx.profile_enable(False)
    ctx.set_device_graphs(True)
    del cans, ms
    err0 = max(float(np.abs(P.t - Q.t).max()) for P, Q in zip(g["init"], g["gt"]))
    err = max(float(np.abs(np.array(P.t[:]) - Q.t).max()) for P, Q in zip(G.poses, g["gt"]))
    peaks, peak_kind = _peaks()
    passes = r.iterations + 1  # one residual pass per iteration + the initial one
    acc_ms = et / passes
    solve_ms = lt / max(1, r.iterations)
    achieved = 32.0 * nmatch / (acc_ms * 1e-3) / 1e9
    E = len(g["edges"])
    out = {"metric": f"global GN iteration ms at N={n_kf}", "value": ms_it, "unit": "ms", "higher_is_better": False,
           "config": {"workload": f"{config}: {n_kf} keyframes, radius-5 m loop x{loops}, {E} bidirectional edges "
                                  f"(k<->k+1..k+{reach}), 512x384, {iters} GN iterations, ray mode, lambda_d 0.1",
                      "iterations_run": r.iterations, "converged": r.converged,
                      "max_translation_error_m": {"init": err0, "final": err}},
           "breakdown_ms_per_iteration": {"accumulate_k_edge_terms": acc_ms, "communication": 0.0,
                                          "solve_k_ldlt": solve_ms,
                                          # assembly, retract, accept + the initial residual pass amortised
                                          "other": ms_it - acc_ms - solve_ms},
           "whole_call_ms": call_ms, "gn_loop_ms": loop_ms,
           "loop": "one CUDA graph per call: conditional WHILE node, body = one GN iteration "
                   "(breakdown from the same call enqueued kernel by kernel: "
                   f"{eager_loop_ms / max(1, r_e.iterations):.3f} ms per iteration)",
           "roofline": {"bound": "hbm", "kernel": "k_edge_terms", "achieved": achieved, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                        "alg_bytes_per_match": 32, "matches_per_launch": nmatch, "peak_kind": peak_kind}}
    if cpu:
        import pyoracle
        k = 2
        sub = g["matches"][:k]
        O = pyoracle.Graph(g["canonicals"], init, g["edges"][:k],
                           [pyoracle.MatchSet(m["pixel_a"], np.arange(H * W), m["confidence"].astype(np.float64),
                                              m["valid"]) for m in sub], H, W)
        t0 = time.perf_counter()
        pyoracle.backend_edge_terms(O, p, 0, k, threads=1)
        per_edge = (time.perf_counter() - t0) / k
        # the reference evaluates every edge twice per iteration (assemble_system + backend_cost)
        out["cpu_baseline"] = {"value": 2 * per_edge * E * 1e3, "unit": "ms", "cores": 1, "kind": "port",
                               "sample": f"{k} of {E} edges timed (FP64 oracle, 1 thread), extrapolated x{E} edges "
                                         "x2 residual passes per iteration (solve excluded)"}
    return out


def bench_backend_sharded(ctx, dev, rank, world, iters=5):
    """BASELINE config 4 sharded across the job's GPUs (--backend-sharded):
    each rank generates and stages only its edges' matches (prepared graph),
    every GN iteration is edge terms -> one NCCL reduce of the E x 72 terms
    -> rank 0 solve -> broadcast.  Per-iteration time split into
    accumulation / communication / solve, max over ranks."""
    import torch
    import torch.distributed as tdist
    import pmxgen
    from paper_2412_12392_b200 import Graph, MatchSet, Pointmap, abi, distributed
    n_kf, reach, loops = 1000, 5, 3
    E = len(pmxgen.loop_edges(n_kf, reach))
    e0, e1 = distributed.shard_range(E, rank, world)
    g = pmxgen.backend_graph(n_kf, reach, 3, loops=loops, edge_range=(e0, e1))
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
    ms = [MatchSet(T(m["pixel_a"]), T(m["confidence"]), T(m["valid"])) for m in g["matches"]]
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = iters
    init = [P.to_struct(abi.pmx_sim3) for P in g["init"]]
    G = Graph(cans, list(init), g["edges"], ms)
    terms_fn, solve_fn, cost_fn, pg = distributed.gpu_prepared_callbacks(ctx, G, p, e0, e1)
    distributed.global_optimize_sharded(init, E, 0, p, terms_fn, solve_fn, cost_fn, torch_device=dev)  # warm-up
    tdist.barrier()
    timers = {}
    t0 = time.perf_counter()
    res = distributed.global_optimize_sharded(init, E, 0, p, terms_fn, solve_fn, cost_fn, torch_device=dev,
                                              timers=timers)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    pg.release()
    vals = torch.tensor([total, timers.get("accumulate", 0.0), timers.get("communication", 0.0),
                         timers.get("solve", 0.0)], dtype=torch.float64, device=dev)
    tdist.all_reduce(vals, op=tdist.ReduceOp.MAX)
    total, acc, comm, solve = (float(v) for v in vals.cpu())
    it = max(1, res.iterations)
    err = max(float(np.abs(np.array(P.t[:]) - Q.t).max()) for P, Q in zip(res.poses, g["gt"]))
    return {"metric": f"global GN iteration ms at N={n_kf} (edge-sharded)", "value": 1e3 * total / it, "unit": "ms",
            "higher_is_better": False, "n_gpus": world, "scaling": "strong",
            "config": {"workload": f"config4: {n_kf} keyframes, loop x{loops}, {E} edges, {iters} GN iterations, "
                                   f"edges sharded {e1 - e0} per rank, NCCL reduce + broadcast per iteration",
                       "iterations_run": res.iterations, "converged": res.converged, "max_translation_error_m": err},
            "breakdown_ms_per_iteration": {"accumulate": 1e3 * acc / (it + 1), "communication": 1e3 * comm / it,
                                           "solve_rank0": 1e3 * solve / it}}


def bench_tracking(ctx, dev):
    """BASELINE config 1: 10 GN iterations on one Sim(3) over 196,608 matches
    (10% outliers) + confidence-weighted fusion."""
    import torch
    import pmxgen
    import pyoracle  # matching for the setup only (not timed)
    from paper_2412_12392_b200 import MatchSet, Pointmap, abi, sim3
    c = pmxgen.config1(seed=1)
    pair = {"X_a": c["X_f_f"], "valid_a": c["valid_f"], "Q_a": c["C_f"], "D_a": c["D_f"],
            "X_b": c["X_k_f"], "valid_b": c["valid_k"], "Q_b": c["C_k"], "D_b": c["D_k"], "height": H, "width": W}
    mp, rp = match_params()
    from paper_2412_12392_b200 import FeatureMap
    Tt = lambda x: torch.from_numpy(np.ascontiguousarray(x.view(np.int16) if x.dtype == np.uint16 else x)).to(dev)
    m = ctx.match_batch([(Pointmap(Tt(pair["X_a"]), Tt(pair["valid_a"]), H, W),
                          Pointmap(Tt(pair["X_b"]), Tt(pair["valid_b"]), H, W),
                          FeatureMap(Tt(pair["D_a"]), Tt(pair["Q_a"]), H, W),
                          FeatureMap(Tt(pair["D_b"]), Tt(pair["Q_b"]), H, W))], params=mp, refine=rp)[0]
    pa, v = pmxgen.inject_outliers(m.pixel_a.cpu().numpy(), m.valid.cpu().numpy(), 0.1, 1, H * W)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
    M = MatchSet(Tt(pa), Tt(q), Tt(v))
    can = Pointmap(Tt(c["canonical"]), Tt(c["canonical_valid"]), H, W)
    src = Pointmap(Tt(c["X_f_f"]), Tt(c["valid_f"]), H, W)
    p = abi.default_solve_pose_params()
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    for _ in range(3):
        r = ctx.track_given_matches(can, src, M, sim3(), params=p)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.track_given_matches(can, src, M, sim3(), params=p)
        ts.append((time.perf_counter() - t0) * 1e3)
    cx, cv, cc = Tt(c["canonical"]).clone(), Tt(c["canonical_valid"]).clone(), Tt(c["canonical_conf"]).clone()
    kf = Pointmap(Tt(c["X_k_f"]), Tt(c["valid_k"]), H, W)
    conf = Tt(c["C_k"])
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ctx.fuse_canonical(cx, cv, cc, kf, conf, r.T_kf, H, W)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        ctx.fuse_canonical(cx, cv, cc, kf, conf, r.T_kf, H, W)
    ev[1].record()
    torch.cuda.synchronize()
    fuse_ms = ev[0].elapsed_time(ev[1]) / 10
    Ttrue = c["T_kf"]
    return {"metric": "tracking GN (10 it) + fusion ms per frame", "value": min(ts) + fuse_ms, "unit": "ms",
            "higher_is_better": False,
            "config": {"workload": "config1: 512x384 frame vs keyframe, 10% outlier matches, 10 GN iterations, "
                                   "lambda_d 0.1, then fusion", "iterations_run": r.iterations, "lost": r.lost,
                       "translation_error_m": float(np.abs(np.array(r.T_kf.t[:]) - Ttrue.t).max())},
            "breakdown_ms": {"track_gn_k_track_gn_call": min(ts), "fusion_k_fuse": fuse_ms},
            "fusion_roofline": {"bound": "hbm", "achieved": 48.0 * H * W / (fuse_ms * 1e-3) / 1e9, "unit": "GB/s",
                                "alg_bytes_per_px": 48}}


def run_pmx(args):
    import torch
    import pmxgen
    from paper_2412_12392_b200 import Context, FeatureMap, MatchSet, Pointmap

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.backend_sharded:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    mine = edge_shard(rank, world)
    sc, poses, edges, make_pair = pmxgen.config2(seed=2)
    host_pairs = [make_pair(e) for e in mine]
    dev = torch.device("cuda", local)

    def to_dev(a, pinned=False):
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16) if a.dtype == np.uint16 else
                             np.ascontiguousarray(a))
        return t.pin_memory() if pinned else t.to(dev)

    def structs(p, place):
        t = {k: place(p[k]) for k in ("X_a", "X_b", "Q_a", "Q_b", "D_a", "D_b", "valid_a", "valid_b")}
        return (t, (Pointmap(t["X_a"], t["valid_a"], H, W), Pointmap(t["X_b"], t["valid_b"], H, W),
                    FeatureMap(t["D_a"], t["Q_a"], H, W), FeatureMap(t["D_b"], t["Q_b"], H, W)))

    dev_pairs = [structs(p, to_dev) for p in host_pairs]
    ctx = Context(local)
    # a real (non-default) stream shared by torch's events and the library
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream)
    mp, rp = match_params()
    outs = [MatchSet.empty(H * W, dev) for _ in mine]
    # resident buffers: the C-ABI argument arrays are built once (no per-step host work)
    batch = ctx.prepare_match_batch([p[1] for p in dev_pairs], outs)
    # warm-up
    for _ in range(args.warmup):
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.arm()
    launches0 = ctx.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for s in range(args.steps):
        ev[s][0].record(stream)
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    gpu_launches = ctx.kernel_launches - launches0
    # per-kernel breakdown from a separate, identical pass with the library's
    # CUDA-event scopes on (kept out of the timed region above)
    ctx.profile_enable(True)
    ctx.profile_reset()
    pe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    pe[0].record(stream)
    for s in range(args.steps):
        ctx.match_batch(batch, params=mp, refine=rp, outs=outs)
    pe[1].record(stream)
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof_ms = pe[0].elapsed_time(pe[1])
    kern = {k: ctx.profile_get(k) for k in KERNEL_BYTES_PER_PX}
    _, exact_px = ctx.profile_get("refine_exact_px")
    ms_local = float(sum(step_ms))
    if dist:
        t = torch.tensor([ms_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    else:
        ms_max = ms_local
    px_total = N_EDGES * H * W  # all ranks
    value = px_total * args.steps / (ms_max / 1e3)

    sharded = None
    if (args.backend_sharded or world > 1) and dist:  # every rank takes part (collectives)
        del dev_pairs, batch
        torch.cuda.empty_cache()
        sharded = bench_backend_sharded(ctx, dev, rank, world)

    # e2e through the public API with host (pinned) buffers: H2D inputs, D2H results
    host_structs = [structs(p, lambda a: to_dev(a, pinned=True)) for p in host_pairs]
    h2d = sum(sum(int(v.numel() * v.element_size()) for v in t.values()) for t, _ in host_structs)
    houts = [MatchSet(torch.empty(H * W, dtype=torch.int32).pin_memory().numpy(),
                      torch.empty(H * W, dtype=torch.float32).pin_memory().numpy(),
                      torch.empty(H * W, dtype=torch.uint8).pin_memory().numpy()) for _ in mine]
    d2h = sum(int(o.pixel_a.nbytes + o.confidence.nbytes + o.valid.nbytes) for o in houts)
    hbatch = [(Pointmap(t["X_a"].numpy(), t["valid_a"].numpy(), H, W), Pointmap(t["X_b"].numpy(), t["valid_b"].numpy(), H, W),
               FeatureMap(t["D_a"].numpy().view(np.uint16), t["Q_a"].numpy(), H, W),
               FeatureMap(t["D_b"].numpy().view(np.uint16), t["Q_b"].numpy(), H, W)) for t, _ in host_structs]
    ctx.match_batch(hbatch, params=mp, refine=rp, outs=houts)  # warm
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.match_batch(hbatch, params=mp, refine=rp, outs=houts)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_local = statistics.mean(e2e_ms)
    if dist:
        t = torch.tensor([e2e_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_local = float(t.item())
    e2e_value = px_total / (e2e_local / 1e3)
    # the host link itself: one pinned 512 MiB host -> device copy (what e2e is bounded by)
    pcie_gbs = None
    try:
        hb = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
        db = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        db.copy_(hb, non_blocking=True)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(3):
            db.copy_(hb, non_blocking=True)
        c1.record(stream)
        torch.cuda.synchronize()
        pcie_gbs = 3 * (512 << 20) / (c0.elapsed_time(c1) / 1e3) / 1e9
        del hb, db
    except Exception:
        pass

    # parity spot-check of the benchmarked outputs vs the host path (same kernels)
    ok = all(np.array_equal(outs[i].pixel_a.cpu().numpy(), houts[i].pixel_a) for i in range(len(mine)))
    valid_frac = float(np.mean([o.valid.float().mean().item() for o in outs]))

    peaks, peak_kind = _peaks()
    if rank == 0:
        px_steps = H * W * len(mine) * args.steps
        breakdown = {}
        for k, (kms, kn) in kern.items():
            nbytes = KERNEL_BYTES_PER_PX.get(k, 117) * px_steps
            breakdown[k] = {"ms_per_step": kms / args.steps, "launches_per_step": kn / args.steps,
                            "share_of_step": kms / prof_ms if prof_ms > 0 else None,
                            "alg_bytes_per_px": KERNEL_BYTES_PER_PX.get(k, 117),
                            "achieved_gbs": nbytes / (kms / 1e3) / 1e9 if kms > 0 else None}
        breakdown["k_match_refine"]["exact_path_px_per_step"] = exact_px / args.steps
        dom = max(breakdown, key=lambda k: breakdown[k]["ms_per_step"])
        achieved = breakdown[dom]["achieved_gbs"]
        traffic = None
        try:
            with open(TRAFFIC_FILE) as f:
                tr = json.load(f)
            # ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch, per b-pixel,
            # scaled to this run's average launch
            traffic = tr[dom]["dram_bytes_per_px"] * px_steps / max(1, kern[dom][1])
        except Exception:
            pass
        cpu = None
        if world == 1 and not args.no_cpu:
            nedge = 6
            secs = cpu_sample(host_pairs[:nedge], 1)
            cpu = {"value": nedge * H * W / secs, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"{nedge} of the 64 config-2 edges, match+refine, FP64 oracle, 1 thread ({secs:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32",
            "data": "synthetic (gen/pmx_gen.cpp, seed 2; radial point noise sigma=0.005)",
            "config": {"workload": "config2: batched match+refine, 64 directed edges, 512x384, 24-d fp16, "
                                   "LM 10 it lambda 1e-8 tol 1e-6 rad, refine {(1,3),(1,3)}",
                       "edges_per_rank": len(mine), "l2": "inputs larger than L2 (1.6 GB per step)",
                       "valid_fraction": valid_frac, "outputs_match_host_path": ok},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": (achieved / peaks["hbm_gbs"]) if achieved else None, "traffic": traffic,
                         "kernel": dom, "alg_bytes_per_launch": breakdown[dom]["alg_bytes_per_px"] * px_steps
                         / max(1, kern[dom][1]), "peak_kind": peak_kind,
                         "path": {"alg_bytes_per_px": ALG_BYTES_PER_PX,
                                  "achieved_gbs": ALG_BYTES_PER_PX * px_steps / (ms_local / 1e3) / 1e9},
                         "note": "issue-bound (FP64 LM + int8 DP4A window search), not HBM-bound: see DESIGN.md"},
            "kernels": breakdown,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_local, "h2d_gbs": h2d / (e2e_local / 1e3) / 1e9,
                    "pinned_copy_gbs": pcie_gbs,
                    "note": "bounded by the host link: the step's inputs cross PCIe once, kernels overlap the copies"},
            "gpu_launches": gpu_launches,
            "clocks": clocks,
        }
        if sharded is not None:
            line["secondary"] = [sharded]
        if world == 1 and not args.no_secondary:
            line["secondary"] = ([sharded] if sharded is not None else []) + \
                [bench_backend(ctx, dev, cpu=not args.no_cpu), bench_tracking(ctx, dev)]
            torch.cuda.empty_cache()
            line["secondary"].append(bench_backend(ctx, dev, cpu=not args.no_cpu, n_kf=1000, reach=5, loops=3,
                                                   iters=5, config="config4"))
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _spawn(args) -> int:
    """--gpus N without torchrun: one process per GPU via torch.distributed.run
    (the driver's own launch line), after checking N devices exist."""
    if args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) visible"}),
                  flush=True)
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {have} visible", file=sys.stderr)
            return 2
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["pmx", "reference"], default="pmx")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-3 / config-1 secondary lines")
    ap.add_argument("--backend-sharded", action="store_true",
                    help="also run config 4 edge-sharded over the job's GPUs (NCCL reduce + broadcast)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_pmx(args)


if __name__ == "__main__":
    main()
