"""GPU parity at the BASELINE configurations themselves (not scaled-down
cases), through the C ABI, against the reference build (oracle/_ref: the
genuine src/*.cpp) when it is present, else the FP64 restatement.

* config 2: the full 64-edge batch (28 consecutive pairs x 2 directions + 8
  long-range pairs, 512x384, 24-d fp16) -> every edge compared with the
  reference's match_pointmaps + feature_refine (src/camera.cpp:195-271);
  bars of BASELINE north_star: >= 99.9% of valid pixels index-equal, every
  mismatch <= 1 px, valid-mask mismatch <= 1e-3.
"""
import os

import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import BASELINE_REFINE, baseline_match_params, compare_matches, pmx_pair
from paper_2412_12392_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = max(1, os.cpu_count() or 1)


def _reference():
    return pyoracle.reference() if pyoracle.have_reference() else _Null()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.fixture(scope="module")
def config2():
    sc, poses, edges, make_pair = pmxgen.config2(seed=2)
    assert len(edges) == 64
    return [make_pair(e) for e in range(len(edges))]


def test_config2_full_batch_vs_reference(ctx, config2):
    mp, rp = baseline_match_params(), abi.refine_params(BASELINE_REFINE)
    gpu = ctx.match_batch([pmx_pair(p) for p in config2], params=mp, refine=rp)
    with _reference():
        ref = pyoracle.match_batch(config2, mp, rp, threads=THREADS)
    worst_eq, total_both, total_eq, total_vm = 1.0, 0, 0, 0
    for e, (g, r) in enumerate(zip(gpu, ref)):
        st = compare_matches(g, r, 512)
        assert st["worst_px"] <= 1, (e, st)
        assert st["valid_mismatch"] <= 1e-3 * st["n"], (e, st)
        worst_eq = min(worst_eq, st["index_equal_frac"])
        total_both += st["both"]
        total_eq += int(round(st["index_equal_frac"] * st["both"]))
        total_vm += st["valid_mismatch"]
        # q = sqrt(Q_a[pa] Q_b[n]) (camera.cpp:230, 269-270): fp32 rounding of the FP64 value
        same = np.asarray(g.pixel_a) == r.pixel_a
        np.testing.assert_allclose(np.asarray(g.confidence)[same], r.confidence[same], rtol=6e-8)
    assert worst_eq >= 0.999 and total_eq / total_both >= 0.999
    print(f"config2: {total_both} px valid in both, index-equal {total_eq / total_both:.7f}, "
          f"worst edge {worst_eq:.7f}, valid mismatches {total_vm}")


# ------------------------------------------------------------------ config 3
@pytest.fixture(scope="module")
def config3(ctx):
    """N = 100 keyframes, 400 edges, 512x384, matches built by the config-2
    matcher on device-generated pair predictions (BASELINE config 3)."""
    return pmxgen.backend_graph_matched(ctx, 100, 4, 3, keep_host=True)


def _pose_err(a, b):
    dt = float(np.abs(np.array(a.t[:]) - np.array(b.t[:])).max())
    Ra, Rb = np.array(a.R[:]).reshape(3, 3), np.array(b.R[:]).reshape(3, 3)
    c = np.clip((np.trace(Ra.T @ Rb) - 1.0) / 2.0, -1.0, 1.0)
    return dt, float(np.arccos(c)), abs(a.s - b.s)


def test_config3_global_optimize_vs_oracle(ctx, config3):
    """Per-iteration poses, iteration count and cost trace of the device GN
    loop (src/backend.cpp:192-256) at the BASELINE config-3 size, against the
    FP64 restatement (pinned to the reference build in test_ref_pins) driven
    through the same control flow: oracle per-edge terms on all host threads,
    numpy assembly + the oracle's LDL^T.  Bars: poses within 1e-5 m / 1e-5
    rad per iteration, same iteration count, costs within 1e-6 relative."""
    import torch
    from helpers import numpy_solve
    from paper_2412_12392_b200 import Graph, MatchSet, Pointmap
    from paper_2412_12392_b200.distributed import global_optimize_sharded
    g = config3
    H, W = g["height"], g["width"]
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = 10
    init = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
    dev = torch.device("cuda")
    cans = [Pointmap(torch.from_numpy(x).to(dev), torch.from_numpy(v).to(dev), H, W) for x, v in g["canonicals"]]
    G = Graph(cans, list(init), g["edges"], g["matches"])
    r = ctx.global_optimize(G, p, trace=True)
    valid = sum(int(m["valid"].sum()) for m in g["matches_host"])
    assert valid > 0.5 * len(g["edges"]) * H * W  # the matcher's valid fraction, not GT projections
    O = pyoracle.Graph(g["canonicals"], list(init), g["edges"],
                       [pyoracle.MatchSet(m["pixel_a"], np.arange(H * W), m["confidence"].astype(np.float64),
                                          m["valid"]) for m in g["matches_host"]], H, W)

    def terms_fn(e0, e1, P):
        O.poses = list(P)
        return pyoracle.backend_edge_terms(O, p, e0, e1, threads=THREADS)

    def cost_fn(terms):
        t = np.asarray(terms)
        return float(sum(t[e, 35] + t[e, 71] for e in range(t.shape[0])))

    ro = global_optimize_sharded(list(init), len(g["edges"]), 0, p, terms_fn, numpy_solve(O, p), cost_fn)
    assert r.iterations == ro.iterations and r.converged == ro.converged, (r.iterations, ro.iterations)
    np.testing.assert_allclose(r.cost_trace, ro.cost_trace, rtol=1e-6)
    assert len(r.pose_trace) == len(ro.pose_trace)
    worst = (0.0, 0.0, 0.0)
    for it, (pg, po) in enumerate(zip(r.pose_trace, ro.pose_trace)):
        for a, b in zip(pg, po):
            e = _pose_err(a, b)
            worst = tuple(max(x, y) for x, y in zip(worst, e))
    assert worst[0] <= 1e-5 and worst[1] <= 1e-5 and worst[2] <= 1e-5, worst
    print(f"config3: {r.iterations} iterations, {valid} valid matches, worst per-iteration pose error "
          f"{worst[0]:.2e} m / {worst[1]:.2e} rad / scale {worst[2]:.2e}")


# ------------------------------------------------------------------ config 4
def test_config4_sampled_edge_terms_vs_oracle(ctx):
    """BASELINE config 4 (N = 1000, 5000 edges, 3 loops): the per-edge
    relative-frame normal-equation terms {H1, g1, c1, H2, g2, c2} of a fixed
    50-edge sample (matches built by the matcher), at the perturbed initial
    poses, against the FP64 restatement (src/backend.cpp:101-142, 175-190).
    Bar: H, g within 1e-4 relative (north_star), costs within 1e-5."""
    import torch
    from paper_2412_12392_b200 import Graph, Pointmap
    e0, e1 = 2500, 2550
    g = pmxgen.backend_graph_matched(ctx, 1000, 5, 3, loops=3, edge_range=(e0, e1), keep_host=True)
    H, W = g["height"], g["width"]
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    init = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
    need = sorted({k for e in range(e0, e1) for k in g["edges"][e]})
    dev = torch.device("cuda")
    blank = np.zeros((H * W, 3), np.float32)
    cans = [(g["canonicals"][k] if k in need else (blank, np.zeros(H * W, np.uint8))) for k in range(len(init))]
    G = Graph([Pointmap(torch.from_numpy(x).to(dev), torch.from_numpy(v).to(dev), H, W) for x, v in cans],
              list(init), g["edges"], g["matches"])
    tg = ctx.backend_edge_terms(G, p, e0, e1).cpu().numpy()
    O = pyoracle.Graph(cans, list(init), g["edges"],
                       [pyoracle.MatchSet(m["pixel_a"], np.arange(len(m["pixel_a"])), m["confidence"].astype(np.float64),
                                          m["valid"]) for m in g["matches_host"]], H, W)
    to = pyoracle.backend_edge_terms(O, p, e0, e1, threads=THREADS)

    def rel(a, b):
        return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))

    worst = 0.0
    for e in range(e1 - e0):
        for d in (0, 36):
            worst = max(worst, rel(tg[e, d:d + 28], to[e, d:d + 28]), rel(tg[e, d + 28:d + 35], to[e, d + 28:d + 35]))
            assert abs(tg[e, d + 35] - to[e, d + 35]) <= 1e-5 * abs(to[e, d + 35])
    assert worst < 1e-4, worst
    print(f"config4 sample: 50 edges, worst relative H/g difference {worst:.2e}")
