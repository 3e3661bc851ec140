"""GPU parity of the decision-critical semantics:

* the strict q > q_min exclusion of robust_weight (src/tracking.cpp:10-13,
  64-65; src/backend.cpp:62-63), exercised with confidences that fall below
  q_min (BASELINE's q >= 1 never triggers it);
* pixel (calibrated) mode normal equations, tracking GN and backend GN
  (src/tracking.cpp:98-113, src/backend.cpp:95-96, 112-113);
* the backend's accept / revert decisions in the end game, where successive
  costs differ by ~1e-12 relative (src/backend.cpp:241-246): decided on FP64
  costs when the fp32-accumulated ones cannot resolve them.
"""
import numpy as np
import pytest

import pmxgen
import pyoracle
from paper_2412_12392_b200 import Graph, MatchSet, Pointmap, abi, sim3

pytestmark = pytest.mark.gpu


def _pose_err(a, b):
    Ra, Rb = np.array(a.R[:]).reshape(3, 3), np.array(b.R[:]).reshape(3, 3)
    ang = np.arccos(np.clip((np.trace(Ra.T @ Rb) - 1) / 2, -1, 1))
    return float(np.abs(np.array(a.t[:]) - np.array(b.t[:])).max()), float(ang), abs(a.s - b.s)


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _K(h, w):
    return abi.pmx_intrinsics(400.0 * w / 512, 400.0 * w / 512, 256.0 * w / 512, 192.0 * h / 384)


def _low_q(q, valid, frac, seed):
    """frac of the valid matches get q in [0.02, 0.3]: below q_min = 0.1 x
    median (median of q in [1, 10] is ~5) -> excluded (robust_weight = inf)."""
    rng = np.random.default_rng(seed)
    q = q.astype(np.float32).copy()
    idx = np.nonzero(valid)[0]
    pick = rng.choice(idx, size=int(frac * idx.size), replace=False)
    q[pick] = rng.uniform(0.02, 0.3, pick.size).astype(np.float32)
    return q


def _frame(seed, h, w):
    c = pmxgen.config1(seed=seed, height=h, width=w)
    pair = {"X_a": c["X_f_f"], "valid_a": c["valid_f"], "Q_a": c["C_f"], "D_a": c["D_f"],
            "X_b": c["X_k_f"], "valid_b": c["valid_k"], "Q_b": c["C_k"], "D_b": c["D_k"], "height": h, "width": w}
    from helpers import BASELINE_REFINE, baseline_match_params
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, baseline_match_params()), pair,
                                abi.refine_params(BASELINE_REFINE))
    pa, v = pmxgen.inject_outliers(m.pixel_a, m.valid, 0.05, seed, h * w)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
    return c, pa, v, q


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_normal_equations_with_exclusions(ctx, mode):
    h, w = 96, 128
    c, pa, v, q = _frame(1, h, w)
    q = _low_q(q, v, 0.2, 1)
    T = pmxgen.Pose(pmxgen.rodrigues([0.01, -0.02, 0.015]), [0.02, -0.01, 0.03], 1.02).to_struct(abi.pmx_sim3)
    wp = abi.default_robust_weight_params()
    wp.distance_weight = 0.1
    wp.q_min = 0.35  # strict q > q_min: the low-q matches carry no information
    K = _K(h, w) if mode == abi.PMX_TRACK_PIXEL else None
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], h, w)
    src = Pointmap(c["X_f_f"], c["valid_f"], h, w)
    Hg, gg, cg, ug = ctx.normal_equations(T, m, can, src, mode, wp, K=K)
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    Ho, go, co, uo = pyoracle.normal_equations(T, om, c["canonical"], c["canonical_valid"], c["X_f_f"],
                                               c["valid_f"], h, w, mode, wp, K=K)
    assert ug == uo and ug < int(v.sum()) - 0.15 * int(v.sum())  # the exclusion branch is live
    assert _rel(Hg, Ho) < 1e-4 and _rel(gg, go) < 1e-4 and abs(cg - co) <= 1e-5 * abs(co)


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_track_given_matches_with_exclusions(ctx, mode):
    """q_min = 0.1 x median of the valid matches' q (tracking.cpp:170-171),
    with 15% of them below it."""
    h, w = 192, 256
    c, pa, v, q = _frame(11, h, w)
    q = _low_q(q, v, 0.15, 2)
    p = abi.default_solve_pose_params()
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(h, w)
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], h, w)
    src = Pointmap(c["X_f_f"], c["valid_f"], h, w)
    rg = ctx.track_given_matches(can, src, m, sim3(), mode=mode, params=p)
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    ro = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], h, w, om,
                                      sim3(), mode=mode, params=p)
    assert not rg.lost and not ro.lost
    assert rg.iterations == ro.iterations
    et, er, es = _pose_err(rg.T_kf, ro.T_kf)
    assert et < 1e-5 and er < 1e-5 and es < 1e-5, (et, er, es)
    np.testing.assert_allclose(list(rg.cost_trace), list(ro.cost_trace[:ro.cost_trace_len]), rtol=1e-6)


def _graph(n_kf=12, reach=3, h=48, w=64, seed=5, low_q=0.0):
    g = pmxgen.backend_graph(n_kf, reach, seed, height=h, width=w, radius=1.0)
    qs = [(_low_q(m["confidence"], m["valid"], low_q, 10 + e) if low_q else m["confidence"])
          for e, m in enumerate(g["matches"])]
    poses = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
    G = Graph([Pointmap(x, v, h, w) for x, v in g["canonicals"]], poses, g["edges"],
              [MatchSet(m["pixel_a"], q, m["valid"]) for m, q in zip(g["matches"], qs)], anchor=0)
    O = pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"],
                       [pyoracle.MatchSet(m["pixel_a"], np.arange(h * w), q.astype(np.float64), m["valid"])
                        for m, q in zip(g["matches"], qs)], h, w)
    return g, G, O


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_backend_with_exclusions(ctx, mode):
    """Per-edge q_min = 0.1 x median (backend.cpp:37-46, 62-63) with 15% of
    every edge's valid matches below it: edge terms and the GN loop."""
    h, w = 48, 64
    g, G, O = _graph(low_q=0.15, h=h, w=w)
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.mode = mode
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(h, w)
    tg = ctx.backend_edge_terms(G, p)
    to = pyoracle.backend_edge_terms(O, p)
    for e in range(len(g["edges"])):
        for d in (0, 36):
            assert _rel(tg[e, d:d + 35], to[e, d:d + 35]) < 1e-4
            assert abs(tg[e, d + 35] - to[e, d + 35]) <= 1e-5 * abs(to[e, d + 35])
    rg = ctx.global_optimize(G, p, trace=True)
    ro, tro = pyoracle.global_optimize(O, p)
    assert rg.iterations == ro.iterations and rg.converged == bool(ro.converged)
    for a, b in zip(G.poses, O.poses):
        et, er, es = _pose_err(a, b)
        assert et < 1e-5 and er < 1e-5 and es < 1e-5, (et, er, es)


def test_backend_end_game_decisions_exact(ctx):
    """update_tol = 0: the loop runs until the accept test reverts a step
    (backend.cpp:242-246) - costs a few 1e-12 apart.  Same iteration count,
    convergence flag, cost trace and final poses as the FP64 oracle, and the
    device loop took at least one decision on FP64 costs."""
    g, G, O = _graph(n_kf=10, reach=3)
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.update_tol = 0.0
    p.max_iterations = 40
    ctx.profile_enable(True)
    ctx.profile_reset()
    rg = ctx.global_optimize(G, p)
    _, fp64_decisions = ctx.profile_get("backend_fp64_decisions")
    ctx.profile_enable(False)
    ro, _ = pyoracle.global_optimize(O, p)
    assert fp64_decisions >= 1
    assert rg.iterations == ro.iterations, (rg.iterations, ro.iterations)
    assert rg.converged == bool(ro.converged)
    np.testing.assert_allclose(rg.cost_trace, list(ro.cost_trace[:ro.cost_trace_len]), rtol=1e-7)
    for a, b in zip(G.poses, O.poses):
        et, er, es = _pose_err(a, b)
        assert et < 1e-6 and er < 1e-6 and es < 1e-6, (et, er, es)


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_backend_end_game_decisions_exact_point_pixel(ctx, mode):
    """update_tol = 0 in point and pixel mode: the generic edge pass carries
    the FP64 cost (FP64-evaluated residuals, block_cost) in its cost slot, so
    the accept / revert end game (backend.cpp:241-246) follows the oracle's
    iterations and cost trace."""
    h, w = 48, 64
    g, G, O = _graph(n_kf=10, reach=3, h=h, w=w)
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.update_tol = 0.0
    p.max_iterations = 30
    p.mode = mode
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(h, w)
    rg = ctx.global_optimize(G, p)
    ro, _ = pyoracle.global_optimize(O, p)
    assert rg.iterations == ro.iterations, (rg.iterations, ro.iterations)
    assert rg.converged == bool(ro.converged)
    np.testing.assert_allclose(rg.cost_trace, list(ro.cost_trace[:ro.cost_trace_len]), rtol=1e-7)
    for a, b in zip(G.poses, O.poses):
        et, er, es = _pose_err(a, b)
        assert et < 1e-6 and er < 1e-6 and es < 1e-6, (et, er, es)


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_track_end_game_decisions_exact_point_pixel(ctx, mode):
    """Tracking's accept / stop decisions in point and pixel mode on FP64
    costs (update_tol = 0, 20 iterations): same iterations and cost trace as
    the oracle."""
    h, w = 96, 128
    c, pa, v, q = _frame(21, h, w)
    p = abi.default_solve_pose_params()
    p.max_iterations = 20
    p.update_tol = 0.0
    p.weights.distance_weight = 0.1
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(h, w)
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], h, w)
    src = Pointmap(c["X_f_f"], c["valid_f"], h, w)
    rg = ctx.track_given_matches(can, src, m, sim3(), mode=mode, params=p)
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    ro = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], h, w, om,
                                      sim3(), mode=mode, params=p)
    assert rg.iterations == ro.iterations, (rg.iterations, ro.iterations)
    np.testing.assert_allclose(list(rg.cost_trace), list(ro.cost_trace[:ro.cost_trace_len]), rtol=1e-9)
