"""GPU parity of frontend tracking (reference src/tracking.cpp:46-247)
against the FP64 oracle through the C ABI.

Bar (BASELINE north_star): Hessians / gradients within 1e-4 relative,
final poses within 1e-5 (translation) and 1e-5 rad (rotation).
"""
import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import BASELINE_REFINE, baseline_match_params, pmx_pair
from paper_2412_12392_b200 import MatchSet, PmxInvalidArgument, Pointmap, abi, sim3

pytestmark = pytest.mark.gpu

H_, W_ = 96, 128


def _frame(seed=1, h=H_, w=W_, outliers=0.1):
    c = pmxgen.config1(seed=seed, height=h, width=w)
    pair = {"X_a": c["X_f_f"], "valid_a": c["valid_f"], "Q_a": c["C_f"], "D_a": c["D_f"],
            "X_b": c["X_k_f"], "valid_b": c["valid_k"], "Q_b": c["C_k"], "D_b": c["D_k"], "height": h, "width": w}
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, baseline_match_params()), pair,
                                abi.refine_params(BASELINE_REFINE))
    pa, v = pmxgen.inject_outliers(m.pixel_a, m.valid, outliers, seed, h * w)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
    return c, pa, v, q


def _pose_err(a, b):
    Ra, Rb = np.array(a.R[:]).reshape(3, 3), np.array(b.R[:]).reshape(3, 3)
    dR = Ra.T @ Rb
    ang = np.arccos(np.clip((np.trace(dR) - 1) / 2, -1, 1))
    return float(np.abs(np.array(a.t[:]) - np.array(b.t[:])).max()), float(ang), abs(a.s - b.s)


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT])
def test_normal_equations_parity(ctx, mode):
    c, pa, v, q = _frame()
    n = H_ * W_
    T = pmxgen.Pose(pmxgen.rodrigues([0.01, -0.02, 0.015]), [0.02, -0.01, 0.03], 1.02).to_struct(abi.pmx_sim3)
    w = abi.default_robust_weight_params()
    w.distance_weight = 0.1
    w.q_min = 0.5
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], H_, W_)
    src = Pointmap(c["X_f_f"], c["valid_f"], H_, W_)
    Hg, gg, cg, ug = ctx.normal_equations(T, m, can, src, mode, w)
    om = pyoracle.MatchSet(pa, np.arange(n), q.astype(np.float64), v)
    Ho, go, co, uo = pyoracle.normal_equations(T, om, c["canonical"], c["canonical_valid"], c["X_f_f"],
                                               c["valid_f"], H_, W_, mode, w)
    assert ug == uo
    assert _rel(Hg, Ho) < 1e-4
    assert _rel(gg, go) < 1e-4
    assert abs(cg - co) / co < 1e-5


def test_residual_blocks_parity(ctx):
    # materialised residual_blocks (tracking.cpp:46-132), FP64 on the device
    c, pa, v, q = _frame()
    n = H_ * W_
    T = pmxgen.Pose(pmxgen.rodrigues([0.01, 0.0, -0.01]), [0.01, 0.02, 0.0], 0.97).to_struct(abi.pmx_sim3)
    K = abi.pmx_intrinsics(400.0 * W_ / 512, 400.0 * W_ / 512, 256.0 * W_ / 512, 192.0 * H_ / 384)
    m = MatchSet(pa, q, v)
    om = pyoracle.MatchSet(pa, np.arange(n), q.astype(np.float64), v)
    can = Pointmap(c["canonical"], c["canonical_valid"], H_, W_)
    src = Pointmap(c["X_f_f"], c["valid_f"], H_, W_)
    for mode in (abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL):
        rg = ctx.residual_blocks(T, m, can, src, mode, K=K)
        ro = pyoracle.residual_blocks(T, om, c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], H_,
                                      W_, mode, K=K)
        assert np.array_equal(rg[4], ro[4])
        for a, b in zip(rg[:4], ro[:4]):
            np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)


def test_pixel_mode_requires_intrinsics(ctx):
    c, pa, v, q = _frame()
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], H_, W_)
    with pytest.raises(PmxInvalidArgument):
        ctx.residual_blocks(sim3(), m, can, can, abi.PMX_TRACK_PIXEL)


def test_track_given_matches_parity(ctx):
    c, pa, v, q = _frame(seed=11, h=192, w=256)
    h, w = 192, 256
    p = abi.default_solve_pose_params()
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    m = MatchSet(pa, q, v)
    can = Pointmap(c["canonical"], c["canonical_valid"], h, w)
    src = Pointmap(c["X_f_f"], c["valid_f"], h, w)
    rg = ctx.track_given_matches(can, src, m, sim3(), params=p)
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    ro = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], h, w, om,
                                      sim3(), params=p)
    assert not rg.lost and not ro.lost
    et, er, es = _pose_err(rg.T_kf, ro.T_kf)
    assert et < 1e-5 and er < 1e-5 and es < 1e-5, (et, er, es)
    # recovers the true relative pose to the realistic two-view accuracy of
    # test_tracking.cpp:225-246 (half-pixel association bias, 10% outliers)
    Ttrue = c["T_kf"]
    assert np.abs(np.array(rg.T_kf.t[:]) - Ttrue.t).max() < 2e-2
    # cost traces agree while both are active
    k = min(len(rg.cost_trace), len(ro.cost_trace))
    np.testing.assert_allclose(rg.cost_trace[:k], ro.cost_trace[:k], rtol=1e-4)
    for a, b in zip(rg.cost_trace[1:], rg.cost_trace[:-1]):
        assert a <= b * (1 + 1e-12) + 1e-300


def test_lost_when_too_few_matches(ctx):
    c, pa, v, q = _frame()
    v2 = np.zeros_like(v)
    v2[:11] = 1
    p = abi.default_solve_pose_params()
    r = ctx.track_given_matches(Pointmap(c["canonical"], None, H_, W_), Pointmap(c["X_f_f"], None, H_, W_),
                                MatchSet(pa, q, v2), sim3(), params=p)
    assert r.lost and r.iterations == 0 and len(r.cost_trace) == 0


def test_exact_sim3_recovery(ctx):
    # test_tracking.cpp:200-223: aligned prediction through a known Sim(3) with scale
    c = pmxgen.config1(seed=4, height=H_, width=W_)
    n = H_ * W_
    T_true = pmxgen.Pose(pmxgen.rodrigues([0.1, -0.08, 0.12]), [0.08, -0.12, 0.05], 1.3)
    X_f = T_true.inverse().act(c["canonical"].astype(np.float64)).astype(np.float32)
    can = c["canonical"]
    # exact correspondences: identity matches, confidence 1
    m = MatchSet(np.arange(n, dtype=np.int32), np.ones(n, np.float32), np.ones(n, np.uint8))
    p = abi.default_solve_pose_params()
    r = ctx.track_given_matches(Pointmap(can, None, H_, W_), Pointmap(X_f, None, H_, W_), m, sim3(), params=p)
    assert not r.lost
    Rg = np.array(r.T_kf.R[:]).reshape(3, 3)
    ang = np.arccos(np.clip((np.trace(Rg.T @ T_true.R) - 1) / 2, -1, 1))
    assert ang < 1e-5 and np.abs(np.array(r.T_kf.t[:]) - T_true.t).max() < 1e-4
    assert abs(r.T_kf.s / T_true.s - 1) < 1e-5


def test_solve_pose_end_to_end_parity(ctx):
    c = pmxgen.config1(seed=2, height=H_, width=W_)
    p = abi.default_solve_pose_params()
    p.matching = baseline_match_params()
    p.refinement = abi.refine_params(BASELINE_REFINE)
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    from paper_2412_12392_b200 import FeatureMap
    args = (Pointmap(c["canonical"], c["canonical_valid"], H_, W_), Pointmap(c["X_f_f"], c["valid_f"], H_, W_),
            Pointmap(c["X_k_f"], c["valid_k"], H_, W_), FeatureMap(c["D_f"], c["C_f"], H_, W_),
            FeatureMap(c["D_k"], c["C_k"], H_, W_))
    rg = ctx.solve_pose(*args, sim3(), params=p)
    ro = abi.pmx_track_result()
    import ctypes as C
    keep = []
    ms = pyoracle.MatchSet.empty(H_ * W_)
    ost = ms.struct()
    pc = pyoracle._pm(c["canonical"], c["canonical_valid"], H_, W_)
    pf = pyoracle._pm(c["X_f_f"], c["valid_f"], H_, W_)
    pk = pyoracle._pm(c["X_k_f"], c["valid_k"], H_, W_)
    ff = pyoracle._fm(c["D_f"], c["C_f"], H_, W_)
    fk = pyoracle._fm(c["D_k"], c["C_k"], H_, W_)
    T0 = sim3()
    pyoracle._check(pyoracle.lib().orc_solve_pose(C.byref(pc), C.byref(pf), C.byref(pk), C.byref(ff), C.byref(fk),
                                                  C.byref(T0), C.c_int(0), C.byref(p), None, C.byref(ro),
                                                  C.byref(ost)))
    same = (np.asarray(rg.matches.pixel_a) == ms.pixel_a).mean()
    assert same > 0.999
    et, er, es = _pose_err(rg.T_kf, ro.T_kf)
    assert et < 1e-5 and er < 1e-5 and es < 1e-5


def test_fuse_canonical_parity(ctx):
    c = pmxgen.config1(seed=3, height=H_, width=W_)
    n = H_ * W_
    T = c["T_kf"].to_struct(abi.pmx_sim3)
    rng = np.random.default_rng(0)
    cv = (rng.random(n) > 0.1).astype(np.uint8)
    cc = c["canonical_conf"].copy()
    cc[::50] = 0.0
    vk = (rng.random(n) > 0.05).astype(np.uint8)
    conf = c["C_k"].copy()
    conf[::77] = -cc[::77]  # c_prev + c <= 0 -> skipped
    gx, gv, gc = c["canonical"].copy(), cv.copy(), cc.copy()
    ctx.fuse_canonical(gx, gv, gc, Pointmap(c["X_k_f"], vk, H_, W_), conf, T, H_, W_)
    ox, ov, oc = pyoracle.fuse_canonical(c["canonical"].astype(np.float64), cv, cc.astype(np.float64), c["X_k_f"],
                                         vk, conf, T, H_, W_)
    assert np.array_equal(gv, ov)
    np.testing.assert_allclose(gx, ox, rtol=2e-7, atol=1e-6)
    np.testing.assert_allclose(gc, oc, rtol=2e-7)


def test_fusion_is_idempotent_and_first_is_exact(ctx):
    # test_tracking.cpp:314-337
    c = pmxgen.config1(seed=5, height=H_, width=W_)
    n = H_ * W_
    X = c["canonical"]
    gx = np.zeros((n, 3), np.float32)
    gv = np.zeros(n, np.uint8)
    gc = np.zeros(n, np.float32)
    ctx.fuse_canonical(gx, gv, gc, Pointmap(X, None, H_, W_), c["canonical_conf"], sim3(), H_, W_)
    assert np.array_equal(gx, X) and gv.all()
    before = gx.copy()
    ctx.fuse_canonical(gx, gv, gc, Pointmap(X, None, H_, W_), c["canonical_conf"], sim3(), H_, W_)
    np.testing.assert_allclose(gx, before, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(gc, 2 * c["canonical_conf"], rtol=1e-6)


def test_track_decisions_match_oracle_at_full_size(ctx):
    """Config-1 size (384 x 512): the accept / stop decisions of the LM loop
    (tracking.cpp:206-223) compare costs a few 1e-12 apart near convergence;
    the loop's FP64 cost sum (ray_cost64) must reproduce the oracle's
    iteration count and cost trace, not just the final pose."""
    h, w = 384, 512
    c = pmxgen.config1(seed=1)
    pa = np.arange(h * w, dtype=np.int32)
    pa, v = pmxgen.inject_outliers(pa, c["valid_k"].copy(), 0.1, 1, h * w)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
    p = abi.default_solve_pose_params()
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    rg = ctx.track_given_matches(Pointmap(c["canonical"], c["canonical_valid"], h, w),
                                 Pointmap(c["X_f_f"], c["valid_f"], h, w), MatchSet(pa, q, v), sim3(), params=p)
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    ro = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], h, w, om,
                                      sim3(), params=p)
    assert rg.iterations == ro.iterations
    n = len(rg.cost_trace)
    assert n >= 3
    np.testing.assert_allclose(rg.cost_trace, np.asarray(ro.cost_trace)[:n], rtol=1e-9)
    et, er, es = _pose_err(rg.T_kf, ro.T_kf)
    assert et < 1e-6 and er < 1e-6 and es < 1e-6, (et, er, es)
