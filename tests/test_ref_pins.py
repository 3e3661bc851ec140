"""Pins the oracle restatement (oracle/liborc.so) to the reference itself:
oracle/_ref/libpmslam_ref.so is /root/reference/proj/src/{lie,camera,
tracking,backend}.cpp compiled UNMODIFIED against the Eigen-API shim
(oracle/eigen_shim, recipe oracle/Makefile target `ref`), behind the same
orc_* ABI.  Every case runs both builds on the same seeded inputs.

Bars: integer / index / validity outputs bit-identical; floating-point
outputs within 1e-12 relative (the shim evaluates Eigen expressions eagerly,
so sums may round differently from Eigen's own kernels at the ulp level), and
the committed golden fixtures are reproduced by the reference build.
"""
import os

import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import BASELINE_REFINE, baseline_match_params
from paper_2412_12392_b200 import abi

pytestmark = pytest.mark.skipif(not pyoracle.have_reference(),
                                reason="oracle/_ref not built (make -C oracle ref needs /root/reference)")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def both(fn, *a, **k):
    """(restatement result, reference result) of the same pyoracle call."""
    o = fn(*a, **k)
    with pyoracle.reference():
        r = fn(*a, **k)
    return o, r


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))), initial=0.0))


def test_reference_build_is_the_reference():
    with pyoracle.reference():
        assert pyoracle.lib().orc_is_reference() == 1
    assert not hasattr(pyoracle.lib(), "orc_is_reference") or pyoracle.lib().orc_is_reference() != 1


@pytest.fixture(scope="module")
def pair():
    return pmxgen.config0(seed=5, height=96, width=128)


@pytest.fixture(scope="module")
def pair_iso():
    return pmxgen.config0(seed=6, height=64, width=96, noise="isotropic")


def test_normalize_rays_bit_identical(pair):
    (ro, do, vo), (rr, dr, vr) = both(pyoracle.normalize_rays, pair["X_a"], pair["valid_a"], 96, 128)
    assert np.array_equal(vo, vr) and np.array_equal(ro, rr) and np.array_equal(do, dr)


def test_interpolate_ray(pair):
    rng = np.random.default_rng(0)
    p = np.c_[rng.uniform(-1, 128, 4000), rng.uniform(-1, 96, 4000)]
    p[:50] = np.floor(p[:50])  # integer pixels and the right / bottom edges
    p[50:60, 0] = 127.0
    p[60:70, 1] = 95.0
    (ro, Jo, oko), (rr, Jr, okr) = both(pyoracle.interpolate_ray, pair["X_a"], pair["valid_a"], 96, 128, p)
    assert np.array_equal(oko, okr) and oko.sum() > 3000
    assert rel(ro, rr) <= 1e-15 and rel(Jo, Jr) <= 1e-13


def test_iterative_project(pair):
    h, w = 96, 128
    x = pair["X_b"][::7]
    idx = np.arange(h * w)[::7]
    p0 = np.c_[idx % w, idx // w].astype(np.float64)
    pp = baseline_match_params().projection
    (po, co, io), (pr, cr, ir) = both(pyoracle.iterative_project, pair["X_a"], pair["valid_a"], h, w, x, p0, pp)
    assert np.array_equal(co, cr) and np.array_equal(io, ir)
    assert rel(po, pr) <= 1e-12


@pytest.mark.parametrize("which", ["radial", "isotropic"])
def test_match_and_refine_bit_identical(pair, pair_iso, which):
    p = pair if which == "radial" else pair_iso
    mp, rp = baseline_match_params(), abi.refine_params(BASELINE_REFINE)
    mo, mr = both(pyoracle.match_pointmaps, p, mp)
    assert np.array_equal(mo.valid, mr.valid) and np.array_equal(mo.pixel_a, mr.pixel_a)
    assert np.array_equal(mo.confidence, mr.confidence) and np.array_equal(mo.pixel_b, mr.pixel_b)
    assert mo.valid.sum() > 0.3 * len(mo)
    fo, fr = both(pyoracle.feature_refine, mo, p, rp)
    assert np.array_equal(fo.pixel_a, fr.pixel_a) and np.array_equal(fo.confidence, fr.confidence)
    assert np.array_equal(fo.valid, fr.valid)


def test_match_default_params_and_seed(pair):
    """The reference defaults (lambda 1e-4, tol 1e-5, levels {(2,2),(1,2)}) and a seeded init."""
    mo, mr = both(pyoracle.match_pointmaps, pair, abi.default_match_params())
    assert np.array_equal(mo.pixel_a, mr.pixel_a) and np.array_equal(mo.valid, mr.valid)
    fo, fr = both(pyoracle.feature_refine, mo, pair, abi.default_refine_params())
    assert np.array_equal(fo.pixel_a, fr.pixel_a)
    seed = pyoracle.MatchSet(np.roll(fo.pixel_a, 3), fo.pixel_b, fo.confidence, fo.valid)
    so, sr = both(pyoracle.match_pointmaps, pair, baseline_match_params(), seed)
    assert np.array_equal(so.pixel_a, sr.pixel_a) and np.array_equal(so.valid, sr.valid)


@pytest.mark.parametrize("name", ["match_radial_48x64.npz", "match_isotropic_48x64.npz"])
def test_reference_reproduces_match_fixture(name):
    z = dict(np.load(os.path.join(GOLD, name)))
    h, w = (int(x) for x in z["shape"])
    p = {"X_a": z["X_a"], "X_b": z["X_b"], "Q_a": z["Q_a"], "Q_b": z["Q_b"], "D_a": z["D_a"], "D_b": z["D_b"],
         "valid_a": z["valid_a"], "valid_b": z["valid_b"], "height": h, "width": w}
    with pyoracle.reference():
        m = pyoracle.match_pointmaps(p, baseline_match_params())
        r = pyoracle.feature_refine(m, p, abi.refine_params(BASELINE_REFINE))
    assert np.array_equal(m.pixel_a, z["lm_pixel_a"]) and np.array_equal(m.valid, z["lm_valid"])
    assert np.array_equal(r.pixel_a, z["pixel_a"]) and np.array_equal(r.confidence, z["confidence"])


def test_match_stats_and_keyframe_decision(pair):
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, baseline_match_params()), pair,
                                abi.refine_params(BASELINE_REFINE))
    so, sr = both(pyoracle.match_stats, m, 96 * 128)
    assert so == sr
    for omega in (0.1, so[1], so[1] + 1e-9, 0.9):
        ko, kr = both(pyoracle.keyframe_decision, m, 96, 128, omega)
        assert ko == kr


@pytest.fixture(scope="module")
def track_case():
    h, w = 64, 96
    c = pmxgen.config1(seed=7, height=h, width=w)
    pair = {"X_a": c["X_f_f"], "valid_a": c["valid_f"], "Q_a": c["C_f"], "D_a": c["D_f"],
            "X_b": c["X_k_f"], "valid_b": c["valid_k"], "Q_b": c["C_k"], "D_b": c["D_k"], "height": h, "width": w}
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, baseline_match_params()), pair,
                                abi.refine_params(BASELINE_REFINE))
    pa, v = pmxgen.inject_outliers(m.pixel_a, m.valid, 0.1, 7, h * w)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64))
    return c, pair, pyoracle.MatchSet(pa, np.arange(h * w), q, v), h, w


def _K(w, h):
    K = abi.pmx_intrinsics()
    K.fx = K.fy = 400.0 * w / 512
    K.cx, K.cy = 256.0 * w / 512, 192.0 * h / 384
    return K


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
@pytest.mark.parametrize("q_min", [0.0, 3.0])
def test_residual_blocks(track_case, mode, q_min):
    c, _, m, h, w = track_case
    T = pmxgen.random_pose(9, 900, 2.0, 0.03, 0.97, 1.03).to_struct(abi.pmx_sim3)
    wp = abi.default_robust_weight_params()
    wp.q_min = q_min  # 3.0 excludes part of q in [1, 10] (tracking.cpp:10-13)
    K = _K(w, h) if mode == abi.PMX_TRACK_PIXEL else None
    o, r = both(pyoracle.residual_blocks, T, m, c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"],
                h, w, mode, wp, K)
    assert np.array_equal(o[4], r[4]) and o[4].sum() > 100  # used
    if q_min > 0:
        assert o[4].sum() < (m.valid == 1).sum() - 50  # the exclusion branch is live
    for a, b in zip(o[:4], r[:4]):
        assert rel(a, b) <= 1e-12


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_solve_pose(track_case, mode):
    c, _, _, h, w = track_case
    pred = {"X_f_f": c["X_f_f"], "valid_f": c["valid_f"], "D_f": c["D_f"], "Q_f": c["C_f"],
            "X_k_f": c["X_k_f"], "valid_k": c["valid_k"], "D_k": c["D_k"], "Q_k": c["C_k"]}
    p = abi.default_solve_pose_params()
    p.matching = baseline_match_params()
    p.refinement = abi.refine_params(BASELINE_REFINE)
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(w, h)
    T0 = pmxgen.Pose().to_struct(abi.pmx_sim3)
    (ro, mo), (rr, mr) = both(pyoracle.solve_pose, c["canonical"], c["canonical_valid"], pred, h, w, T0, mode, p)
    assert np.array_equal(mo.pixel_a, mr.pixel_a) and np.array_equal(mo.valid, mr.valid)
    assert ro.lost == rr.lost == 0 and ro.iterations == rr.iterations and ro.iterations >= 2
    assert ro.cost_trace_len == rr.cost_trace_len
    assert rel(ro.cost_trace[:ro.cost_trace_len], rr.cost_trace[:rr.cost_trace_len]) <= 1e-10
    assert rel(ro.T_kf.R[:], rr.T_kf.R[:]) <= 1e-10 and rel(ro.T_kf.t[:], rr.T_kf.t[:]) <= 1e-10
    assert abs(ro.T_kf.s - rr.T_kf.s) <= 1e-10


def test_solve_pose_pixel_mode_without_K_raises(track_case):
    c, _, _, h, w = track_case
    pred = {"X_f_f": c["X_f_f"], "valid_f": c["valid_f"], "D_f": c["D_f"], "Q_f": c["C_f"],
            "X_k_f": c["X_k_f"], "valid_k": c["valid_k"], "D_k": c["D_k"], "Q_k": c["C_k"]}
    T0 = pmxgen.Pose().to_struct(abi.pmx_sim3)
    for use_ref in (False, True):
        with (pyoracle.reference() if use_ref else _null()):
            with pytest.raises(pyoracle.OracleError) as e:
                pyoracle.solve_pose(c["canonical"], c["canonical_valid"], pred, h, w, T0, abi.PMX_TRACK_PIXEL)
            assert e.value.code == abi.PMX_ERR_INVALID_ARGUMENT


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def test_fuse_canonical_bit_identical(track_case):
    c, _, _, h, w = track_case
    T = pmxgen.random_pose(3, 910, 3.0, 0.05, 0.95, 1.05).to_struct(abi.pmx_sim3)
    conf0 = c["canonical_conf"].astype(np.float64)
    conf0[::11] = 0.0  # c_prev <= 0 branch
    cv = c["canonical_valid"].copy()
    cv[::13] = 0
    o, r = both(pyoracle.fuse_canonical, c["canonical"].astype(np.float64), cv, conf0, c["X_k_f"], c["valid_k"],
                c["C_k"], T, h, w)
    for a, b in zip(o, r):
        assert np.array_equal(a, b)


@pytest.fixture(scope="module")
def graph():
    h, w = 24, 32
    g = pmxgen.backend_graph(7, 2, 31, height=h, width=w, radius=1.0)
    ms = [pyoracle.MatchSet(m["pixel_a"], np.arange(h * w), m["confidence"].astype(np.float64), m["valid"])
          for m in g["matches"]]
    return g, ms, h, w


def _graph(g, ms, h, w, poses=None):
    return pyoracle.Graph(g["canonicals"], poses or [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"], ms,
                          h, w)


@pytest.mark.parametrize("mode", [abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL])
def test_assemble_system_and_cost(graph, mode):
    g, ms, h, w = graph
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.mode = mode
    if mode == abi.PMX_TRACK_PIXEL:
        p.has_intrinsics = 1
        p.intrinsics = _K(w, h)
    (Ho, go), (Hr, gr) = both(pyoracle.assemble_system, _graph(g, ms, h, w), p)
    assert np.array_equal(Ho != 0, Hr != 0)  # same sparsity (gauge included)
    assert rel(Ho, Hr) <= 1e-12 * max(1.0, np.abs(Ho).max()) and rel(go, gr) <= 1e-12 * max(1.0, np.abs(go).max())
    co, cr = both(pyoracle.backend_cost, _graph(g, ms, h, w), p)
    assert abs(co - cr) <= 1e-12 * abs(co)


def test_global_optimize_trace(graph):
    g, ms, h, w = graph
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = 6
    Go, Gr = _graph(g, ms, h, w), _graph(g, ms, h, w)
    ro, to = pyoracle.global_optimize(Go, p)
    with pyoracle.reference():
        rr, tr = pyoracle.global_optimize(Gr, p)
    assert ro.iterations == rr.iterations and ro.converged == rr.converged and ro.iterations >= 2
    assert rel(ro.cost_trace[:ro.cost_trace_len], rr.cost_trace[:rr.cost_trace_len]) <= 1e-10
    assert len(to) == len(tr)
    for it in range(len(to)):
        for a, b in zip(to[it], tr[it]):
            assert rel(a.t[:], b.t[:]) <= 1e-10 and rel(a.R[:], b.R[:]) <= 1e-10 and abs(a.s - b.s) <= 1e-10
    for a, b in zip(Go.poses, Gr.poses):
        assert rel(a.t[:], b.t[:]) <= 1e-10


def test_reference_reproduces_backend_fixture():
    z = dict(np.load(os.path.join(GOLD, "backend_6kf_24x32.npz")))
    h, w = (int(x) for x in z["shape"])
    n = z["init"].shape[0]
    E = z["edges"].shape[0]

    def pose(row):
        T = abi.pmx_sim3()
        T.R[:] = list(row[:9])
        T.t[:] = list(row[9:12])
        T.s = float(row[12])
        return T

    G = pyoracle.Graph([(z[f"can{k}"], None) for k in range(n)], [pose(r) for r in z["init"]],
                       [tuple(e) for e in z["edges"]],
                       [pyoracle.MatchSet(z[f"pa{e}"], np.arange(h * w), z[f"q{e}"].astype(np.float64), z[f"v{e}"])
                        for e in range(E)], h, w)
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    with pyoracle.reference():
        res, _ = pyoracle.global_optimize(G, p)
    assert res.iterations == int(z["iterations"][0])
    assert rel(res.cost_trace[:res.cost_trace_len], z["cost_trace"]) <= 1e-10
    final = np.array([list(T.R) + list(T.t) + [T.s] for T in G.poses])
    assert rel(final, z["final"]) <= 1e-10


def test_reference_reproduces_track_fixture():
    """The track fixture is the oracle's match-given GN; the reference has no
    such entry, so its GN loop is pinned through solve_pose above and the
    fixture's residual blocks at the fixture's final pose are compared here."""
    z = dict(np.load(os.path.join(GOLD, "track_48x64.npz")))
    h, w = (int(x) for x in z["shape"])
    m = pyoracle.MatchSet(z["pixel_a"], np.arange(h * w), z["confidence"].astype(np.float64), z["valid"])
    T = abi.pmx_sim3()
    T.R[:] = list(z["R"])
    T.t[:] = list(z["t"])
    T.s = float(z["s"][0])
    wp = abi.default_robust_weight_params()
    wp.distance_weight = 0.1
    o, r = both(pyoracle.residual_blocks, T, m, z["canonical"], z["canonical_valid"], z["X_f_f"], z["valid_f"], h, w,
                abi.PMX_TRACK_RAY, wp)
    assert np.array_equal(o[4], r[4])
    for a, b in zip(o[:4], r[:4]):
        assert rel(a, b) <= 1e-12


def test_sim3_helpers():
    rng = np.random.default_rng(3)
    for k in range(50):
        tau = rng.normal(0, [0.3] * 3 + [0.5] * 3 + [0.2])
        if k % 5 == 0:
            tau[3:6] *= 1e-9  # small-angle branches
        if k % 7 == 0:
            tau[6] = 0.0
        o, r = both(pyoracle.sim3_exp, tau)
        assert rel(o.R[:], r.R[:]) <= 1e-14 and rel(o.t[:], r.t[:]) <= 1e-14 and o.s == r.s
        lo, lr = both(pyoracle.sim3_log, o)
        assert rel(lo, lr) <= 1e-12
        b = pyoracle.sim3_exp(rng.normal(0, 0.4, 7))
        co, cr = both(pyoracle.sim3_compose, o, b)
        assert rel(co.R[:], cr.R[:]) <= 1e-14 and rel(co.t[:], cr.t[:]) <= 1e-14
        io, ir = both(pyoracle.sim3_inverse, o)
        assert rel(io.t[:], ir.t[:]) <= 1e-14
        ao, ar = both(pyoracle.sim3_adjoint, o)
        assert rel(ao, ar) <= 1e-14


def test_robust_weight():
    for q, s2, qm in [(2.0, 1e-3, 0.5), (0.5, 1e-3, 0.5), (0.4, 1e-2, 0.5), (3.0, 4.0, 0.0)]:
        o, r = both(lambda *a: pyoracle.lib().orc_robust_weight(*a), q, s2, qm)
        assert o == r
