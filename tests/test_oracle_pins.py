"""Pins the CPU oracle (oracle/, FP64 restatement of the reference hot path)
against the reference's own known-answer and property tests.

The reference cannot be built here (Eigen3 absent) and ships no golden
vectors, so these ports of /root/reference/proj/tests/test_{camera,tracking,
backend}.cpp — same properties, same tolerances — are what pins the oracle
before it is trusted as the GPU parity checker.  Scenes come from
gen/pmx_gen.cpp instead of the reference's box-room renderer (which would
need libstdc++'s implementation-defined distributions).
"""
import ctypes as C
import math

import numpy as np
import pytest

import pmxgen
import pyoracle
from paper_2412_12392_b200 import abi

RNG = np.random.default_rng(7)


def S3(R=None, t=None, s=1.0):
    return pmxgen.Pose(R, t, s).to_struct(abi.pmx_sim3)


def to_pose(T):
    return pmxgen.Pose.from_struct(T)


def noiseless_pair(ia, Ta, ib, Tb, h=48, w=64, seed=11):
    sc = pmxgen.Scene(seed, h, w, f=400.0 * w / 512, cx=256.0 * w / 512, cy=192.0 * h / 384, point_sigma=0.0)
    return sc, sc.pair(ia, Ta, ib, Tb)


def small_motion(k):
    return pmxgen.Pose(pmxgen.rodrigues([0.0, 0.01 * k, 0.005 * k]), [0.03 * k, -0.01 * k, 0.0], 1.0)


# ------------------------------------------------------------ camera.cpp

def test_normalize_rays_known_values():  # test_camera.cpp:34-44
    X = np.array([[0, 0, 2], [1, 1, 1], [0, 0, 0]], np.float32)
    rays, dist, valid = pyoracle.normalize_rays(X, None, 1, 3)
    assert np.linalg.norm(rays[0] - [0, 0, 1]) <= 1e-15 and dist[0] == pytest.approx(2.0)
    assert np.linalg.norm(rays[1] - np.ones(3) / math.sqrt(3)) <= 1e-15
    assert dist[1] == pytest.approx(math.sqrt(3.0))
    assert valid[2] == 0


def test_normalize_rays_reconstruction():  # test_camera.cpp:46-53
    _, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(1))
    rays, dist, valid = pyoracle.normalize_rays(p["X_a"], None, 48, 64)
    assert valid.all()
    assert np.abs(np.linalg.norm(rays, axis=1) - 1).max() <= 1e-9
    rec = rays * dist[:, None]
    assert (np.linalg.norm(rec - p["X_a"], axis=1) <= 1e-9 * dist).all()


def test_interpolate_ray_jacobian_matches_fd():  # test_camera.cpp:66-87
    _, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(1))
    pts = np.stack([RNG.uniform(1, 62, 100), RNG.uniform(1, 46, 100)], 1)
    r0, J, ok = pyoracle.interpolate_ray(p["X_a"], None, 48, 64, pts)
    assert ok.all()
    eps = 1e-6
    for axis in range(2):
        hi, lo = pts.copy(), pts.copy()
        hi[:, axis] += eps
        lo[:, axis] -= eps
        fd = (pyoracle.interpolate_ray(p["X_a"], None, 48, 64, hi)[0] -
              pyoracle.interpolate_ray(p["X_a"], None, 48, 64, lo)[0]) / (2 * eps)
        an = J[:, 3 * axis:3 * axis + 3]
        err = np.linalg.norm(an - fd, axis=1)
        assert (err <= 1e-5 * np.maximum(1.0, np.linalg.norm(fd, axis=1))).all()


def test_iterative_project_exact_seed_is_fixed_point():  # test_camera.cpp:89-98
    _, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(1))
    u, v = 20, 17
    x = p["X_a"][v * 64 + u]
    pix, conv, it = pyoracle.iterative_project(p["X_a"], None, 48, 64, x, [u, v])
    assert conv[0] and np.hypot(pix[0, 0] - u, pix[0, 1] - v) <= 0.5


def test_iterative_project_converges_from_5px():  # test_camera.cpp:100-117
    h, w = 96, 128
    _, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(1), h, w)
    uu, vv = np.meshgrid(np.arange(w), np.arange(h))
    uu, vv = uu.ravel(), vv.ravel()
    p0 = np.stack([np.clip(uu + 5, 0, w - 1), np.clip(vv + 5, 0, h - 1)], 1)
    pix, conv, it = pyoracle.iterative_project(p["X_a"], None, h, w, p["X_a"], p0)
    ok = conv.astype(bool) & (it <= 10) & (np.hypot(pix[:, 0] - uu, pix[:, 1] - vv) <= 1.0)
    assert ok.mean() >= 0.99


def test_self_pair_identity_init_is_identity():  # test_camera.cpp:119-132
    _, p = noiseless_pair(0, pmxgen.Pose(), 0, pmxgen.Pose())
    m = pyoracle.match_pointmaps(p)
    assert m.valid.all()
    assert (m.pixel_a == np.arange(48 * 64)).all()


def _gt_pair(h=96, w=128):
    sc, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(2), h, w)
    gt = sc.gt_matches(0, pmxgen.Pose(), 1, small_motion(2))
    return p, gt


def test_matches_ground_truth_and_confidence():  # test_camera.cpp:134-158
    h, w = 96, 128
    p, gt = _gt_pair(h, w)
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(p), p)
    both = (m.valid == 1) & (gt["valid"] == 1)
    assert both.sum() > 1000
    pa, pg = m.pixel_a[both], gt["pixel_a"][both]
    d = np.hypot(pa % w - pg % w, pa // w - pg // w)
    assert (d <= 1.0).mean() >= 0.95
    q = np.sqrt(p["Q_a"][pa].astype(np.float64) * p["Q_b"][both].astype(np.float64))
    np.testing.assert_allclose(m.confidence[both], q, rtol=1e-9)


def test_recall_with_identity_init():  # test_camera.cpp:160-175
    p, gt = _gt_pair()
    m = pyoracle.match_pointmaps(p)
    g = gt["valid"] == 1
    assert g.sum() > 1000 and (m.valid[g] == 1).mean() >= 0.95


def test_gross_depth_outliers_invalidated():  # test_camera.cpp:177-196
    _, p = noiseless_pair(0, pmxgen.Pose(), 1, small_motion(1))
    sel = RNG.random(48 * 64) < 0.2
    p = dict(p, X_b=p["X_b"].copy())
    p["X_b"][sel] *= 3.0
    m = pyoracle.match_pointmaps(p)
    assert sel.sum() > 100 and (m.valid[sel] == 1).mean() <= 0.02


def test_seeded_matching_keeps_valid_count():  # test_camera.cpp:198-217
    sc = pmxgen.Scene(11, 48, 64, f=50.0, cx=32.0, cy=24.0, point_sigma=0.0)
    p01 = sc.pair(1, small_motion(1), 0, pmxgen.Pose())
    p02 = sc.pair(2, small_motion(2), 0, pmxgen.Pose())
    seed = pyoracle.match_pointmaps(p01)
    unseeded = pyoracle.match_pointmaps(p02)
    seeded = pyoracle.match_pointmaps(p02, init=seed)
    assert seeded.valid.sum() >= 0.95 * unseeded.valid.sum()


def test_feature_refine_planted_peak_and_flat_tie():  # test_camera.cpp:219-247
    h, w, d = 16, 16, 4
    Fa = np.zeros((h * w, d), np.float16)
    Fb = np.zeros((h * w, d), np.float16)
    Fa[:, 1] = 1
    Fb[:, 0] = 1
    gu = gv = 8
    peak = gv * w + gu + 2
    Fa[peak] = 0
    Fa[peak, 0] = 1
    q = np.ones(h * w, np.float32)
    pair = {"D_a": Fa.view(np.uint16), "D_b": Fb.view(np.uint16), "Q_a": q, "Q_b": q, "height": h, "width": w}
    m = pyoracle.MatchSet([gv * w + gu], [5 * w + 5], [1.0], [1])
    assert pyoracle.feature_refine(m, pair).pixel_a[0] == peak
    flat = np.full((h * w, d), 0.5, np.float16).view(np.uint16)
    pair = dict(pair, D_a=flat, D_b=flat)
    assert pyoracle.feature_refine(m, pair).pixel_a[0] == gv * w + gu


def test_feature_refine_keeps_maximal_match():  # test_camera.cpp:249-261
    _, p = noiseless_pair(0, pmxgen.Pose(), 0, pmxgen.Pose())
    m = pyoracle.match_pointmaps(p)
    r = pyoracle.feature_refine(m, p)
    assert (r.pixel_a == m.pixel_a).all()


# ----------------------------------------------------------- tracking.cpp

def test_robust_weight_known_answers():  # test_tracking.cpp:54-60
    L = pyoracle.lib()
    L.orc_robust_weight.restype = C.c_double
    q_min = 0.05
    rw = lambda q, s2, qm: L.orc_robust_weight(C.c_double(q), C.c_double(s2), C.c_double(qm))
    assert rw(2 * q_min, 1.0, q_min) == pytest.approx(1.0 / (2 * q_min))
    assert math.isinf(rw(q_min, 1.0, q_min))
    assert math.isinf(rw(0.0, 1.0, q_min))
    assert rw(0.5, 1e-3, 0.0) == pytest.approx(2e-3)


def _aligned(T_true, h=48, w=64, seed=21):
    sc = pmxgen.Scene(seed, h, w, f=400.0 * w / 512, cx=256.0 * w / 512, cy=192.0 * h / 384, point_sigma=0.0)
    can = sc.image(0, pmxgen.Pose(), pmxgen.Pose(), want=("X",))["X"]
    X_f = T_true.inverse().act(can.astype(np.float64)).astype(np.float32)
    n = h * w
    m = pyoracle.MatchSet(np.arange(n), np.arange(n), np.ones(n), np.ones(n, np.uint8))
    return can, X_f, m


def test_residuals_vanish_at_true_pose():  # test_tracking.cpp:84-105
    T = pmxgen.Pose(pmxgen.rodrigues([0.15, -0.1, 0.2]), [0.1, -0.2, 0.05], 1.3)
    can, X_f, m = _aligned(T)
    # exact correspondences in double: express X_f through T in FP64 on fp32 inputs
    for mode in (abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT):
        res, jac, wt, info, used = pyoracle.residual_blocks(T.to_struct(abi.pmx_sim3), m, can, None, X_f, None, 48,
                                                            64, mode)
        assert used.sum() > 500
        # fp32 storage of X_f limits exactness to ~1e-7 (the reference's 1e-9 assumes FP64 points)
        assert np.abs(res[used == 1]).max() <= 1e-6


def _fd_subset():
    sc = pmxgen.Scene(21, 48, 64, f=50.0, cx=32.0, cy=24.0, point_sigma=0.0)
    T01 = small_motion(1)
    can = sc.image(0, pmxgen.Pose(), pmxgen.Pose(), want=("X",))["X"]
    p = sc.pair(1, T01, 0, pmxgen.Pose())
    m = pyoracle.match_pointmaps(p)
    idx = np.arange(0, 48 * 64, 37)
    idx = idx[m.valid[idx] == 1]
    sub = pyoracle.MatchSet(m.pixel_a[idx], idx, m.confidence[idx], m.valid[idx])
    return can, p["X_a"], sub, T01


def test_residual_jacobians_match_fd():  # test_tracking.cpp:107-148
    can, X_f, sub, T_true = _fd_subset()
    assert len(sub) >= 40
    K = abi.pmx_intrinsics(50.0, 50.0, 32.0, 24.0)
    eps = 1e-6
    for mode in (abi.PMX_TRACK_RAY, abi.PMX_TRACK_POINT, abi.PMX_TRACK_PIXEL):
        configs = 0
        for trial in range(4):
            tau = RNG.uniform(-0.05, 0.05, 7)
            T = pyoracle.sim3_compose(pyoracle.sim3_exp(tau), T_true.to_struct(abi.pmx_sim3))
            r0, J, w, info, used = pyoracle.residual_blocks(T, sub, can, None, X_f, None, 48, 64, mode, K=K)
            for axis in range(7):
                d = np.zeros(7)
                d[axis] = eps
                Th = pyoracle.sim3_compose(pyoracle.sim3_exp(d), T)
                Tl = pyoracle.sim3_compose(pyoracle.sim3_exp(-d), T)
                rh = pyoracle.residual_blocks(Th, sub, can, None, X_f, None, 48, 64, mode, K=K)
                rl = pyoracle.residual_blocks(Tl, sub, can, None, X_f, None, 48, 64, mode, K=K)
                ok = (used == 1) & (rh[4] == 1) & (rl[4] == 1)
                fd = (rh[0] - rl[0]) / (2 * eps)
                an = J[:, :, axis]
                err = np.linalg.norm(fd - an, axis=1)
                assert (err[ok] <= 1e-5 * np.maximum(1.0, np.linalg.norm(an, axis=1)[ok])).all()
                configs += ok.sum()
        assert configs >= 100 * 7


def test_distance_rows_restore_rank_under_pure_rotation():  # test_tracking.cpp:150-188
    h, w = 48, 64
    sc = pmxgen.Scene(33, h, w, f=50.0, cx=32.0, cy=24.0, point_sigma=0.0)
    Rrot = pmxgen.Pose(pmxgen.rodrigues([0.0, 0.02, 0.01]), [0, 0, 0], 1.0)
    can = sc.image(0, pmxgen.Pose(), pmxgen.Pose(), want=("X",))["X"]
    p = sc.pair(1, Rrot, 0, pmxgen.Pose())
    m = pyoracle.match_pointmaps(p)
    assert m.valid.sum() > 500
    res, J, wt, info, used = pyoracle.residual_blocks(Rrot.to_struct(abi.pmx_sim3), m, can, None, p["X_a"], None,
                                                      h, w, abi.PMX_TRACK_RAY)
    u = used == 1
    Hr = np.einsum("n,nra,nrb->ab", np.ones(u.sum()), J[u][:, :3] * wt[u][:, :3, None], J[u][:, :3])
    Hf = np.einsum("nra,nrb->ab", J[u] * wt[u][:, :, None], J[u])
    er, ef = np.linalg.eigvalsh(Hr), np.linalg.eigvalsh(Hf)
    assert er[0] <= 1e-10 * er[-1]
    assert ef[0] >= 1e-8 * ef[-1]


def _track(can, X_f, m, init=None, mode=abi.PMX_TRACK_RAY, params=None):
    return pyoracle.track_given_matches(can, None, X_f, None, 48, 64, m, init or S3(), mode, params)


def test_self_tracking_is_identity():  # test_tracking.cpp:190-198
    can, X_f, m = _aligned(pmxgen.Pose())
    r = _track(can, can, m)
    assert not r.lost
    assert np.linalg.norm(pyoracle.sim3_log(r.T_kf)) <= 1e-8


def test_exact_sim3_recovery_with_scale():  # test_tracking.cpp:200-223
    T = pmxgen.Pose(pmxgen.rodrigues([0.1, -0.08, 0.12]), [0.08, -0.12, 0.05], 1.3)
    can, X_f, m = _aligned(T)
    r = _track(can, X_f, m)
    assert not r.lost
    err = pyoracle.sim3_log(pyoracle.sim3_compose(pyoracle.sim3_inverse(T.to_struct(abi.pmx_sim3)), r.T_kf))
    # fp32 storage of the prediction bounds exact recovery near 1e-7 (reference: FP64 points, 1e-6 / 1e-8)
    assert np.linalg.norm(err[:3]) <= 1e-6 and np.linalg.norm(err[3:6]) <= 1e-6
    assert abs(r.T_kf.s / T.s - 1) <= 1e-6
    tr = list(r.cost_trace[:r.cost_trace_len])
    for a, b in zip(tr[1:], tr[:-1]):
        assert a <= b * (1 + 1e-12) + 1e-300


def test_tracking_equivariance():  # test_tracking.cpp:248-270
    T = pmxgen.Pose(pmxgen.rodrigues([0.1, -0.08, 0.12]), [0.08, -0.12, 0.05], math.exp(0.1))
    can, X_f, m = _aligned(T)
    base = _track(can, X_f, m)
    G = pmxgen.Pose(pmxgen.rodrigues([0.4, -0.2, 0.1]), [0.2, -0.1, 0.3], math.exp(0.15))
    can_g = G.act(can.astype(np.float64)).astype(np.float32)
    X_g = G.act(X_f.astype(np.float64)).astype(np.float32)
    Tb = to_pose(base.T_kf)
    init = (G * Tb * G.inverse()).to_struct(abi.pmx_sim3)
    moved = _track(can_g, X_g, m, init=init)
    exp = (G * Tb * G.inverse()).to_struct(abi.pmx_sim3)
    d = pyoracle.sim3_log(pyoracle.sim3_compose(pyoracle.sim3_inverse(exp), moved.T_kf))
    assert np.linalg.norm(d) <= 1e-5  # fp32 re-expression of the inputs


def test_fusion_first_exact_then_idempotent():  # test_tracking.cpp:314-337
    h, w = 48, 64
    X = RNG.standard_normal((h * w, 3)).astype(np.float32) + np.array([0, 0, 3], np.float32)
    C0 = RNG.uniform(0.5, 1.0, h * w).astype(np.float32)
    cx, cv, cc = pyoracle.fuse_canonical(np.zeros((h * w, 3)), np.zeros(h * w, np.uint8), np.zeros(h * w), X, None,
                                         C0, S3(), h, w)
    assert np.abs(cx - X).max() <= 1e-15 and np.allclose(cc, C0)
    cx2, cv2, cc2 = pyoracle.fuse_canonical(cx, cv, cc, X, None, C0, S3(), h, w)
    assert np.abs(cx2 - cx).max() <= 1e-12 and np.allclose(cc2, 2 * C0)


def test_fusion_50_observations_rmse():  # test_tracking.cpp:339-379
    h, w, n_obs, sigma = 24, 32, 50, 0.05
    rng = np.random.default_rng(3)
    gt = (rng.normal(0, sigma, (h * w, 3)) + [0, 0, 2.0]) * 10.0
    cx, cv, cc = np.zeros((h * w, 3)), np.zeros(h * w, np.uint8), np.zeros(h * w)
    ones = np.ones(h * w, np.float32)
    single = None
    for obs in range(n_obs):
        noise = rng.normal(0, sigma, (h * w, 3))
        noisy = (gt + noise).astype(np.float32)
        if obs == 0:
            single = math.sqrt((noise ** 2).sum() / (h * w))
        cx, cv, cc = pyoracle.fuse_canonical(cx, cv, cc, noisy, None, ones, S3(), h, w)
        assert np.allclose(cc, obs + 1.0)
    fused = math.sqrt(((cx - gt) ** 2).sum() / (h * w))
    ideal = single / math.sqrt(n_obs)
    assert ideal / 1.5 <= fused <= 1.5 * ideal


def test_keyframe_decision_thresholds():  # test_tracking.cpp:381-410
    full = pyoracle.MatchSet(np.arange(100), np.arange(100), np.ones(100), np.ones(100, np.uint8))
    assert not pyoracle.keyframe_decision(full, 10, 10, 0.333)
    sparse = pyoracle.MatchSet(np.arange(30), np.arange(30), np.ones(30), np.ones(30, np.uint8))
    assert pyoracle.keyframe_decision(sparse, 10, 10, 0.333)
    collapsed = pyoracle.MatchSet(np.zeros(90), np.arange(90), np.ones(90), np.ones(90, np.uint8))
    assert pyoracle.keyframe_decision(collapsed, 10, 10, 0.333)


# ------------------------------------------------------------ backend.cpp

def consistent_graph(poses, h=6, w=8, loop_edge=False, seed=7):  # test_backend.cpp:39-64
    rng = np.random.default_rng(seed)
    n = h * w
    world = np.stack([2 * rng.uniform(-1, 1, n), 2 * rng.uniform(-1, 1, n), 4 + 1.5 * rng.uniform(-1, 1, n)], 1)
    cans = [(P.inverse().act(world).astype(np.float32), None) for P in poses]
    edges = [(k - 1, k) for k in range(1, len(poses))]
    if loop_edge and len(poses) > 2:
        edges.append((0, len(poses) - 1))
    ident = np.arange(n)
    ms = [pyoracle.MatchSet(ident, ident, np.ones(n), np.ones(n, np.uint8)) for _ in edges]
    return pyoracle.Graph(cans, [P.to_struct(abi.pmx_sim3) for P in poses], edges, ms, h, w)


def orbit(n, seed=3):
    return [pmxgen.Pose(pmxgen.rodrigues([0.0, 0.15 * k, 0.05 * k]), [0.3 * math.sin(0.3 * k), 0.1 * k, 0.2 * k], 1.0)
            for k in range(n)]


def test_stationary_point():  # test_backend.cpp:100-105
    g = consistent_graph(orbit(4), 8, 8)
    H, grad = pyoracle.assemble_system(g)
    # fp32-stored canonicals leave ~1e-7 relative point noise (reference: FP64
    # points, |g| <= 1e-10): require |g| to be tiny relative to the gradient of
    # a 1e-3 perturbation of the same configuration
    g.poses[2] = pyoracle.sim3_compose(pyoracle.sim3_exp(np.full(7, 1e-3)), g.poses[2])
    _, grad_p = pyoracle.assemble_system(g)
    assert np.abs(grad).max() <= 1e-2 * np.abs(grad_p).max()


def _perturbed(n=3, h=6, w=8, seed=5):
    g = consistent_graph(orbit(n), h, w)
    rng = np.random.default_rng(seed)
    for k in range(1, n):
        g.poses[k] = pyoracle.sim3_compose(pyoracle.sim3_exp(rng.uniform(-0.05, 0.05, 7)), g.poses[k])
    return g


def test_assemble_matches_bruteforce_dense_stacking():  # test_backend.cpp:107-173
    g = _perturbed()
    p = abi.default_backend_params()
    H, grad = pyoracle.assemble_system(g, p)
    n = len(g.poses)
    dim = 7 * n
    Hb = np.zeros((dim, dim))
    gb = np.zeros(dim)
    for e, (i, j) in enumerate(g.edges):
        m = g.matches[e]
        med = np.sort(m.confidence[m.valid == 1])[(m.valid == 1).sum() // 2]
        w = abi.default_robust_weight_params()
        w.q_min = w.q_min_fraction * med
        sw = pyoracle.MatchSet(m.pixel_b, m.pixel_a, m.confidence, m.valid)
        for ref, src, ms in ((i, j, sw), (j, i, m)):
            Trel = pyoracle.sim3_compose(pyoracle.sim3_inverse(g.poses[ref]), g.poses[src])
            res, J, wt, info, used = pyoracle.residual_blocks(Trel, ms, g.canonicals[ref][0], None,
                                                              g.canonicals[src][0], None, g.h, g.w, 0, w)
            adj = pyoracle.sim3_adjoint(pyoracle.sim3_inverse(g.poses[ref]))
            for k in np.nonzero(used)[0]:
                for r in range(4):
                    if wt[k, r] <= 0:
                        continue
                    row = np.zeros(dim)
                    jr = J[k, r] @ adj
                    row[7 * ref:7 * ref + 7] = -jr
                    row[7 * src:7 * src + 7] = jr
                    Hb += wt[k, r] * np.outer(row, row)
                    gb += wt[k, r] * row * res[k, r]
    # gauge: anchor rows/cols -> identity, gradient 0
    Hb[:7, :] = 0
    Hb[:, :7] = 0
    Hb[:7, :7] = np.eye(7)
    gb[:7] = 0
    assert np.abs(H - Hb).max() <= 1e-10 * np.abs(Hb).max()
    assert np.abs(grad - gb).max() <= 1e-10 * max(np.abs(gb).max(), 1e-300)
    assert np.allclose(H, H.T, rtol=0, atol=1e-12 * np.abs(H).max())


def test_gradient_matches_fd_of_cost():  # test_backend.cpp:175-204
    g = _perturbed()
    p = abi.default_backend_params()
    H, grad = pyoracle.assemble_system(g, p)
    eps = 1e-6
    for k in (1, 2):
        for a in range(7):
            d = np.zeros(7)
            d[a] = eps
            base = list(g.poses)
            g.poses = list(base)
            g.poses[k] = pyoracle.sim3_compose(pyoracle.sim3_exp(d), base[k])
            hi = pyoracle.backend_cost(g, p)
            g.poses[k] = pyoracle.sim3_compose(pyoracle.sim3_exp(-d), base[k])
            lo = pyoracle.backend_cost(g, p)
            g.poses = base
            fd = (hi - lo) / (2 * eps)
            assert abs(fd - grad[7 * k + a]) <= 1e-5 * max(1.0, abs(fd))


def test_hessian_sparsity_follows_edges():  # test_backend.cpp:206-239
    g = consistent_graph(orbit(5), 6, 8)
    g.edges = [(0, 1), (1, 2), (3, 4)]
    g.matches = g.matches[:3]
    H, grad = pyoracle.assemble_system(g)
    blk = lambda i, j: np.abs(H[7 * i:7 * i + 7, 7 * j:7 * j + 7]).max()
    assert blk(1, 2) > 0 and blk(3, 4) > 0
    assert blk(1, 3) == 0 and blk(2, 4) == 0 and blk(0, 1) == 0
    assert np.array_equal(H[:7, :7], np.eye(7))


def test_consistent_graph_fixed_point():  # test_backend.cpp:241-264
    poses = orbit(5, 9)
    g = consistent_graph(poses)
    anchor = list(g.poses[0].R), list(g.poses[0].t), g.poses[0].s
    res, trace = pyoracle.global_optimize(g)
    assert res.converged and res.iterations == 1
    assert (list(g.poses[0].R), list(g.poses[0].t), g.poses[0].s) == anchor
    for a, P in zip(g.poses, poses):
        d = pyoracle.sim3_log(pyoracle.sim3_compose(pyoracle.sim3_inverse(P.to_struct(abi.pmx_sim3)), a))
        assert np.linalg.norm(d) <= 1e-6


def ate_rmse(est, gt):
    """Sim(3)-aligned ATE (Umeyama) over camera centres."""
    X = np.array([p.t for p in est])
    Y = np.array([p.t for p in gt])
    mx, my = X.mean(0), Y.mean(0)
    Xc, Yc = X - mx, Y - my
    U, S, Vt = np.linalg.svd(Yc.T @ Xc / len(X))
    D = np.eye(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        D[2, 2] = -1
    R = U @ D @ Vt
    s = np.trace(np.diag(S) @ D) / (Xc ** 2).sum(1).mean()
    t = my - s * R @ mx
    return math.sqrt(((s * (X @ R.T) + t - Y) ** 2).sum(1).mean())


def test_drift_corrected_by_loop_edge():  # test_backend.cpp:266-306
    n = 20
    poses = [pmxgen.Pose(pmxgen.rodrigues([0, 2 * math.pi * k / n, 0]),
                         [2 * math.sin(2 * math.pi * k / n), 0, 2 - 2 * math.cos(2 * math.pi * k / n)], 1.0)
             for k in range(n)]
    g = consistent_graph(poses, 8, 8, loop_edge=True)
    drift = pyoracle.sim3_exp(np.array([0.01, -0.006, 0.008, 0.004, -0.006, 0.005, 0.004]))
    dr = [poses[0].to_struct(abi.pmx_sim3)]
    for k in range(1, n):
        rel = pyoracle.sim3_compose(pyoracle.sim3_inverse(poses[k - 1].to_struct(abi.pmx_sim3)),
                                    poses[k].to_struct(abi.pmx_sim3))
        dr.append(pyoracle.sim3_compose(dr[-1], pyoracle.sim3_compose(rel, drift)))
    g.poses = dr
    pre = ate_rmse([to_pose(P) for P in g.poses], poses)
    assert pre > 1e-3
    res, trace = pyoracle.global_optimize(g)
    assert res.converged
    post = ate_rmse([to_pose(P) for P in g.poses], poses)
    assert post <= 0.1 * pre
    tr = list(res.cost_trace[:res.cost_trace_len])
    for a, b in zip(tr[1:], tr[:-1]):
        assert a <= b * (1 + 1e-12) + 1e-300


def test_gauge_invariance():  # test_backend.cpp:308-338
    poses = orbit(5, 13)
    rng = np.random.default_rng(13)
    noise = [rng.uniform(-0.03, 0.03, 7) for _ in range(5)]

    def rel_after(G):
        moved = [G * P for P in poses]
        g = consistent_graph(moved)
        for k in range(1, 5):
            g.poses[k] = (G * to_pose(pyoracle.sim3_exp(noise[k])) * poses[k]).to_struct(abi.pmx_sim3)
        assert pyoracle.global_optimize(g)[0].converged
        return [pyoracle.sim3_compose(pyoracle.sim3_inverse(g.poses[0]), g.poses[k]) for k in range(1, 5)]

    G = to_pose(pyoracle.sim3_exp(np.array([0.5, -0.3, 0.8, 0.4, -0.2, 0.6, 0.2])))
    base, moved = rel_after(pmxgen.Pose()), rel_after(G)
    for a, b in zip(base, moved):
        assert np.linalg.norm(pyoracle.sim3_log(pyoracle.sim3_compose(pyoracle.sim3_inverse(a), b))) <= 1e-6


def test_pure_rotation_distance_restores_rank():  # test_backend.cpp:340-372
    poses = [pmxgen.Pose(), pmxgen.Pose(pmxgen.rodrigues([0.0, 0.25, 0.1]), [0, 0, 0], 1.0)]
    g = consistent_graph(poses, 8, 8)
    rot = np.zeros(7)
    rot[3:6] = [0.01, -0.008, 0.006]
    g.poses[1] = pyoracle.sim3_compose(pyoracle.sim3_exp(rot), g.poses[1])
    weak = abi.default_backend_params()
    weak.weights.distance_weight = 0.0
    Hw, _ = pyoracle.assemble_system(g, weak)
    Hf, _ = pyoracle.assemble_system(g)
    ew, ef = np.linalg.eigvalsh(Hw[7:, 7:]), np.linalg.eigvalsh(Hf[7:, 7:])
    assert ew[0] <= 1e-10 * ew[-1] and ef[0] >= 1e-8 * ef[-1]
    assert pyoracle.global_optimize(g)[0].converged


def test_sparse_ldlt_matches_numpy_and_zero_pivot():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((21, 21))
    A = A @ A.T + np.eye(21)
    b = rng.standard_normal(21)
    x, ok = pyoracle.ldlt_solve(A, b)
    assert ok and np.allclose(x, np.linalg.solve(A, b), rtol=1e-10)
    Z = np.zeros((14, 14))
    Z[7:, 7:] = np.eye(7)
    assert not pyoracle.ldlt_solve(Z, np.ones(14))[1]


def test_sim3_exp_log_roundtrip():  # test_lie.cpp (exp/log consistency used on the path)
    for tau in (np.array([0.1, -0.2, 0.3, 0.2, -0.1, 0.05, 0.3]), np.array([0.1, 0.2, 0.3, 0, 0, 0, 0]),
                np.array([0.1, 0.2, 0.3, 1e-10, 0, 0, 1e-10])):
        np.testing.assert_allclose(pyoracle.sim3_log(pyoracle.sim3_exp(tau)), tau, atol=1e-12)
