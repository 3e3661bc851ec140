"""GPU parity of backend global optimisation (reference src/backend.cpp:29-256)
against the FP64 oracle through the C ABI.

Bar (BASELINE north_star): H, g within 1e-4 relative; final poses within
1e-5 (translation) and 1e-5 rad (rotation).
"""
import numpy as np
import pytest

import pmxgen
import pyoracle
from paper_2412_12392_b200 import Graph, MatchSet, Pointmap, abi

pytestmark = pytest.mark.gpu


def _graph(n_kf=8, reach=2, h=48, w=64, seed=3, **kw):
    g = pmxgen.backend_graph(n_kf, reach, seed, height=h, width=w, radius=1.0, **kw)
    poses = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
    cans = [Pointmap(x, v, h, w) for x, v in g["canonicals"]]
    ms = [MatchSet(m["pixel_a"], m["confidence"], m["valid"]) for m in g["matches"]]
    G = Graph(cans, poses, g["edges"], ms, anchor=0)
    O = pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"],
                       [pyoracle.MatchSet(m["pixel_a"], np.arange(h * w), m["confidence"].astype(np.float64),
                                          m["valid"]) for m in g["matches"]], h, w)
    return g, G, O


def _params():
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    return p


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_edge_terms_parity(ctx):
    g, G, O = _graph()
    p = _params()
    tg = ctx.backend_edge_terms(G, p)
    to = pyoracle.backend_edge_terms(O, p)
    for e in range(len(g["edges"])):
        for d in (0, 36):
            assert _rel(tg[e, d:d + 28], to[e, d:d + 28]) < 1e-4
            assert _rel(tg[e, d + 28:d + 35], to[e, d + 28:d + 35]) < 1e-4
            assert abs(tg[e, d + 35] - to[e, d + 35]) <= 1e-5 * abs(to[e, d + 35])


def test_assemble_system_parity(ctx):
    g, G, O = _graph()
    p = _params()
    Hg, gg = ctx.assemble_system(G, p)
    Ho, go = pyoracle.assemble_system(O, p)
    # sparsity pattern identical (anchor gauge + edge list), values 1e-4 relative
    assert np.array_equal(Hg != 0, Ho != 0)
    assert _rel(Hg, Ho) < 1e-4
    assert _rel(gg, go) < 1e-4
    np.testing.assert_allclose(Hg, Hg.T, rtol=0, atol=1e-9 * np.abs(Hg).max())
    np.testing.assert_array_equal(Hg[:7, :7], np.eye(7))
    assert np.all(gg[:7] == 0)


def test_backend_cost_parity(ctx):
    g, G, O = _graph()
    p = _params()
    assert abs(ctx.backend_cost(G, p) - pyoracle.backend_cost(O, p)) <= 1e-5 * pyoracle.backend_cost(O, p)


def _pose_err(a, b):
    Ra, Rb = np.array(a.R[:]).reshape(3, 3), np.array(b.R[:]).reshape(3, 3)
    ang = np.arccos(np.clip((np.trace(Ra.T @ Rb) - 1) / 2, -1, 1))
    return float(np.abs(np.array(a.t[:]) - np.array(b.t[:])).max()), float(ang)


@pytest.mark.parametrize("n_kf,reach", [(8, 2), (20, 4)])
def test_global_optimize_parity(ctx, n_kf, reach):
    g, G, O = _graph(n_kf=n_kf, reach=reach)
    p = _params()
    rg = ctx.global_optimize(G, p, trace=True)
    ro, tro = pyoracle.global_optimize(O, p)
    assert rg.converged == bool(ro.converged)
    for a, b in zip(G.poses, O.poses):
        et, er = _pose_err(a, b)
        assert et < 1e-5 and er < 1e-5, (et, er)
    # anchor bit-identical
    assert list(G.poses[0].R) == list(g["init"][0].to_struct(abi.pmx_sim3).R)
    # per-iteration poses agree while both traces are active
    for it in range(min(len(rg.pose_trace), len(tro))):
        for a, b in zip(rg.pose_trace[it], tro[it]):
            et, er = _pose_err(a, b)
            assert et < 1e-5 and er < 1e-5
    # drift reduced towards ground truth
    err = [np.abs(np.array(P.t[:]) - T.t).max() for P, T in zip(G.poses, g["gt"])]
    err0 = [np.abs(I.t - T.t).max() for I, T in zip(g["init"], g["gt"])]
    assert max(err) < 0.5 * max(err0)


def test_consistent_graph_is_fixed_point(ctx):
    # test_backend.cpp:241-264 (noise-free canonicals at the true poses)
    h, w = 24, 32
    rng = np.random.default_rng(7)
    n = h * w
    world = np.stack([rng.uniform(-2, 2, n), rng.uniform(-2, 2, n), 4 + 1.5 * rng.uniform(-1, 1, n)], 1)
    poses = [pmxgen.Pose(pmxgen.rodrigues([0, 0.05 * k, 0.02 * k]), [0.1 * k, 0, 0.02 * k], 1.0) for k in range(5)]
    cans = [(poses[k].inverse().act(world).astype(np.float32), None) for k in range(5)]
    edges = [(k, k + 1) for k in range(4)]
    ident = np.arange(n, dtype=np.int32)
    ms = [MatchSet(ident, np.ones(n, np.float32), np.ones(n, np.uint8)) for _ in edges]
    G = Graph([Pointmap(x, None, h, w) for x, _ in cans], [P.to_struct(abi.pmx_sim3) for P in poses], edges, ms)
    p = abi.default_backend_params()
    r = ctx.global_optimize(G, p)
    assert r.converged
    for a, b in zip(G.poses, poses):
        et, er = _pose_err(a, b.to_struct(abi.pmx_sim3))
        assert et < 1e-5 and er < 1e-5
    assert list(G.poses[0].t) == list(poses[0].t)


def test_ldlt_solve_matches_numpy_and_flags_zero_pivot(ctx):
    rng = np.random.default_rng(1)
    for n in (7, 70, 333):
        A = rng.standard_normal((n, n))
        A = A @ A.T + n * np.eye(n)
        b = rng.standard_normal(n)
        x, ok = ctx.ldlt_solve(A, b)
        assert ok
        np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
        xo, oko = pyoracle.ldlt_solve(A, b)
        assert oko
        np.testing.assert_allclose(x, xo, rtol=1e-9, atol=1e-12)
    A = np.zeros((14, 14))
    A[7:, 7:] = np.eye(7)
    x, ok = ctx.ldlt_solve(A, np.ones(14))
    assert not ok
    assert not pyoracle.ldlt_solve(A, np.ones(14))[1]


def test_solve_terms_equals_global_step(ctx):
    # the edge-sharded building blocks reproduce one assemble+solve step
    g, G, O = _graph()
    p = _params()
    terms = ctx.backend_edge_terms(G, p)
    tau, cost, solved = ctx.backend_solve_terms(G, terms, p)
    assert solved
    H, grad = ctx.assemble_system(G, p)
    np.testing.assert_allclose(tau, np.linalg.solve(H, -grad), rtol=1e-6, atol=1e-10)
    assert abs(cost - ctx.backend_cost(G, p)) <= 1e-12 * cost


def test_prepared_graph_matches_stateless_entry_points(ctx):
    # pmx_graph_prepare: staged once, then terms / solve at changing poses
    import torch
    g, G, O = _graph()
    p = _params()
    pg = ctx.prepare_graph(G, p)
    t_pg = pg.edge_terms(G.poses).cpu().numpy()
    np.testing.assert_allclose(t_pg, ctx.backend_edge_terms(G, p), rtol=0, atol=0)
    tau, cost, solved = pg.solve(G.poses, torch.from_numpy(t_pg).cuda())
    tau_ref, cost_ref, solved_ref = ctx.backend_solve_terms(G, t_pg, p)
    assert solved and solved_ref and cost == cost_ref
    np.testing.assert_allclose(tau.cpu().numpy(), tau_ref, rtol=1e-9, atol=1e-12)
    # a sub-range of edges only stages / compacts its own edges
    half = len(g["edges"]) // 2
    pg2 = ctx.prepare_graph(G, p, half, len(g["edges"]))
    np.testing.assert_array_equal(pg2.edge_terms(G.poses).cpu().numpy(), t_pg[half:])
    pg.release()
    pg2.release()


def test_sharded_driver_single_rank_nccl_matches_global_optimize(ctx):
    # the edge-sharded loop (distributed.py) on one rank over NCCL, with the
    # prepared-graph callbacks, converges to the device loop's poses
    import os
    import torch
    import torch.distributed as dist
    from paper_2412_12392_b200 import distributed
    g, G, O = _graph(n_kf=10, reach=3)
    p = _params()
    init = [abi.pmx_sim3.from_buffer_copy(T) for T in G.poses]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        terms_fn, solve_fn, cost_fn, pg = distributed.gpu_prepared_callbacks(ctx, G, p, 0, len(g["edges"]))
        res = distributed.global_optimize_sharded(init, len(g["edges"]), 0, p, terms_fn, solve_fn, cost_fn,
                                                  torch_device=torch.device("cuda", 0))
        pg.release()
    finally:
        dist.destroy_process_group()
    r = ctx.global_optimize(G, p)
    assert res.converged == r.converged
    for a, b in zip(res.poses, G.poses):
        assert np.abs(np.array(a.t[:]) - np.array(b.t[:])).max() < 1e-7
        assert np.abs(np.array(a.R[:]) - np.array(b.R[:])).max() < 1e-7


def test_banded_solver_matches_dense_solve(ctx):
    # a long ring of keyframes takes the banded form of K9 (folded order +
    # block cyclic reduction): its step equals the dense solve of the system
    g, G, O = _graph(n_kf=400, reach=2, h=12, w=16)
    p = _params()
    terms = ctx.backend_edge_terms(G, p)
    tau, cost, solved = ctx.backend_solve_terms(G, terms, p)
    assert solved
    H, grad = ctx.assemble_system(G, p)
    ref = np.linalg.solve(H, -grad)
    np.testing.assert_allclose(tau, ref, rtol=1e-6, atol=1e-9 * np.abs(ref).max())
    r = ctx.global_optimize(G, p)
    assert r.converged and r.iterations >= 1


@pytest.mark.parametrize("n_kf,reach", [(20, 4), (400, 2)])
def test_graph_loop_equals_enqueued_loop(ctx, n_kf, reach):
    # the GN loop as one CUDA graph (conditional WHILE node, stops on the
    # device) runs exactly the kernels of the enqueued loop: identical poses,
    # iterations and cost trace, for the frontal (20 kf) and banded (400 kf) solvers
    h, w = (48, 64) if n_kf < 100 else (12, 16)
    p = _params()
    p.damping_retries = 3
    out = []
    for graphs in (True, False):
        ctx.set_device_graphs(graphs)
        _, G, _ = _graph(n_kf=n_kf, reach=reach, h=h, w=w)
        r = ctx.global_optimize(G, p, trace=True)
        out.append((r, [(list(P.R), list(P.t), P.s) for P in G.poses]))
    ctx.set_device_graphs(True)
    (ra, pa), (rb, pb) = out
    assert ra.iterations == rb.iterations and ra.converged == rb.converged
    assert list(ra.cost_trace) == list(rb.cost_trace)
    assert pa == pb
    if n_kf < 100:
        assert ra.iterations < p.max_iterations  # converged before the cap: the graph stopped early


@pytest.mark.parametrize("n_kf,reach,h,w", [(8, 2, 48, 64), (400, 2, 12, 16)])
def test_damping_retry_on_zero_pivot(ctx, n_kf, reach, h, w):
    # a keyframe whose edges carry no valid match has an all-zero 7x7 block:
    # the undamped factorisation meets an exact zero pivot and fails, the
    # retry with lambda = damping_init on every diagonal succeeds
    # (backend.cpp:208-227) - frontal (8 kf) and banded (400 kf) solvers
    g = pmxgen.backend_graph(n_kf, reach, 3, height=h, width=w, radius=1.0)
    lone = n_kf // 2
    ms, oms = [], []
    for (i, j), m in zip(g["edges"], g["matches"]):
        valid = np.zeros_like(m["valid"]) if lone in (i, j) else m["valid"]
        ms.append(MatchSet(m["pixel_a"], m["confidence"], valid))
        oms.append(pyoracle.MatchSet(m["pixel_a"], np.arange(h * w), m["confidence"].astype(np.float64), valid))
    poses = [T.to_struct(abi.pmx_sim3) for T in g["init"]]
    G = Graph([Pointmap(x, v, h, w) for x, v in g["canonicals"]], poses, g["edges"], ms, anchor=0)
    p = _params()
    p.max_iterations = 2
    terms = ctx.backend_edge_terms(G, p)
    tau, cost, solved = ctx.backend_solve_terms(G, terms, p)
    assert solved
    np.testing.assert_array_equal(tau[7 * lone:7 * lone + 7], 0.0)  # g = 0 on the lone keyframe
    r = ctx.global_optimize(G, p)
    assert r.iterations >= 1
    if n_kf < 100:  # the oracle at the small size: same retry semantics, same poses
        O = pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"], oms, h, w)
        pyoracle.global_optimize(O, p)
        for a, b in zip(G.poses, O.poses):
            et, er = _pose_err(a, b)
            assert et < 1e-5 and er < 1e-5, (et, er)
    assert list(G.poses[lone].t) == list(g["init"][lone].to_struct(abi.pmx_sim3).t) or \
        np.abs(np.array(G.poses[lone].t[:]) - g["init"][lone].t).max() < 1e-12


@pytest.mark.parametrize("graphs", [True, False])
def test_zero_iterations_leaves_poses(ctx, graphs):
    # max_iterations = 0: the initial cost only, poses untouched (no loop graph is built)
    ctx.set_device_graphs(graphs)
    try:
        g, G, O = _graph(n_kf=8, reach=2)
        p = _params()
        p.max_iterations = 0
        before = [(list(P.R), list(P.t), P.s) for P in G.poses]
        r = ctx.global_optimize(G, p)
        assert r.iterations == 0
        assert [(list(P.R), list(P.t), P.s) for P in G.poses] == before
        assert len(r.cost_trace) == 1 and r.cost_trace[0] > 0
    finally:
        ctx.set_device_graphs(True)


@pytest.mark.parametrize("with_nccl", [False, True])
def test_device_sharded_loop_single_rank(with_nccl):
    """pmx_graph_optimize_sharded (the device-resident edge-sharded GN loop)
    on one rank, with and without an NCCL communicator (reduce / broadcast
    on one rank), equals global_optimize: same iterations, cost trace and
    bit-identical poses."""
    from paper_2412_12392_b200 import Context
    from paper_2412_12392_b200.distributed import device_sharded_optimize
    c = Context(0)
    try:
        if with_nccl:
            c.nccl_init(c.nccl_unique_id(), 0, 1)
        g, G, O = _graph(n_kf=20, reach=4)
        p = _params()
        p.max_iterations = 10
        ref = Graph(G.canonicals, list(G.poses), G.edges, G.matches, anchor=0)
        rr = c.global_optimize(ref, p, trace=True)
        rs, poses, tm, pg = device_sharded_optimize(c, G, p, 0, 1, trace=True)
        pg.release()
        assert rs.iterations == rr.iterations and rs.converged == rr.converged
        np.testing.assert_array_equal(rs.cost_trace, rr.cost_trace)
        for a, b in zip(poses, ref.poses):
            assert list(a.R) == list(b.R) and list(a.t) == list(b.t) and a.s == b.s
        assert len(rs.pose_trace) == len(rr.pose_trace)
        assert tm["accumulate"] > 0 and tm["solve"] > 0 and (tm["communication"] > 0) == with_nccl
    finally:
        c.close()
