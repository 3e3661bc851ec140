"""World-size-2 gloo test of the edge-sharded backend driver
(paper_2412_12392_b200/distributed.py) on CPU: the per-edge terms come from
the oracle (test-only), the solve is a numpy restatement of K8/K9; the
sharded result must equal the oracle's single-process global_optimize."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import pmxgen
import pyoracle
from paper_2412_12392_b200 import abi
from paper_2412_12392_b200.distributed import global_optimize_sharded, shard_range

H, W = 24, 32


def make_graph():
    g = pmxgen.backend_graph(8, 2, 5, height=H, width=W, radius=1.0)
    return pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"],
                          [pyoracle.MatchSet(m["pixel_a"], np.arange(H * W), m["confidence"].astype(np.float64),
                                             m["valid"]) for m in g["matches"]], H, W)


def numpy_solve(graph, params):
    """Rank-0 solve from per-edge terms: adjoint sandwich (backend.cpp:114-141),
    gauge (144-155), damping retries (208-230) with the oracle's LDL^T."""
    def solve(terms, P):
        t = np.asarray(terms)
        n = len(P)
        dim = 7 * n
        Hm = np.zeros((dim, dim))
        gv = np.zeros(dim)
        iu = np.triu_indices(7)
        adj = [pyoracle.sim3_adjoint(pyoracle.sim3_inverse(T)) for T in P]
        for e, (i, j) in enumerate(graph.edges):
            H1 = np.zeros((7, 7)); H1[iu] = t[e, :28]; H1 = H1 + np.triu(H1, 1).T
            H2 = np.zeros((7, 7)); H2[iu] = t[e, 36:64]; H2 = H2 + np.triu(H2, 1).T
            S = adj[i].T @ H1 @ adj[i] + adj[j].T @ H2 @ adj[j]
            g = -adj[i].T @ t[e, 28:35] + adj[j].T @ t[e, 64:71]
            for (a, b, sg) in ((i, i, 1), (i, j, -1), (j, i, -1), (j, j, 1)):
                Hm[7 * a:7 * a + 7, 7 * b:7 * b + 7] += sg * S
            gv[7 * i:7 * i + 7] += g
            gv[7 * j:7 * j + 7] -= g
        a = graph.anchor
        Hm[7 * a:7 * a + 7, :] = 0
        Hm[:, 7 * a:7 * a + 7] = 0
        Hm[7 * a:7 * a + 7, 7 * a:7 * a + 7] = np.eye(7)
        gv[7 * a:7 * a + 7] = 0
        lam = 0.0
        for _ in range(params.damping_retries + 1):
            x, ok = pyoracle.ldlt_solve(Hm + lam * np.eye(dim), -gv)
            if ok and np.isfinite(x).all() and np.abs(x).max() < 1e3:
                return x, True
            lam = params.damping_init if lam == 0.0 else lam * 10
        return np.zeros(dim), False
    return solve


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = make_graph()
    params = abi.default_backend_params()
    params.weights.distance_weight = 0.1

    def terms_fn(e0, e1, P):
        g.poses = list(P)
        return pyoracle.backend_edge_terms(g, params, e0, e1)

    def cost_fn(terms):
        t = np.asarray(terms)
        return float(sum(t[e, 35] + t[e, 71] for e in range(t.shape[0])))

    res = global_optimize_sharded(list(g.poses), len(g.edges), 0, params, terms_fn, numpy_solve(g, params), cost_fn)
    if rank == 0:
        q.put((res.iterations, res.converged, res.cost_trace,
               [(list(T.R), list(T.t), T.s) for T in res.poses]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 5000):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world) for r in range(world)]
            covered = [e for a, b in got for e in range(a, b)]
            assert covered == list(range(n))


def test_sharded_backend_equals_single_process_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    it, conv, trace, poses = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = make_graph()
    params = abi.default_backend_params()
    params.weights.distance_weight = 0.1
    ro, _ = pyoracle.global_optimize(g, params)
    assert conv == bool(ro.converged) and it == ro.iterations
    np.testing.assert_allclose(trace, list(ro.cost_trace[:ro.cost_trace_len]), rtol=1e-9)
    for (R, t, s), T in zip(poses, g.poses):
        np.testing.assert_allclose(R, list(T.R), atol=1e-9)
        np.testing.assert_allclose(t, list(T.t), atol=1e-9)
        assert abs(s - T.s) < 1e-9
