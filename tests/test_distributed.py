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
from helpers import numpy_solve
from paper_2412_12392_b200.distributed import global_optimize_sharded, shard_range

H, W = 24, 32


def make_graph():
    g = pmxgen.backend_graph(8, 2, 5, height=H, width=W, radius=1.0)
    return pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"],
                          [pyoracle.MatchSet(m["pixel_a"], np.arange(H * W), m["confidence"].astype(np.float64),
                                             m["valid"]) for m in g["matches"]], H, W)


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


def _match_worker(rank, world, port, q):
    """One rank of the edge-sharded batched matcher (bench.py's config-2
    path): its contiguous edge shard, matched by the CPU oracle here (the
    checker; the GPU runs the same shard through libpmx_cuda.so), gathered
    to rank 0 with the edge ids."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import BASELINE_REFINE, baseline_match_params
    n_edges = 7
    pairs = [pmxgen.config0(seed=40 + e, height=24, width=32) for e in range(n_edges)]
    e0, e1 = shard_range(n_edges, rank, world)
    mine = pyoracle.match_batch(pairs[e0:e1], baseline_match_params(), abi.refine_params(BASELINE_REFINE))
    payload = [(e0 + k, m.pixel_a.tolist(), m.valid.tolist()) for k, m in enumerate(mine)]
    out = [None] * world
    dist.all_gather_object(out, payload)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_matching_shards_cover_every_edge_once(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_match_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = sorted(e for shard in out for e, _, _ in shard)
    assert got == list(range(7))  # every edge exactly once
    from helpers import BASELINE_REFINE, baseline_match_params
    pairs = [pmxgen.config0(seed=40 + e, height=24, width=32) for e in range(7)]
    ref = pyoracle.match_batch(pairs, baseline_match_params(), abi.refine_params(BASELINE_REFINE))
    for shard in out:
        for e, pa, v in shard:  # reassembled in edge order = the single-process batch
            assert np.array_equal(np.array(pa, np.int32), ref[e].pixel_a) and np.array_equal(np.array(v), ref[e].valid)
