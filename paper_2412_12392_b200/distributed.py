"""Edge-sharded multi-GPU paths (one process per GPU, torch.distributed).

Batched matching shards by graph edge with no data-path collective
(``shard_range``).  The backend (reference src/backend.cpp:192-256) shards
the per-edge normal-equation accumulation (K7, the HBM-bound part) by edge:

  every rank:  terms[e0:e1] = relative-frame {H, g, cost} of its edges
  reduce    :  one sum-reduce of the zero-padded E x 72 FP64 buffer to rank 0
               (NCCL over NVLink; gloo in the CPU tests)
  rank 0    :  cost, adjoint sandwich + dense 7N x 7N assembly + gauge, damped
               LDL^T solve (K8/K9)
  broadcast :  {solved, accept/stop, tau (7N)}; all ranks retract the
               replicated FP64 poses with the same host routine.

Each Gauss-Newton iteration is exactly one reduce + one broadcast: the terms
evaluated at the trial poses give both the accept test and, if accepted, the
next iteration's system (the reference evaluates residuals twice).

The compute callbacks are pluggable so the control flow is testable on CPU
(tests/test_distributed.py drives it with the oracle over gloo); on GPUs
``gpu_callbacks`` binds them to libpmx_cuda.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Sequence

import numpy as np

from . import abi

TERMS = abi.PMX_EDGE_TERMS


def shard_range(n: int, rank: int, world: int):
    """Contiguous block of [0, n) owned by `rank` (edges of batched matching / backend)."""
    per = (n + world - 1) // world
    return min(n, rank * per), min(n, (rank + 1) * per)


def retract(T: abi.pmx_sim3, tau7: np.ndarray) -> abi.pmx_sim3:
    """Exp(tau) * T in FP64 via the library's host routine (identical on every rank)."""
    lib = abi.load_library()
    out = abi.pmx_sim3()
    t = np.ascontiguousarray(tau7, np.float64)
    lib.pmx_sim3_retract(C.byref(T), abi.ptr(t), C.byref(out))
    return out


@dataclass
class ShardedResult:
    iterations: int = 0
    converged: bool = False
    cost_trace: List[float] = field(default_factory=list)
    poses: list = field(default_factory=list)
    # poses after every iteration (the reverted ones for a rejected step), as
    # pmx_global_optimize's pose_trace
    pose_trace: list = field(default_factory=list)


def global_optimize_sharded(poses: Sequence, num_edges: int, anchor: int, params: abi.pmx_backend_params,
                            terms_fn: Callable, solve_fn: Callable, cost_fn: Callable, torch_device=None,
                            group=None, timers: dict | None = None) -> ShardedResult:
    """global_optimize (backend.cpp:192-256) with edge-sharded accumulation.

    terms_fn(e0, e1, poses) -> (e1-e0, 72) FP64 tensor/array of this rank's edges
    solve_fn(terms, poses)  -> (tau[7N] np.ndarray, solved: bool)      (rank 0)
    cost_fn(terms)          -> float, directed-constraint costs summed in edge order (rank 0)
    timers                  -> optional dict accumulating seconds per phase ("accumulate",
                               "communication", "solve"), device-synchronised at phase ends
    """
    import time as _time
    import torch
    import torch.distributed as dist

    single = not (dist.is_available() and dist.is_initialized())  # one process: no collectives
    rank, world = (0, 1) if single else (dist.get_rank(group), dist.get_world_size(group))
    n = len(poses)
    P = [abi.pmx_sim3.from_buffer_copy(T) for T in poses]
    res = ShardedResult(poses=P)
    if n < 2 or num_edges == 0:  # backend.cpp:195-198
        res.converged = True
        return res
    dev = torch_device if torch_device is not None else torch.device("cpu")
    e0, e1 = shard_range(num_edges, rank, world)

    def sync():
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)

    def tick(phase, t0):
        if timers is not None:
            sync()
            timers[phase] = timers.get(phase, 0.0) + _time.perf_counter() - t0
        return _time.perf_counter()

    def reduce_terms(P):
        t0 = _time.perf_counter()
        full = torch.zeros((num_edges, TERMS), dtype=torch.float64, device=dev)
        if e1 > e0:
            local = terms_fn(e0, e1, P)
            full[e0:e1] = torch.as_tensor(local, dtype=torch.float64, device=dev)
        t0 = tick("accumulate", t0)
        if not single:
            dist.reduce(full, dst=0, group=group)
        tick("communication", t0)
        return full

    def bcast(vec: np.ndarray) -> np.ndarray:
        t0 = _time.perf_counter()
        t = torch.as_tensor(vec, dtype=torch.float64, device=dev).clone()
        if not single:
            dist.broadcast(t, src=0, group=group)
        out = t.cpu().numpy()
        tick("communication", t0)
        return out

    terms = reduce_terms(P)
    cost = cost_fn(terms) if rank == 0 else 0.0
    res.cost_trace.append(cost)
    for it in range(params.max_iterations):
        res.iterations += 1
        msg = np.zeros(1 + 7 * n)
        if rank == 0:
            t0 = _time.perf_counter()
            tau, solved = solve_fn(terms, P)
            tick("solve", t0)
            msg[0] = 1.0 if solved else 0.0
            msg[1:] = tau
        msg = bcast(msg)
        if msg[0] == 0.0:  # state intact, not converged (backend.cpp:228-230)
            res.poses = P
            return res
        tau = msg[1:]
        previous = P
        P = [T if k == anchor else retract(T, tau[7 * k:7 * k + 7]) for k, T in enumerate(P)]
        terms_new = reduce_terms(P)
        flag = np.zeros(2)
        if rank == 0:
            cost_new = cost_fn(terms_new)
            flag[0] = 0.0 if cost_new > cost * (1.0 + 1e-12) + 1e-300 else 1.0
            flag[1] = cost_new
        flag = bcast(flag)
        if flag[0] == 0.0:  # revert (backend.cpp:242-246)
            P = previous
            res.pose_trace.append(list(P))
            break
        res.pose_trace.append(list(P))
        cost = flag[1]
        terms = terms_new
        res.cost_trace.append(cost)
        if float(np.sqrt((tau ** 2).sum())) < params.update_tol:
            break
    res.converged = True
    res.poses = P
    return res


def gpu_callbacks(ctx, graph, params):
    """Bind the sharded driver to libpmx_cuda.so for a device-resident Graph."""
    import torch

    def terms_fn(e0, e1, P):
        graph.poses = list(P)
        return ctx.backend_edge_terms(graph, params, e0, e1)

    def solve_fn(terms, P):
        graph.poses = list(P)
        tau, _cost, solved = ctx.backend_solve_terms(graph, terms, params)
        return (tau.cpu().numpy() if isinstance(tau, torch.Tensor) else tau), solved

    def cost_fn(terms):
        t = terms.detach().cpu().numpy() if isinstance(terms, torch.Tensor) else np.asarray(terms)
        c = 0.0
        for e in range(t.shape[0]):  # directed-constraint order of backend.cpp:179-188
            c += t[e, 35]
            c += t[e, 71]
        return c

    return terms_fn, solve_fn, cost_fn


def gpu_prepared_callbacks(ctx, graph, params, begin: int, end: int, rank: int = 0):
    """Bind the sharded driver to a prepared graph (pmx_graph_prepare): the
    rank's edges [begin, end) are staged and compacted once; every iteration
    is then edge terms on the device -> NCCL reduce -> rank 0 solve on the
    device (frontal plan built once) -> broadcast, with no re-staging.
    Rank 0 needs the full topology (all edges, any match sets)."""
    pg = ctx.prepare_graph(graph, params, begin, end)

    def terms_fn(e0, e1, P):
        assert (e0, e1) == (begin, end), "prepared range mismatch"
        return pg.edge_terms(list(P))

    def solve_fn(terms, P):
        tau, _cost, solved = pg.solve(list(P), terms.contiguous())
        return tau.cpu().numpy(), solved

    def cost_fn(terms):
        t = terms.detach().cpu().numpy()
        return float(np.sum(t[:, 35]) + np.sum(t[:, 71])) if t.size else 0.0

    return terms_fn, solve_fn, cost_fn, pg


def device_sharded_optimize(ctx, graph, params, rank: int, world: int, trace: bool = False):
    """The edge-sharded backend as one device-resident loop per rank
    (pmx_graph_optimize_sharded): the context's NCCL communicator is created
    from a unique id broadcast over torch.distributed, each rank prepares
    its contiguous edge shard, and every GN iteration runs on the device
    (reduce of the terms to rank 0, solve on rank 0, broadcasts of state and
    tau) with no host round trip.  Returns (OptimizeResult, poses, timings,
    prepared graph)."""
    import torch.distributed as dist
    if world > 1:
        uid = [ctx.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], rank, world)
    e0, e1 = shard_range(len(graph.edges), rank, world)
    pg = ctx.prepare_graph(graph, params, e0, e1)
    res, poses, timings = pg.optimize_sharded(list(graph.poses), params, trace=trace)
    return res, poses, timings, pg
