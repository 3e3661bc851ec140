"""Diagnose GPU-vs-oracle drift on the small backend golden fixture:
per max_iterations final-pose diff, cost traces, and relative error of the
per-edge terms at the initial state."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import pyoracle
from paper_2412_12392_b200 import Context, Graph, MatchSet, Pointmap, abi
from test_golden import _graph_parts, load

z = load("backend_6kf_24x32.npz")
h, w, poses, cans, edges, ms = _graph_parts(z)
ctx = Context(0)
for it in range(1, 11):
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = it
    G = Graph([Pointmap(c, None, h, w) for c in cans], list(poses), edges, [MatchSet(pa, q, v) for pa, q, v in ms])
    r = ctx.global_optimize(G, p)
    O = pyoracle.Graph([(c, None) for c in cans], list(poses), edges,
                       [pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v) for pa, q, v in ms], h, w)
    ro, _ = pyoracle.global_optimize(O, p)
    fg = np.array([list(T.R) + list(T.t) + [T.s] for T in G.poses])
    fo = np.array([list(T.R) + list(T.t) + [T.s] for T in O.poses])
    print(f"maxit {it}: gpu it {r.iterations} conv {r.converged} | oracle it {ro.iterations} conv {ro.converged} | "
          f"dt {np.abs(fg[:, 9:12] - fo[:, 9:12]).max():.3e} dR {np.abs(fg[:, :9] - fo[:, :9]).max():.3e}")
    print("   cost gpu", list(r.cost_trace)[:12])
    print("   cost orc", list(ro.cost_trace)[:12])
p = abi.default_backend_params()
p.weights.distance_weight = 0.1
G = Graph([Pointmap(c, None, h, w) for c in cans], list(poses), edges, [MatchSet(pa, q, v) for pa, q, v in ms])
O = pyoracle.Graph([(c, None) for c in cans], list(poses), edges,
                   [pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v) for pa, q, v in ms], h, w)
tg = np.asarray(ctx.backend_edge_terms(G, p))
to = np.asarray(pyoracle.backend_edge_terms(O, p))
print("terms shape", tg.shape, to.shape)
rel = np.abs(tg - to) / (np.abs(to).max(axis=1, keepdims=True) + 1e-300)
print("max rel err per edge (vs edge max |term|)", rel.max(axis=1))
