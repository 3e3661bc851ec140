"""Small, fixed workloads for `ncu --set full` captures (dev tool).

python tools/ncu_target.py match [edges]   -> 2 match_batch calls over config-2 edges
python tools/ncu_target.py backend [kf]    -> 2 GN iterations of a config-3-shaped graph
python tools/ncu_target.py all             -> every hot kernel once or twice: matching (5 config-2
                                              edges), tracking + fusion (config 1), backend config 3
                                              (matcher-built matches, frontal solver), banded solver
                                              (N = 1000 topology)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen")]

import torch  # noqa: E402

import pmxgen  # noqa: E402
from paper_2412_12392_b200 import Context, FeatureMap, Graph, MatchSet, Pointmap, abi  # noqa: E402

H, W = 384, 512
dev = torch.device("cuda")


def T(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)


mode = sys.argv[1]
ctx = Context(0)
if mode == "all":
    sys.path[:0] = [os.path.join(ROOT, "oracle")]
    from paper_2412_12392_b200 import sim3
    # matching
    sc, poses, edges, mk = pmxgen.config2(seed=2)
    pairs = []
    for e in range(5):
        p = mk(e)
        pairs.append((Pointmap(T(p["X_a"]), T(p["valid_a"]), H, W), Pointmap(T(p["X_b"]), T(p["valid_b"]), H, W),
                      FeatureMap(T(p["D_a"]), T(p["Q_a"]), H, W), FeatureMap(T(p["D_b"]), T(p["Q_b"]), H, W)))
    mp = abi.default_match_params()
    mp.projection.lambda_init = 1e-8
    mp.projection.angle_tol = 1e-6
    rp = abi.refine_params([(1, 3), (1, 3)])
    outs = [MatchSet.empty(H * W, dev) for _ in range(5)]
    for _ in range(2):
        ctx.match_batch(pairs, params=mp, refine=rp, outs=outs)
    # tracking + fusion (config 1)
    c = pmxgen.config1(seed=1)
    pr = (Pointmap(T(c["X_f_f"]), T(c["valid_f"]), H, W), Pointmap(T(c["X_k_f"]), T(c["valid_k"]), H, W),
          FeatureMap(T(c["D_f"]), T(c["C_f"]), H, W), FeatureMap(T(c["D_k"]), T(c["C_k"]), H, W))
    m = ctx.match_batch([pr], params=mp, refine=rp)[0]
    tp = abi.default_solve_pose_params()
    tp.max_iterations = 10
    tp.weights.distance_weight = 0.1
    can = Pointmap(T(c["canonical"]), T(c["canonical_valid"]), H, W)
    r = ctx.track_given_matches(can, pr[0], m, sim3(), params=tp)
    cx, cv, cc = T(c["canonical"]).clone(), T(c["canonical_valid"]).clone(), T(c["canonical_conf"]).clone()
    ctx.fuse_canonical(cx, cv, cc, pr[1], T(c["C_k"]), r.T_kf, H, W)
    # backend config 3 (matcher-built matches), 3 iterations (frontal solver);
    # enqueued kernel by kernel (ncu does not profile kernels of conditional graphs)
    g = pmxgen.backend_graph_matched(ctx, 100, 4, 3)
    ctx.set_device_graphs(False)
    cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
    bp = abi.default_backend_params()
    bp.weights.distance_weight = 0.1
    bp.max_iterations = 3
    ctx.global_optimize(Graph(cans, [P.to_struct(abi.pmx_sim3) for P in g["init"]], g["edges"], g["matches"]), bp)
    del cans, g
    # banded solver: the N = 1000 topology, matches on a few edges only
    g = pmxgen.backend_graph(1000, 5, 3, height=48, width=64, loops=3, edge_range=(0, 40))
    cans = [Pointmap(T(x), T(v), 48, 64) for x, v in g["canonicals"]]
    ms = [MatchSet(T(mm["pixel_a"]), T(mm["confidence"]), T(mm["valid"])) for mm in g["matches"]]
    bp.max_iterations = 1
    ctx.global_optimize(Graph(cans, [P.to_struct(abi.pmx_sim3) for P in g["init"]], g["edges"], ms), bp)
    torch.cuda.synchronize()
    print("all ok")
elif mode == "match":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    sc, poses, edges, mk = pmxgen.config2(seed=2)
    pairs = []
    for e in range(n):
        p = mk(e)
        pairs.append((Pointmap(T(p["X_a"]), T(p["valid_a"]), H, W), Pointmap(T(p["X_b"]), T(p["valid_b"]), H, W),
                      FeatureMap(T(p["D_a"]), T(p["Q_a"]), H, W), FeatureMap(T(p["D_b"]), T(p["Q_b"]), H, W)))
    mp = abi.default_match_params()
    mp.projection.lambda_init = 1e-8
    mp.projection.angle_tol = 1e-6
    rp = abi.refine_params([(1, 3), (1, 3)])
    outs = [MatchSet.empty(H * W, dev) for _ in range(n)]
    for _ in range(2):
        ctx.match_batch(pairs, params=mp, refine=rp, outs=outs)
    torch.cuda.synchronize()
    print("valid", float(np.mean([o.valid.float().mean().item() for o in outs])))
else:
    kf = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    ctx.set_device_graphs(False)  # kernels enqueued one by one (the conditional-graph loop hides them from -k)
    g = pmxgen.backend_graph(kf, 4, 3)
    cans = [Pointmap(T(x), T(v), H, W) for x, v in g["canonicals"]]
    ms = [MatchSet(T(m["pixel_a"]), T(m["confidence"]), T(m["valid"])) for m in g["matches"]]
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    p.max_iterations = 2
    init = [P.to_struct(abi.pmx_sim3) for P in g["init"]]
    r = ctx.global_optimize(Graph(cans, list(init), g["edges"], ms), p)
    torch.cuda.synchronize()
    print("iterations", r.iterations)
