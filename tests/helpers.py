"""Shared test helpers: build pair / graph structures for both the CUDA path
(paper_2412_12392_b200) and the oracle (oracle/pyoracle.py, test-only)."""
from __future__ import annotations

import numpy as np

from paper_2412_12392_b200 import FeatureMap, MatchSet, Pointmap, abi

BASELINE_LM = dict(lambda_init=1e-8, angle_tol=1e-6)  # BASELINE config 0 schedule
BASELINE_REFINE = [(1, 3), (1, 3)]                    # "radius-3 window, 2 refine steps"


def baseline_match_params():
    p = abi.default_match_params()
    p.projection.lambda_init = BASELINE_LM["lambda_init"]
    p.projection.angle_tol = BASELINE_LM["angle_tol"]
    return p


def pmx_pair(pair):
    h, w = pair["height"], pair["width"]
    Xa = Pointmap(pair["X_a"], pair.get("valid_a"), h, w)
    Xb = Pointmap(pair["X_b"], pair.get("valid_b"), h, w)
    Fa = FeatureMap(pair["D_a"], pair["Q_a"], h, w)
    Fb = FeatureMap(pair["D_b"], pair["Q_b"], h, w)
    return Xa, Xb, Fa, Fb


def to_torch_pair(pair, device="cuda"):
    import torch
    out = dict(pair)
    for k in ("X_a", "X_b", "Q_a", "Q_b", "valid_a", "valid_b"):
        if pair.get(k) is not None:
            out[k] = torch.from_numpy(np.ascontiguousarray(pair[k])).to(device)
    for k in ("D_a", "D_b"):
        out[k] = torch.from_numpy(np.ascontiguousarray(pair[k]).view(np.int16)).to(device)
    return out


def compare_matches(gpu: MatchSet, orc, width: int):
    """Parity statistics of a GPU MatchSet against an oracle MatchSet."""
    ga = np.asarray(gpu.pixel_a)
    gv = np.asarray(gpu.valid).astype(bool)
    oa = orc.pixel_a
    ov = orc.valid.astype(bool)
    both = gv & ov
    eq = ga[both] == oa[both]
    du = np.abs(ga[both] % width - oa[both] % width)
    dv = np.abs(ga[both] // width - oa[both] // width)
    worst = int(np.max(np.maximum(du, dv))) if both.any() else 0
    return {
        "n": int(ga.shape[0]),
        "valid_gpu": int(gv.sum()),
        "valid_orc": int(ov.sum()),
        "valid_mismatch": int((gv != ov).sum()),
        "both": int(both.sum()),
        "index_equal_frac": float(eq.mean()) if both.any() else 1.0,
        "worst_px": worst,
        "all_index_equal": bool((ga == oa).all()),
    }


def numpy_solve(graph, params):
    """Rank-0 solve from per-edge terms: adjoint sandwich (backend.cpp:114-141),
    gauge (144-155), damping retries (208-230) with the oracle's LDL^T."""
    import pyoracle  # test-only checker

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


