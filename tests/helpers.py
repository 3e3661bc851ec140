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
