"""Generates tests/golden/*.npz: small seeded BASELINE-shaped cases.

Matching and backend outputs come from the GENUINE reference sources
(oracle/_ref/libpmslam_ref.so: /root/reference/proj/src/*.cpp compiled
against the Eigen-API shim) when that build exists, else from the FP64
restatement; tests/test_ref_pins.py checks that both produce these fixtures
bit for bit (matching) / within 1e-10 (backend).  The track fixture is the
restatement's match-given GN (the reference has no such entry; its
residuals are pinned to the reference in test_ref_pins).
Regenerate with:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "gen"), os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import pmxgen  # noqa: E402
import pyoracle  # noqa: E402
from helpers import BASELINE_REFINE, baseline_match_params  # noqa: E402
from paper_2412_12392_b200 import abi  # noqa: E402


def match_case(name, seed, h, w, noise):
    p = pmxgen.config0(seed=seed, height=h, width=w, noise=noise)
    mp = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    m = pyoracle.match_pointmaps(p, mp)
    r = pyoracle.feature_refine(m, p, rp)
    np.savez_compressed(os.path.join(HERE, name), X_a=p["X_a"], X_b=p["X_b"], Q_a=p["Q_a"], Q_b=p["Q_b"],
                        D_a=p["D_a"], D_b=p["D_b"], valid_a=p["valid_a"], valid_b=p["valid_b"],
                        lm_pixel_a=m.pixel_a, lm_valid=m.valid, pixel_a=r.pixel_a, valid=r.valid,
                        confidence=r.confidence, shape=np.array([h, w]))


def track_case(name, seed, h, w):
    c = pmxgen.config1(seed=seed, height=h, width=w)
    pair = {"X_a": c["X_f_f"], "valid_a": c["valid_f"], "Q_a": c["C_f"], "D_a": c["D_f"],
            "X_b": c["X_k_f"], "valid_b": c["valid_k"], "Q_b": c["C_k"], "D_b": c["D_k"], "height": h, "width": w}
    m = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, baseline_match_params()), pair,
                                abi.refine_params(BASELINE_REFINE))
    pa, v = pmxgen.inject_outliers(m.pixel_a, m.valid, 0.1, seed, h * w)
    q = np.sqrt(c["C_f"][np.clip(pa, 0, None)].astype(np.float64) * c["C_k"].astype(np.float64)).astype(np.float32)
    p = abi.default_solve_pose_params()
    p.max_iterations = 10
    p.weights.distance_weight = 0.1
    om = pyoracle.MatchSet(pa, np.arange(h * w), q.astype(np.float64), v)
    T0 = pmxgen.Pose().to_struct(abi.pmx_sim3)
    r = pyoracle.track_given_matches(c["canonical"], c["canonical_valid"], c["X_f_f"], c["valid_f"], h, w, om, T0,
                                     params=p)
    np.savez_compressed(os.path.join(HERE, name), canonical=c["canonical"], canonical_valid=c["canonical_valid"],
                        X_f_f=c["X_f_f"], valid_f=c["valid_f"], pixel_a=pa, valid=v, confidence=q,
                        R=np.array(r.T_kf.R[:]), t=np.array(r.T_kf.t[:]), s=np.array([r.T_kf.s]),
                        iterations=np.array([r.iterations]), cost_trace=np.array(r.cost_trace[:r.cost_trace_len]),
                        shape=np.array([h, w]))


def backend_case(name, seed, n_kf, reach, h, w):
    g = pmxgen.backend_graph(n_kf, reach, seed, height=h, width=w, radius=1.0)
    O = pyoracle.Graph(g["canonicals"], [T.to_struct(abi.pmx_sim3) for T in g["init"]], g["edges"],
                       [pyoracle.MatchSet(m["pixel_a"], np.arange(h * w), m["confidence"].astype(np.float64),
                                          m["valid"]) for m in g["matches"]], h, w)
    p = abi.default_backend_params()
    p.weights.distance_weight = 0.1
    res, _ = pyoracle.global_optimize(O, p)
    arrays = {}
    for k, (x, v) in enumerate(g["canonicals"]):
        arrays[f"can{k}"] = x
    for e, m in enumerate(g["matches"]):
        arrays[f"pa{e}"] = m["pixel_a"]
        arrays[f"q{e}"] = m["confidence"]
        arrays[f"v{e}"] = m["valid"]
    init = np.array([list(T.R.ravel()) + list(T.t) + [T.s] for T in g["init"]])
    final = np.array([list(T.R) + list(T.t) + [T.s] for T in O.poses])
    np.savez_compressed(os.path.join(HERE, name), edges=np.array(g["edges"]), init=init, final=final,
                        iterations=np.array([res.iterations]), converged=np.array([res.converged]),
                        cost_trace=np.array(res.cost_trace[:res.cost_trace_len]), shape=np.array([h, w]), **arrays)


if __name__ == "__main__":
    import contextlib
    src = pyoracle.reference() if pyoracle.have_reference() else contextlib.nullcontext()
    with src:
        match_case("match_radial_48x64.npz", 21, 48, 64, "radial")
        match_case("match_isotropic_48x64.npz", 22, 48, 64, "isotropic")
        backend_case("backend_6kf_24x32.npz", 24, 6, 2, 24, 32)
    track_case("track_48x64.npz", 23, 48, 64)
    print("golden fixtures written to", HERE, "(reference build)" if pyoracle.have_reference() else "(restatement)")
