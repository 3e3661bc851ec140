"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/liborc.so, the FP64 CPU restatement of the reference
hot path (see oracle/oracle.hpp).  Imported only by tests/, by
__graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
``--impl reference`` leg.  The product package never imports this module.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2412_12392_b200 import abi
from paper_2412_12392_b200.abi import ptr

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liborc.so")
# The genuine reference sources (src/{lie,camera,tracking,backend}.cpp)
# compiled against the Eigen-API shim behind the same orc_* ABI
# (oracle/Makefile target `ref`): the pin of the restatement.
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libpmslam_ref.so")
_libs = {}
_active = "restatement"


def have_reference() -> bool:
    """True when oracle/_ref/libpmslam_ref.so was built (it is built from
    /root/reference, and travels to the GPU box with the snapshot)."""
    return os.path.exists(REF_LIB_PATH)


def lib():
    if _active not in _libs:
        if _active == "reference":
            path = REF_LIB_PATH
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} not built (make -C oracle ref, needs /root/reference)")
        else:
            path = LIB_PATH
            if not os.path.exists(path):
                subprocess.check_call(["make", "-s", "-C", _HERE])
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_robust_weight.restype = C.c_double
        L.orc_robust_weight.argtypes = [C.c_double] * 3
        _libs[_active] = L
    return _libs[_active]


@contextlib.contextmanager
def reference():
    """Route every pyoracle call inside the block to the genuine reference
    build (oracle/_ref) instead of the restatement."""
    global _active
    prev, _active = _active, "reference"
    try:
        yield
    finally:
        _active = prev


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _check(code):
    if code != 0:
        raise OracleError(code, lib().orc_last_error().decode())


def _pm(xyz, valid, h, w):
    return abi.pointmap(np.ascontiguousarray(xyz, np.float32), None if valid is None else np.ascontiguousarray(valid, np.uint8), h, w)


def _fm(desc, conf, h, w):
    d = np.ascontiguousarray(desc, np.uint16)
    return abi.featuremap(d, np.ascontiguousarray(conf, np.float32), h, w, d.shape[-1] if d.ndim > 1 else d.size // (h * w))


class MatchSet:
    """Host FP64 MatchSet (reference camera.hpp:80-89), SoA numpy."""

    def __init__(self, pixel_a, pixel_b, confidence, valid):
        self.pixel_a = np.ascontiguousarray(pixel_a, np.int32)
        self.pixel_b = np.ascontiguousarray(pixel_b, np.int32)
        self.confidence = np.ascontiguousarray(confidence, np.float64)
        self.valid = np.ascontiguousarray(valid, np.uint8)

    @staticmethod
    def empty(n):
        return MatchSet(np.full(n, -1, np.int32), np.full(n, -1, np.int32), np.zeros(n), np.zeros(n, np.uint8))

    def struct(self):
        return abi.matchset(self.pixel_a, self.pixel_b, self.confidence, self.valid,
                            cls=abi.orc_matchset)

    def __len__(self):
        return self.pixel_a.shape[0]


def normalize_rays(xyz, valid, h, w):
    n = h * w
    rays = np.empty((n, 3)); dist = np.empty(n); v = np.empty(n, np.uint8)
    pm = _pm(xyz, valid, h, w)
    _check(lib().orc_normalize_rays(C.byref(pm), ptr(rays), ptr(dist), ptr(v)))
    return rays, dist, v


def interpolate_ray(xyz, valid, h, w, p):
    p = np.ascontiguousarray(p, np.float64).reshape(-1, 2)
    n = p.shape[0]
    ray = np.empty((n, 3)); J = np.empty((n, 6)); ok = np.empty(n, np.uint8)
    pm = _pm(xyz, valid, h, w)
    _check(lib().orc_interpolate_ray(C.byref(pm), C.c_int64(n), ptr(p), ptr(ray), ptr(J), ptr(ok)))
    return ray, J, ok


def iterative_project(xyz, valid, h, w, x, p0, params=None):
    x = np.ascontiguousarray(x, np.float32).reshape(-1, 3)
    p0 = np.ascontiguousarray(p0, np.float64).reshape(-1, 2)
    n = x.shape[0]
    pix = np.empty((n, 2)); conv = np.empty(n, np.uint8); it = np.empty(n, np.int32)
    pm = _pm(xyz, valid, h, w)
    params = params or abi.default_match_params().projection
    _check(lib().orc_iterative_project(C.byref(pm), C.c_int64(n), ptr(x), ptr(p0), C.byref(params),
                                       ptr(pix), ptr(conv), ptr(it)))
    return pix, conv, it


def median_scene_distance(xyz, valid, h, w):
    out = C.c_double()
    pm = _pm(xyz, valid, h, w)
    _check(lib().orc_median_scene_distance(C.byref(pm), C.byref(out)))
    return out.value


def match_pointmaps(pair, params=None, init: MatchSet | None = None):
    h, w = pair["height"], pair["width"]
    Xa = _pm(pair["X_a"], pair.get("valid_a"), h, w)
    Xb = _pm(pair["X_b"], pair.get("valid_b"), h, w)
    Fa = _fm(pair["D_a"], pair["Q_a"], h, w)
    Fb = _fm(pair["D_b"], pair["Q_b"], h, w)
    out = MatchSet.empty(h * w)
    o = out.struct()
    i = init.struct() if init is not None else None
    params = params or abi.default_match_params()
    _check(lib().orc_match_pointmaps(C.byref(Xa), C.byref(Xb), C.byref(Fa), C.byref(Fb),
                                     C.byref(i) if i is not None else None, C.byref(params), C.byref(o)))
    return out


def feature_refine(m: MatchSet, pair, params=None):
    h, w = pair["height"], pair["width"]
    Fa = _fm(pair["D_a"], pair["Q_a"], h, w)
    Fb = _fm(pair["D_b"], pair["Q_b"], h, w)
    out = MatchSet.empty(len(m))
    o = out.struct(); i = m.struct()
    params = params or abi.default_refine_params()
    _check(lib().orc_feature_refine(C.byref(i), C.byref(Fa), C.byref(Fb), C.byref(params), C.byref(o)))
    return out


def pair_struct(pair, keep):
    h, w = pair["height"], pair["width"]
    arrs = [np.ascontiguousarray(pair["X_a"], np.float32), np.ascontiguousarray(pair["X_b"], np.float32),
            np.ascontiguousarray(pair["D_a"], np.uint16), np.ascontiguousarray(pair["D_b"], np.uint16),
            np.ascontiguousarray(pair["Q_a"], np.float32), np.ascontiguousarray(pair["Q_b"], np.float32)]
    va = pair.get("valid_a"); vb = pair.get("valid_b")
    va = None if va is None else np.ascontiguousarray(va, np.uint8)
    vb = None if vb is None else np.ascontiguousarray(vb, np.uint8)
    keep.extend(arrs + [va, vb])
    d = arrs[2].shape[-1]
    return abi.pmx_pair(abi.pointmap(arrs[0], va, h, w), abi.pointmap(arrs[1], vb, h, w),
                        abi.featuremap(arrs[2], arrs[4], h, w, d), abi.featuremap(arrs[3], arrs[5], h, w, d),
                        None)


def match_batch(pairs, params=None, refine=None, threads=1):
    keep = []
    n = len(pairs)
    arr = (abi.pmx_pair * n)(*[pair_struct(p, keep) for p in pairs])
    outs = [MatchSet.empty(p["height"] * p["width"]) for p in pairs]
    oarr = (abi.orc_matchset * n)(*[o.struct() for o in outs])
    params = params or abi.default_match_params()
    _check(lib().orc_match_batch(C.c_int32(n), arr, None, C.byref(params),
                                 C.byref(refine) if refine is not None else None, oarr, C.c_int32(threads)))
    return outs


def match_stats(m: MatchSet, num_pixels_a):
    vc = C.c_int64(); uf = C.c_double()
    s = m.struct()
    _check(lib().orc_match_stats(C.byref(s), C.c_int32(num_pixels_a), C.byref(vc), C.byref(uf)))
    return vc.value, uf.value


def keyframe_decision(m: MatchSet, h, w, omega):
    out = C.c_int32(); s = m.struct()
    _check(lib().orc_keyframe_decision(C.byref(s), C.c_int32(h), C.c_int32(w), C.c_double(omega), C.byref(out)))
    return bool(out.value)


def residual_blocks(T, m: MatchSet, X_ref, valid_ref, X_src, valid_src, h, w, mode=abi.PMX_TRACK_RAY,
                    params=None, K=None):
    n = len(m)
    res = np.zeros((n, 4)); jac = np.zeros((n, 4, 7)); wt = np.zeros((n, 4)); info = np.zeros(n)
    used = np.zeros(n, np.uint8)
    pr = _pm(X_ref, valid_ref, h, w); ps = _pm(X_src, valid_src, h, w)
    s = m.struct()
    params = params or abi.default_robust_weight_params()
    _check(lib().orc_residual_blocks(C.byref(T), C.byref(s), C.byref(pr), C.byref(ps), C.c_int(mode),
                                     C.byref(params), C.byref(K) if K is not None else None,
                                     ptr(res), ptr(jac), ptr(wt), ptr(info), ptr(used)))
    return res, jac, wt, info, used


def normal_equations(T, m: MatchSet, X_ref, valid_ref, X_src, valid_src, h, w, mode=abi.PMX_TRACK_RAY,
                     params=None, K=None):
    H = np.zeros((7, 7)); g = np.zeros(7); cost = C.c_double(); used = C.c_int64()
    pr = _pm(X_ref, valid_ref, h, w); ps = _pm(X_src, valid_src, h, w)
    s = m.struct()
    params = params or abi.default_robust_weight_params()
    _check(lib().orc_normal_equations(C.byref(T), C.byref(s), C.byref(pr), C.byref(ps), C.c_int(mode),
                                      C.byref(params), C.byref(K) if K is not None else None,
                                      ptr(H), ptr(g), C.byref(cost), C.byref(used)))
    return H, g, cost.value, used.value


def track_given_matches(canonical, valid_c, X_f_f, valid_f, h, w, m: MatchSet, init, mode=abi.PMX_TRACK_RAY,
                        params=None):
    res = abi.pmx_track_result()
    pc = _pm(canonical, valid_c, h, w); pf = _pm(X_f_f, valid_f, h, w)
    s = m.struct()
    params = params or abi.default_solve_pose_params()
    _check(lib().orc_track_given_matches(C.byref(pc), C.byref(pf), C.byref(s), C.byref(init), C.c_int(mode),
                                         C.byref(params), C.byref(res)))
    return res


def fuse_canonical(canon_xyz, canon_valid, canon_conf, X_k_f, valid_k, conf, T, h, w):
    cx = np.ascontiguousarray(canon_xyz, np.float64).copy()
    cv = np.ascontiguousarray(canon_valid, np.uint8).copy()
    cc = np.ascontiguousarray(canon_conf, np.float64).copy()
    pk = _pm(X_k_f, valid_k, h, w)
    c32 = np.ascontiguousarray(conf, np.float32)
    _check(lib().orc_fuse_canonical(C.c_int32(h), C.c_int32(w), ptr(cx), ptr(cv), ptr(cc), C.byref(pk),
                                    ptr(c32), C.byref(T)))
    return cx, cv, cc


class Graph:
    """Host graph for the oracle: canonicals [(xyz, valid)], poses [pmx_sim3],
    edges [(i, j)], matches [MatchSet]."""

    def __init__(self, canonicals, poses, edges, matches, h, w, anchor=0):
        self.canonicals = [(np.ascontiguousarray(x, np.float32), None if v is None else np.ascontiguousarray(v, np.uint8))
                           for x, v in canonicals]
        self.poses = list(poses)
        self.edges = list(edges)
        self.matches = list(matches)
        self.h, self.w, self.anchor = h, w, anchor

    def struct(self, keep):
        n = len(self.canonicals)
        cans = (abi.pmx_pointmap * n)(*[abi.pointmap(x, v, self.h, self.w) for x, v in self.canonicals])
        poses = (abi.pmx_sim3 * n)(*self.poses)
        ei = np.array([e[0] for e in self.edges], np.int32)
        ej = np.array([e[1] for e in self.edges], np.int32)
        ms = (abi.orc_matchset * len(self.edges))(*[m.struct() for m in self.matches])
        keep.extend([cans, poses, ei, ej, ms])
        return abi.orc_graph(n, cans, poses, self.anchor, len(self.edges), ptr(ei), ptr(ej), ms)


def assemble_system(g: Graph, params=None):
    keep = []
    gs = g.struct(keep)
    dim = 7 * len(g.canonicals)
    H = np.zeros((dim, dim)); grad = np.zeros(dim)
    params = params or abi.default_backend_params()
    _check(lib().orc_assemble_system(C.byref(gs), C.byref(params), ptr(H), ptr(grad)))
    return H, grad


def backend_cost(g: Graph, params=None):
    keep = []
    gs = g.struct(keep)
    out = C.c_double()
    params = params or abi.default_backend_params()
    _check(lib().orc_backend_cost(C.byref(gs), C.byref(params), C.byref(out)))
    return out.value


def backend_edge_terms(g: Graph, params=None, begin=0, end=None, threads=1):
    keep = []
    gs = g.struct(keep)
    end = len(g.edges) if end is None else end
    out = np.zeros((end - begin, abi.PMX_EDGE_TERMS))
    params = params or abi.default_backend_params()
    _check(lib().orc_backend_edge_terms(C.byref(gs), C.byref(params), C.c_int32(begin), C.c_int32(end),
                                        ptr(out), C.c_int32(threads)))
    return out


def global_optimize(g: Graph, params=None):
    keep = []
    gs = g.struct(keep)
    params = params or abi.default_backend_params()
    res = abi.pmx_optimize_result()
    n = len(g.canonicals)
    trace = (abi.pmx_sim3 * (max(1, params.max_iterations) * n))()
    _check(lib().orc_global_optimize(C.byref(gs), C.byref(params), C.byref(res), trace))
    poses = [gs.poses[k] for k in range(n)]
    g.poses = [abi.pmx_sim3.from_buffer_copy(p) for p in poses]
    rows = res.iterations if res.converged else max(0, res.iterations - 1)  # a failed iteration records nothing
    tr = [[abi.pmx_sim3.from_buffer_copy(trace[it * n + k]) for k in range(n)] for it in range(rows)]
    return res, tr


def ldlt_solve(A, b):
    A = np.ascontiguousarray(A, np.float64); b = np.ascontiguousarray(b, np.float64)
    n = b.shape[0]
    x = np.zeros(n); ok = C.c_int32()
    _check(lib().orc_ldlt_solve(C.c_int32(n), ptr(A), ptr(b), ptr(x), C.byref(ok)))
    return x, bool(ok.value)


def sim3_exp(tau):
    t = np.ascontiguousarray(tau, np.float64); out = abi.pmx_sim3()
    _check(lib().orc_sim3_exp(ptr(t), C.byref(out)))
    return out


def sim3_log(T):
    out = np.zeros(7)
    _check(lib().orc_sim3_log(C.byref(T), ptr(out)))
    return out


def sim3_compose(a, b):
    out = abi.pmx_sim3()
    _check(lib().orc_sim3_compose(C.byref(a), C.byref(b), C.byref(out)))
    return out


def sim3_inverse(a):
    out = abi.pmx_sim3()
    _check(lib().orc_sim3_inverse(C.byref(a), C.byref(out)))
    return out


def sim3_adjoint(a):
    out = np.zeros((7, 7))
    _check(lib().orc_sim3_adjoint(C.byref(a), ptr(out)))
    return out


# --------------------------------------------------------------------------
# Neighbours of the path, restated in numpy (FP64).

def accept_loop_edge(pair, omega_l, params=None, refine=None):
    """accept_loop_edge, reference src/retrieval.cpp:226-251: match + refine,
    then every valid match whose endpoint descriptors have dot < 0.5
    (FP64, retrieval.cpp:238-244) is invalidated; accepted iff
    valid_fraction() >= omega_l (camera.cpp:16-19).  Returns (accepted, MatchSet)."""
    m = feature_refine(match_pointmaps(pair, params), pair, refine or abi.default_refine_params())
    Da = np.asarray(pair["D_a"], np.uint16).view(np.float16).astype(np.float64)
    Db = np.asarray(pair["D_b"], np.uint16).view(np.float16).astype(np.float64)
    valid = m.valid.astype(bool)
    idx = np.nonzero(valid)[0]
    dots = np.einsum("ij,ij->i", Da[m.pixel_a[idx]], Db[m.pixel_b[idx]])  # exact: fp16 products in FP64
    valid[idx[dots < 0.5]] = False
    m.valid = valid.astype(np.uint8)
    frac = valid.sum() / len(valid) if len(valid) else 0.0
    return bool(frac >= omega_l), m


def constrain_to_rays(xyz, valid, h, w, K):
    """constrain_to_rays, reference src/pipeline.cpp:32-46 (z <= 0 invalidates)."""
    xyz = np.array(xyz, np.float32).reshape(-1, 3)
    valid = np.array(valid, np.uint8)
    u = np.tile(np.arange(w), h)
    v = np.repeat(np.arange(h), w)
    z = xyz[:, 2].astype(np.float64)
    keep = (valid != 0) & (z > 0.0)
    valid[(valid != 0) & ~(z > 0.0)] = 0
    x = z * ((u - K.cx) / K.fx)
    y = z * ((v - K.cy) / K.fy)
    out = xyz.copy()
    out[keep, 0] = x[keep].astype(np.float32)
    out[keep, 1] = y[keep].astype(np.float32)
    out[keep, 2] = z[keep].astype(np.float32)
    return out, valid


PAIR_MAGIC = b"PMPAIR01"


def write_pair_record(X_i, X_j, C_i, C_j, D_i, D_j, Q_i, Q_j) -> bytes:
    """RecordingPredictor::predict's record, reference src/pipeline.cpp:582-594:
    magic, then float32 X_i, X_j (HW x 3), C_i, C_j, D_i, D_j (HW x dim,
    pixel-major = Eigen column order), Q_i, Q_j."""
    parts = [np.ascontiguousarray(a, np.float32).ravel() for a in (X_i, X_j, C_i, C_j, D_i, D_j, Q_i, Q_j)]
    return PAIR_MAGIC + b"".join(p.tobytes() for p in parts)


def read_pair_record(buf: bytes, h, w, dim):
    """StreamPredictor::predict, reference src/pipeline.cpp:642-676."""
    if buf[:8] != PAIR_MAGIC:
        raise ValueError("StreamPredictor: bad magic")
    hw = h * w
    sizes = [3 * hw, 3 * hw, hw, hw, dim * hw, dim * hw, hw, hw]
    if len(buf) < 8 + 4 * sum(sizes):
        raise ValueError("StreamPredictor: truncated record")
    a = np.frombuffer(buf, np.float32, count=sum(sizes), offset=8)
    out, o = {}, 0
    for name, n in zip(("X_i", "X_j", "C_i", "C_j", "D_i", "D_j", "Q_i", "Q_j"), sizes):
        out[name] = a[o:o + n].copy()
        o += n
    out["X_i"] = out["X_i"].reshape(hw, 3)
    out["X_j"] = out["X_j"].reshape(hw, 3)
    out["D_i"] = out["D_i"].reshape(hw, dim)
    out["D_j"] = out["D_j"].reshape(hw, dim)
    out["valid_i"] = np.isfinite(out["X_i"]).all(axis=1).astype(np.uint8)  # allFinite (pipeline.cpp:541)
    out["valid_j"] = np.isfinite(out["X_j"]).all(axis=1).astype(np.uint8)
    return out


def solve_pose(canonical, valid_c, pred, h, w, init, mode=abi.PMX_TRACK_RAY, params=None,
               seed: MatchSet | None = None):
    """solve_pose, reference src/tracking.cpp:149-226: match the frame's own
    pointmap (a = frame, b = keyframe image) + refine + LM-damped GN.
    pred: X_f_f / valid_f / D_f / Q_f and X_k_f / valid_k / D_k / Q_k."""
    res = abi.pmx_track_result()
    pc = _pm(canonical, valid_c, h, w)
    pf = _pm(pred["X_f_f"], pred.get("valid_f"), h, w)
    pk = _pm(pred["X_k_f"], pred.get("valid_k"), h, w)
    Ff = _fm(pred["D_f"], pred["Q_f"], h, w)
    Fk = _fm(pred["D_k"], pred["Q_k"], h, w)
    out = MatchSet.empty(h * w)
    o = out.struct()
    s = seed.struct() if seed is not None else None
    params = params or abi.default_solve_pose_params()
    _check(lib().orc_solve_pose(C.byref(pc), C.byref(pf), C.byref(pk), C.byref(Ff), C.byref(Fk), C.byref(init),
                                C.c_int(mode), C.byref(params), C.byref(s) if s is not None else None,
                                C.byref(res), C.byref(o)))
    return res, out
