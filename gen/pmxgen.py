"""Deterministic synthetic inputs for the BASELINE configs (bench/test infra).

Thin numpy wrapper over gen/libpmx_gen.so (counter-based splitmix64 RNG +
explicit Box-Muller, FP64 ray casting).  The BASELINE configs name synthetic
512x384 pointmaps; there is no dataset.  Resolved ambiguities (SURVEY.md
Appendix B) are recorded in DESIGN.md §3 and in the docstrings below.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpmx_gen.so")
_lib = None

H, W, F, CX, CY, DIM = 384, 512, 400.0, 256.0, 192.0, 24


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.check_call(["make", "-s", "-C", _HERE])
        _lib = C.CDLL(_LIB_PATH)
        _lib.gen_image.restype = C.c_int
        _lib.gen_gt_matches.restype = C.c_int
    return _lib


def _threads():
    return max(1, min(32, os.cpu_count() or 1))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Pose:
    """Sim(3) x -> s R x + t (FP64), the reference's Sim3Pose (lie.hpp:36-70)."""

    def __init__(self, R=None, t=None, s=1.0):
        self.R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64).reshape(3, 3)
        self.t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64).reshape(3)
        self.s = float(s)

    def __mul__(self, o: "Pose") -> "Pose":  # lie.cpp:131-140
        return Pose(self.R @ o.R, self.s * (self.R @ o.t) + self.t, self.s * o.s)

    def inverse(self) -> "Pose":  # lie.cpp:121-129
        Ri = self.R.T
        si = 1.0 / self.s
        return Pose(Ri, -si * (Ri @ self.t), si)

    def act(self, x):
        return self.s * (np.asarray(x) @ self.R.T) + self.t

    def to_struct(self, struct_cls):
        T = struct_cls()
        for i, v in enumerate(self.R.reshape(-1)):
            T.R[i] = float(v)
        for i in range(3):
            T.t[i] = float(self.t[i])
        T.s = self.s
        return T

    @staticmethod
    def from_struct(T) -> "Pose":
        return Pose(np.array(T.R[:]).reshape(3, 3), np.array(T.t[:]), T.s)

    def __repr__(self):
        return f"Pose(R={self.R.tolist()}, t={self.t.tolist()}, s={self.s})"


def rodrigues(omega) -> np.ndarray:
    omega = np.asarray(omega, dtype=np.float64)
    th = float(np.linalg.norm(omega))
    K = np.array([[0, -omega[2], omega[1]], [omega[2], 0, -omega[0]], [-omega[1], omega[0], 0]])
    if th < 1e-12:
        return np.eye(3) + K
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * (K @ K)


def uniform(seed, stream, n):
    out = np.empty(n, dtype=np.float64)
    _load().gen_uniform(C.c_uint64(seed), C.c_uint64(stream), C.c_int64(n), _p(out))
    return out


def gauss(seed, stream, n):
    out = np.empty(n, dtype=np.float64)
    _load().gen_gauss(C.c_uint64(seed), C.c_uint64(stream), C.c_int64(n), _p(out))
    return out


def unit_vector(seed, stream):
    g = gauss(seed, stream, 3)
    return g / np.linalg.norm(g)


def random_pose(seed, stream, max_rot_deg, max_trans, scale_lo, scale_hi) -> Pose:
    """Axis uniform on S^2, angle U[0, max]; translation direction uniform,
    magnitude U[0, max]; scale U[lo, hi] (BASELINE configs 0/1)."""
    u = uniform(seed, stream, 3)
    axis = unit_vector(seed, stream + 1)
    tdir = unit_vector(seed, stream + 2)
    R = rodrigues(axis * math.radians(max_rot_deg) * u[0])
    return Pose(R, tdir * max_trans * u[1], scale_lo + (scale_hi - scale_lo) * u[2])


def perturb_pose(T: Pose, seed, stream, rot_deg, trans, scale_frac) -> Pose:
    """Fixed-magnitude perturbation along random directions (configs 3/4):
    rotation rot_deg about a random axis, translation `trans` in a random
    direction, scale x exp(+-scale_frac)."""
    axis = unit_vector(seed, stream)
    tdir = unit_vector(seed, stream + 1)
    sign = 1.0 if uniform(seed, stream + 2, 1)[0] < 0.5 else -1.0
    dR = rodrigues(axis * math.radians(rot_deg))
    return Pose(dR @ T.R, T.t + tdir * trans, T.s * math.exp(sign * scale_frac))


class Scene:
    """The config-0 surface z = 2 + 0.3 sin(3x) cos(2y) + a x + b y over the
    reference camera's normalised coordinates; tilt a, b ~ U[-0.2, 0.2].

    Point noise N(0, point_sigma^2): ``noise="radial"`` (default) perturbs
    the distance along each view's own viewing ray, the reference's noise
    model (src/synth.cpp:221-226); ``noise="isotropic"`` adds it per
    coordinate (a rough ray field; an adversarial parity case)."""

    def __init__(self, seed: int, height=H, width=W, f=F, cx=CX, cy=CY, dim=DIM,
                 point_sigma=0.005, desc_sigma=0.05, noise="radial", surface="depthmap"):
        ab = uniform(seed, 7, 2) * 0.4 - 0.2
        self.seed, self.height, self.width, self.dim = seed, height, width, dim
        self.f, self.cx, self.cy = f, cx, cy
        self.params = np.array([seed, ab[0], ab[1], f, cx, cy, height, width, dim,
                                point_sigma, desc_sigma, 0 if noise == "radial" else 1,
                                0 if surface == "depthmap" else 1],
                               dtype=np.float64)

    def image(self, image_id: int, T_wk: Pose, T_frame: Pose, salt: int = 0,
              want=("X", "valid", "Q", "D")):
        from paper_2412_12392_b200.abi import pmx_sim3
        n = self.height * self.width
        X = np.empty((n, 3), np.float32) if "X" in want else None
        valid = np.empty(n, np.uint8) if "valid" in want else None
        Q = np.empty(n, np.float32) if "Q" in want else None
        D = np.empty((n, self.dim), np.uint16) if "D" in want else None
        a, b = T_wk.to_struct(pmx_sim3), T_frame.to_struct(pmx_sim3)
        _load().gen_image(_p(self.params), C.c_int64(image_id), C.byref(a), C.byref(b),
                          C.c_uint64(salt), _p(X), _p(valid), _p(Q), _p(D), None,
                          C.c_int(_threads()))
        return {"X": X, "valid": valid, "Q": Q, "D": D}

    def pair(self, ia: int, T_wa: Pose, ib: int, T_wb: Pose, salt: int = 0):
        """Pair prediction of edge (a, b) in frame a (what MASt3R predicts):
        X_a = camera a's points in frame a, X_b_in_a = camera b's points in
        frame a, per-image Q, pair-predicted fp16 descriptors (ids on camera
        a's pixel grid, gen_pair_desc)."""
        return pair_from_cameras(Camera(self, ia, T_wa), Camera(self, ib, T_wb), salt)

    def gt_matches(self, ia, T_wa, ib, T_wb, subpixel=False):
        from paper_2412_12392_b200.abi import pmx_sim3
        n = self.height * self.width
        pa = np.empty(n, np.int32)
        q = np.empty(n, np.float32)
        v = np.empty(n, np.uint8)
        sp = np.empty((n, 2), np.float64) if subpixel else None
        a, b = T_wa.to_struct(pmx_sim3), T_wb.to_struct(pmx_sim3)
        _load().gen_gt_matches(_p(self.params), C.c_int64(ia), C.byref(a), C.c_int64(ib),
                               C.byref(b), _p(pa), _p(q), _p(v), _p(sp), C.c_int(_threads()))
        out = {"pixel_a": pa, "confidence": q, "valid": v}
        if subpixel:
            out["subpixel"] = sp
        return out


# ------------------------------------------------------------------ configs

def config0(seed: int = 0, height=H, width=W, noise="radial"):
    """BASELINE config 0: one pair, camera j under a random relative Sim(3)
    (rotation <= 5 deg, translation <= 0.1, scale in [0.9, 1.1])."""
    sc = Scene(seed, height, width, f=F * width / W, cx=CX * width / W, cy=CY * height / H, noise=noise)
    T_ij = random_pose(seed, 100, 5.0, 0.1, 0.9, 1.1)
    pair = sc.pair(0, Pose(), 1, T_ij)
    pair["T_ij"] = T_ij
    pair["scene"] = sc
    return pair


def config1(seed: int = 1, height=H, width=W):
    """BASELINE config 1: keyframe (reference camera) + frame under T_kf
    (rotation <= 3 deg, translation <= 0.05, scale in [0.95, 1.05]).
    Returns canonical (keyframe own view, noisy), C~, the frame prediction
    (X_f_f, X_k_f, C_f, C_k, F_f, F_k) and the true T_kf."""
    sc = Scene(seed, height, width, f=F * width / W, cx=CX * width / W, cy=CY * height / H)
    T_kf = random_pose(seed, 200, 3.0, 0.05, 0.95, 1.05)
    kf = sc.image(0, Pose(), Pose(), salt=10)
    pred = sc.pair(1, T_kf, 0, Pose(), salt=20)  # a = frame, b = keyframe image
    return {"scene": sc, "T_kf": T_kf,
            "canonical": kf["X"], "canonical_valid": kf["valid"], "canonical_conf": kf["Q"],
            "X_f_f": pred["X_a"], "valid_f": pred["valid_a"], "C_f": pred["Q_a"], "D_f": pred["D_a"],
            "X_k_f": pred["X_b"], "valid_k": pred["valid_b"], "C_k": pred["Q_b"], "D_k": pred["D_b"],
            "height": height, "width": width}


def inject_outliers(pixel_a: np.ndarray, valid: np.ndarray, frac: float, seed: int, hw: int):
    """Config 1: `frac` of entries get a uniform-random pixel_a and are flagged valid."""
    n = pixel_a.shape[0]
    u = uniform(seed, 300, n)
    r = uniform(seed, 301, n)
    pa = pixel_a.copy()
    v = valid.copy()
    sel = u < frac
    pa[sel] = np.minimum((r[sel] * hw).astype(np.int64), hw - 1).astype(np.int32)
    v[sel] = 1
    return pa, v


def trajectory_config2(seed: int = 2, n_kf: int = 32):
    """32 keyframes on a smooth lateral arc over the surface (small yaw/pitch
    wobble).  Returns camera->world poses (the reference camera = world)."""
    poses = []
    for k in range(n_kf):
        s = k / (n_kf - 1)
        t = np.array([1.2 * (s - 0.5), 0.25 * math.sin(math.pi * s), 0.05 * math.sin(2 * math.pi * s)])
        w = np.array([0.03 * math.sin(2 * math.pi * s), -0.04 * (s - 0.5), 0.02 * math.cos(math.pi * s)])
        poses.append(Pose(rodrigues(w), t, 1.0))
    return poses


def edges_config2(seed: int = 2, n_kf: int = 32, n_consecutive: int = 28, n_long: int = 8,
                  min_overlap: float = 0.4, poses=None, scene=None):
    """64 directed edges: 28 consecutive pairs x both directions + 8 long-range
    pairs (|i-j| >= 3) with GT overlap >= 40%, chosen deterministically."""
    edges = []
    for k in range(n_consecutive):
        edges.append((k, k + 1))
        edges.append((k + 1, k))
    poses = poses or trajectory_config2(seed, n_kf)
    sc = scene or Scene(seed, 48, 64, f=F * 64 / W, cx=CX * 64 / W, cy=CY * 48 / H, surface="heightfield")
    u = uniform(seed, 400, 4096)
    k = 0
    longs = []
    while len(longs) < n_long and k + 1 < len(u):
        i = int(u[k] * n_kf) % n_kf
        j = int(u[k + 1] * n_kf) % n_kf
        k += 2
        if abs(i - j) < 3 or (i, j) in longs:
            continue
        gt = sc.gt_matches(i, poses[i], j, poses[j])
        if gt["valid"].mean() >= min_overlap:
            longs.append((i, j))
    return edges + longs


def loop_trajectory(n_kf: int, radius: float = 5.0, loops: int = 1, seed: int = 3):
    """Keyframes on `loops` turns of a circle of radius `radius` (m) in the
    reference camera's XY plane, looking down +Z at the surface; the radius
    shrinks by 4% per extra loop (multi-loop, config 4)."""
    poses = []
    for k in range(n_kf):
        a = 2 * math.pi * loops * k / n_kf
        r = radius * (1.0 - 0.04 * (loops * k // n_kf))
        t = np.array([r * math.cos(a), r * math.sin(a), 0.02 * math.sin(3 * a)])
        R = rodrigues(np.array([0.0, 0.0, a]))
        poses.append(Pose(R, t, 1.0))
    return poses


def loop_edges(n_kf: int, reach: int):
    """Cyclic neighbours k <-> k+1 .. k+reach (the wrap-around edges are the
    loop closures): n_kf * reach bidirectional edges."""
    return [(k, (k + d) % n_kf) for k in range(n_kf) for d in range(1, reach + 1)]


def gt_from_cameras(ca: "Camera", cb: "Camera"):
    """Ground-truth matches of edge (a, b) from cached world points (gen_gt_from_points)."""
    from paper_2412_12392_b200.abi import pmx_sim3
    n = ca.scene.height * ca.scene.width
    pa = np.empty(n, np.int32)
    q = np.empty(n, np.float32)
    v = np.empty(n, np.uint8)
    a = ca.T.to_struct(pmx_sim3)
    _load().gen_gt_from_points(_p(ca.scene.params), C.byref(a), _p(cb.P), _p(cb.valid), _p(ca.Q), _p(cb.Q),
                               _p(pa), _p(q), _p(v), C.c_int(_threads()))
    return {"pixel_a": pa, "confidence": q, "valid": v}


def backend_graph(n_kf: int, reach: int, seed: int, height=H, width=W, loops: int = 1,
                  radius: float = 5.0, rot_deg=2.0, trans=0.05, scale_frac=0.03,
                  edges=None, edge_range=None):
    """Configs 3/4: GT loop poses, canonical pointmaps (own view + noise),
    edges with ground-truth matches (pixel_a in i, pixel_b in j, dense), and
    perturbed initial poses (anchor = keyframe 0, unperturbed)."""
    sc = Scene(seed, height, width, f=F * width / W, cx=CX * width / W, cy=CY * height / H, surface="heightfield")
    gt = loop_trajectory(n_kf, radius, loops, seed)
    cams = [Camera(sc, k, gt[k]) for k in range(n_kf)]
    canon = [(c.express(c.T, 1000 + k), c.valid) for k, c in enumerate(cams)]
    edges = edges if edges is not None else loop_edges(n_kf, reach)
    e0, e1 = edge_range if edge_range is not None else (0, len(edges))
    empty = {"pixel_a": np.empty(0, np.int32), "confidence": np.empty(0, np.float32), "valid": np.empty(0, np.uint8)}
    # edge_range: only these edges' matches (one rank's shard); the others are empty
    matches = [gt_from_cameras(cams[i], cams[j]) if e0 <= e < e1 else empty for e, (i, j) in enumerate(edges)]
    init = [gt[0]] + [perturb_pose(gt[k], seed, 5000 + 3 * k, rot_deg, trans, scale_frac)
                      for k in range(1, n_kf)]
    return {"scene": sc, "gt": gt, "init": init, "canonicals": canon, "edges": edges,
            "matches": matches, "height": height, "width": width}


class Camera:
    """A ray-cast camera (world points cached) for many-edge configs."""

    def __init__(self, scene: Scene, image_id: int, T_wk: Pose):
        from paper_2412_12392_b200.abi import pmx_sim3
        n = scene.height * scene.width
        self.scene, self.image_id, self.T = scene, image_id, T_wk
        self.P = np.empty((n, 3), np.float64)
        self.valid = np.empty(n, np.uint8)
        self.Q = np.empty(n, np.float32)
        a = T_wk.to_struct(pmx_sim3)
        _load().gen_camera(_p(scene.params), C.c_int64(image_id), C.byref(a), _p(self.P), _p(self.valid),
                           _p(self.Q), None, C.c_int(_threads()))

    def express(self, T_frame: Pose, salt: int) -> np.ndarray:
        from paper_2412_12392_b200.abi import pmx_sim3
        X = np.empty(self.P.shape, np.float32)
        a, b = self.T.to_struct(pmx_sim3), T_frame.to_struct(pmx_sim3)
        _load().gen_express(_p(self.scene.params), C.c_int64(self.image_id), C.byref(a), C.byref(b),
                            C.c_uint64(salt), _p(self.P), _p(self.valid), _p(X), C.c_int(_threads()))
        return X


def pair_from_cameras(ca: Camera, cb: Camera, salt: int):
    """Pair prediction of edge (a, b) in frame a from cached cameras."""
    from paper_2412_12392_b200.abi import pmx_sim3
    sc = ca.scene
    n = sc.height * sc.width
    Da = np.empty((n, sc.dim), np.uint16)
    Db = np.empty((n, sc.dim), np.uint16)
    a = ca.T.to_struct(pmx_sim3)
    _load().gen_pair_desc(_p(sc.params), C.c_int64(ca.image_id), C.byref(a), _p(ca.valid), C.c_int64(cb.image_id),
                          _p(cb.P), _p(cb.valid), _p(Da), _p(Db), C.c_int(_threads()))
    return {"X_a": ca.express(ca.T, salt), "valid_a": ca.valid, "Q_a": ca.Q, "D_a": Da,
            "X_b": cb.express(ca.T, salt + 1), "valid_b": cb.valid, "Q_b": cb.Q, "D_b": Db,
            "height": sc.height, "width": sc.width}


def config2(seed: int = 2, height=H, width=W, n_kf: int = 32, edges=None):
    """BASELINE config 2: 32 keyframes on a smooth trajectory, 64 directed edges.
    Returns (scene, cameras, edges, make_pair(e))."""
    sc = Scene(seed, height, width, f=F * width / W, cx=CX * width / W, cy=CY * height / H, surface="heightfield")
    poses = trajectory_config2(seed, n_kf)
    edges = edges if edges is not None else edges_config2(seed, n_kf, poses=poses)
    cams = {}

    def cam(k):
        if k not in cams:
            cams[k] = Camera(sc, k, poses[k])
        return cams[k]

    def make_pair(e):
        a, b = edges[e]
        return pair_from_cameras(cam(a), cam(b), salt=2 * e)

    return sc, poses, edges, make_pair


# ------------------------------------------------- device pair predictions
_CU_PATH = os.path.join(_HERE, "libpmx_gen_cuda.so")
_cu = None


def _load_cuda():
    global _cu
    if _cu is None:
        if not os.path.exists(_CU_PATH):
            subprocess.check_call(["make", "-s", "-C", _HERE, "libpmx_gen_cuda.so"])
        _cu = C.CDLL(_CU_PATH)
        _cu.gen_cuda_express.restype = C.c_int
        _cu.gen_cuda_pair_desc.restype = C.c_int
    return _cu


def _tp(t):
    return C.c_void_p(t.data_ptr())


class DeviceCamera:
    """A Camera's world points / validity / Q resident on the GPU (torch)."""

    def __init__(self, cam: Camera, device):
        import torch
        self.cam = cam
        self.P = torch.from_numpy(cam.P).to(device)
        self.valid = torch.from_numpy(cam.valid).to(device)
        self.Q = torch.from_numpy(cam.Q).to(device)


def device_pair(ca: DeviceCamera, cb: DeviceCamera, salt: int, stream=None):
    """Pair prediction of edge (a, b) in frame a generated on the GPU
    (gen/pmx_gen_cuda.cu, the device twin of pair_from_cameras)."""
    import torch
    from paper_2412_12392_b200.abi import pmx_sim3
    sc = ca.cam.scene
    n = sc.height * sc.width
    dev = ca.P.device
    s = C.c_void_p(stream.cuda_stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream)
    Ta = ca.cam.T.to_struct(pmx_sim3)
    Tb = cb.cam.T.to_struct(pmx_sim3)
    X_a = torch.empty((n, 3), dtype=torch.float32, device=dev)
    X_b = torch.empty((n, 3), dtype=torch.float32, device=dev)
    D_a = torch.empty((n, sc.dim), dtype=torch.int16, device=dev)
    D_b = torch.empty((n, sc.dim), dtype=torch.int16, device=dev)
    L = _load_cuda()
    for rc in (L.gen_cuda_express(_p(sc.params), C.c_int64(ca.cam.image_id), C.byref(Ta), C.byref(Ta),
                                  C.c_uint64(salt), _tp(ca.P), _tp(ca.valid), _tp(X_a), s),
               L.gen_cuda_express(_p(sc.params), C.c_int64(cb.cam.image_id), C.byref(Tb), C.byref(Ta),
                                  C.c_uint64(salt + 1), _tp(cb.P), _tp(cb.valid), _tp(X_b), s),
               L.gen_cuda_pair_desc(_p(sc.params), C.c_int64(ca.cam.image_id), C.byref(Ta), _tp(ca.valid),
                                    C.c_int64(cb.cam.image_id), _tp(cb.P), _tp(cb.valid), _tp(D_a), _tp(D_b), s)):
        if rc != 0:
            raise RuntimeError(f"gen_cuda: CUDA error {rc}")
    return {"X_a": X_a, "valid_a": ca.valid, "Q_a": ca.Q, "D_a": D_a,
            "X_b": X_b, "valid_b": cb.valid, "Q_b": cb.Q, "D_b": D_b, "height": sc.height, "width": sc.width}


MATCHED_SALT = 1_000_000


def backend_graph_matched(ctx, n_kf: int, reach: int, seed: int, height=H, width=W, loops: int = 1,
                          radius: float = 5.0, rot_deg=2.0, trans=0.05, scale_frac=0.03, edge_range=None,
                          chunk: int = 64, device=None, keep_host: bool = False):
    """Configs 3/4 with matches "precomputed as in config 2" (BASELINE.json):
    every edge's pair prediction (camera i's and camera j's points in frame
    i + pair descriptors, generated on the GPU) is matched by the product's
    batched matcher (LM lambda 1e-8, tol 1e-6 rad, refine {(1,3),(1,3)}), and
    the resulting MatchSets (pixel_a in i, pixel_b = index in j, q, valid)
    are the backend's frozen matches.  Canonicals, poses, edges and the
    perturbed initial poses are those of backend_graph.  Returns the
    backend_graph dict with "matches" as device MatchSets (and host numpy
    copies under "matches_host" when keep_host)."""
    import torch
    from paper_2412_12392_b200 import FeatureMap, MatchSet, Pointmap, abi
    device = device or torch.device("cuda", torch.cuda.current_device())
    sc = Scene(seed, height, width, f=F * width / W, cx=CX * width / W, cy=CY * height / H, surface="heightfield")
    gt = loop_trajectory(n_kf, radius, loops, seed)
    edges = loop_edges(n_kf, reach)
    e0, e1 = edge_range if edge_range is not None else (0, len(edges))
    need = sorted({k for e in range(e0, e1) for k in edges[e]})
    # an edge shard only ray-casts its own keyframes; the others get empty
    # (all-invalid) canonicals, which no edge of the shard reads
    cams = {k: Camera(sc, k, gt[k]) for k in need}
    blank = (np.zeros((height * width, 3), np.float32), np.zeros(height * width, np.uint8))
    canon = [(cams[k].express(cams[k].T, 1000 + k), cams[k].valid) if k in cams else blank for k in range(n_kf)]
    dcams = {k: DeviceCamera(cams[k], device) for k in need}
    mp = abi.default_match_params()
    mp.projection.lambda_init = 1e-8
    mp.projection.angle_tol = 1e-6
    rp = abi.refine_params([(1, 3), (1, 3)])
    n = height * width
    empty = MatchSet(torch.empty(0, dtype=torch.int32, device=device), torch.empty(0, dtype=torch.float32, device=device),
                     torch.empty(0, dtype=torch.uint8, device=device))
    matches = [empty] * len(edges)
    for c0 in range(e0, e1, chunk):
        c1 = min(e1, c0 + chunk)
        preds = [device_pair(dcams[edges[e][0]], dcams[edges[e][1]], MATCHED_SALT + 2 * e) for e in range(c0, c1)]
        outs = [MatchSet.empty(n, device) for _ in range(c0, c1)]
        ctx.match_batch([(Pointmap(p["X_a"], p["valid_a"], height, width), Pointmap(p["X_b"], p["valid_b"], height, width),
                          FeatureMap(p["D_a"], p["Q_a"], height, width), FeatureMap(p["D_b"], p["Q_b"], height, width))
                         for p in preds], params=mp, refine=rp, outs=outs)
        for k, e in enumerate(range(c0, c1)):
            matches[e] = outs[k]
        del preds
    torch.cuda.synchronize(device)
    init = [gt[0]] + [perturb_pose(gt[k], seed, 5000 + 3 * k, rot_deg, trans, scale_frac) for k in range(1, n_kf)]
    out = {"scene": sc, "gt": gt, "init": init, "canonicals": canon, "edges": edges, "matches": matches,
           "height": height, "width": width, "matcher": "config-2 matcher (device pair predictions)"}
    if keep_host:
        out["matches_host"] = [{"pixel_a": m.pixel_a.cpu().numpy(), "confidence": m.confidence.cpu().numpy(),
                                "valid": m.valid.cpu().numpy()} for m in matches]
    return out
