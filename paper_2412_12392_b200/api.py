"""Python mirror of the reference's matching / tracking / optimiser API.

Same names, argument meaning and error behaviour as the CPU reference
``pmslam`` (/root/reference/proj/include/pmslam/{camera,tracking,backend}.hpp),
executed by ``libpmx_cuda.so`` through the C ABI of ``include/pmx.h``:

=====================  ==================================================
reference              here
=====================  ==================================================
normalize_rays         Context.normalize_rays        (camera.hpp:100)
iterative_project      Context.iterative_project     (camera.hpp:123)
match_pointmaps        Context.match_pointmaps       (camera.hpp:135)
feature_refine         Context.feature_refine        (camera.hpp:147)
(loop-edge matching)   Context.match_batch           (retrieval.cpp:232)
residual_blocks        Context.residual_blocks       (tracking.hpp:56)
(GN normal equations)  Context.normal_equations      (tracking.cpp:188)
solve_pose             Context.solve_pose            (tracking.hpp:105)
(GN on given matches)  Context.track_given_matches   (tracking.cpp:165)
fuse_canonical         Context.fuse_canonical        (tracking.hpp:112)
keyframe_decision      Context.keyframe_decision     (tracking.hpp:117)
assemble_system        Context.assemble_system       (backend.hpp:57)
backend_cost           Context.backend_cost          (backend.hpp:72)
global_optimize        Context.global_optimize       (backend.hpp:69)
=====================  ==================================================

Arrays are numpy (host memory: the call stages them H2D and returns host
results) or torch CUDA tensors (device memory: results stay on the device).
The reference's std::invalid_argument / std::domain_error surface as
``ValueError`` / ``ArithmeticError`` (``PmxError`` subclasses).  There is no
CPU fallback: a missing extension or device raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any, List, Optional, Sequence

import numpy as np

from . import abi
from .abi import ptr


class PmxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pmx status {code}: {msg}")
        self.code = code


class PmxInvalidArgument(PmxError, ValueError):
    pass


class PmxDomainError(PmxError, ArithmeticError):
    pass


def _is_dev(a) -> bool:
    return a is not None and hasattr(a, "is_cuda") and a.is_cuda


@dataclass
class Pointmap:
    """H x W grid of points, row-major (camera.hpp:17-31): xyz (HW, 3) fp32, valid (HW,) u8 or None."""
    xyz: Any
    valid: Any
    height: int
    width: int

    def struct(self):
        return abi.pointmap(self.xyz, self.valid, self.height, self.width)


@dataclass
class FeatureMap:
    """Per-pixel fp16 descriptors (HW, dim) + match confidence Q (HW,) (camera.hpp:55-71)."""
    descriptors: Any
    match_confidence: Any
    height: int
    width: int

    @property
    def dim(self) -> int:
        return int(self.descriptors.shape[-1])

    def struct(self):
        return abi.featuremap(self.descriptors, self.match_confidence, self.height, self.width, self.dim)


@dataclass
class MatchSet:
    """SoA MatchSet (camera.hpp:73-89); pixel_b None = dense (pixel_b[k] == k)."""
    pixel_a: Any
    confidence: Any
    valid: Any
    pixel_b: Any = None

    def __len__(self):
        return int(self.pixel_a.shape[0])

    def struct(self):
        return abi.matchset(self.pixel_a, self.pixel_b, self.confidence, self.valid)

    @staticmethod
    def empty(n: int, device=None, dense: bool = True) -> "MatchSet":
        if device is not None:
            import torch
            pb = None if dense else torch.empty(n, dtype=torch.int32, device=device)
            return MatchSet(torch.empty(n, dtype=torch.int32, device=device),
                            torch.empty(n, dtype=torch.float32, device=device),
                            torch.empty(n, dtype=torch.uint8, device=device), pb)
        pb = None if dense else np.empty(n, np.int32)
        return MatchSet(np.empty(n, np.int32), np.empty(n, np.float32), np.empty(n, np.uint8), pb)

    def valid_count(self) -> int:  # camera.cpp:10-14
        v = self.valid
        return int(v.sum().item() if hasattr(v, "sum") and _is_dev(v) else np.count_nonzero(v))


@dataclass
class TrackResult:  # tracking.hpp:93-99
    T_kf: Any
    iterations: int
    lost: bool
    cost_trace: List[float]
    matches: Optional[MatchSet] = None


@dataclass
class OptimizeResult:  # backend.hpp:59-63
    iterations: int
    converged: bool
    cost_trace: List[float]
    pose_trace: List[list] = field(default_factory=list)


@dataclass
class Graph:
    """Keyframe graph (backend.hpp:18-32) by index: canonicals[k] = Pointmap,
    poses[k] = pmx_sim3 (T_WC, updated in place by global_optimize), edges
    [(i, j)], matches[e] = MatchSet (pixel_a in i, pixel_b in j)."""
    canonicals: Sequence[Pointmap]
    poses: list
    edges: Sequence[tuple]
    matches: Sequence[MatchSet]
    anchor: int = 0

    def struct(self, keep: list):
        n = len(self.canonicals)
        cans = (abi.pmx_pointmap * max(1, n))(*[c.struct() for c in self.canonicals])
        poses = (abi.pmx_sim3 * max(1, n))(*self.poses)
        ei = np.ascontiguousarray([e[0] for e in self.edges], np.int32)
        ej = np.ascontiguousarray([e[1] for e in self.edges], np.int32)
        ms = (abi.pmx_matchset * max(1, len(self.edges)))(*[m.struct() for m in self.matches])
        keep.extend([cans, poses, ei, ej, ms])
        return abi.pmx_graph(n, cans, poses, self.anchor, len(self.edges), ptr(ei), ptr(ej), ms)


class Context:
    """One pmx context (device + stream).  ``stream`` may be a torch.cuda.Stream
    (or raw cudaStream_t int) the library enqueues on."""

    def __init__(self, device: int = 0, stream=None):
        self.lib = abi.load_library()
        h = C.c_void_p()
        code = self.lib.pmx_create(int(device), C.byref(h))
        if code != abi.PMX_OK:
            raise PmxError(code, f"pmx_create(device={device}) failed (no sm_100 device?)")
        self.h = h
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "h", None):
            self.lib.pmx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self.lib.pmx_set_stream(self.h, C.c_void_p(raw)))

    def synchronize(self):
        self._check(self.lib.pmx_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.pmx_kernel_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        self._check(self.lib.pmx_profile_enable(self.h, int(on)))

    def nccl_unique_id(self) -> bytes:
        """128-byte NCCL unique id (rank 0) for nccl_init on every rank."""
        buf = (C.c_uint8 * 128)()
        self._check(self.lib.pmx_nccl_unique_id(self.h, buf))
        return bytes(buf)

    def nccl_init(self, uid: bytes, rank: int, nranks: int):
        """The context's NCCL communicator (edge-sharded backend)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self.lib.pmx_nccl_init(self.h, buf, C.c_int32(rank), C.c_int32(nranks)))

    def set_device_graphs(self, on: bool = True):
        """Device loops as one CUDA graph with a conditional WHILE node (default)."""
        self._check(self.lib.pmx_set_device_graphs(self.h, int(on)))

    def profile_reset(self):
        self._check(self.lib.pmx_profile_reset(self.h))

    def profile_get(self, kernel: str):
        """(total ms, launches) of a bracketed hot kernel since the last reset."""
        t, n = C.c_double(), C.c_int64()
        self._check(self.lib.pmx_profile_get(self.h, kernel.encode(), C.byref(t), C.byref(n)))
        return t.value, n.value

    def _check(self, code):
        if code == abi.PMX_OK:
            return
        msg = self.lib.pmx_last_error(self.h).decode()
        if code == abi.PMX_ERR_INVALID_ARGUMENT:
            raise PmxInvalidArgument(code, msg)
        if code == abi.PMX_ERR_DOMAIN:
            raise PmxDomainError(code, msg)
        raise PmxError(code, msg)

    @staticmethod
    def _mem(*arrays):
        dev = [_is_dev(a) for a in arrays if a is not None]
        if any(dev) and not all(dev):
            raise PmxInvalidArgument(abi.PMX_ERR_INVALID_ARGUMENT, "mixed host and device arrays")
        return abi.PMX_MEM_DEVICE if dev and all(dev) else abi.PMX_MEM_HOST

    # ---------------------------------------------------------- matching
    def normalize_rays(self, pm: Pointmap):
        n = pm.height * pm.width
        mem = self._mem(pm.xyz, pm.valid)
        if mem == abi.PMX_MEM_DEVICE:
            import torch
            dv = pm.xyz.device
            rays = torch.empty((n, 3), dtype=torch.float64, device=dv)
            dist = torch.empty(n, dtype=torch.float64, device=dv)
            valid = torch.empty(n, dtype=torch.uint8, device=dv)
        else:
            rays, dist, valid = np.empty((n, 3)), np.empty(n), np.empty(n, np.uint8)
        s = pm.struct()
        self._check(self.lib.pmx_normalize_rays(self.h, mem, C.byref(s), ptr(rays), ptr(dist), ptr(valid)))
        return rays, dist, valid

    def interpolate_ray(self, pm: Pointmap, p):
        """interpolate_ray (camera.cpp:58-100) at continuous pixels p (n x 2):
        (ray n x 3, jacobian n x 6 column-major 3x2, ok n)."""
        p = np.ascontiguousarray(p, np.float64).reshape(-1, 2)
        n = p.shape[0]
        ray, jac, ok = np.empty((n, 3)), np.empty((n, 6)), np.empty(n, np.uint8)
        s = pm.struct()
        self._check(self.lib.pmx_interpolate_ray(self.h, abi.PMX_MEM_HOST, C.byref(s), C.c_int64(n), ptr(p), ptr(ray),
                                                 ptr(jac), ptr(ok)))
        return ray, jac, ok

    def median_scene_distance(self, pm: Pointmap) -> float:
        """median_scene_distance (camera.cpp:178-191), exact FP64."""
        out = np.zeros(1)
        s = pm.struct()
        self._check(self.lib.pmx_median_scene_distance(self.h, abi.PMX_MEM_HOST, C.byref(s), ptr(out)))
        return float(out[0])

    def iterative_project(self, pm: Pointmap, x, p0, params=None):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, 3)
        p0 = np.ascontiguousarray(p0, np.float64).reshape(-1, 2)
        n = x.shape[0]
        pix, conv, it = np.empty((n, 2)), np.empty(n, np.uint8), np.empty(n, np.int32)
        params = params or abi.default_match_params().projection
        s = pm.struct()
        self._check(self.lib.pmx_iterative_project(self.h, abi.PMX_MEM_HOST, C.byref(s), C.c_int64(n), ptr(x),
                                                   ptr(p0), C.byref(params), ptr(pix), ptr(conv), ptr(it)))
        return pix, conv, it

    def match_pointmaps(self, X_a: Pointmap, X_b_in_a: Pointmap, F_a: FeatureMap, F_b: FeatureMap,
                        init: Optional[MatchSet] = None, params=None) -> MatchSet:
        return self.match_batch([(X_a, X_b_in_a, F_a, F_b, init)], params=params, refine=None)[0]

    def feature_refine(self, matches: MatchSet, F_a: FeatureMap, F_b: FeatureMap, params=None) -> MatchSet:
        mem = self._mem(matches.pixel_a, F_a.descriptors)
        n = len(matches)
        dev = matches.pixel_a.device if mem == abi.PMX_MEM_DEVICE else None
        out = MatchSet.empty(n, dev, dense=matches.pixel_b is None)
        params = params or abi.default_refine_params()
        i, o, fa, fb = matches.struct(), out.struct(), F_a.struct(), F_b.struct()
        self._check(self.lib.pmx_feature_refine(self.h, mem, C.byref(i), C.byref(fa), C.byref(fb), C.byref(params),
                                                C.byref(o)))
        if matches.pixel_b is not None and out.pixel_b is None:
            out.pixel_b = matches.pixel_b
        return out

    def prepare_match_batch(self, pairs, outs: Optional[List[MatchSet]] = None) -> "PreparedBatch":
        """Build the C-ABI pair/output arrays of a batch once (for buffers that
        stay resident and are matched repeatedly, e.g. a benchmark loop)."""
        return PreparedBatch(self, pairs, outs)

    def match_batch(self, pairs, params=None, refine=None, outs: Optional[List[MatchSet]] = None) -> List[MatchSet]:
        """Fused match_pointmaps (+ feature_refine when ``refine`` is given)
        over independent pairs (X_a, X_b_in_a, F_a, F_b[, init]), or over a
        PreparedBatch (then ``outs`` is the batch's own)."""
        if isinstance(pairs, PreparedBatch):
            b = pairs
            params = params or abi.default_match_params()
            self._check(self.lib.pmx_match_batch(self.h, b.mem, C.c_int32(b.n), b.arr, C.byref(params),
                                                 C.byref(refine) if refine is not None else None, b.oarr))
            return b.outs
        keep = []
        structs = []
        mem = None
        for p in pairs:
            X_a, X_b, F_a, F_b = p[:4]
            init = p[4] if len(p) > 4 else None
            m = self._mem(X_a.xyz, X_b.xyz, F_a.descriptors, F_b.descriptors)
            if mem is not None and m != mem:
                raise PmxInvalidArgument(abi.PMX_ERR_INVALID_ARGUMENT, "mixed host and device pairs")
            mem = m
            ip = None
            if init is not None:
                ist = init.struct()
                keep.append(ist)
                ip = C.pointer(ist)
            structs.append(abi.pmx_pair(X_a.struct(), X_b.struct(), F_a.struct(), F_b.struct(), ip))
        n = len(structs)
        if outs is None:
            outs = []
            for p in pairs:
                dev = p[1].xyz.device if mem == abi.PMX_MEM_DEVICE else None
                outs.append(MatchSet.empty(p[1].height * p[1].width, dev))
        arr = (abi.pmx_pair * max(1, n))(*structs)
        oarr = (abi.pmx_matchset * max(1, n))(*[o.struct() for o in outs])
        params = params or abi.default_match_params()
        self._check(self.lib.pmx_match_batch(self.h, mem if mem is not None else abi.PMX_MEM_HOST, C.c_int32(n), arr,
                                             C.byref(params), C.byref(refine) if refine is not None else None, oarr))
        return outs

    def accept_loop_edges(self, pairs, omega_l: float, params=None, refine=None, outs=None):
        """accept_loop_edge (retrieval.cpp:226-251) over candidate edges
        (X_i_i, X_j_in_i, F_i, F_j): match + refine + descriptor-agreement
        gate + valid_fraction >= omega_l.  Returns (accepted bools, gated
        MatchSets)."""
        keep, structs, mem = [], [], None
        for p in pairs:
            X_a, X_b, F_a, F_b = p[:4]
            m = self._mem(X_a.xyz, X_b.xyz, F_a.descriptors, F_b.descriptors)
            if mem is not None and m != mem:
                raise PmxInvalidArgument(abi.PMX_ERR_INVALID_ARGUMENT, "mixed host and device pairs")
            mem = m
            structs.append(abi.pmx_pair(X_a.struct(), X_b.struct(), F_a.struct(), F_b.struct(), None))
        n = len(structs)
        if outs is None:
            outs = [MatchSet.empty(p[1].height * p[1].width, p[1].xyz.device if mem == abi.PMX_MEM_DEVICE else None)
                    for p in pairs]
        arr = (abi.pmx_pair * max(1, n))(*structs)
        oarr = (abi.pmx_matchset * max(1, n))(*[o.struct() for o in outs])
        acc = (C.c_int32 * max(1, n))()
        params = params or abi.default_match_params()
        refine = refine if refine is not None else abi.default_refine_params()
        self._check(self.lib.pmx_accept_loop_edges(self.h, mem if mem is not None else abi.PMX_MEM_HOST, C.c_int32(n),
                                                   arr, C.c_double(omega_l), C.byref(params), C.byref(refine), oarr,
                                                   acc))
        return [bool(acc[i]) for i in range(n)], outs

    def ingest_pair_record(self, record, height: int, width: int, dim: int, device=None):
        """Unpack one PMPAIR01 record (pipeline.cpp:642-676; bytes / uint8
        array on the host, or a uint8 CUDA tensor) into the matcher's
        layouts.  Returns (dict of arrays / tensors, inexact fp16 count)."""
        import torch
        hw = height * width
        on_dev = isinstance(record, torch.Tensor) and record.is_cuda
        if on_dev:
            dev, rec_ptr, nbytes = record.device, record.data_ptr(), record.numel()
            mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)
        else:
            buf = np.frombuffer(record, np.uint8) if isinstance(record, (bytes, bytearray)) else np.asarray(record)
            rec_ptr, nbytes = buf.ctypes.data, buf.nbytes
            npdt = {torch.float32: np.float32, torch.uint8: np.uint8, torch.int16: np.uint16}
            mk = lambda shape, dt: np.empty(shape, npdt[dt])
        out = {"X_i": mk((hw, 3), torch.float32), "valid_i": mk((hw,), torch.uint8),
               "X_j": mk((hw, 3), torch.float32), "valid_j": mk((hw,), torch.uint8),
               "C_i": mk((hw,), torch.float32), "C_j": mk((hw,), torch.float32),
               "D_i": mk((hw, dim), torch.int16), "D_j": mk((hw, dim), torch.int16),
               "Q_i": mk((hw,), torch.float32), "Q_j": mk((hw,), torch.float32)}
        rec = abi.pmx_pair_record(*[ptr(out[k]) for k, _ in abi.pmx_pair_record._fields_])
        bad = C.c_int64()
        self._check(self.lib.pmx_ingest_pair_record(self.h, abi.PMX_MEM_DEVICE if on_dev else abi.PMX_MEM_HOST,
                                                    C.c_void_p(rec_ptr), C.c_int64(nbytes), C.c_int32(height),
                                                    C.c_int32(width), C.c_int32(dim), C.byref(rec), C.byref(bad)))
        return out, int(bad.value)

    def constrain_to_rays(self, xyz, valid, height: int, width: int, K):
        """constrain_to_rays (pipeline.cpp:32-46) in place; K: pmx_intrinsics."""
        mem = self._mem(xyz)
        self._check(self.lib.pmx_constrain_to_rays(self.h, mem, C.c_int32(height), C.c_int32(width), ptr(xyz),
                                                   ptr(valid), C.byref(K)))

    def match_stats(self, m: MatchSet, num_pixels_a: int):
        vc, uf = C.c_int64(), C.c_double()
        s = m.struct()
        self._check(self.lib.pmx_match_stats(self.h, self._mem(m.pixel_a), C.byref(s), C.c_int32(num_pixels_a),
                                             C.byref(vc), C.byref(uf)))
        return vc.value, uf.value

    def keyframe_decision(self, m: MatchSet, height: int, width: int, omega_k: float) -> bool:
        out = C.c_int32()
        s = m.struct()
        self._check(self.lib.pmx_keyframe_decision(self.h, self._mem(m.pixel_a), C.byref(s), C.c_int32(height),
                                                   C.c_int32(width), C.c_double(omega_k), C.byref(out)))
        return bool(out.value)

    # ---------------------------------------------------------- tracking
    def residual_blocks(self, T, matches: MatchSet, X_ref: Pointmap, X_src: Pointmap, mode=abi.PMX_TRACK_RAY,
                        params=None, K=None):
        n = len(matches)
        res, jac, wt, info, used = (np.zeros((n, 4)), np.zeros((n, 4, 7)), np.zeros((n, 4)), np.zeros(n),
                                    np.zeros(n, np.uint8))
        s, r, x = matches.struct(), X_ref.struct(), X_src.struct()
        params = params or abi.default_robust_weight_params()
        self._check(self.lib.pmx_residual_blocks(self.h, abi.PMX_MEM_HOST, C.byref(T), C.byref(s), C.byref(r),
                                                 C.byref(x), C.c_int(mode), C.byref(params),
                                                 C.byref(K) if K is not None else None, ptr(res), ptr(jac), ptr(wt),
                                                 ptr(info), ptr(used)))
        return res, jac, wt, info, used

    def normal_equations(self, T, matches: MatchSet, X_ref: Pointmap, X_src: Pointmap, mode=abi.PMX_TRACK_RAY,
                         params=None, K=None):
        H, g, cost, used = np.zeros((7, 7)), np.zeros(7), C.c_double(), C.c_int64()
        s, r, x = matches.struct(), X_ref.struct(), X_src.struct()
        params = params or abi.default_robust_weight_params()
        mem = self._mem(matches.pixel_a, X_ref.xyz, X_src.xyz)
        self._check(self.lib.pmx_normal_equations(self.h, mem, C.byref(T), C.byref(s), C.byref(r), C.byref(x),
                                                  C.c_int(mode), C.byref(params),
                                                  C.byref(K) if K is not None else None, ptr(H), ptr(g),
                                                  C.byref(cost), C.byref(used)))
        return H, g, cost.value, used.value

    def track_given_matches(self, canonical: Pointmap, X_f_f: Pointmap, matches: MatchSet, init,
                            mode=abi.PMX_TRACK_RAY, params=None) -> TrackResult:
        res = abi.pmx_track_result()
        c, f, m = canonical.struct(), X_f_f.struct(), matches.struct()
        params = params or abi.default_solve_pose_params()
        mem = self._mem(canonical.xyz, X_f_f.xyz, matches.pixel_a)
        self._check(self.lib.pmx_track_given_matches(self.h, mem, C.byref(c), C.byref(f), C.byref(m),
                                                     C.byref(init), C.c_int(mode), C.byref(params), C.byref(res)))
        return TrackResult(abi.pmx_sim3.from_buffer_copy(res.T_kf), res.iterations, bool(res.lost),
                           list(res.cost_trace[:res.cost_trace_len]), matches)

    def solve_pose(self, canonical: Pointmap, X_f_f: Pointmap, X_k_f: Pointmap, F_f: FeatureMap,
                   F_k: FeatureMap, init, mode=abi.PMX_TRACK_RAY, params=None,
                   match_seed: Optional[MatchSet] = None) -> TrackResult:
        res = abi.pmx_track_result()
        params = params or abi.default_solve_pose_params()
        mem = self._mem(canonical.xyz, X_f_f.xyz, X_k_f.xyz)
        dev = X_k_f.xyz.device if mem == abi.PMX_MEM_DEVICE else None
        out = MatchSet.empty(X_k_f.height * X_k_f.width, dev)
        c, f, k, ff, fk, o = (canonical.struct(), X_f_f.struct(), X_k_f.struct(), F_f.struct(), F_k.struct(),
                              out.struct())
        seed = match_seed.struct() if match_seed is not None else None
        self._check(self.lib.pmx_solve_pose(self.h, mem, C.byref(c), C.byref(f), C.byref(k), C.byref(ff), C.byref(fk),
                                            C.byref(init), C.c_int(mode), C.byref(params),
                                            C.byref(seed) if seed is not None else None, C.byref(res), C.byref(o)))
        return TrackResult(abi.pmx_sim3.from_buffer_copy(res.T_kf), res.iterations, bool(res.lost),
                           list(res.cost_trace[:res.cost_trace_len]), out)

    def fuse_canonical(self, canonical_xyz, canonical_valid, canonical_conf, X_k_f: Pointmap, confidence, T_kf,
                       height: int, width: int):
        """In place on (canonical_xyz, canonical_valid, canonical_conf)."""
        mem = self._mem(canonical_xyz, X_k_f.xyz)
        k = X_k_f.struct()
        self._check(self.lib.pmx_fuse_canonical(self.h, mem, C.c_int32(height), C.c_int32(width), ptr(canonical_xyz),
                                                ptr(canonical_valid), ptr(canonical_conf), C.byref(k),
                                                ptr(confidence), C.byref(T_kf)))

    # ----------------------------------------------------------- backend
    def _graph_mem(self, g: Graph):
        arrays = [c.xyz for c in g.canonicals] + [m.pixel_a for m in g.matches]
        return self._mem(*arrays) if arrays else abi.PMX_MEM_HOST

    def assemble_system(self, g: Graph, params=None):
        keep = []
        gs = g.struct(keep)
        dim = 7 * len(g.canonicals)
        H, grad = np.zeros((dim, dim)), np.zeros(dim)
        params = params or abi.default_backend_params()
        mem = self._graph_mem(g)
        if mem == abi.PMX_MEM_DEVICE:
            import torch
            dev = g.canonicals[0].xyz.device
            Hd = torch.empty((dim, dim), dtype=torch.float64, device=dev)
            gd = torch.empty(dim, dtype=torch.float64, device=dev)
            self._check(self.lib.pmx_assemble_system(self.h, mem, C.byref(gs), C.byref(params), ptr(Hd), ptr(gd)))
            return Hd, gd
        self._check(self.lib.pmx_assemble_system(self.h, mem, C.byref(gs), C.byref(params), ptr(H), ptr(grad)))
        return H, grad

    def backend_cost(self, g: Graph, params=None) -> float:
        keep = []
        gs = g.struct(keep)
        out = C.c_double()
        params = params or abi.default_backend_params()
        self._check(self.lib.pmx_backend_cost(self.h, self._graph_mem(g), C.byref(gs), C.byref(params), C.byref(out)))
        return out.value

    def backend_edge_terms(self, g: Graph, params=None, begin: int = 0, end: Optional[int] = None):
        keep = []
        gs = g.struct(keep)
        end = len(g.edges) if end is None else end
        out = np.zeros((end - begin, abi.PMX_EDGE_TERMS))
        params = params or abi.default_backend_params()
        mem = self._graph_mem(g)
        if mem == abi.PMX_MEM_DEVICE:
            import torch
            outd = torch.zeros((end - begin, abi.PMX_EDGE_TERMS), dtype=torch.float64,
                               device=g.canonicals[0].xyz.device)
            self._check(self.lib.pmx_backend_edge_terms(self.h, mem, C.byref(gs), C.byref(params), C.c_int32(begin),
                                                        C.c_int32(end), ptr(outd)))
            return outd
        self._check(self.lib.pmx_backend_edge_terms(self.h, mem, C.byref(gs), C.byref(params), C.c_int32(begin),
                                                    C.c_int32(end), ptr(out)))
        return out

    def backend_solve_terms(self, g: Graph, terms, params=None):
        keep = []
        gs = g.struct(keep)
        dim = 7 * len(g.canonicals)
        params = params or abi.default_backend_params()
        cost, solved = C.c_double(), C.c_int32()
        if _is_dev(terms):
            import torch
            tau = torch.zeros(dim, dtype=torch.float64, device=terms.device)
            self._check(self.lib.pmx_backend_solve_terms(self.h, abi.PMX_MEM_DEVICE, C.byref(gs), C.byref(params),
                                                         ptr(terms), ptr(tau), C.byref(cost), C.byref(solved)))
        else:
            terms = np.ascontiguousarray(terms, np.float64)
            tau = np.zeros(dim)
            self._check(self.lib.pmx_backend_solve_terms(self.h, abi.PMX_MEM_HOST, C.byref(gs), C.byref(params),
                                                         ptr(terms), ptr(tau), C.byref(cost), C.byref(solved)))
        return tau, cost.value, bool(solved.value)

    def prepare_graph(self, g: Graph, params=None, begin: int = 0, end: Optional[int] = None) -> "PreparedGraph":
        """Stage g once for repeated edge-term / solve calls at changing poses
        (edges [begin, end) compacted; the edge-sharded backend's handle)."""
        return PreparedGraph(self, g, params or abi.default_backend_params(), begin,
                             len(g.edges) if end is None else end)

    def global_optimize(self, g: Graph, params=None, trace: bool = False) -> OptimizeResult:
        keep = []
        gs = g.struct(keep)
        params = params or abi.default_backend_params()
        res = abi.pmx_optimize_result()
        n = len(g.canonicals)
        tr = (abi.pmx_sim3 * max(1, params.max_iterations * n))() if trace else None
        self._check(self.lib.pmx_global_optimize(self.h, self._graph_mem(g), C.byref(gs), C.byref(params),
                                                 C.byref(res), tr))
        g.poses = [abi.pmx_sim3.from_buffer_copy(gs.poses[k]) for k in range(n)]
        pt = []
        if trace:
            # a failed iteration (no damped solve succeeded, backend.cpp:228-230)
            # records no poses: the trace has iterations - 1 rows then
            rows = res.iterations if res.converged else max(0, res.iterations - 1)
            pt = [[abi.pmx_sim3.from_buffer_copy(tr[it * n + k]) for k in range(n)] for it in range(rows)]
        return OptimizeResult(res.iterations, bool(res.converged), list(res.cost_trace[:res.cost_trace_len]), pt)

    def ldlt_solve(self, A, b):
        A = np.ascontiguousarray(A, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(b.shape[0])
        ok = C.c_int32()
        self._check(self.lib.pmx_ldlt_solve(self.h, abi.PMX_MEM_HOST, C.c_int32(b.shape[0]), ptr(A), ptr(b), ptr(x),
                                            C.byref(ok)))
        return x, bool(ok.value)


def sim3(R=None, t=None, s=1.0) -> abi.pmx_sim3:
    T = abi.pmx_sim3()
    R = np.eye(3) if R is None else np.asarray(R, np.float64)
    for i, v in enumerate(R.reshape(-1)):
        T.R[i] = float(v)
    t = np.zeros(3) if t is None else np.asarray(t, np.float64)
    for i in range(3):
        T.t[i] = float(t[i])
    T.s = float(s)
    return T


class PreparedBatch:
    """pmx_pair / pmx_matchset arrays of one batch, built once (see
    Context.prepare_match_batch).  Holds references to every buffer."""

    def __init__(self, ctx: "Context", pairs, outs: Optional[List[MatchSet]] = None):
        self.keep = []
        structs = []
        mem = None
        for p in pairs:
            X_a, X_b, F_a, F_b = p[:4]
            init = p[4] if len(p) > 4 else None
            m = ctx._mem(X_a.xyz, X_b.xyz, F_a.descriptors, F_b.descriptors)
            if mem is not None and m != mem:
                raise PmxInvalidArgument(abi.PMX_ERR_INVALID_ARGUMENT, "mixed host and device pairs")
            mem = m
            ip = None
            if init is not None:
                ist = init.struct()
                self.keep.append(ist)
                ip = C.pointer(ist)
            structs.append(abi.pmx_pair(X_a.struct(), X_b.struct(), F_a.struct(), F_b.struct(), ip))
        self.n = len(structs)
        self.mem = mem if mem is not None else abi.PMX_MEM_HOST
        if outs is None:
            outs = [MatchSet.empty(p[1].height * p[1].width, p[1].xyz.device if self.mem == abi.PMX_MEM_DEVICE
                                   else None) for p in pairs]
        self.pairs, self.outs = list(pairs), outs
        self.arr = (abi.pmx_pair * max(1, self.n))(*structs)
        self.oarr = (abi.pmx_matchset * max(1, self.n))(*[o.struct() for o in outs])


class PreparedGraph:
    """pmx_graph_prepare handle: device-resident graph of one edge range.
    edge_terms(poses) -> (end-begin, 72) float64 CUDA tensor;
    solve(poses, terms) -> (tau (7N,) float64 CUDA tensor, cost, solved)."""

    def __init__(self, ctx: "Context", g: Graph, params, begin: int, end: int):
        import torch
        self.ctx, self.begin, self.end, self.n = ctx, begin, end, len(g.canonicals)
        self._keep = []
        gs = g.struct(self._keep)
        self._g = g
        self.device = g.canonicals[0].xyz.device if _is_dev(g.canonicals[0].xyz) else torch.device("cuda")
        h = C.c_void_p()
        ctx._check(ctx.lib.pmx_graph_prepare(ctx.h, ctx._graph_mem(g), C.byref(gs), C.byref(params), C.c_int32(begin),
                                             C.c_int32(end), C.byref(h)))
        self.h = h

    def _poses(self, poses):
        arr = (abi.pmx_sim3 * max(1, self.n))(*poses)
        self._keep_p = arr
        return arr

    def edge_terms(self, poses):
        import torch
        out = torch.empty((self.end - self.begin, abi.PMX_EDGE_TERMS), dtype=torch.float64, device=self.device)
        self.ctx._check(self.ctx.lib.pmx_graph_edge_terms(self.ctx.h, self.h, self._poses(poses), ptr(out)))
        self.ctx.synchronize()
        return out

    def solve(self, poses, terms):
        import torch
        tau = torch.empty(7 * self.n, dtype=torch.float64, device=self.device)
        cost, solved = C.c_double(), C.c_int32()
        self.ctx._check(self.ctx.lib.pmx_graph_solve(self.ctx.h, self.h, self._poses(poses), ptr(terms), ptr(tau),
                                                     C.byref(cost), C.byref(solved)))
        return tau, cost.value, bool(solved.value)

    def optimize_sharded(self, poses, params=None, trace: bool = False):
        """pmx_graph_optimize_sharded: the whole GN loop of global_optimize
        with this rank's edges, NCCL reduce / broadcast on the device.
        Returns (OptimizeResult, poses, timings {accumulate, communication,
        solve} in device ms)."""
        P = self._poses(poses)
        res = abi.pmx_optimize_result()
        mi = (params or abi.default_backend_params()).max_iterations
        tr = (abi.pmx_sim3 * max(1, mi * self.n))() if trace else None
        tm = (C.c_double * 3)()
        self.ctx._check(self.ctx.lib.pmx_graph_optimize_sharded(self.ctx.h, self.h, P, C.byref(res), tr, tm))
        rows = res.iterations if res.converged else max(0, res.iterations - 1)
        pt = [[abi.pmx_sim3.from_buffer_copy(tr[it * self.n + k]) for k in range(self.n)] for it in range(rows)] \
            if trace else []
        out = [abi.pmx_sim3.from_buffer_copy(P[k]) for k in range(self.n)]
        return (OptimizeResult(res.iterations, bool(res.converged), list(res.cost_trace[:res.cost_trace_len]), pt),
                out, {"accumulate": tm[0], "communication": tm[1], "solve": tm[2]})

    def release(self):
        if getattr(self, "h", None):
            self.ctx._check(self.ctx.lib.pmx_graph_release(self.ctx.h, self.h))
            self.h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass
