"""ctypes mirror of include/pmx.h (the C-ABI drop-in boundary).

The structs here are byte-for-byte the POD types of ``include/pmx.h``; the
loader binds ``paper_2412_12392_b200/csrc/libpmx_cuda.so`` (built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2412_12392_b200/csrc``) and
fails loudly when it is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMX_LIB (dev only): load a variant build of the library instead (tools/variants.sh)
LIB_PATH = os.environ.get("PMX_LIB") or os.path.join(_HERE, "csrc", "libpmx_cuda.so")

PMX_OK = 0
PMX_ERR_INVALID_ARGUMENT = 1
PMX_ERR_DOMAIN = 2
PMX_ERR_CUDA = 3
PMX_ERR_NO_DEVICE = 4
PMX_ERR_OUT_OF_MEMORY = 5
PMX_ERR_NCCL = 6

PMX_MEM_HOST = 0
PMX_MEM_DEVICE = 1

PMX_TRACK_RAY = 0
PMX_TRACK_POINT = 1
PMX_TRACK_PIXEL = 2

PMX_MAX_REFINE_LEVELS = 8
PMX_MAX_TRACE = 64
PMX_EDGE_TERMS = 72


class pmx_pointmap(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32),
                ("xyz", C.c_void_p), ("valid", C.c_void_p)]


class pmx_featuremap(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("dim", C.c_int32),
                ("descriptors", C.c_void_p), ("match_confidence", C.c_void_p)]


class pmx_matchset(C.Structure):
    _fields_ = [("count", C.c_int64), ("pixel_a", C.c_void_p), ("pixel_b", C.c_void_p),
                ("confidence", C.c_void_p), ("valid", C.c_void_p)]


class orc_matchset(C.Structure):  # oracle/oracle_capi.h (FP64 confidences)
    _fields_ = [("count", C.c_int64), ("pixel_a", C.c_void_p), ("pixel_b", C.c_void_p),
                ("confidence", C.c_void_p), ("valid", C.c_void_p)]


class pmx_sim3(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("s", C.c_double)]


class pmx_iter_proj_params(C.Structure):
    _fields_ = [("lambda_init", C.c_double), ("lambda_up", C.c_double),
                ("lambda_down", C.c_double), ("angle_tol", C.c_double),
                ("max_iterations", C.c_int32)]


class pmx_match_params(C.Structure):
    _fields_ = [("projection", pmx_iter_proj_params),
                ("invalidation_median_fraction", C.c_double)]


class pmx_refine_params(C.Structure):
    _fields_ = [("num_levels", C.c_int32),
                ("stride", C.c_int32 * PMX_MAX_REFINE_LEVELS),
                ("radius", C.c_int32 * PMX_MAX_REFINE_LEVELS)]


class pmx_intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double)]


class pmx_robust_weight_params(C.Structure):
    _fields_ = [("sigma2_point", C.c_double), ("sigma2_ray", C.c_double),
                ("sigma2_pixel", C.c_double), ("q_min", C.c_double),
                ("q_min_fraction", C.c_double), ("huber_delta", C.c_double),
                ("distance_weight", C.c_double)]


class pmx_solve_pose_params(C.Structure):
    _fields_ = [("weights", pmx_robust_weight_params), ("matching", pmx_match_params),
                ("refinement", pmx_refine_params), ("refine_features", C.c_int32),
                ("max_iterations", C.c_int32), ("update_tol", C.c_double),
                ("min_valid_matches", C.c_int32), ("has_intrinsics", C.c_int32),
                ("intrinsics", pmx_intrinsics)]


class pmx_track_result(C.Structure):
    _fields_ = [("T_kf", pmx_sim3), ("iterations", C.c_int32), ("lost", C.c_int32),
                ("cost_trace_len", C.c_int32), ("cost_trace", C.c_double * PMX_MAX_TRACE)]


class pmx_backend_params(C.Structure):
    _fields_ = [("weights", pmx_robust_weight_params), ("mode", C.c_int32),
                ("has_intrinsics", C.c_int32), ("intrinsics", pmx_intrinsics),
                ("max_iterations", C.c_int32), ("update_tol", C.c_double),
                ("damping_init", C.c_double), ("damping_retries", C.c_int32)]


class pmx_graph(C.Structure):
    _fields_ = [("num_keyframes", C.c_int32), ("canonicals", C.POINTER(pmx_pointmap)),
                ("poses", C.POINTER(pmx_sim3)), ("anchor_index", C.c_int32),
                ("num_edges", C.c_int32), ("edge_i", C.c_void_p), ("edge_j", C.c_void_p),
                ("edge_matches", C.POINTER(pmx_matchset))]


class orc_graph(C.Structure):
    _fields_ = [("num_keyframes", C.c_int32), ("canonicals", C.POINTER(pmx_pointmap)),
                ("poses", C.POINTER(pmx_sim3)), ("anchor_index", C.c_int32),
                ("num_edges", C.c_int32), ("edge_i", C.c_void_p), ("edge_j", C.c_void_p),
                ("edge_matches", C.POINTER(orc_matchset))]


class pmx_optimize_result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("cost_trace_len", C.c_int32), ("cost_trace", C.c_double * PMX_MAX_TRACE)]


class pmx_pair(C.Structure):
    _fields_ = [("X_a", pmx_pointmap), ("X_b_in_a", pmx_pointmap),
                ("F_a", pmx_featuremap), ("F_b", pmx_featuremap),
                ("init", C.POINTER(pmx_matchset))]


class pmx_pair_record(C.Structure):  # PMPAIR01 record unpacked (pipeline.cpp:642-676)
    _fields_ = [("X_i", C.c_void_p), ("valid_i", C.c_void_p), ("X_j", C.c_void_p), ("valid_j", C.c_void_p),
                ("C_i", C.c_void_p), ("C_j", C.c_void_p), ("D_i", C.c_void_p), ("D_j", C.c_void_p),
                ("Q_i", C.c_void_p), ("Q_j", C.c_void_p)]


# Every symbol include/pmx.h declares (checked by tests/test_abi.py).
PMX_SYMBOLS = [
    "pmx_default_match_params", "pmx_default_refine_params",
    "pmx_default_robust_weight_params", "pmx_default_solve_pose_params",
    "pmx_default_backend_params", "pmx_sim3_identity", "pmx_abi_version",
    "pmx_create", "pmx_destroy", "pmx_last_error", "pmx_set_stream", "pmx_get_stream",
    "pmx_synchronize", "pmx_kernel_launch_count", "pmx_normalize_rays", "pmx_interpolate_ray",
    "pmx_median_scene_distance",
    "pmx_iterative_project", "pmx_match_pointmaps", "pmx_feature_refine",
    "pmx_match_batch", "pmx_match_stats", "pmx_keyframe_decision",
    "pmx_residual_blocks", "pmx_normal_equations", "pmx_track_given_matches",
    "pmx_solve_pose", "pmx_fuse_canonical", "pmx_assemble_system", "pmx_backend_cost",
    "pmx_global_optimize", "pmx_backend_edge_terms", "pmx_backend_solve_terms",
    "pmx_ldlt_solve", "pmx_profile_enable", "pmx_profile_reset", "pmx_profile_get",
    "pmx_sim3_retract", "pmx_sim3_relative", "pmx_accept_loop_edges", "pmx_ingest_pair_record",
    "pmx_constrain_to_rays", "pmx_graph_prepare", "pmx_graph_edge_terms", "pmx_graph_solve",
    "pmx_graph_release", "pmx_set_device_graphs", "pmx_nccl_unique_id", "pmx_nccl_init",
    "pmx_graph_optimize_sharded",
]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpmx_cuda.so.  Raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"pmx CUDA extension not built: {path} is missing "
            "(run __graft_entry__.build() or make -C paper_2412_12392_b200/csrc)")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    lib.pmx_last_error.restype = C.c_char_p
    lib.pmx_get_stream.restype = C.c_void_p
    lib.pmx_kernel_launch_count.restype = C.c_int64
    lib.pmx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.pmx_accept_loop_edges.argtypes = [C.c_void_p, C.c_int, C.c_int32, C.c_void_p, C.c_double, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p]
    lib.pmx_ingest_pair_record.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                           C.c_int32, C.c_void_p, C.POINTER(C.c_int64)]
    lib.pmx_graph_prepare.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                      C.POINTER(C.c_void_p)]
    lib.pmx_graph_edge_terms.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.pmx_graph_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    lib.pmx_graph_release.argtypes = [C.c_void_p, C.c_void_p]
    lib.pmx_constrain_to_rays.argtypes = [C.c_void_p, C.c_int, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    for name in PMX_SYMBOLS:
        if os.environ.get("PMX_LIB") and not hasattr(lib, name):
            continue  # dev variant builds of older sources may lack newer entries
        fn = getattr(lib, name)
        if name not in ("pmx_last_error", "pmx_get_stream", "pmx_kernel_launch_count",
                        "pmx_create") and not name.startswith("pmx_default") \
                and name != "pmx_sim3_identity":
            fn.restype = C.c_int
    if path == LIB_PATH:
        _lib = lib
    return lib


def default_match_params() -> pmx_match_params:
    p = pmx_match_params()
    p.projection.lambda_init = 1e-4
    p.projection.lambda_up = 10.0
    p.projection.lambda_down = 0.3
    p.projection.angle_tol = 1e-5
    p.projection.max_iterations = 10
    p.invalidation_median_fraction = 0.1
    return p


def refine_params(levels) -> pmx_refine_params:
    p = pmx_refine_params()
    p.num_levels = len(levels)
    for i, (s, r) in enumerate(levels):
        p.stride[i] = s
        p.radius[i] = r
    return p


def default_refine_params() -> pmx_refine_params:
    return refine_params([(2, 2), (1, 2)])  # camera.hpp:142


def default_robust_weight_params() -> pmx_robust_weight_params:
    return pmx_robust_weight_params(1e-2, 1e-3, 4.0, 0.0, 0.1, 1.345, 0.01)  # tracking.hpp:26-34


def default_solve_pose_params() -> pmx_solve_pose_params:
    p = pmx_solve_pose_params()
    p.weights = default_robust_weight_params()
    p.matching = default_match_params()
    p.refinement = default_refine_params()
    p.refine_features = 1
    p.max_iterations = 20
    p.update_tol = 1e-6
    p.min_valid_matches = 12
    p.has_intrinsics = 0
    return p


def default_backend_params() -> pmx_backend_params:
    p = pmx_backend_params()
    p.weights = default_robust_weight_params()
    p.mode = PMX_TRACK_RAY
    p.has_intrinsics = 0
    p.max_iterations = 10
    p.update_tol = 1e-6
    p.damping_init = 1e-6
    p.damping_retries = 3
    return p


# ------------------------------------------------------------ struct helpers

def ptr(a):
    """Address of a numpy array or torch tensor as a c_void_p (None -> NULL).
    (A bare Python int would be passed to C as a 32-bit int.)"""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def pointmap(xyz, valid, height: int, width: int) -> pmx_pointmap:
    return pmx_pointmap(height, width, ptr(xyz), ptr(valid))


def featuremap(desc, conf, height: int, width: int, dim: int) -> pmx_featuremap:
    return pmx_featuremap(height, width, dim, ptr(desc), ptr(conf))


def matchset(pixel_a, pixel_b, conf, valid, count=None, cls=pmx_matchset):
    n = count if count is not None else int(pixel_a.shape[0])
    return cls(n, ptr(pixel_a), ptr(pixel_b), ptr(conf), ptr(valid))
