"""CPU checks of the drop-in boundary: libpmx_cuda.so loads without a GPU,
exports every symbol include/pmx.h declares, the ctypes mirror matches the
header, and the product fails loudly (no CPU fallback) without a device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2412_12392_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pmx.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmx_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(abi.LIB_PATH):
        subprocess.check_call(["make", "-s", "-j8", "-C", os.path.dirname(abi.LIB_PATH)])
    return abi.load_library()


def test_header_and_python_mirror_agree():
    assert header_symbols() == sorted(abi.PMX_SYMBOLS)


def test_library_exports_every_header_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pmx_[a-z0-9_]+)", out))
    assert set(header_symbols()) <= exported


def test_struct_layouts_match_c():
    # sizes of the POD structs as the C compiler lays them out
    src = "#include <stdio.h>\n#include \"pmx.h\"\nint main(){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\"," \
          "sizeof(pmx_pointmap),sizeof(pmx_featuremap),sizeof(pmx_matchset),sizeof(pmx_sim3)," \
          "sizeof(pmx_solve_pose_params),sizeof(pmx_track_result),sizeof(pmx_backend_params)," \
          "sizeof(pmx_graph),sizeof(pmx_pair));}"
    exe = "/tmp/pmx_sizes"
    subprocess.run(["gcc", "-x", "c", "-I", os.path.dirname(HEADER), "-o", exe, "-"], input=src, text=True,
                   check=True)
    got = [int(x) for x in subprocess.check_output([exe]).split()]
    want = [C.sizeof(t) for t in (abi.pmx_pointmap, abi.pmx_featuremap, abi.pmx_matchset, abi.pmx_sim3,
                                 abi.pmx_solve_pose_params, abi.pmx_track_result, abi.pmx_backend_params,
                                 abi.pmx_graph, abi.pmx_pair)]
    assert got == want


def test_defaults_match_reference(lib):
    p = abi.pmx_match_params()
    lib.pmx_default_match_params(C.byref(p))
    assert (p.projection.lambda_init, p.projection.angle_tol, p.projection.max_iterations,
            p.invalidation_median_fraction) == (1e-4, 1e-5, 10, 0.1)  # camera.hpp:102-131
    r = abi.pmx_refine_params()
    lib.pmx_default_refine_params(C.byref(r))
    assert r.num_levels == 2 and list(r.stride[:2]) == [2, 1] and list(r.radius[:2]) == [2, 2]  # camera.hpp:142
    b = abi.pmx_backend_params()
    lib.pmx_default_backend_params(C.byref(b))
    assert (b.max_iterations, b.update_tol, b.damping_init, b.damping_retries) == (10, 1e-6, 1e-6, 3)
    assert b.weights.distance_weight == 0.01 and b.weights.huber_delta == 1.345  # tracking.hpp:26-34


def test_host_sim3_helpers_match_oracle(lib):
    import pyoracle
    tau = np.array([0.1, -0.2, 0.3, 0.2, -0.1, 0.05, 0.3])
    T = pyoracle.sim3_exp(np.array([0.5, 0.1, -0.2, 0.3, 0.2, -0.4, 0.1]))
    out = abi.pmx_sim3()
    lib.pmx_sim3_retract(C.byref(T), abi.ptr(tau), C.byref(out))
    ref = pyoracle.sim3_compose(pyoracle.sim3_exp(tau), T)
    np.testing.assert_allclose(list(out.R), list(ref.R), atol=1e-14)
    np.testing.assert_allclose(list(out.t), list(ref.t), atol=1e-14)
    lib.pmx_sim3_relative(C.byref(T), C.byref(ref), C.byref(out))
    rel = pyoracle.sim3_compose(pyoracle.sim3_inverse(T), ref)
    np.testing.assert_allclose(list(out.t), list(rel.t), atol=1e-13)


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    assert lib.pmx_create(0, C.byref(h)) == abi.PMX_ERR_NO_DEVICE
    from paper_2412_12392_b200 import Context, PmxError
    with pytest.raises(PmxError):
        Context(0)


def test_missing_extension_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="not built"):
        abi.load_library(str(tmp_path / "libpmx_cuda.so"))
