"""The rows SURVEY §8(f) ranks next to the hot path:

  * accept_loop_edge (reference src/retrieval.cpp:226-251): the caller of
    batched matching for loop edges — match + refine + descriptor-agreement
    gate + valid_fraction >= omega_l;
  * PMPAIR01 pair records (src/pipeline.cpp:510-676): the stream format that
    feeds the path, unpacked on the device;
  * constrain_to_rays (src/pipeline.cpp:32-46): the calibrated-mode transform
    applied to pointmaps before they reach the path.

CPU tests pin the numpy restatements (oracle/pyoracle.py) by known answers;
GPU tests compare the CUDA path with them through the C ABI.
"""
import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import BASELINE_REFINE, baseline_match_params, pmx_pair
from paper_2412_12392_b200 import abi


def _record_inputs(seed=7, h=24, w=32, dim=24):
    rng = np.random.default_rng(seed)
    hw = h * w
    X_i = rng.normal(size=(hw, 3)).astype(np.float32)
    X_j = rng.normal(size=(hw, 3)).astype(np.float32)
    X_i[3, 1] = np.nan  # non-finite points are invalid (allFinite)
    X_j[5, 2] = np.inf
    D = rng.normal(size=(2, hw, dim)).astype(np.float16).astype(np.float32)  # fp16-exact descriptors
    C = rng.uniform(1, 10, size=(4, hw)).astype(np.float32)
    return dict(X_i=X_i, X_j=X_j, C_i=C[0], C_j=C[1], D_i=D[0], D_j=D[1], Q_i=C[2], Q_j=C[3]), h, w, dim


def test_pair_record_roundtrip_oracle():
    inp, h, w, dim = _record_inputs()
    rec = pyoracle.write_pair_record(**inp)
    assert rec[:8] == b"PMPAIR01" and len(rec) == 8 + 4 * h * w * (3 + 3 + 1 + 1 + dim + dim + 1 + 1)
    out = pyoracle.read_pair_record(rec, h, w, dim)
    for k, v in inp.items():
        np.testing.assert_array_equal(out[k], v)
    assert out["valid_i"][3] == 0 and out["valid_j"][5] == 0 and out["valid_i"].sum() == h * w - 1
    with pytest.raises(ValueError):
        pyoracle.read_pair_record(b"PMENC001" + rec[8:], h, w, dim)
    with pytest.raises(ValueError):
        pyoracle.read_pair_record(rec[:-4], h, w, dim)


def test_constrain_to_rays_oracle_known_answer():
    K = abi.pmx_intrinsics(2.0, 4.0, 1.0, 0.5)
    xyz = np.array([[9, 9, 2.0], [9, 9, -1.0], [9, 9, 3.0], [7, 7, 1.0]], np.float32)
    valid = np.array([1, 1, 0, 1], np.uint8)
    out, v = pyoracle.constrain_to_rays(xyz, valid, 2, 2, K)
    # pixel (u, v): 0 -> (0, 0), 3 -> (1, 1); z * ((u - cx) / fx, (v - cy) / fy, 1)
    np.testing.assert_array_equal(out[0], np.float32([2 * (0 - 1) / 2, 2 * (0 - 0.5) / 4, 2]))
    np.testing.assert_array_equal(out[3], np.float32([1 * (1 - 1) / 2, 1 * (1 - 0.5) / 4, 1]))
    assert list(v) == [1, 0, 0, 1]
    np.testing.assert_array_equal(out[1], xyz[1])  # z <= 0: invalidated, untouched
    np.testing.assert_array_equal(out[2], xyz[2])  # invalid: untouched


def test_accept_loop_edge_oracle_gate():
    pair = pmxgen.config0(seed=11, height=48, width=64)
    params = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    ok, m = pyoracle.accept_loop_edge(pair, 0.5, params, rp)
    base = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, params), pair, rp)
    assert ok and m.valid.sum() <= base.valid.sum()
    # a pair whose b descriptors are all zero disagrees everywhere: no match survives
    bad = dict(pair)
    bad["D_b"] = np.zeros_like(pair["D_b"])
    ok2, m2 = pyoracle.accept_loop_edge(bad, 0.01, params, rp)
    assert not ok2 and m2.valid.sum() == 0


@pytest.mark.gpu
def test_accept_loop_edges_gpu_parity(ctx):
    params = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    pairs = [pmxgen.config0(seed=s, height=96, width=128) for s in (21, 22)]
    bad = dict(pairs[1])
    bad["D_b"] = np.zeros_like(pairs[1]["D_b"])
    pairs.append(bad)
    acc, outs = ctx.accept_loop_edges([pmx_pair(p) for p in pairs], 0.5, params, rp)
    for p, a, o in zip(pairs, acc, outs):
        ok, m = pyoracle.accept_loop_edge(p, 0.5, params, rp)
        assert a == ok
        np.testing.assert_array_equal(np.asarray(o.valid), m.valid)
        v = m.valid.astype(bool)
        np.testing.assert_array_equal(np.asarray(o.pixel_a)[v], m.pixel_a[v])
    assert acc[:2] == [True, True] and acc[2] is False


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_ingest_pair_record_gpu(ctx, on_device):
    import torch
    inp, h, w, dim = _record_inputs(seed=3)
    inp["D_j"][7, 2] = np.float32(0.1)  # not fp16-representable: counted
    rec = pyoracle.write_pair_record(**inp)
    ref = pyoracle.read_pair_record(rec, h, w, dim)
    src = torch.frombuffer(bytearray(rec), dtype=torch.uint8).cuda() if on_device else rec
    out, inexact = ctx.ingest_pair_record(src, h, w, dim)
    get = (lambda t: t.cpu().numpy()) if on_device else (lambda t: t)
    assert inexact == 1
    for k in ("X_i", "X_j", "C_i", "C_j", "Q_i", "Q_j", "valid_i", "valid_j"):
        np.testing.assert_array_equal(get(out[k]), ref[k], err_msg=k)
    for k in ("D_i", "D_j"):
        np.testing.assert_array_equal(get(out[k]).view(np.float16), ref[k].astype(np.float16), err_msg=k)


@pytest.mark.gpu
def test_constrain_to_rays_gpu():
    import torch
    from paper_2412_12392_b200 import Context
    ctx = Context(0)
    pair = pmxgen.config0(seed=4, height=48, width=64)
    K = abi.pmx_intrinsics(400.0 * 64 / 512, 400.0 * 64 / 512, 32.0, 24.0)
    xyz = pair["X_a"].copy()
    xyz[::7, 2] *= -1  # some non-positive depths
    valid = pair["valid_a"].copy()
    ref_xyz, ref_v = pyoracle.constrain_to_rays(xyz, valid, 48, 64, K)
    hx, hv = xyz.copy(), valid.copy()
    ctx.constrain_to_rays(hx, hv, 48, 64, K)  # host memory path
    np.testing.assert_array_equal(hx.reshape(-1, 3), ref_xyz)
    np.testing.assert_array_equal(hv, ref_v)
    dx, dv = torch.from_numpy(xyz.copy()).cuda(), torch.from_numpy(valid.copy()).cuda()
    ctx.constrain_to_rays(dx, dv, 48, 64, K)  # device path
    np.testing.assert_array_equal(dx.cpu().numpy().reshape(-1, 3), ref_xyz)
    np.testing.assert_array_equal(dv.cpu().numpy(), ref_v)
    ctx.close()
