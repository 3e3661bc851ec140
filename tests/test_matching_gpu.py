"""GPU parity of iterative projective matching + refinement (reference
src/camera.cpp:39-271) against the FP64 oracle, through the C ABI.

Bar (BASELINE north_star): match indices bit-exact on >= 99.9% of valid
pixels, every mismatch within 1 px; confidences q = sqrt(Q_a Q_b) exact to
fp32 rounding.
"""
import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import (BASELINE_REFINE, baseline_match_params, compare_matches, pmx_pair, to_torch_pair)
from paper_2412_12392_b200 import FeatureMap, MatchSet, Pointmap, abi

pytestmark = pytest.mark.gpu


def _check(stats, min_equal=0.999, max_valid_mismatch_frac=1e-3):
    assert stats["worst_px"] <= 1, stats
    assert stats["index_equal_frac"] >= min_equal, stats
    assert stats["valid_mismatch"] <= max_valid_mismatch_frac * stats["n"], stats


@pytest.mark.parametrize("shape,noise", [((96, 128), "radial"), ((384, 512), "radial"), ((96, 128), "isotropic")])
def test_match_pointmaps_parity(ctx, shape, noise):
    pair = pmxgen.config0(seed=3, height=shape[0], width=shape[1], noise=noise)
    params = baseline_match_params()
    orc = pyoracle.match_pointmaps(pair, params)
    Xa, Xb, Fa, Fb = pmx_pair(pair)
    gpu = ctx.match_pointmaps(Xa, Xb, Fa, Fb, params=params)
    st = compare_matches(gpu, orc, shape[1])
    _check(st)
    # q is written even for invalid matches (camera.cpp:229-230)
    both = np.asarray(gpu.pixel_a) == orc.pixel_a
    np.testing.assert_allclose(np.asarray(gpu.confidence)[both], orc.confidence[both], rtol=1e-7)


@pytest.mark.parametrize("levels", [BASELINE_REFINE, [(2, 2), (1, 2)]])
def test_match_and_refine_parity(ctx, levels):
    pair = pmxgen.config0(seed=5)
    params = baseline_match_params()
    rp = abi.refine_params(levels)
    orc = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, params), pair, rp)
    Xa, Xb, Fa, Fb = pmx_pair(pair)
    gpu = ctx.match_batch([(Xa, Xb, Fa, Fb)], params=params, refine=rp)[0]
    _check(compare_matches(gpu, orc, pair["width"]))


def test_device_memory_path_matches_host_path(ctx):
    import torch
    pair = pmxgen.config0(seed=6, height=96, width=128)
    params = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    Xa, Xb, Fa, Fb = pmx_pair(pair)
    host = ctx.match_batch([(Xa, Xb, Fa, Fb)], params=params, refine=rp)[0]
    tp = to_torch_pair(pair)
    dXa, dXb, dFa, dFb = pmx_pair(tp)
    dev = ctx.match_batch([(dXa, dXb, dFa, dFb)], params=params, refine=rp)[0]
    torch.cuda.synchronize()
    assert np.array_equal(dev.pixel_a.cpu().numpy(), host.pixel_a)
    assert np.array_equal(dev.valid.cpu().numpy(), host.valid)
    assert np.array_equal(dev.confidence.cpu().numpy(), host.confidence)


def test_batched_pairs_equal_single_calls(ctx):
    params = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    pairs = [pmxgen.config0(seed=s, height=96, width=128) for s in (10, 11, 12)]
    batch = ctx.match_batch([pmx_pair(p) for p in pairs], params=params, refine=rp)
    for p, b in zip(pairs, batch):
        single = ctx.match_batch([pmx_pair(p)], params=params, refine=rp)[0]
        assert np.array_equal(single.pixel_a, b.pixel_a)
        assert np.array_equal(single.valid, b.valid)


def test_seeded_matching_parity(ctx):
    # camera.cpp:202-210: seed map keyed by pixel_b, last valid write wins
    pair = pmxgen.config0(seed=7, height=96, width=128)
    n = 96 * 128
    params = baseline_match_params()
    rng = np.random.default_rng(0)
    pa = rng.integers(-5, n + 5, size=n + 300).astype(np.int32)
    pb = np.concatenate([np.arange(n), rng.integers(-3, n + 3, size=300)]).astype(np.int32)
    valid = (rng.random(n + 300) < 0.8).astype(np.uint8)
    conf = np.ones(n + 300)
    orc_init = pyoracle.MatchSet(pa, pb, conf, valid)
    orc = pyoracle.match_pointmaps(pair, params, init=orc_init)
    Xa, Xb, Fa, Fb = pmx_pair(pair)
    init = MatchSet(pa, conf.astype(np.float32), valid, pb)
    gpu = ctx.match_pointmaps(Xa, Xb, Fa, Fb, init=init, params=params)
    st = compare_matches(gpu, orc, 128)
    _check(st)


def test_invalid_and_degenerate_pixels(ctx):
    # invalid b pixels -> pixel_a = -1, q = 0, invalid; zero points; NaN points
    pair = pmxgen.config0(seed=8, height=48, width=64)
    n = 48 * 64
    rng = np.random.default_rng(1)
    vb = (rng.random(n) > 0.1).astype(np.uint8)
    va = (rng.random(n) > 0.05).astype(np.uint8)
    Xb = pair["X_b"].copy()
    Xb[::97] = 0.0
    Xb[5::101] = np.nan
    pair = dict(pair, valid_a=va, valid_b=vb, X_b=Xb)
    params = baseline_match_params()
    orc = pyoracle.match_pointmaps(pair, params)
    Xa, Xb_, Fa, Fb = pmx_pair(pair)
    gpu = ctx.match_pointmaps(Xa, Xb_, Fa, Fb, params=params)
    assert np.array_equal(np.asarray(gpu.pixel_a)[vb == 0], np.full((vb == 0).sum(), -1))
    _check(compare_matches(gpu, orc, 64))
    assert np.array_equal(np.asarray(gpu.pixel_a), orc.pixel_a)


def test_gross_outliers_invalidated(ctx):
    # test_camera.cpp:177-196 on the CUDA path: 20% x3 depth outliers -> <= 2% valid
    pair = pmxgen.config0(seed=9, height=96, width=128)
    rng = np.random.default_rng(2)
    sel = rng.random(96 * 128) < 0.2
    Xb = pair["X_b"].copy()
    Xb[sel] *= 3.0
    pair = dict(pair, X_b=Xb)
    Xa, Xb_, Fa, Fb = pmx_pair(pair)
    gpu = ctx.match_pointmaps(Xa, Xb_, Fa, Fb)
    assert np.asarray(gpu.valid)[sel].mean() <= 0.02


def test_feature_refine_planted_peak_and_ties(ctx):
    # test_camera.cpp:219-247
    h, w, d = 16, 16, 8
    Fa = np.zeros((h * w, d), np.float32)
    Fb = np.zeros((h * w, d), np.float32)
    Fa[:, 1] = 1.0
    Fb[:, 0] = 1.0
    gu, gv = 8, 8
    peak = gv * w + gu + 2
    Fa[peak] = 0.0
    Fa[peak, 0] = 1.0
    q = np.ones(h * w, np.float32)
    m = MatchSet(np.array([gv * w + gu], np.int32), np.ones(1, np.float32), np.ones(1, np.uint8),
                 np.array([5 * w + 5], np.int32))
    FA = FeatureMap(Fa.astype(np.float16).view(np.uint16), q, h, w)
    FB = FeatureMap(Fb.astype(np.float16).view(np.uint16), q, h, w)
    out = ctx.feature_refine(m, FA, FB)
    assert int(out.pixel_a[0]) == peak
    flat = FeatureMap(np.full((h * w, d), 0.5, np.float16).view(np.uint16), q, h, w)
    out = ctx.feature_refine(m, flat, flat)
    assert int(out.pixel_a[0]) == gv * w + gu


def test_feature_refine_exact_near_ties(ctx):
    # candidates whose exact scores differ by one fp16 product ulp: the fp32
    # filter must defer to the exact FP64 re-check (strict '>' semantics).
    h, w, d = 12, 12, 24
    rng = np.random.default_rng(3)
    base = rng.standard_normal(d)
    base /= np.linalg.norm(base)
    Fa = np.tile(base, (h * w, 1)).astype(np.float16)
    # perturb a few pixels by one fp16 ulp in one component
    for idx in (30, 31, 42, 55, 66):
        k = idx % d
        Fa[idx, k] = np.nextafter(Fa[idx, k], np.float16(2.0))
    Fb = np.tile(base, (h * w, 1)).astype(np.float16)
    q = np.ones(h * w, np.float32)
    n = h * w
    pa = np.arange(n, dtype=np.int32)
    m = MatchSet(pa, np.ones(n, np.float32), np.ones(n, np.uint8), pa.copy())
    pair = {"D_a": Fa.view(np.uint16), "D_b": Fb.view(np.uint16), "Q_a": q, "Q_b": q, "height": h, "width": w}
    for levels in ([(1, 3), (1, 3)], [(2, 2), (1, 2)]):
        rp = abi.refine_params(levels)
        gpu = ctx.feature_refine(m, FeatureMap(pair["D_a"], q, h, w), FeatureMap(pair["D_b"], q, h, w), rp)
        orc = pyoracle.feature_refine(pyoracle.MatchSet(pa, pa, np.ones(n), np.ones(n, np.uint8)), pair, rp)
        assert np.array_equal(np.asarray(gpu.pixel_a), orc.pixel_a)


def test_iterative_project_parity(ctx):
    pair = pmxgen.config0(seed=4, height=96, width=128)
    h, w = 96, 128
    rng = np.random.default_rng(4)
    idx = rng.integers(0, h * w, 2000)
    x = pair["X_b"][idx]
    p0 = np.stack([idx % w + rng.uniform(-6, 6, idx.size), idx // w + rng.uniform(-6, 6, idx.size)], 1)
    params = baseline_match_params().projection
    pix_o, conv_o, it_o = pyoracle.iterative_project(pair["X_a"], None, h, w, x, p0, params)
    pm = Pointmap(pair["X_a"], None, h, w)
    pix_g, conv_g, it_g = ctx.iterative_project(pm, x, p0, params)
    assert (conv_g == conv_o).mean() >= 0.999
    assert (it_g == it_o).mean() >= 0.999
    same = conv_g == conv_o
    np.testing.assert_allclose(pix_g[same], pix_o[same], atol=1e-9)


def test_normalize_rays_parity(ctx):
    pair = pmxgen.config0(seed=2, height=48, width=64)
    X = pair["X_a"].copy()
    X[3] = 0.0
    X[7] = np.inf
    valid = np.ones(48 * 64, np.uint8)
    valid[11] = 0
    r_o, d_o, v_o = pyoracle.normalize_rays(X, valid, 48, 64)
    r_g, d_g, v_g = ctx.normalize_rays(Pointmap(X, valid, 48, 64))
    assert np.array_equal(v_g, v_o)
    assert np.array_equal(r_g, r_o)  # bit-exact: same FP64 ops, IEEE div / sqrt
    assert np.array_equal(d_g[v_o == 1], d_o[v_o == 1])


def test_match_stats_and_keyframe_decision(ctx):
    # camera.cpp:10-28, tracking.cpp:249-257 (test_tracking.cpp:381+)
    h, w = 10, 10
    full = MatchSet(np.arange(100, dtype=np.int32), np.ones(100, np.float32), np.ones(100, np.uint8),
                    np.arange(100, dtype=np.int32))
    assert not ctx.keyframe_decision(full, h, w, 0.333)
    sparse = MatchSet(np.arange(30, dtype=np.int32), np.ones(30, np.float32), np.ones(30, np.uint8),
                      np.arange(30, dtype=np.int32))
    assert ctx.keyframe_decision(sparse, h, w, 0.333)
    collapsed = MatchSet(np.zeros(90, np.int32), np.ones(90, np.float32), np.ones(90, np.uint8),
                         np.arange(90, dtype=np.int32))
    assert ctx.keyframe_decision(collapsed, h, w, 0.333)
    rng = np.random.default_rng(5)
    pa = rng.integers(-2, 120, 500).astype(np.int32)
    v = (rng.random(500) < 0.7).astype(np.uint8)
    m = MatchSet(pa, np.ones(500, np.float32), v, np.arange(500, dtype=np.int32))
    vc, uf = ctx.match_stats(m, 100)
    vo, uo = pyoracle.match_stats(pyoracle.MatchSet(pa, np.arange(500), np.ones(500), v), 100)
    assert vc == vo and uf == uo


def _fused_vs_oracle(ctx, pairs, levels=BASELINE_REFINE, exact=True):
    params = baseline_match_params()
    rp = abi.refine_params(levels)
    gpu = ctx.match_batch([pmx_pair(p) for p in pairs], params=params, refine=rp)
    for p, g in zip(pairs, gpu):
        orc = pyoracle.feature_refine(pyoracle.match_pointmaps(p, params), p, rp)
        st = compare_matches(g, orc, p["width"])
        _check(st)
        if exact:
            assert st["all_index_equal"], st


def test_fused_refine_descriptor_overflow_takes_exact_path(ctx):
    # |descriptor| > 1 + 2^-8 has no exact int8 image: the whole pair takes the
    # exact path of the fused kernel (qbad), same results
    pair = pmxgen.config0(seed=31, height=48, width=64)
    big = dict(pair)
    big["D_a"] = (pair["D_a"].view(np.float16) * np.float16(3.0)).view(np.uint16)
    big["D_b"] = (pair["D_b"].view(np.float16) * np.float16(3.0)).view(np.uint16)
    _fused_vs_oracle(ctx, [big, pair])


def test_fused_refine_flat_descriptors_all_ties(ctx):
    # every candidate ties: no pixel is decided by the integer scores; the
    # exact path keeps the centre (strict '>' scan, camera.cpp:250-263)
    pair = pmxgen.config0(seed=32, height=48, width=64)
    flat = dict(pair)
    one = np.zeros_like(pair["D_a"].view(np.float16))
    one[:, 0] = np.float16(1.0)
    flat["D_a"] = one.view(np.uint16)
    flat["D_b"] = one.copy().view(np.uint16)
    _fused_vs_oracle(ctx, [flat])


@pytest.mark.parametrize("dim", [16, 32])
def test_fused_refine_other_descriptor_dims(ctx, dim):
    # no int8 fast path for dim != 24: per-pixel exact refinement in the same kernel
    pair = pmxgen.config0(seed=33, height=48, width=64)
    rng = np.random.default_rng(dim)
    for k in ("D_a", "D_b"):
        d = rng.normal(size=(48 * 64, dim))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pair[k] = d.astype(np.float16).view(np.uint16)
    pair["D_b"] = pair["D_a"].copy()  # b descriptors equal the a ones at the same pixel
    _fused_vs_oracle(ctx, [pair])


def test_ragged_batch_mixed_sizes(ctx):
    # pairs of different sizes (and a < b grids) in one batch: scratch and tiles by the largest
    pairs = [pmxgen.config0(seed=34, height=48, width=64), pmxgen.config0(seed=35, height=96, width=128),
             pmxgen.config0(seed=36, height=24, width=32)]
    a = pmxgen.config0(seed=37, height=48, width=64)
    b = pmxgen.config0(seed=37, height=40, width=56)
    mixed = dict(a)  # X_b / F_b on a smaller grid than X_a / F_a
    for k in ("X_b", "valid_b", "D_b", "Q_b"):
        mixed[k] = b[k]
    mixed["height_b"], mixed["width_b"] = 40, 56
    _fused_vs_oracle(ctx, pairs)
    params = baseline_match_params()
    rp = abi.refine_params(BASELINE_REFINE)
    from paper_2412_12392_b200 import FeatureMap, Pointmap
    Xa = Pointmap(mixed["X_a"], mixed["valid_a"], 48, 64)
    Xb = Pointmap(mixed["X_b"], mixed["valid_b"], 40, 56)
    Fa = FeatureMap(mixed["D_a"], mixed["Q_a"], 48, 64)
    Fb = FeatureMap(mixed["D_b"], mixed["Q_b"], 40, 56)
    g = ctx.match_batch([(Xa, Xb, Fa, Fb)] + [pmx_pair(p) for p in pairs[:1]], params=params, refine=rp)
    assert len(g[0].pixel_a) == 40 * 56 and np.asarray(g[0].pixel_a).max() < 48 * 64
    ok = np.asarray(g[0].valid).astype(bool)
    assert ok.mean() > 0.2  # an unrelated view still matches its geometric neighbourhood


def test_empty_batch_and_all_invalid_pair(ctx):
    assert ctx.match_batch([], params=baseline_match_params()) == []
    pair = pmxgen.config0(seed=38, height=24, width=32)
    dead = dict(pair, valid_a=np.zeros_like(pair["valid_a"]), valid_b=np.zeros_like(pair["valid_b"]))
    g = ctx.match_batch([pmx_pair(dead)], params=baseline_match_params(), refine=abi.refine_params(BASELINE_REFINE))[0]
    assert not np.asarray(g.valid).any() and (np.asarray(g.pixel_a) == -1).all()


def _sphere_points(n, radius, seed):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return (radius * d).astype(np.float32)


@pytest.mark.parametrize("case", ["config0", "sphere_ties", "even_count", "with_invalid", "empty"])
def test_median_scene_distance_exact(ctx, case):
    """median_scene_distance (camera.cpp:178-191) is the FP64 rank-floor(n/2)
    norm; the device selects it exactly, including many FP64 norms that share
    one fp32 key (points on a sphere: > 64 ties, the bisection path)."""
    h, w = 96, 128
    valid = None
    if case == "config0":
        xyz = pmxgen.config0(seed=8, height=h, width=w)["X_a"]
    elif case in ("sphere_ties", "even_count"):
        xyz = _sphere_points(h * w, 2.0, 9)
        if case == "even_count":
            valid = np.ones(h * w, np.uint8)
            valid[::97] = 0
    elif case == "with_invalid":
        xyz = pmxgen.config0(seed=10, height=h, width=w)["X_a"].copy()
        valid = (np.arange(h * w) % 3 != 0).astype(np.uint8)
        xyz[::5] = 0.0  # |p| < 1e-12 is excluded too
    else:
        xyz = np.zeros((h * w, 3), np.float32)
    got = ctx.median_scene_distance(Pointmap(xyz, valid, h, w))
    want = pyoracle.median_scene_distance(xyz, valid, h, w)
    assert got == want, (got, want)


def test_interpolate_ray_entry(ctx):
    pair = pmxgen.config0(seed=12, height=96, width=128)
    rng = np.random.default_rng(1)
    p = np.c_[rng.uniform(-1, 128, 3000), rng.uniform(-1, 96, 3000)]
    p[:20] = np.floor(p[:20])
    p[20:30, 0] = 127.0
    ray, J, ok = ctx.interpolate_ray(Pointmap(pair["X_a"], pair["valid_a"], 96, 128), p)
    with (pyoracle.reference() if pyoracle.have_reference() else _nullctx()):
        oray, oJ, ook = pyoracle.interpolate_ray(pair["X_a"], pair["valid_a"], 96, 128, p)
    assert np.array_equal(ok, ook) and ok.sum() > 2000
    np.testing.assert_allclose(ray[ok == 1], oray[ook == 1], rtol=0, atol=4e-16)
    np.testing.assert_allclose(J[ok == 1], oJ[ook == 1], rtol=1e-12, atol=1e-14)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.mark.parametrize("shapes", [[(37, 53)], [(9, 7), (2, 33), (1, 40)], [(37, 53), (31, 33), (9, 7)]])
def test_odd_sizes_match_and_refine(ctx, shapes):
    """Odd and tiny images (widths not multiples of the 32-pixel tile, odd
    pixel counts so the int8 image slots sit at odd offsets, windows that
    cross every border, a one-row image) through the fused batch kernel, in
    one batch: same indices / validity as the reference restatement."""
    pairs = [pmxgen.config0(seed=41 + i, height=h, width=w) for i, (h, w) in enumerate(shapes)]
    params, rp = baseline_match_params(), abi.refine_params(BASELINE_REFINE)
    gpu = ctx.match_batch([pmx_pair(p) for p in pairs], params=params, refine=rp)
    for g, p in zip(gpu, pairs):
        orc = pyoracle.feature_refine(pyoracle.match_pointmaps(p, params), p, rp)
        st = compare_matches(g, orc, p["width"])
        assert st["all_index_equal"] and st["valid_mismatch"] == 0, (p["height"], p["width"], st)


@pytest.mark.parametrize("shape", [(96, 128), (384, 512)])
def test_reference_default_parameters_parity(ctx, shape):
    """The reference's own defaults (LM lambda 1e-4, angle tol 1e-5 rad,
    refine levels {(2,2),(1,2)}; inc/camera.hpp:103-107, 142) rather than the
    BASELINE schedule: same indices / validity as the restatement."""
    pair = pmxgen.config0(seed=17, height=shape[0], width=shape[1])
    params, rp = abi.default_match_params(), abi.default_refine_params()
    orc = pyoracle.feature_refine(pyoracle.match_pointmaps(pair, params), pair, rp)
    gpu = ctx.match_batch([pmx_pair(pair)], params=params, refine=rp)[0]
    _check(compare_matches(gpu, orc, shape[1]))
