"""The host-buffer matching path (PMX_MEM_HOST, run_match_batch): pipelined
chunk schedule (full chunks, then 4/2/1/1-style halving), DMA for the large
arrays and, for pinned device-mapped host memory, the SM copy kernel
(k_copy_segs) for valid masks and confidences - including arrays at odd byte
offsets.  Outputs must equal the device-resident path and the pageable host
path bit for bit (same kernels on the same bytes)."""
import numpy as np
import pytest

import pmxgen
from helpers import BASELINE_REFINE, baseline_match_params, to_torch_pair
from paper_2412_12392_b200 import FeatureMap, MatchSet, Pointmap, abi

pytestmark = pytest.mark.gpu
H, W = 96, 128


def _pairs(n):
    sc, poses, edges, mk = pmxgen.config2(seed=5, height=H, width=W)
    return [mk(e) for e in range(n)]


def _pinned(a, offset=0):
    """A pinned copy of `a`, starting `offset` bytes into its allocation."""
    import torch
    a = np.ascontiguousarray(a)
    buf = torch.empty(a.nbytes + offset, dtype=torch.uint8).pin_memory().numpy()
    out = buf[offset:offset + a.nbytes].view(a.dtype).reshape(a.shape)
    out[...] = a
    return out


def _struct(p, conv):
    return (Pointmap(conv(p["X_a"]), conv(p["valid_a"], 1), H, W), Pointmap(conv(p["X_b"]), conv(p["valid_b"], 3), H, W),
            FeatureMap(conv(p["D_a"]), conv(p["Q_a"], 4), H, W), FeatureMap(conv(p["D_b"]), conv(p["Q_b"]), H, W))


def _outs(n, pinned):
    def arr(dt):
        return _pinned(np.zeros(H * W, dt)) if pinned else np.zeros(H * W, dt)
    return [MatchSet(arr(np.int32), arr(np.float32), arr(np.uint8)) for _ in range(n)]


@pytest.mark.parametrize("n", [1, 6, 11])
def test_host_paths_equal_device_path(ctx, n):
    import torch
    pairs = _pairs(n)
    mp, rp = baseline_match_params(), abi.refine_params(BASELINE_REFINE)
    dev = []
    for p in pairs:
        t = to_torch_pair(p)
        dev.append((Pointmap(t["X_a"], t["valid_a"], H, W), Pointmap(t["X_b"], t["valid_b"], H, W),
                    FeatureMap(t["D_a"], t["Q_a"], H, W), FeatureMap(t["D_b"], t["Q_b"], H, W)))
    ref = ctx.match_batch(dev, params=mp, refine=rp)
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches
    pageable = ctx.match_batch([_struct(p, lambda a, o=0: np.ascontiguousarray(a)) for p in pairs], params=mp, refine=rp,
                               outs=_outs(n, False))
    l1 = ctx.kernel_launches
    pinned = ctx.match_batch([_struct(p, _pinned) for p in pairs], params=mp, refine=rp, outs=_outs(n, True))
    l2 = ctx.kernel_launches
    assert l2 - l1 > l1 - l0  # the pinned call added its k_copy_segs launches
    for r, a, b in zip(ref, pageable, pinned):
        rv = r.valid.cpu().numpy()
        assert rv.sum() > 0.5 * H * W
        for o in (a, b):
            np.testing.assert_array_equal(np.asarray(o.valid), rv)
            np.testing.assert_array_equal(np.asarray(o.pixel_a), r.pixel_a.cpu().numpy())
            np.testing.assert_array_equal(np.asarray(o.confidence), r.confidence.cpu().numpy())
