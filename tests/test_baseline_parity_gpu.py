"""GPU parity at the BASELINE configurations themselves (not scaled-down
cases), through the C ABI, against the reference build (oracle/_ref: the
genuine src/*.cpp) when it is present, else the FP64 restatement.

* config 2: the full 64-edge batch (28 consecutive pairs x 2 directions + 8
  long-range pairs, 512x384, 24-d fp16) -> every edge compared with the
  reference's match_pointmaps + feature_refine (src/camera.cpp:195-271);
  bars of BASELINE north_star: >= 99.9% of valid pixels index-equal, every
  mismatch <= 1 px, valid-mask mismatch <= 1e-3.
"""
import os

import numpy as np
import pytest

import pmxgen
import pyoracle
from helpers import BASELINE_REFINE, baseline_match_params, compare_matches, pmx_pair
from paper_2412_12392_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = max(1, os.cpu_count() or 1)


def _reference():
    return pyoracle.reference() if pyoracle.have_reference() else _Null()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@pytest.fixture(scope="module")
def config2():
    sc, poses, edges, make_pair = pmxgen.config2(seed=2)
    assert len(edges) == 64
    return [make_pair(e) for e in range(len(edges))]


def test_config2_full_batch_vs_reference(ctx, config2):
    mp, rp = baseline_match_params(), abi.refine_params(BASELINE_REFINE)
    gpu = ctx.match_batch([pmx_pair(p) for p in config2], params=mp, refine=rp)
    with _reference():
        ref = pyoracle.match_batch(config2, mp, rp, threads=THREADS)
    worst_eq, total_both, total_eq, total_vm = 1.0, 0, 0, 0
    for e, (g, r) in enumerate(zip(gpu, ref)):
        st = compare_matches(g, r, 512)
        assert st["worst_px"] <= 1, (e, st)
        assert st["valid_mismatch"] <= 1e-3 * st["n"], (e, st)
        worst_eq = min(worst_eq, st["index_equal_frac"])
        total_both += st["both"]
        total_eq += int(round(st["index_equal_frac"] * st["both"]))
        total_vm += st["valid_mismatch"]
        # q = sqrt(Q_a[pa] Q_b[n]) (camera.cpp:230, 269-270): fp32 rounding of the FP64 value
        same = np.asarray(g.pixel_a) == r.pixel_a
        np.testing.assert_allclose(np.asarray(g.confidence)[same], r.confidence[same], rtol=6e-8)
    assert worst_eq >= 0.999 and total_eq / total_both >= 0.999
    print(f"config2: {total_both} px valid in both, index-equal {total_eq / total_both:.7f}, "
          f"worst edge {worst_eq:.7f}, valid mismatches {total_vm}")
