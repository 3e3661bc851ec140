"""Runs last (file order): under a range-checked build of the library
(-DPMX_CHECKED: tools/variants.sh checked, selected with PMX_LIB), every
gather index the hot kernels used during the whole GPU test session must
have been inside its array.  compute-sanitizer is not available on this
pool; this is the substitute (tools/gpu_checked.sh)."""
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.skipif("checked" not in os.environ.get("PMX_LIB", ""), reason="release build (no range checks)")
def test_no_range_violations_in_the_session(ctx):
    _, violations = ctx.profile_get("checked_violations")
    assert violations == 0, f"{violations} out-of-range gather indices"
