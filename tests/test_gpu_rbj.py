"""RBJ peaking-EQ stress set (reported next to fp32 sequential
filtering, not gated at 1e-4).  The property checked: the GPU path (fp32 data, fp32/fp64
carries) is never much worse than a plain fp32 sequential filter on the same inputs, and
every output is finite.  The full-size report is tools/rbj_stress.py ->
profiles/r02_rbj_stress.txt."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_rbj_stress_not_worse_than_fp32_sequential():
    import rbj_stress
    rows = rbj_stress.run(batch=16, length=1 << 14, seed=99)
    for d in rows:
        for k in ("gpu_y", "gpu_gx", "gpu_gb", "gpu_ga"):
            assert np.isfinite(d[k]), (k, d)
        assert d["gpu_y"] <= max(10 * d["seq32_y"], 1e-4), d
    print("\n" + rbj_stress.report(rows))
