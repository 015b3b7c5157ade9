"""The measured-and-rejected kernel variants stay exact.

They live only in the variants build (libaccspmm_variants.so, -DACCSPMM_VARIANTS; the product
library ships one kernel family per width and precision), so the check runs in a subprocess
with ACCSPMM_LIB=variants: every ACCSPMM_KCFG variant (2 warps per CTA, FP16 PRMT fragments,
k4/k8 swap, values two ahead, 3/4-stage rings, L2::256B value loads, value evict-first, value
staging by bulk copy, hybrid TMA + cp.async gather, the 3-byte TF32 image of B "B3" and its
ring/occupancy variants, the 64-bit decode, lane-0 / all-lane TMA issue, hot-column plans with
evict-first blocks at every tag level, register-direct gather) computes the same product -- integer data bit-exact with split windows, N = 64 and 256
(per-slice maps), floats within tolerance."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _worker_kcfgs():
    """The worker's variant list (read from its source: importing it would load the variants
    library into this process)."""
    import ast
    tree = ast.parse(open(os.path.join(HERE, "_variants_worker.py")).read())
    for node in tree.body:
        if isinstance(node, ast.Assign) and getattr(node.targets[0], "id", "") == "KCFGS":
            return ast.literal_eval(node.value)
    raise AssertionError("KCFGS not found")


def test_measurement_variants_stay_exact():
    from paper_2501_09251_b200 import _build
    _build.build(variants=True)
    env = dict(os.environ, ACCSPMM_LIB="variants")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variants_worker.py")], env=env,
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(rows) == 2 * len(_worker_kcfgs()), r.stdout[-2000:]
    bad = [x for x in rows if not x["ok"]]
    assert not bad, bad
