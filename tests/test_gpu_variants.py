"""The measured-and-rejected kernel variants stay exact.

They live only in the variants build (libaccspmm_variants.so, -DACCSPMM_VARIANTS; the product
library ships one kernel family per width and precision), so the check runs in a subprocess
with ACCSPMM_LIB=variants: every ACCSPMM_KCFG variant (2 warps per CTA, FP16 PRMT fragments,
k4/k8 swap, values two ahead, 3/4-stage rings, L2::256B value loads, register-direct gather)
computes the same product -- integer data bit-exact with split windows, N = 64 and 256
(per-slice maps), floats within tolerance."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_measurement_variants_stay_exact():
    from paper_2501_09251_b200 import _build
    _build.build(variants=True)
    env = dict(os.environ, ACCSPMM_LIB="variants")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variants_worker.py")], env=env,
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(rows) == 22, r.stdout[-2000:]
    bad = [x for x in rows if not x["ok"]]
    assert not bad, bad
