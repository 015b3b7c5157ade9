"""Runs every measured kernel variant of the variants build (ACCSPMM_LIB=variants) on the
fixture of test_gpu_variants.py and prints one JSON line per case.  Spawned by that test: the
product library (libaccspmm.so) contains no variants and reads no ACCSPMM_* knobs."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
assert os.environ.get("ACCSPMM_LIB") == "variants"

import numpy as np  # noqa: E402

import gen  # noqa: E402
import paper_2501_09251_b200 as acc  # noqa: E402
from gpu_util import assert_bit_exact, assert_within, run  # noqa: E402

KCFGS = ["20", "46", "47", "48", "49", "50", "51", "52", "53", "54", "55", "56", "57", "10", "11", "12"]


def main():
    assert acc.LIB_PATH.endswith("libaccspmm_variants.so"), acc.LIB_PATH
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=3, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    vf = gen.values_uniform(A.nnz, 4)
    Bf = gen.dense_normal(A.K, 128, 5)
    for precision in ("tf32", "fp16"):
        for kcfg in KCFGS:
            os.environ["ACCSPMM_KCFG"] = kcfg
            res = {"kcfg": kcfg, "precision": precision, "ok": True}
            try:
                for N in (64, 256):
                    B = gen.dense_int(A.K, N, 2)
                    C, p = run(A, v, B, precision, balance="on", unit_cap=32)
                    assert p.info["n_split_windows"] > 0
                    assert_bit_exact(C, A, v, B, precision)
                Cf, _ = run(A, vf, Bf, precision)
                assert_within(Cf, A, vf, Bf, precision)
            except AssertionError as e:
                res.update(ok=False, err=repr(e)[:400])
            print(json.dumps(res), flush=True)
    os.environ.pop("ACCSPMM_KCFG", None)
    _ = np


if __name__ == "__main__":
    main()
