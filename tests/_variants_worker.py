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

KCFGS = ["20", "46", "47", "48", "49", "50", "51", "52", "53", "54", "55", "56", "57", "58", "59", "60", "61", "62", "63", "64", "65", "66", "68", "69", "70", "73", "77", "78", "79", "80", "85", "87", "93", "10", "11", "12",
         "b3", "hot"]


def main():
    kcfgs = sys.argv[1:] or KCFGS   # a subset on the command line (A/B scripts check new variants first)
    assert acc.LIB_PATH.endswith("libaccspmm_variants.so"), acc.LIB_PATH
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=3, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    vf = gen.values_uniform(A.nnz, 4)
    Bf = gen.dense_normal(A.K, 128, 5)
    for precision in ("tf32", "fp16"):
        for kcfg in kcfgs:
            # "b3": the default kernel reading the 3-byte TF32 image of B (ACCSPMM_B3=1); 58-61
            # are B3 variants (the knob is on for them, off for the others)
            # "hot": hot-column plans (R22) with every tag level exercised: a 1 MiB hot set and
            # hot/cold policies at any B size
            os.environ["ACCSPMM_KCFG"] = "-1" if kcfg in ("b3", "hot") else kcfg
            os.environ["ACCSPMM_HOT_MB"] = "1" if kcfg == "hot" else "64"
            os.environ["ACCSPMM_HOT_L2_MB"] = "0" if kcfg == "hot" else "96"
            hot = {"hot_cols": "on"} if kcfg == "hot" else {}
            os.environ["ACCSPMM_B3"] = "1" if kcfg in ("b3", "58", "59", "60", "61") else "0"
            res = {"kcfg": kcfg, "precision": precision, "ok": True}
            try:
                for N in (64, 256):
                    B = gen.dense_int(A.K, N, 2)
                    C, p = run(A, v, B, precision, balance="on", unit_cap=32, **hot)
                    assert p.info["n_split_windows"] > 0
                    if kcfg == "b3" and precision == "tf32":
                        assert p.b_bytes(N) == 3, p.b_bytes(N)   # the B3 path really ran
                    assert_bit_exact(C, A, v, B, precision)
                Cf, _ = run(A, vf, Bf, precision, **hot)
                assert_within(Cf, A, vf, Bf, precision)
            except AssertionError as e:
                res.update(ok=False, err=repr(e)[:400])
            print(json.dumps(res), flush=True)
    os.environ.pop("ACCSPMM_KCFG", None)
    os.environ.pop("ACCSPMM_B3", None)
    os.environ.pop("ACCSPMM_HOT_MB", None)
    os.environ.pop("ACCSPMM_HOT_L2_MB", None)
    _ = np


if __name__ == "__main__":
    main()
