"""Per-phase cycle trace of the tcgen05 kernel (variants build, ACCSPMM_KCFG=68) on Reddit-shaped."""
import ctypes
import os
import sys

os.environ["ACCSPMM_LIB"] = "variants"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2501_09251_b200 as acc

cfg, A = gen.make_config("reddit")
vals = gen.values_uniform(A.nnz, 1)
Bd = torch.from_numpy(gen.dense_normal(A.K, 128, 2)).cuda()
lib = acc.load_library()
for wh in [int(x) for x in sys.argv[1:]] or [32]:
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, window_rows=wh, kernel="tcgen05", reorder="auto", build="device")
    C = torch.empty((A.M, 128), device="cuda")
    os.environ["ACCSPMM_KCFG"] = "-1"
    p.execute(Bd, C)
    os.environ["ACCSPMM_KCFG"] = "68"
    p.execute(Bd, C)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (64 * 16))()
    lib.accspmm_debug_tc05_trace(buf)
    t = np.array(buf, dtype=np.float64).reshape(64, 16)
    U = p.export_units()[:64]
    nblk = (U[:, 3] - U[:, 2]).astype(np.float64)
    per = t.sum(0) / nblk.sum()
    names_p = ["acc_free wait", "ready wait", "mma+commit", "chunk+tma", "-", "-", "-", "loop/advance"]
    names_t = ["empty wait", "full_t wait", "lds+sttm", "decode", "wait::st+arrive", "epilogue", "loop top", "-"]
    print("wh", wh, "blocks", int(nblk.sum()), "cycles per block:")
    print("  producer   ", {n: round(v, 1) for n, v in zip(names_p, per[:8]) if n != "-"})
    print("  transposer ", {n: round(v, 1) for n, v in zip(names_t, per[8:]) if n != "-"})
    os.environ["ACCSPMM_KCFG"] = "-1"
    del p
