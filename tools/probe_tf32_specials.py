"""Diagnostic: how does the hardware cvt.rna.tf32.f32 treat non-finite inputs? (GPU box)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_09251_b200 as acc
chunk = 1 << 28
inp = torch.empty(chunk, dtype=torch.int32, device="cuda")
out = torch.empty(chunk, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
tot = {"finite": 0, "inf": 0, "nan": 0}
examples = []
rules = {"trunc": 0, "canon7fffffff": 0, "rna_wrap": 0, "other": 0, "nan_total": 0}
for c in range(16):
    host = (np.arange(chunk, dtype=np.uint64) + c * chunk).astype(np.uint32)
    inp.copy_(torch.from_numpy(host.view(np.int32)))
    acc.accspmm_debug_round_tf32(inp.data_ptr(), out.data_ptr(), chunk, s)
    dev = out.cpu().numpy().view(np.uint32)
    ref = ((host.astype(np.uint64) + 0x1000) & 0xFFFFE000).astype(np.uint32)
    x = host.view(np.float32)
    bad = dev != ref
    fin = np.isfinite(x); isn = np.isnan(x); isi = np.isinf(x)
    tot["finite"] += int((bad & fin).sum()); tot["inf"] += int((bad & isi).sum()); tot["nan"] += int((bad & isn).sum())
    h = host[isn]; d = dev[isn]
    rules["nan_total"] += h.size
    rules["trunc"] += int((d == (h & 0xFFFFE000)).sum())
    rules["canon7fffffff"] += int((d == 0x7FFFFFFF).sum())
    rules["rna_wrap"] += int((d == ((h.astype(np.uint64) + 0x1000) & 0xFFFFE000).astype(np.uint32)).sum())
    # is output NaN for every NaN input?
    dn = d.view(np.float32)
    rules.setdefault("out_is_nan", 0); rules["out_is_nan"] += int(np.isnan(dn).sum())
    idx = np.nonzero(bad)[0][:3]
    for i in idx:
        examples.append((hex(int(host[i])), hex(int(dev[i])), hex(int(ref[i]))))
    sel = np.array([0x7F800001, 0x7F800FFF, 0x7F801000, 0x7FC00000, 0x7FFFFFFF, 0xFF800001, 0xFFC00000, 0x7F800000, 0x7F7FFFFF], dtype=np.uint64)
    for v in sel:
        if c * chunk <= v < (c + 1) * chunk:
            examples.append(("probe", hex(int(v)), hex(int(dev[int(v) - c * chunk]))))
print("mismatches by class:", tot)
print("nan rules:", rules)
for e in examples[:60]: print(e)
