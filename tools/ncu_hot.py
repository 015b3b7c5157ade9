"""Hot SASS lines of an ncu report (run here): top-N instructions by stall samples, with the
dominant stall reasons per line.  usage: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv, io, subprocess, sys


def main(path, n=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    print("total samples", tot, "instructions", len(data))
    idx = {id(d): i for i, d in enumerate(data)}
    top = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:n]
    for d in sorted(top, key=lambda d: idx[id(d)]):
        s = float(d["Warp Stall Sampling (All Samples)"] or 0)
        rs = sorted(((h[6:], float(d[h] or 0)) for h in hdr if h.startswith("stall_") and "(" not in h),
                    key=lambda x: -x[1])
        why = " ".join(f"{k}:{int(v)}" for k, v in rs[:3] if v > 0)
        print(f"{idx[id(d)]:5d} {100*s/tot:5.1f}%  ex={d['Instructions Executed']:>10}  {d['Source'].strip()[:70]:70s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
