"""Static check of a cubin/object: in every kernel, uniform registers that are read but never
written (ptxas miscompiles of this kind raise 'illegal instruction' at run time).
usage: python tools/check_sass_ur.py file.o|file.so"""
import re, subprocess, sys

def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    bad = 0
    for fn in out.split("Function : ")[1:]:
        name = fn.split("\n", 1)[0].strip()
        written, read = set(), set()
        for line in fn.splitlines():
            m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)\s+([^;]*);", line)
            if not m:
                continue
            ops = [o.strip() for o in m.group(3).split(",")]
            op = m.group(2)
            # "OP UPn, URm, ..." (e.g. ULOP3 with a predicate output): URm is written too
            if len(ops) > 1 and re.fullmatch(r"U?P(\d+|T)", ops[0]) and re.fullmatch(r"UR\d+", ops[1]):
                ops = [ops[1]] + ops[2:]
            urs = [re.findall(r"\bUR(\d+)\b", o) for o in ops]
            if ops and urs[0] and not op.startswith(("ST", "LDGSTS", "RED", "ATOM", "UTMA", "SYNCS", "BAR", "UBLKCP", "UTMALDG", "UTMAPF")):
                for r in urs[0]:
                    written.add(int(r))
                    if ".128" in op:
                        written.update({int(r) + 1, int(r) + 2, int(r) + 3})
                    elif ".64" in op or ".WIDE" in op:
                        written.add(int(r) + 1)
                rest = urs[1:]
            else:
                rest = urs
            for lst in rest:
                read.update(int(r) for r in lst)
            if op.startswith(("LDGSTS", "LDG", "STG")):
                for r in re.findall(r"desc\[UR(\d+)\]", m.group(3)):
                    read.update({int(r), int(r) + 1})
        missing = sorted(r for r in read - written if r < 63)
        if missing:
            bad += 1
            print(name[:110], "reads unwritten UR", missing)
    print("kernels with unwritten uniform reads:", bad)

if __name__ == "__main__":
    main(sys.argv[1])
