"""Dynamic SASS profile from an ncu source-page CSV (ncu -i rep --page source
--csv --print-source sass): executed warp instructions and stall samples per
opcode, per kernel.  Runs here (no GPU).

    python tools/sass_profile.py gpurun_out/r02b/sass_c4.csv [top]
"""
import csv
import collections
import re
import sys


def load(path):
    kernels, cur, hdr = [], None, None
    with open(path, newline="") as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "Kernel Name":
                cur = {"name": row[1], "rows": []}
                kernels.append(cur)
                hdr = None
                continue
            if hdr is None:
                hdr = row
                continue
            cur["rows"].append(dict(zip(hdr, row)))
    return kernels


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def opcode(src):
    s = re.sub(r"^@!?U?P[0-9T]+\s+", "", src.strip())
    return s.split(" ")[0].split(".")[0] if s else ""


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    for k in load(path):
        cnt, stall = collections.Counter(), collections.Counter()
        tot = 0.0
        samples = 0.0
        for r in k["rows"]:
            op = opcode(r.get("Source", ""))
            n = num(r.get("Instructions Executed", "0"))
            cnt[op] += n
            tot += n
            s = num(r.get("Warp Stall Sampling (All Samples)", "0"))
            stall[op] += s
            samples += s
        print(k["name"][:100])
        print(f"  executed warp instructions: {tot:.4g}; stall samples {samples:.4g}")
        for op, n in cnt.most_common(top):
            print(f"  {op:10s} {n:14.4g} {100 * n / tot:6.2f}%   samples {100 * stall[op] / max(1, samples):6.2f}%")


if __name__ == "__main__":
    main()
