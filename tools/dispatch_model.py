"""Dispatch model of a hot-kernel iteration from its SASS (runs here, no GPU).

Finds the largest basic block of a pass3 kernel (the unrolled S+1-step body),
counts its instructions by opcode and prices them with the per-instruction
dispatch costs measured by tools/ubench.py on the B200 (cycles per warp-
instruction per SMSP at 4 warps/SMSP): packed FFMA2/FADD2/FMUL2 2.2, MUFU 2.9
(its increment on an FFMA2 stream), everything else 1.1.  With --extra N the
per-iteration instructions outside the body (staging, flush; from the ncu
source page) are added at 1.1.  Prints predicted cycles per 64 pair-lines and
the implied roofline fraction (16.8 cycles = the FP32/8 roofline at 1965 MHz).

    python tools/dispatch_model.py paper_1407_2343_b200/build/obj/inst_S10.o \
        '_ZN5plgpu16nlm_pass3_kernelILi10ELi3ELi2ELi2ELi2ELb0EEEvNS_9Pass3DescE' --pairs 110 --extra 326
"""
import argparse
import re
import subprocess
from collections import Counter

COST = {"FFMA2": 2.2, "FADD2": 2.2, "FMUL2": 2.2, "MUFU": 2.9}
ROOF = 16.8  # cycles per 64 pair-lines at the FP32/8 roofline


def body_ops(obj: str, fn: str) -> Counter:
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True,
                          check=True).stdout
    ops = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if m:
            ops.append(re.sub(r"^@!?U?P\w+\s+", "", m.group(1)).split()[0].split(".")[0])
    best, start = (0, 0, 0), 0
    for i, op in enumerate(ops + ["BRA"]):
        if op in ("BRA", "EXIT", "WARPSYNC", "CALL", "RET", "BAR"):
            best = max(best, (i - start, start, i))
            start = i + 1
    return Counter(ops[best[1]:best[2]])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("obj")
    ap.add_argument("fn")
    ap.add_argument("--pairs", type=int, required=True, help="unique pairs per body (R * S)")
    ap.add_argument("--lines", type=int, default=2, help="lines per lane (pair-lines = 32 * lines)")
    ap.add_argument("--extra", type=int, default=0, help="instructions per iteration outside the body")
    a = ap.parse_args()
    c = body_ops(a.obj, a.fn)
    cyc = sum(n * COST.get(op, 1.1) for op, n in c.items()) + 1.1 * a.extra
    per64 = cyc / a.pairs * (2 / a.lines)
    print("body:", dict(c.most_common(12)))
    print(f"instructions {sum(c.values())} (+{a.extra}), dispatch cycles {cyc:.0f}, "
          f"{per64:.1f} cycles per 64 pair-lines -> frac <= {ROOF / per64:.3f}")


if __name__ == "__main__":
    main()
