"""SASS evidence for profiles/r02_sass.md: per kernel of the built library,
counts of the instructions that show which hardware paths it uses (TMA bulk
copies, mbarriers, named barriers, wide streaming loads/stores, shared
atomics, tensor-core MMA).  No GPU needed.

    python tools/sass_evidence.py [paper_2107_01391_b200/librecsort_b200.so] > profiles/r02_sass.md
"""
import collections
import re
import subprocess
import sys

SO = sys.argv[1] if len(sys.argv) > 1 else "paper_2107_01391_b200/librecsort_b200.so"
COLS = [("UBLKCP", r"\bUBLKCP"), ("SYNCS (mbarrier)", r"\bSYNCS"), ("STG.E.EF.ENL2.256", r"STG\.E\.EF\.ENL2\.256"),
        ("LDG.E.EF.128", r"LDG\.E\.EF\.128"), ("ATOMS", r"\bATOMS"), ("BAR.SYNC id>0", r"BAR\.SYNC(?:\.DEFER_BLOCKING)? 0x[1-9a-f]"),
        ("BAR.ARV", r"BAR\.ARV"), ("MATCH", r"\bMATCH"), ("tensor core (HMMA/UTC*MMA)", r"\bHMMA|\bUTC\w*MMA")]


def main():
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    archs = sorted(set(re.findall(r"arch = (sm_\w+)", out)))
    per = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur:
            for name, pat in COLS:
                if re.search(pat, line):
                    per[cur][name] += 1
    print("# SASS evidence (cuobjdump -sass of the built library; `python tools/sass_evidence.py`)\n")
    print(f"Target architectures in the fatbin: {archs}\n")
    print("| kernel | " + " | ".join(n for n, _ in COLS) + " |")
    print("|---|" + "---|" * len(COLS))
    tot = collections.Counter()
    for fn, c in per.items():
        if not any(c.values()):
            continue
        short = re.sub(r"^_ZN3rsb\d+", "", fn)[:60]
        print(f"| {short} | " + " | ".join(str(c[n]) for n, _ in COLS) + " |")
        tot.update(c)
    print("| **all kernels** | " + " | ".join(str(tot[n]) for n, _ in COLS) + " |")
    print("\nNo tensor-core instructions are expected: nothing on this path is a contraction (DESIGN.md).")


if __name__ == "__main__":
    main()
