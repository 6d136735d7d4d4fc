#!/usr/bin/env python
"""Instruction-class counts per kernel of the built librlhead.so (cuobjdump
-sass): the evidence that the GEMMs run on tcgen05 / TMEM / TMA (the SASS
mnemonics B200_PROFILING.md names) and that the HBM kernels use the
intended vector/ballot/match instructions. Writes a markdown table.

    python scripts/sass_summary.py > profiles/r2/sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2509_15965_b200", "librlhead.so")

CLASSES = [
    ("UTCHMMA", r"UTCHMMA"),            # tcgen05.mma (kind::f16)
    ("UTCHMMA.2CTA", r"UTCHMMA\S*2CTA"),
    ("UTCBAR", r"UTCBAR"),              # tcgen05.commit -> mbarrier
    ("UTMALDG", r"UTMALDG"),            # TMA tensor load
    ("UTMASTG", r"UTMASTG"),            # TMA tensor store
    ("UTMAREDG", r"UTMAREDG"),          # TMA tensor reduce (dW += box)
    ("UBLKCP", r"UBLKCP"),              # 1-D bulk copy (fused reduce-scatter rows to peers)
    ("UTMACCTL.PF", r"UTMACCTL\.PF"),  # TMA descriptor prefetch
    ("LDTM", r"\bLDTM"),                # tcgen05.ld (TMEM -> registers)
    ("UTCATOMSWS", r"UTCATOMSWS"),      # tcgen05.alloc/dealloc
    ("SYNCS", r"\bSYNCS"),              # mbarrier ops
    ("MUFU.EX2", r"MUFU\.EX2"),
    ("LDG.128", r"LDG\.E\.128|LDG\.E\.EF\.128|LDG\.E\.LU\.128"),
    ("STG.128", r"STG\.E\.128|STG\.E\.EF\.128"),
    ("VOTE", r"\bVOTE"),
    ("MATCH", r"\bMATCH"),
    ("SHFL", r"\bSHFL"),
    ("DADD/DFMA", r"\bD(ADD|FMA|MUL)"),
]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        return out.stdout.splitlines()
    except Exception:
        return names


def main():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True,
                          text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None or "/*" not in line:
            continue
        ins = line.split("*/", 1)[-1] if line.strip().startswith("/*") else line
        for name, pat in CLASSES:
            if re.search(pat, ins):
                funcs[cur][name] += 1
        funcs[cur]["total"] += 1
    names = demangle(list(funcs))
    cols = [c for c, _ in CLASSES]
    print("# SASS instruction classes per kernel (`cuobjdump -sass librlhead.so`)\n")
    print("Built with `-gencode arch=compute_100a,code=sm_100a`; `python scripts/sass_summary.py`.\n")
    print("| kernel | " + " | ".join(cols) + " | total |")
    print("|---" * (len(cols) + 2) + "|")
    for (raw, cnt), nice in zip(funcs.items(), names):
        nice = re.sub(r"\(.*$", "", nice).replace("rlh::", "")
        nice = nice.replace("|", "/")
        print(f"| `{nice}` | " + " | ".join(str(cnt.get(c, 0)) for c in cols) +
              f" | {cnt['total']} |")
    return 0


if __name__ == "__main__":
    sys.exit(main())
