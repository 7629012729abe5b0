"""Per-kernel SASS instruction summary of the built libdiagmm.so (static counts).

Proves which kernels issue tcgen05 / TMA / TMEM instructions and which run on
the FMA pipes:  python tools/sass_summary.py > profiles/r02_sass_summary.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2506_11449_b200" / "_lib" / "libdiagmm.so"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS",
        "FHFMA", "FFMA", "FFMA2", "DFMA", "HFMA2", "LDS", "STS", "LDG", "STG", "SHFL", "BAR"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op, mod = m.group(1), m.group(2) or ""
            funcs[cur][op] += 1
            if op in ("UTCHMMA", "UTMALDG", "UTMASTG") and "2CTA" in mod:
                funcs[cur][op + ".2CTA"] += 1
            if op == "LDS" and ".128" in mod:
                funcs[cur]["LDS.128"] += 1
    names = demangle(list(funcs))
    print(f"# static SASS instruction counts per kernel, {LIB.name} (cuobjdump -sass), sm_100a")
    print("# columns: " + " ".join(KEYS + ["UTCHMMA.2CTA", "LDS.128"]))
    for f, c in sorted(funcs.items(), key=lambda kv: names[kv[0]]):
        short = re.sub(r"\(.*", "", names[f])
        short = re.sub(r"\bdiagmm::", "", short)
        tot = sum(v for k, v in c.items() if "." not in k)
        cols = " ".join(f"{k}={c[k]}" for k in KEYS + ["UTCHMMA.2CTA", "LDS.128"] if c[k])
        print(f"{short:70s} total={tot:6d} {cols}")


if __name__ == "__main__":
    sys.exit(main())
