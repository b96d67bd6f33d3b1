"""SASS instruction census of liblyc.so per kernel (cuobjdump -sass): the
tensor-core, TMA and async-copy mnemonics that evidence the sm_100a paths.

    python scripts/sass_census.py [> profiles/rNN_sass_census.txt]
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2602_04541_b200" / "liblyc.so"
WATCH = ["HMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "UTCCP", "LDTM", "STTM", "UTMALDG", "UTMASTG",
         "UTMAPF", "UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "ELECT", "REDG", "ATOMG", "SHFL", "MUFU"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                          check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs.setdefault(cur, Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]+)?", line)
        if cur and m:
            funcs[cur][m.group(1)] += 1
            funcs[cur]["_total"] += 1
    demangled = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True,
                               text=True).stdout.splitlines()
        demangled = dict(zip(funcs, names))
    except OSError:
        pass
    print(f"# SASS census of {LIB.name} (cuobjdump -sass, sm_100a)")
    print("# columns: " + " ".join(WATCH) + " total")
    for f, c in sorted(funcs.items(), key=lambda kv: -kv[1]["_total"]):
        name = demangled.get(f, f)
        name = re.sub(r"\(.*", "", name)
        print(f"{name[:70]:70s} " + " ".join(f"{w}={c[w]}" for w in WATCH if c[w]) +
              f" total={c['_total']}")


if __name__ == "__main__":
    sys.exit(main())
