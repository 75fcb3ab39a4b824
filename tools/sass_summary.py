"""Per-kernel SASS opcode counts of libnnb.so (cuobjdump -sass): the static evidence
that each kernel issues the instructions its design claims (DMMA for the FP64 tensor
path, UTMALDG/UBLKCP for TMA, UTCxMMA/UTCBAR for tcgen05, SYNCS for mbarriers).

    python tools/sass_summary.py [path/to/libnnb.so] > profiles/r02_sass_summary.txt
"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

OPS = ["DMMA", "DFMA", "DADD", "DMUL", "UTMALDG", "UTMASTG", "UBLKCP", "UTCQMMA", "UTCIMMA", "UTCHMMA", "UTCBAR",
       "LDTM", "STTM", "SYNCS", "BAR", "LDS", "STS", "LDG", "STG", "SHFL", "ATOM", "RED", "LDSM", "MEMBAR"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2212_02406_b200/libnnb.so"
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels = OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            kernels[cur][m.group(1)] += 1
            kernels[cur]["_total"] += 1
    demangled = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout
        demangled = dict(zip(kernels, names.splitlines()))
    except Exception:
        pass
    print(f"# SASS opcode counts per kernel, {so} (cuobjdump -sass; static instruction counts)")
    print("# columns: " + " ".join(OPS) + " total")
    for k, c in kernels.items():
        name = demangled.get(k, k)
        name = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", ""))[:140]
        row = " ".join(f"{op}={c[op]}" for op in OPS if c[op])
        print(f"{name}\n    {row} total={c['_total']}")


if __name__ == "__main__":
    main()
