"""SASS instruction-class summary of libqsim.so per kernel (evidence for
profiles/): TMA (UTMALDG / UTMASTG / UBLKCP / UTMAPF), mbarrier (SYNCS),
FP64 (DFMA / DMUL / DADD), shared memory (LDS / STS), global (LDG / STG),
shuffles (SHFL) and tensor-core instructions (none expected: the path is not a
dense contraction).  Usage: python tools/sass_summary.py [lib] > profiles/r2_sass_summary.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_quant_ph_0201042_b200/libqsim.so"
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
CLASSES = {
    "UTMALDG": r"\bUTMALDG\b", "UTMASTG": r"\bUTMASTG\b", "UBLKCP": r"\bUBLKCP\b", "UTMAPF": r"\bUTMAPF\b",
    "SYNCS": r"\bSYNCS\.", "DFMA": r"\bDFMA\b", "DMUL": r"\bDMUL\b", "DADD": r"\bDADD\b", "LDS": r"\bLDS\b",
    "STS": r"\bSTS\b", "LDG": r"\bLDG\b", "STG": r"\bSTG\b", "SHFL": r"\bSHFL\b", "RED/ATOM": r"\b(RED|ATOM)G?\b",
    "UTC*MMA/HMMA": r"\b(UTC\w*MMA|HMMA|DMMA)\b",
}
funcs = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs.setdefault(cur, collections.Counter())
        continue
    if cur and "/*" in line:
        for k, pat in CLASSES.items():
            if re.search(pat, line):
                funcs[cur][k] += 1


def short(name):
    """Kernel name and template arguments from the mangled symbol."""
    for m in re.finditer(r"(\d+)(k_)", name):
        digits, k = m.group(1), m.start(2)
        L = None
        for i in range(len(digits)):   # the length prefix is a suffix of the digit run (hash digits precede it)
            cand = int(digits[i:])
            if k + cand < len(name) and name[k + cand] in "EI" and re.fullmatch(r"k_[a-z0-9_]+", name[k:k + cand]):
                L = cand
                break
        if L is None:
            continue
        base = name[k:k + L]
        rest = name[k + L:]
        args = re.findall(r"L([ib])(\d+)E", rest[:40]) if rest.startswith("I") else []
        return base + (f"<{','.join(v for _, v in args)}>" if args else "")
    return name[:40]


agg = collections.OrderedDict()
for f, c in funcs.items():
    k = short(f)
    agg.setdefault(k, collections.Counter()).update(c)
cols = list(CLASSES)
print("| kernel | " + " | ".join(cols) + " |")
print("|---" * (len(cols) + 1) + "|")
for k, c in agg.items():
    print(f"| {k} | " + " | ".join(str(c.get(x, 0)) for x in cols) + " |")
