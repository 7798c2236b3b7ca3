"""Groups ncu SASS-level stall samples and executed instructions of
decode_kernel by phase (line ranges between PROF_MARK barriers) and by
helper source file (softplus.cuh = log_add)."""
import collections
import csv
import re
import sys

sys.path.insert(0, "profiles")
from sass_lines import line_map  # noqa: E402

ncu_csv, sass, func, src = sys.argv[1:5]
marks = []
for i, l in enumerate(open(src), 1):
    m = re.search(r"PROF_MARK\((\d+)\);", l)
    if m and "#define" not in l:
        marks.append((i, int(m.group(1))))
names = {0: "init+F/G tables", 1: "P1 windows/eos", 2: "P2 phi/factors", 3: "P3 bulk+keys",
         4: "P4 theta", 5: "P5 contenders", 6: "P6 recursion", 7: "P7 rank", 8: "fallback",
         9: "P8 walk", 10: "P9 end detect", 11: "finalize"}


SRC_LINES = open(src).read().split("\n")
KSTART = next(i for i, l in enumerate(SRC_LINES, 1) if "decode_kernel(const" in l)
FUNCS = [(i, re.search(r"(\w+)\(", l).group(1)) for i, l in enumerate(SRC_LINES, 1)
         if re.match(r"^(__device__|template|static|SP_HD)", l) is None and
         re.match(r"^__device__.*\(|^(\w+ )+\w+\(.*", l) and i < KSTART and "(" in l]


def helper_of(line):
    name = "helper"
    for i, l in enumerate(SRC_LINES[:line], 1):
        m = re.match(r"^__device__ (?:__forceinline__ )?[\w:<>\*& ]+?(\w+)\(", l)
        if m:
            name = "fn:" + m.group(1)
    return name


def phase_of(line):
    if line < KSTART:
        return helper_of(line)
    for ln, k in marks:
        if line <= ln:
            return names.get(k, str(k))
    return "tail"


amap = line_map(sass, func)
rows = list(csv.reader(open(ncu_csv)))
hdr = rows[1]
ia, isamp, iinst = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
base = int(rows[2][ia], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0])
for r in rows[2:]:
    try:
        a = int(r[ia], 16) - base
        s, n = float(r[isamp] or 0), float(r[iinst] or 0)
    except (ValueError, IndexError):
        continue
    f, l = amap.get(a, ("?", 0))
    key = phase_of(l) if f == src.split("/")[-1] else f
    agg[key][0] += s
    agg[key][1] += n
ts = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"{'phase':20s} {'stall%':>7s} {'inst%':>7s}   (total {ti:.3g} warp-instructions)")
for k, (s, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:20s} {100*s/ts:7.1f} {100*n/ti:7.1f}")
