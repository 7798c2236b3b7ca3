"""Stall-reason breakdown per phase from an ncu SASS source page (csv)."""
import collections
import csv
import re
import sys

sys.path.insert(0, "profiles")
from sass_lines import line_map  # noqa: E402

ncu_csv, sass, func, src = sys.argv[1:5]
marks = [(i, int(m.group(1))) for i, l in enumerate(open(src), 1)
         for m in [re.search(r"PROF_MARK\((\d+)\);", l)] if m and "#define" not in l]
names = {0: "init", 1: "P1", 2: "P2", 3: "P3", 4: "P4", 5: "P5", 6: "P6", 7: "P7", 8: "fb",
         9: "P8", 10: "P9", 11: "fin"}


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
ia = hdr.index("Address")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(h) for h in reasons]
base = int(rows[2][ia], 16)
agg = collections.defaultdict(lambda: collections.Counter())
for r in rows[2:]:
    try:
        a = int(r[ia], 16) - base
    except (ValueError, IndexError):
        continue
    f, l = amap.get(a, ("?", 0))
    ph = phase_of(l) if f == src.split("/")[-1] else f
    for h, i in zip(reasons, idx):
        try:
            agg[ph][h] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(sum(c.values()) for c in agg.values())
for ph, c in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
    s = sum(c.values())
    top = ", ".join(f"{k[6:]} {100*v/tot:.1f}" for k, v in c.most_common(5))
    print(f"{ph:22s} {100*s/tot:5.1f}%  [{top}]")
