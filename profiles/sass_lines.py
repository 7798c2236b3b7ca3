"""Joins an ncu SASS source page (csv) with nvdisasm -g line info to rank
source lines by warp-stall samples and executed instructions."""
import collections
import csv
import re
import sys


def line_map(sass_path, func):
    cur = None
    amap = {}
    infn = False
    for ln in open(sass_path):
        if ln.startswith("//---------------------"):
            infn = func in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            amap[int(m.group(1), 16)] = cur
    return amap


def main(ncu_csv, sass_path, func, src_path, top=40):
    amap = line_map(sass_path, func)
    rows = list(csv.reader(open(ncu_csv)))
    hdr = rows[1]
    ia, isamp, iinst = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Instructions Executed")
    agg = collections.defaultdict(lambda: [0, 0])
    tot_s = tot_i = 0
    base = int(rows[2][ia], 16)
    for r in rows[2:]:
        try:
            a = int(r[ia], 16) - base
            s, n = float(r[isamp] or 0), float(r[iinst] or 0)
        except (ValueError, IndexError):
            continue
        key = amap.get(a, ("?", 0))
        agg[key][0] += s
        agg[key][1] += n
        tot_s += s
        tot_i += n
    src = {}
    try:
        src = {i + 1: l.rstrip() for i, l in enumerate(open(src_path))}
    except OSError:
        pass
    print(f"total samples {tot_s:.0f}, instructions {tot_i:.3g}")
    for (f, l), (s, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        text = src.get(l, "") if f == src_path.split("/")[-1] else ""
        print(f"{100*s/tot_s:5.1f}% smp {100*n/tot_i:5.1f}% inst  {f}:{l:<5d} {text.strip()[:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
