"""Per-kernel SASS opcode census of libbl_b200.so (cuobjdump -sass): the
evidence of which hardware paths each kernel uses -- tcgen05 MMA (UTCHMMA /
UTCQMMA), TMA (UTMALDG / UTMASTG), TMEM loads/stores (LDTM / STTM), legacy
warp MMA (HMMA), packed fp32 FMA (FFMA2), exp2 (MUFU.EX2), fp64 (DFMA /
DADD / DMUL), mbarrier ops (SYNCS).
python profiles/sass_summary.py [paper_2101_05600_b200/libbl_b200.so]"""
import collections
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "HMMA", "FFMA2", "MUFU.EX2",
       "DFMA", "DADD", "DMUL", "SYNCS", "LDG", "STG", "LDS", "STS"]


def main(path):
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, counts = None, collections.OrderedDict()
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            counts.setdefault(cur, collections.Counter())
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if not m:
            continue
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                counts[cur][o] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True,
                               text=True).stdout.splitlines()
    print("%-58s " % "kernel" + " ".join("%8s" % o for o in OPS))
    for (k, c), dn in zip(counts.items(), demangled):
        name = dn
        if name.endswith(")"):  # drop the parameter list (the last balanced parentheses)
            depth = 0
            for i in range(len(name) - 1, -1, -1):
                depth += {")": 1, "(": -1}.get(name[i], 0)
                if depth == 0:
                    name = name[:i]
                    break
        name = name.replace("(anonymous namespace)::", "")[:58]
        print("%-58s " % name + " ".join("%8d" % c[o] for o in OPS))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2101_05600_b200/libbl_b200.so")
