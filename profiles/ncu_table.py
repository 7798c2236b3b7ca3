"""Summarise an ncu report: one line per captured kernel with duration,
DRAM bytes, tensor-pipe and DRAM utilisation.
usage: python profiles/ncu_table.py gpurun_out/prof_gemm.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "rd",
    "dram__bytes_write.sum": "wr",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    for r in rows[2:]:
        out = {"kernel": r[name_i].split("(")[0].replace("(anonymous namespace)::", "")[-40:]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    x = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    x = v
                out[short] = round(x, 2) if isinstance(x, float) else x
        print(out)


if __name__ == "__main__":
    main(sys.argv[1])
