"""Runs bench.py's config-3 prefix-score leg alone (vocab 5000, TMA slab):
prints kernel ms and K1 GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_05600_b200 as bl  # noqa: E402

r = bench.run_prefix_c3(torch, bl, torch.device("cuda", 0), bench.peaks())
print("c3 kernel %.2f ms  %.0f GB/s  frac %.3f" % (r["kernel_ms"], r["k1_gbs"], r["frac"]))
