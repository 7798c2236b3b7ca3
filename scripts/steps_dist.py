"""Distribution of decode steps per segment on the bench workload (C2),
and the kernel time with segments ordered by step count (tail check)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05600_b200 as bl  # noqa: E402
import bench  # noqa: E402

n = 2880
g = bench.flat_grids(torch, n, 1000, torch.device("cuda"))
cfg = bl.DecoderConfig(beam_width=10, ctc_weight=0.3, margin_m1=5, margin_m2=20, eos_mode="both")
dec = bl.Decoder(bl.UniformScorer(499), cfg)
stride = 249 * 500 * 4
descs = [(f"s{i}", 249, 500, g.data_ptr() + i * stride) for i in range(n)]
for _ in range(2):
    res = dec.decode_raw(descs, on_device=True)
st = np.array([r.steps_taken for r in res])
print("kernel_ms", dec.last_stats["kernel_ms"])
print("steps: mean %.1f p50 %d p90 %d p99 %d max %d" % (st.mean(), *np.percentile(st, [50, 90, 99]), st.max()))
order = np.argsort(-st)  # longest first
d2 = [descs[i] for i in order]
for _ in range(2):
    dec.decode_raw(d2, on_device=True)
print("longest-first kernel_ms", dec.last_stats["kernel_ms"])
