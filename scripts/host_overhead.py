"""Host-side overhead of one bench-shaped decode call: wall time of
bl_decode (C: plan + launch + sync + result assembly) and of the Python
export, vs the kernel time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05600_b200 as bl  # noqa: E402
import bench  # noqa: E402
from paper_2101_05600_b200 import api  # noqa: E402

n = 2880
g = bench.flat_grids(torch, n, 1000, torch.device("cuda"))
cfg = bl.DecoderConfig(beam_width=10, ctc_weight=0.3, margin_m1=5, margin_m2=20, eos_mode="both")
dec = bl.Decoder(bl.UniformScorer(499), cfg)
stride = 249 * 500 * 4
descs = [(f"s{i}", 249, 500, g.data_ptr() + i * stride) for i in range(n)]
orig = api.Decoder._collect
tc = []


def timed_collect(self, h, counters, ids):
    t = time.perf_counter()
    r = orig(self, h, counters, ids)
    tc.append(time.perf_counter() - t)
    return r


api.Decoder._collect = timed_collect
for _ in range(2):
    dec.decode_raw(descs, on_device=True)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    dec.decode_raw(descs, on_device=True)
    t1 = time.perf_counter()
    print("wall %.2f ms  kernel %.2f ms  python collect %s" %
          ((t1 - t0) * 1e3, dec.last_stats["kernel_ms"],
           "%.2f ms" % (tc[-1] * 1e3) if tc else "bulk path (bl_decode_into)"))
