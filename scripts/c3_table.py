"""Experiment: the C3 decode shape with PER-HYPOTHESIS scorer rows (a
bigram table with a row for every context token, all rows the flat
distribution) instead of the uniform scorer's one shared row, one launch
and step-granular: isolates the cost of per-hypothesis rows in the search
kernel from the network kernels. python scripts/c3_table.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_05600_b200 as bl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2880
V = bench.VOCAB
dev = torch.device("cuda", 0)
g = bench.segment_grids(torch, 0, n, dev, 100000)
row = list(np.full(V, -np.log(V)))
stride = bench.T_ENC * V * 4
descs = [(f"t{i}", bench.T_ENC, V, g.data_ptr() + i * stride) for i in range(n)]
rng = np.random.default_rng(5)
noisy = [list(np.log(r / r.sum())) for r in rng.exponential(size=(V - 1, V))]
for kind in ("uniform", "table", "table_noisy"):
    for step in (False, True):
        if kind == "uniform":
            sc = bl.UniformScorer(V - 1)
        else:
            sc = bl.TableScorer(V - 1, 2)
            sc._entries = {(t,): (row if kind == "table" else noisy[t]) for t in range(V - 1)}
            sc._rebuild()
        dec = bl.Decoder(sc, bl.DecoderConfig(beam_width=bench.BEAM), step_mode=step)
        torch.cuda.synchronize()
        for _ in range(2):
            dec.decode_raw(descs, on_device=True)
        st = dec.last_stats
        print(f"{kind:8s} step={int(step)}: kernel {st['kernel_ms']:.1f} ms  filter_keys/step "
              f"{st['filter_keys'] / max(1, st['steps']):.1f}  contenders/step "
              f"{st['contenders'] / max(1, st['steps']):.1f}", flush=True)
