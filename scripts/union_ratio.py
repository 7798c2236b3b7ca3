"""Distinct ancestor entries (union over the live beam) vs nb*l, from the
recorded prefixes of a Transformer-scored decode."""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05600_b200 as bl  # noqa: E402
from paper_2101_05600_b200 import encoder as enc  # noqa: E402
from paper_2101_05600_b200 import transformer as tr  # noqa: E402

e = enc.Encoder(enc.SMALL, enc.random_weights(enc.SMALL, seed=0))
grid, mem = e.forward(torch.from_numpy(enc.synthetic_fbank(4, 1000, seed=2)), memory=True)
dec = bl.Decoder(tr.TransformerScorer(tr.SMALL, tr.random_weights(tr.SMALL, seed=1)),
                 bl.DecoderConfig(beam_width=10, margin_m1=5, margin_m2=20))
dec.set_record(True)
descs = [(f"s{i}", 249, 500, grid[i].data_ptr()) for i in range(4)]
dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(), mem_frames=249)
by = collections.defaultdict(list)
for u, p, _ in dec.records():
    by[(u, len(p))].append(p)
tot_u, tot_n = 0, 0
for (u, l), ps in sorted(by.items()):
    union = sum(len({q[:k] for q in ps}) for k in range(l + 1))   # positions 0..l
    tot_u += union
    tot_n += len(ps) * (l + 1)
    if u == 0 and l in (5, 20, 50, 100, 200):
        print("l", l, "nb", len(ps), "union", union, "nb*l", len(ps) * (l + 1))
print("overall union / (nb*l) = %.3f" % (tot_u / tot_n))
