"""BASELINE config 2's knobs (vocab 500, M2 = 20, beam 10) on N segments
(default 2880) from HBM: kernel ms of one call (bench.py's c2_vocab500 leg
alone). python scripts/c2_leg.py [N]"""
import os
import sys

sys.path.insert(0, os.environ.get("BL_PKG_ROOT",
                                  os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2101_05600_b200 as bl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2880
T, V = 249, 500
dev = torch.device("cuda", 0)
g = torch.empty((n, T, V), dtype=torch.float32, device=dev)
gen = torch.Generator(device=dev)
gen.manual_seed(1000)
for s0 in range(0, n, 256):
    x = torch.empty((min(n, s0 + 256) - s0, T, V), dtype=torch.float64, device=dev)
    x.exponential_(generator=gen)
    g[s0:s0 + x.shape[0]] = torch.log(x / x.sum(-1, keepdim=True)).float()
dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=10, margin_m2=20))
descs = [(f"c2_{i}", T, V, g.data_ptr() + i * T * V * 4) for i in range(n)]
torch.cuda.synchronize()
kms = []
for k in range(4):
    dec.decode_raw(descs, on_device=True)
    if k:
        kms.append(dec.last_stats["kernel_ms"])
print("c2 %d segments: kernel %.2f ms (min %.2f)" % (n, sum(kms) / len(kms), min(kms)))
