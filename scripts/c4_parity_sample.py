"""Parity at the exact headline workload beyond bench.py's per-run gate:
segments [a, b) of the bench's 8 h recording (the same seeded grids,
T_enc 249, vocab 5000, beam 10, default knobs, 5-best) decoded on the GPU
inside the full 2880-segment call, and by the unmodified reference
(oracle/_ref) on all host cores; tokens, label times, steps, triggers and
joints compared (the n-best lists are pinned by tests/test_gpu_parity.py). python scripts/c4_parity_sample.py [a b]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_05600_b200 as bl  # noqa: E402
import pyoracle as po  # noqa: E402

a = int(sys.argv[1]) if len(sys.argv) > 1 else 0
b = int(sys.argv[2]) if len(sys.argv) > 2 else 32
dev = torch.device("cuda", 0)
n = 2880
g = bench.segment_grids(torch, 0, n, dev, 100000)
dec = bl.Decoder(bl.UniformScorer(bench.VOCAB - 1), bl.DecoderConfig(beam_width=bench.BEAM),
                 nbest=bench.NBEST)
stride = bench.T_ENC * bench.VOCAB * 4
descs = [(f"s{i}", bench.T_ENC, bench.VOCAB, g.data_ptr() + i * stride) for i in range(n)]
res = list(dec.decode_raw(descs, on_device=True))
host = [g[i].cpu().numpy() for i in range(a, b)]
t0 = time.perf_counter()
want, _ = po.Ref().decode(host, po.ScorerSpec("uniform", bench.VOCAB - 1),
                          po.config(beam_width=bench.BEAM), batch_size=128,
                          ids=[f"s{i}" for i in range(a, b)], threads=os.cpu_count())
wall = time.perf_counter() - t0
bad = 0
for i, w in zip(range(a, b), want):
    r = res[i]
    ok = (r.tokens == w.tokens and r.label_times == w.label_times and r.steps_taken == w.steps
          and r.eos_trigger == w.eos_trigger and abs(r.joint_logp - w.joint_logp) <= 1e-9)
    bad += 0 if ok else 1
print(f"segments [{a}, {b}) of the 2880-segment headline call vs oracle/_ref "
      f"({os.cpu_count()} threads, {wall:.0f} s): {b - a - bad} identical, {bad} mismatches")
sys.exit(1 if bad else 0)
