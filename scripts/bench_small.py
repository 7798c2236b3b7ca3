"""Small fixed workload for kernel profiling: 64 flat segments, T=249,
vocab 500, B=10, M2=20 (the bench config's per-utterance shape)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2101_05600_b200 as bl
rng = np.random.default_rng(1)
G = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 64):
    p = rng.exponential(size=(249, 500))
    G.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
utts = [bl.Utterance(f"b{i}", bl.PosteriorGrid(g)) for i, g in enumerate(G)]
dec = bl.Decoder(bl.UniformScorer(499), bl.DecoderConfig(beam_width=10, margin_m2=20))
for _ in range(2):
    dec.decode(utts)
print(dec.last_stats)
