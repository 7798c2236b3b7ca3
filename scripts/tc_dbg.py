import sys, numpy as np
sys.path.insert(0, ".")
import paper_2101_05600_b200 as bl
V = 5000
rng = np.random.default_rng(0)
G = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    p = rng.exponential(size=(int(sys.argv[2]) if len(sys.argv) > 2 else 40, V)); G.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
d = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=10))
r = d.decode([bl.Utterance(f"u{i}", bl.PosteriorGrid(g)) for i, g in enumerate(G)])
print("ok", [len(x.tokens) for x in r], d.last_stats["fallback_steps"], d.last_stats["kernel_ms"])
