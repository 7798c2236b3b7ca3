import sys, numpy as np
sys.path.insert(0, ".")
import paper_2101_05600_b200 as bl
rng = np.random.default_rng(0)
for V in (8, 500, 5000):
    for T in (499, 1000, 1500, 2000, 3000):
        p = rng.exponential(size=(T, V)); g = np.log(p / p.sum(1, keepdims=True)).astype(np.float32)
        try:
            r = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=10, margin_m2=20)).decode([bl.Utterance("x", bl.PosteriorGrid(g))])
            print(V, T, "ok", r[0].steps_taken)
        except Exception as e:
            print(V, T, "ERR", type(e).__name__, str(e)[:80])
