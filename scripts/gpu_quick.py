import sys, time, os
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import paper_2101_05600_b200 as bl
import pyoracle as po
ref = po.Ref()
def cmp(got, want, tol=1e-9):
    bad = 0
    for g, w in zip(got, want):
        if g.tokens != w.tokens or g.label_times != w.label_times or g.steps_taken != w.steps or g.eos_trigger != w.eos_trigger or abs(g.joint_logp - w.joint_logp) > tol:
            bad += 1
            if bad <= 3: print("MISMATCH", g.id, g.tokens[:10], w.tokens[:10], g.steps_taken, w.steps, g.eos_trigger, w.eos_trigger, g.joint_logp, w.joint_logp)
    return bad
corp = ref.random_corpus(5, 60, 10, 60, 3)
ids = [c[0] for c in corp]; grids = [c[1] for c in corp]
utts = [bl.Utterance(i, bl.PosteriorGrid(g)) for i, g in corp]
for exact in (True, False):
  for kw in [{}, dict(margin_m1=bl.NO_MARGIN), dict(margin_m2=3), dict(ctc_weight=1.0), dict(ctc_weight=0.0), dict(eos_mode="ctc", beam_width=5), dict(beam_width=10, margin_m2=20), dict(eos_mode="baseline")]:
    cfg = bl.DecoderConfig(**kw)
    pc = po.config(**kw)
    want, wc = ref.decode(grids, po.ScorerSpec("uniform", 3), pc, batch_size=16, ids=ids)
    dec = bl.Decoder(bl.UniformScorer(3), cfg, exact=exact)
    cnt = bl.DecodeCounters()
    got = dec.decode(utts, cnt)
    print("exact" if exact else "fast", kw, "bad", cmp(got, want), "counters", (cnt.steps, cnt.scorer_queries, cnt.ctc_frames_evaluated), wc, dec.last_stats)
# bench-like
rng = np.random.default_rng(1)
G = []
for i in range(64):
    p = rng.exponential(size=(249, 500)); G.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
utts = [bl.Utterance(f"b{i}", bl.PosteriorGrid(g)) for i, g in enumerate(G)]
cfg = bl.DecoderConfig(beam_width=10, margin_m2=20)
dec = bl.Decoder(bl.UniformScorer(499), cfg)
for rep in range(3):
    t = time.time(); got = dec.decode(utts); el = time.time() - t
    print("bench-like U=64 V=500 B=10 M2=20: wall %.3f s, kernel %.3f ms" % (el, dec.last_stats["kernel_ms"]), dec.last_stats)
t = time.time()
want, wc = ref.decode(G[:8], po.ScorerSpec("uniform", 499), po.config(beam_width=10, margin_m2=20), batch_size=8, ids=[u.id for u in utts[:8]])
print("ref 8 utts: %.2f s" % (time.time() - t), "bad", cmp(got[:8], want))
