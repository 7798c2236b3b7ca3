"""Dev parity sweep on the GPU vs the compiled reference (oracle/_ref)."""
import math
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import numpy as np

import paper_2101_05600_b200 as bl
import pyoracle as po

ref = po.Ref()


def cmp(got, want, tol=1e-9):
    bad = 0
    for g, w in zip(got, want):
        if (g.tokens != w.tokens or g.label_times != w.label_times or g.steps_taken != w.steps
                or g.eos_trigger != w.eos_trigger or abs(g.joint_logp - w.joint_logp) > tol):
            bad += 1
            if bad <= 3:
                print("  MISMATCH", g.id, g.tokens[:8], w.tokens[:8], g.steps_taken, w.steps,
                      g.eos_trigger, w.eos_trigger, g.joint_logp, w.joint_logp)
    return bad


def run(name, corpus, spec_bl, spec_po, kw, batch=16, exact_modes=(False, True)):
    ids = [c[0] for c in corpus]
    grids = [c[1] for c in corpus]
    want, wc = ref.decode(grids, spec_po, po.config(**kw), batch_size=batch, ids=ids)
    utts = [bl.Utterance(i, bl.PosteriorGrid(g)) for i, g in corpus]
    for exact in exact_modes:
        dec = bl.Decoder(spec_bl, bl.DecoderConfig(**kw), exact=exact)
        cnt = bl.DecodeCounters()
        got = dec.decode(utts, cnt)
        b = cmp(got, want)
        cok = (cnt.steps, cnt.scorer_queries, cnt.ctc_frames_evaluated) == tuple(wc)
        st = dec.last_stats
        print(f"{name:28s} {'exact' if exact else 'fast ':5s} {kw} bad={b} counters_ok={cok} "
              f"kernel={st['kernel_ms']:.2f}ms fallback={st['fallback_steps']} "
              f"cont/step={st['contenders'] / max(1, st['steps']):.1f}")


corp = ref.random_corpus(5, 60, 10, 60, 3)
for kw in [{}, dict(margin_m1=bl.NO_MARGIN), dict(margin_m2=3), dict(ctc_weight=1.0),
           dict(ctc_weight=0.0), dict(eos_mode="ctc", beam_width=5),
           dict(beam_width=10, margin_m2=20), dict(eos_mode="baseline")]:
    run("random C=3", corp, bl.UniformScorer(3), po.ScorerSpec("uniform", 3), kw)

planted = ref.synth_corpus(7, 40, 500, 500, 5, "planted")
run("planted T=500 (C7)", planted, bl.UniformScorer(5), po.ScorerSpec("uniform", 5),
    dict(margin_m1=5, margin_m2=20))
run("planted T=500 unrestricted", planted[:10], bl.UniformScorer(5), po.ScorerSpec("uniform", 5),
    dict(margin_m1=bl.NO_MARGIN, margin_m2=bl.NO_MARGIN))

# EOS pathology (acceptance C6): loop grid + LoopScorer
def loop_grid(seed, t):
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(t):
        p = np.array([0.90 * rng.uniform(0.9, 1.1), 0.03 * rng.uniform(0.9, 1.1), 0.07])
        rows.append(np.log(p / p.sum()))
    return np.array(rows, dtype=np.float32)
lg = [(f"loop{s}", loop_grid(s, 100)) for s in range(1, 21)]
for mode in ("baseline", "both"):
    run("loop C6 " + mode, lg, bl.LoopScorer(2, 0, 0.9), po.ScorerSpec("loop", 2, loop_token=0, p_loop=0.9),
        dict(ctc_weight=0.3, margin_m1=bl.NO_MARGIN, max_steps_ratio=0.25, eos_mode=mode))

# table scorer, order 3
rng = np.random.default_rng(3)
C = 4
ents = []
for ctx in [(), (0,), (1,), (2, 3), (0, 0), (3, 1), (1, 2)]:
    p = rng.exponential(size=C + 1)
    lp = list(np.log(p / p.sum()))
    ents.append((ctx, lp))
ts = bl.TableScorer(C, 3)
for ctx, lp in ents:
    ts.add_entry(ctx, lp)
tcorp = ref.random_corpus(11, 30, 10, 50, C)
run("table order3", tcorp, ts, po.ScorerSpec("table", C, order=3, entries=ents), dict(beam_width=6))

# all-blank grid + sharpened grids (fp32 underflow guard)
blank = [("blank", np.array([[-1e30, -1e30, 0.0]] * 8, dtype=np.float32))]
run("all-blank", blank, bl.UniformScorer(2), po.ScorerSpec("uniform", 2), {})
sharp = []
for i, (uid, g) in enumerate(ref.synth_corpus(21, 12, 80, 120, 20, "planted")):
    h = g.astype(np.float64) * 12.0
    h = h - np.log(np.exp(h - h.max(1, keepdims=True)).sum(1, keepdims=True)) - h.max(1, keepdims=True)
    sharp.append((uid, h.astype(np.float32)))
run("sharpened x12", sharp, bl.UniformScorer(20), po.ScorerSpec("uniform", 20), dict(beam_width=8, margin_m2=20))

# bench-like
G = []
for i in range(64):
    p = rng.exponential(size=(249, 500))
    G.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
utts = [bl.Utterance(f"b{i}", bl.PosteriorGrid(g)) for i, g in enumerate(G)]
dec = bl.Decoder(bl.UniformScorer(499), bl.DecoderConfig(beam_width=10, margin_m2=20))
for rep in range(3):
    t = time.time()
    got = dec.decode(utts)
    el = time.time() - t
    print("bench-like U=64 V=500 B=10 M2=20: wall %.3f s, kernel %.3f ms, fallback %d" % (
        el, dec.last_stats["kernel_ms"], dec.last_stats["fallback_steps"]))
t = time.time()
want, wc = ref.decode(G[:8], po.ScorerSpec("uniform", 499), po.config(beam_width=10, margin_m2=20),
                      batch_size=8, ids=[u.id for u in utts[:8]])
print("ref 8 utts: %.2f s" % (time.time() - t), "bad", cmp(got[:8], want))
