"""Randomised parity sweep: the device decoder against the compiled reference
(oracle/_ref, unmodified batched_beam_search) over the configuration space —
beam 1..32, vocabularies 2..500, ragged lengths 1..100, both margins, all
three eos modes, ctc weights 0..1, eos M/C/Dend, max-steps ratios, uniform /
loop / n-gram table scorers, random / planted / blank-heavy grids, optionally
sharpened — in the three decoder modes (certified fp32 bulk, fp64 decisions,
step-granular). Tokens, label times, steps and triggers identical; joint
within 1e-9; counters equal."""
import os

import numpy as np
import pytest

import paper_2101_05600_b200 as bl
import pyoracle as po

pytestmark = pytest.mark.gpu
CASES = int(os.environ.get("BL_FUZZ_CASES", "64"))


def _case(k, ref):
    rng = np.random.default_rng(7000 + k)
    C = int(rng.choice([1, 2, 3, 5, 8, 17, 40, 120, 499]))
    B = int(rng.choice([1, 2, 3, 4, 7, 10, 16, 24, 32]))
    n = int(rng.integers(1, 7))
    style = str(rng.choice(["random", "planted", "blank_heavy"]))
    t_lo = int(rng.integers(1, 40))
    t_hi = t_lo + int(rng.integers(0, 60))
    items = ref.synth_corpus(int(rng.integers(1, 1 << 30)), n, t_lo, t_hi, C, style)
    if rng.random() < 0.3:  # peaky posteriors: log-domain plateau ties
        k_sh = float(rng.choice([4.0, 10.0]))
        out = []
        for u, g in items:
            h = g.astype(np.float64) * k_sh
            m = h.max(1, keepdims=True)
            out.append((u, (h - m - np.log(np.exp(h - m).sum(1, keepdims=True)))
                        .astype(np.float32)))
        items = out
    kw = dict(beam_width=B, ctc_weight=float(rng.choice([0.0, 0.3, 0.5, 1.0])),
              eos_m=int(rng.integers(1, 5)), eos_dend=float(rng.choice([-30.0, -10.0, -3.0])),
              eos_c=int(rng.integers(0, 4)), margin_m1=int(rng.integers(0, 8)),
              margin_m2=int(rng.choice([bl.NO_MARGIN, 3, 10, 25])),
              eos_mode=str(rng.choice(["baseline", "ctc", "both"])),
              max_steps_ratio=float(rng.choice([1.0, 0.6, 0.25])))
    kind = str(rng.choice(["uniform", "loop", "table"])) if C >= 2 else "uniform"
    if kind == "uniform":
        spec, sc = po.ScorerSpec("uniform", C), bl.UniformScorer(C)
    elif kind == "loop":
        tok, p = int(rng.integers(0, C)), float(rng.choice([0.6, 0.9, 0.99]))
        spec, sc = po.ScorerSpec("loop", C, loop_token=tok, p_loop=p), bl.LoopScorer(C, tok, p)
    else:
        order = int(rng.integers(2, 4))
        ents = []
        for _ in range(int(rng.integers(1, 12))):
            ctx = tuple(int(x) for x in rng.integers(0, C, size=int(rng.integers(0, order))))
            pr = rng.exponential(size=C + 1)
            ents.append((ctx, list(np.log(pr / pr.sum()))))
        ents = list({c: (c, lp) for c, lp in ents}.values())
        spec = po.ScorerSpec("table", C, order=order, entries=ents)
        sc = bl.TableScorer(C, order)
        for ctx, lp in ents:
            sc.add_entry(ctx, lp)
    mode = str(rng.choice(["fast", "exact", "step"]))
    return items, kw, spec, sc, mode


@pytest.mark.parametrize("k", range(CASES))
def test_random_config_vs_reference(ref, k):
    items, kw, spec, sc, mode = _case(k, ref)
    ids = [u for u, _ in items]
    want, wc = ref.decode([g for _, g in items], spec, po.config(**kw), ids=ids)
    cnt = bl.DecodeCounters()
    dec = bl.Decoder(sc, bl.DecoderConfig(**kw), exact=mode == "exact", step_mode=mode == "step")
    got = dec.decode([bl.Utterance(u, bl.PosteriorGrid(g)) for u, g in items], cnt)
    assert [g.id for g in got] == ids
    for g, w in zip(got, want):
        assert g.tokens == w.tokens, (kw, mode, g.id)
        assert g.label_times == w.label_times, (kw, mode, g.id)
        assert g.steps_taken == w.steps and g.eos_trigger == w.eos_trigger, (kw, mode, g.id)
        assert abs(g.joint_logp - w.joint_logp) <= 1e-9, (kw, mode, g.id)
    assert (cnt.steps, cnt.scorer_queries, cnt.ctc_frames_evaluated) == tuple(wc)


LARGE_CASES = int(os.environ.get("BL_FUZZ_LARGE_CASES", "16"))


@pytest.mark.parametrize("k", range(LARGE_CASES))
def test_random_large_vocab_vs_reference(ref, k):
    """Large vocabularies (the on-chip key filter): V 1024 / 2048 / 5000,
    beams up to 24, ragged lengths, both margins, all eos modes, uniform /
    loop scorers, random / planted / blank-heavy / sharpened grids; host grids
    (TMA slab, kMode 2), step-granular, and separately allocated device grids
    (no dense slab: the __ldg filter variant, kMode 1)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9100 + k)
    C = int(rng.choice([1023, 2047, 4999]))
    B = int(rng.choice([1, 3, 4, 10, 16, 24]))
    n = int(rng.integers(1, 5))
    style = str(rng.choice(["random", "planted", "blank_heavy"]))
    t_lo = int(rng.integers(2, 30))
    items = ref.synth_corpus(int(rng.integers(1, 1 << 30)), n, t_lo, t_lo + int(rng.integers(0, 40)),
                             C, style)
    if rng.random() < 0.3:
        out = []
        for u, g in items:
            h = g.astype(np.float64) * 6.0
            m = h.max(1, keepdims=True)
            out.append((u, (h - m - np.log(np.exp(h - m).sum(1, keepdims=True)))
                        .astype(np.float32)))
        items = out
    kw = dict(beam_width=B, ctc_weight=float(rng.choice([0.3, 0.5, 1.0])),
              eos_m=int(rng.integers(1, 4)), eos_c=int(rng.integers(0, 3)),
              margin_m1=int(rng.integers(0, 8)),
              margin_m2=int(rng.choice([bl.NO_MARGIN, 5, 20])),
              eos_mode=str(rng.choice(["baseline", "ctc", "both"])))
    if rng.random() < 0.5:
        spec, sc = po.ScorerSpec("uniform", C), bl.UniformScorer(C)
    else:
        tok, p = int(rng.integers(0, C)), float(rng.choice([0.6, 0.9]))
        spec, sc = po.ScorerSpec("loop", C, loop_token=tok, p_loop=p), bl.LoopScorer(C, tok, p)
    mode = str(rng.choice(["host", "step", "nondense"]))
    ids = [u for u, _ in items]
    want, wc = ref.decode([g for _, g in items], spec, po.config(**kw), ids=ids)
    cnt = bl.DecodeCounters()
    dec = bl.Decoder(sc, bl.DecoderConfig(**kw), step_mode=mode == "step")
    if mode == "nondense":
        dev = [torch.from_numpy(g).cuda() for _, g in items]
        torch.cuda.synchronize()
        got = list(dec.decode_raw([(u, g.shape[0], g.shape[1], d.data_ptr())
                                   for (u, g), d in zip(items, dev)], on_device=True,
                                  counters=cnt))
    else:
        got = dec.decode([bl.Utterance(u, bl.PosteriorGrid(g)) for u, g in items], cnt)
    for g, w in zip(got, want):
        assert g.tokens == w.tokens, (kw, mode, g.id)
        assert g.label_times == w.label_times, (kw, mode, g.id)
        assert g.steps_taken == w.steps and g.eos_trigger == w.eos_trigger, (kw, mode, g.id)
        assert abs(g.joint_logp - w.joint_logp) <= 1e-9, (kw, mode, g.id)
    assert (cnt.steps, cnt.scorer_queries, cnt.ctc_frames_evaluated) == tuple(wc)
