"""Transformer attention-decoder scorer (SURVEY.md §8 a'2).

* Network numerics (unpinned by the reference): every row the device scorer
  produced for a live hypothesis, recorded with its prefix, against the
  torch-CPU decoder (oracle/torch_decoder.py) run NON-incrementally on the
  same prefix and the same encoder memory: max |d logp| <= 0.05 with bf16
  rounding emulated (checks the KV-cache ancestor addressing too).
* Search parity (pinned): the reference decoder (oracle/_ref, unmodified
  batched_beam_search) driven by a replay scorer that answers each
  (utterance, prefix) query with the device's row gives identical tokens,
  label times, steps, triggers (joint within 1e-9), with zero replay misses
  (a miss = the reference asked for a prefix the device never scored).
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2101_05600_b200 as bl
from paper_2101_05600_b200 import encoder as enc
from paper_2101_05600_b200 import transformer as tr
from paper_2101_05600_b200.api import lib

TINY_ENC = enc.EncoderSpec(80, 128, 2, 256, 2, 64)
TINY_DEC = tr.DecoderSpec(128, 2, 256, 2, 64)


def test_decoder_weight_count_matches_library():
    for spec in (tr.SMALL, tr.LARGE, TINY_DEC):
        assert lib().bl_transformer_num_weights(C.byref(spec.c())) == spec.num_weights()
    bad = tr.DecoderSpec(100, 2, 256, 2, 64)
    assert lib().bl_transformer_num_weights(C.byref(bad.c())) == 0


def test_torch_decoder_reference_is_normalised():
    from torch_decoder import decoder_scores
    w = tr.random_weights(TINY_DEC, seed=3)
    mem = np.random.default_rng(0).standard_normal((20, 128)).astype(np.float32)
    rows = decoder_scores(TINY_DEC, w, mem, [(), (1,), (1, 5, 7)])
    assert rows.shape == (3, 64)
    np.testing.assert_allclose(np.exp(rows).sum(1), 1.0, atol=1e-9)


def test_replay_scorer_without_entries_is_uniform(ref):
    """The shim's replay scorer: unanswered queries count as misses and fall
    back to the uniform row, so an empty table decodes like UniformScorer."""
    import pyoracle as po
    items = ref.random_corpus(5, 4, 10, 30, 3)
    grids, ids = [g for _, g in items], [u for u, _ in items]
    want, wc = ref.decode(grids, po.ScorerSpec("uniform", 3), po.config(), ids=ids)
    ref.replay_misses(reset=True)
    got, gc = ref.decode(grids, po.ScorerSpec("replay", 3, replay_ids=ids), po.config(), ids=ids)
    assert [r.tokens for r in got] == [r.tokens for r in want]
    assert ref.replay_misses() == wc[1] > 0


# ---------------------------------------------------------------- GPU tests
def _setup(espec, dspec, n, frames, seed):
    torch = pytest.importorskip("torch")
    e = enc.Encoder(espec, enc.random_weights(espec, seed=seed))
    fb = torch.from_numpy(enc.synthetic_fbank(n, frames, espec.idim, seed=seed + 1))
    grid, mem = e.forward(fb, memory=True)
    w = tr.random_weights(dspec, seed=seed + 2)
    return grid, mem, w


def _decode(grid, mem, scorer, cfg, record=True, nbest=1):
    torch = pytest.importorskip("torch")
    dec = bl.Decoder(scorer, cfg, nbest=nbest)
    dec.set_record(record)
    n, T, V = grid.shape
    descs = [(f"s{i}", T, V, grid[i].data_ptr()) for i in range(n)]
    torch.cuda.synchronize()
    res = dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(), mem_frames=T)
    return dec, list(res), [d[0] for d in descs]


@pytest.mark.gpu
@pytest.mark.parametrize("beam,frames", [(1, 200), (4, 200), (10, 200), (16, 200), (20, 200),
                                         (10, 1000), (20, 1000)])
def test_transformer_rows_vs_torch(beam, frames):
    """beam <= 16: union-of-ancestors self-attention (mma.sync); beam 20:
    the per-hypothesis warp kernel (csrc/decoder_net.cu use_union_self_attn).
    1000 frames (T2 = 249 memory rows, 128 per stage): the staged source
    attention runs several stages per warp with the cross-warp merge, and the
    self-attention union list spans several stages late in the decode."""
    from torch_decoder import decoder_scores
    grid, mem, w = _setup(TINY_ENC, TINY_DEC, 3, frames, seed=5)
    sc = tr.TransformerScorer(TINY_DEC, w)
    dec, res, ids = _decode(grid, mem, sc, bl.DecoderConfig(beam_width=beam))
    recs = dec.records()
    assert len(recs) > 0
    memh = mem.float().cpu().numpy()
    rng = np.random.default_rng(0)
    worst = 0.0
    for u in range(grid.shape[0]):
        mine = [r for r in recs if r[0] == u]
        pick = [mine[i] for i in sorted(rng.choice(len(mine), min(len(mine), 25), replace=False))]
        want = decoder_scores(TINY_DEC, w, memh[u], [p for _, p, _ in pick], emulate_bf16=True)
        got = np.stack([r for _, _, r in pick])
        np.testing.assert_allclose(np.exp(got).sum(1), 1.0, atol=1e-12)
        worst = max(worst, float(np.abs(got - want).max()))
    assert worst <= 0.05, worst


@pytest.mark.gpu
@pytest.mark.parametrize("espec,dspec,n,frames,beam,m2", [
    (TINY_ENC, TINY_DEC, 4, 200, 4, bl.NO_MARGIN),
    (TINY_ENC, TINY_DEC, 3, 400, 6, 10),
    (enc.SMALL, tr.SMALL, 2, 1000, 10, 20),
])
def test_transformer_search_vs_reference_replay(ref, espec, dspec, n, frames, beam, m2):
    import pyoracle as po
    grid, mem, w = _setup(espec, dspec, n, frames, seed=7)
    kw = dict(beam_width=beam, margin_m1=5, margin_m2=m2)
    sc = tr.TransformerScorer(dspec, w)
    dec, res, ids = _decode(grid, mem, sc, bl.DecoderConfig(**kw))
    recs = dec.records()
    spec = po.ScorerSpec("replay", dspec.vocab - 1, replay_ids=ids,
                         entries=[(u, p, r) for u, p, r in recs])
    host = grid.cpu().numpy()
    ref.replay_misses(reset=True)
    want, _ = ref.decode([host[i] for i in range(n)], spec, po.config(**kw), ids=ids)
    assert ref.replay_misses() == 0
    for g, r in zip(res, want):
        assert g.tokens == r.tokens and g.label_times == r.label_times, (g.id, g.tokens, r.tokens)
        assert g.steps_taken == r.steps and g.eos_trigger == r.eos_trigger
        assert abs(g.joint_logp - r.joint_logp) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("var,val", [("BL_FUSED_LOG_SOFTMAX", "1"), ("BL_NO_GRAPH", "1"),
                                     ("BL_LOG_SOFTMAX", "rows")])
def test_scorer_modes_vs_reference_replay(var, val):
    """The replay parity above in a fresh process (each switch is read once
    per process) for the alternative scorer-step paths: BL_FUSED_LOG_SOFTMAX
    (normaliser partials in the output GEMM's epilogue, attf rows
    materialised after it), BL_NO_GRAPH (the step's kernels launched
    directly instead of one CUDA graph per step), BL_LOG_SOFTMAX=rows (fp64
    att rows materialised by the warp normaliser and read by the search,
    instead of the staged normaliser's fp32 rows + fp64 log-normaliser)."""
    env = dict(os.environ, **{var: val})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider",
                        __file__ + "::test_transformer_search_vs_reference_replay"],
                       env=env, cwd=os.path.dirname(os.path.dirname(__file__)),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_transformer_large_vocab_tma_step_mode_vs_reference(ref):
    """Librispeech-size model (d=512, 8 heads, vocab 5000): the search runs its
    TMA-streamed slab path in step mode with per-hypothesis network rows."""
    import pyoracle as po
    grid, mem, w = _setup(enc.LARGE, tr.LARGE, 2, 300, seed=13)
    kw = dict(beam_width=4, margin_m1=5, margin_m2=10)
    dec, res, ids = _decode(grid, mem, tr.TransformerScorer(tr.LARGE, w), bl.DecoderConfig(**kw))
    recs = dec.records()
    spec = po.ScorerSpec("replay", tr.LARGE.vocab - 1, replay_ids=ids,
                         entries=[(u, p, r) for u, p, r in recs])
    host = grid.cpu().numpy()
    ref.replay_misses(reset=True)
    want, _ = ref.decode([host[i] for i in range(grid.shape[0])], spec, po.config(**kw), ids=ids)
    assert ref.replay_misses() == 0
    for g, r in zip(res, want):
        assert g.tokens == r.tokens and g.label_times == r.label_times
        assert g.steps_taken == r.steps and g.eos_trigger == r.eos_trigger
        assert abs(g.joint_logp - r.joint_logp) <= 1e-9


@pytest.mark.gpu
def test_transformer_scorer_needs_memory():
    torch = pytest.importorskip("torch")
    w = tr.random_weights(TINY_DEC, seed=1)
    sc = tr.TransformerScorer(TINY_DEC, w)
    dec = bl.Decoder(sc, bl.DecoderConfig(beam_width=2))
    g = torch.full((5, 64), -np.log(64.0), device="cuda")
    with pytest.raises(ValueError):
        dec.decode_raw([("x", 5, 64, g.data_ptr())], on_device=True)
    with pytest.raises(ValueError):
        tr.TransformerScorer(TINY_DEC, w[:-1])
