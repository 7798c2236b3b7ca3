"""Long-recording chaining (segment -> slice -> encode -> batched decode),
SURVEY.md §8 f.3: every segment's result equals the CPU oracle decoding the
grid the device encoder produced for that segment alone (uniform scorer), and
with the Transformer scorer equals decoding each segment on its own."""
import numpy as np
import pytest

import paper_2101_05600_b200 as bl
from paper_2101_05600_b200 import encoder as enc
from paper_2101_05600_b200 import transformer as tr
from paper_2101_05600_b200.recognize import recognize

pytestmark = pytest.mark.gpu
ESPEC = enc.EncoderSpec(80, 128, 2, 256, 2, 64)
DSPEC = tr.DecoderSpec(128, 2, 256, 2, 64)


def _recording(T, seed=3):
    return enc.synthetic_fbank(1, T, 80, seed=seed)[0]


def test_recognize_hard_segments_vs_oracle(oracle):
    import pyoracle as po
    torch = pytest.importorskip("torch")
    fb = _recording(5200)
    e = enc.Encoder(ESPEC, enc.random_weights(ESPEC, seed=4))
    kw = dict(beam_width=5, margin_m2=15)
    dec = bl.Decoder(bl.UniformScorer(63), bl.DecoderConfig(**kw))
    out = recognize(fb, e, dec, "talk")
    segs = bl.hard_segments(5200, 1000, 1000, "talk")
    assert [s for s, _ in out] == segs and len({s.end - s.start for s in segs}) == 2
    for s, r in out:
        assert r.id == f"talk:{s.start}-{s.end}"
        g = e.forward(torch.from_numpy(fb[s.start:s.end][None].copy())).cpu().numpy()[0]
        want, _ = po.Oracle().decode([g], po.ScorerSpec("uniform", 63), po.config(**kw),
                                     ids=[r.id])
        assert r.tokens == want[0].tokens and r.steps_taken == want[0].steps
        assert abs(r.joint_logp - want[0].joint_logp) <= 1e-9


def test_recognize_transformer_scorer_equals_per_segment():
    torch = pytest.importorskip("torch")
    fb = _recording(3100, seed=5)
    e = enc.Encoder(ESPEC, enc.random_weights(ESPEC, seed=6))
    sc = tr.TransformerScorer(DSPEC, tr.random_weights(DSPEC, seed=7))
    kw = dict(beam_width=4, margin_m2=15)
    out = recognize(fb, e, bl.Decoder(sc, bl.DecoderConfig(**kw)), "m", 600, 800)
    assert len(out) == 4
    for s, r in out:
        g, mem = e.forward(torch.from_numpy(fb[s.start:s.end][None].copy()), memory=True)
        one = bl.Decoder(sc, bl.DecoderConfig(**kw)).decode_raw(
            [(r.id, g.shape[1], g.shape[2], g.data_ptr())], on_device=True,
            memory=mem.data_ptr(), mem_frames=g.shape[1])[0]
        assert one.tokens == r.tokens and one.steps_taken == r.steps_taken
        assert abs(one.joint_logp - r.joint_logp) <= 1e-9


def test_recognize_vad_segments():
    rng = np.random.default_rng(1)
    T = 2600
    vad = rng.normal(0, 1, (T, 2)).astype(np.float32)
    vad[300:1400, 0] += 4.0      # speech evidence on node 0
    vad[1700:2500, 0] += 4.0
    segs = bl.vad_segments(vad, [0], [1], 0.0, 9, 200, 700, "v")
    assert len(segs) >= 2 and all(s.source == "vad" for s in segs)
    e = enc.Encoder(ESPEC, enc.random_weights(ESPEC, seed=8))
    dec = bl.Decoder(bl.UniformScorer(63), bl.DecoderConfig(beam_width=3))
    out = recognize(_recording(T), e, dec, segments=segs)
    assert [s for s, _ in out] == segs
    assert all(r.steps_taken >= 1 for _, r in out)


def test_model_file_and_native_chain(tmp_path):
    """BLM1 model file (bl_model_save): the encoder loaded from it and the
    decoder loaded through the reference's model-load hook
    (make_scorer("transformer:PATH"), scorer.hpp:84) decode a long recording
    through the native chain (bl_recognize) exactly like the in-memory
    weights through the Python chain (recognize.py)."""
    from paper_2101_05600_b200 import model as bm
    ew, dw = enc.random_weights(ESPEC, seed=11), tr.random_weights(DSPEC, seed=12)
    path = str(tmp_path / "m.blm")
    bm.save_model(path, ESPEC, ew, DSPEC, dw)
    fb = _recording(3100, seed=13)
    kw = dict(beam_width=4, margin_m2=15)
    want = recognize(fb, enc.Encoder(ESPEC, ew),
                     bl.Decoder(tr.TransformerScorer(DSPEC, dw), bl.DecoderConfig(**kw)),
                     "m", 600, 800)
    e2 = bm.load_encoder(path)
    sc2 = bl.make_scorer("transformer:" + path, DSPEC.vocab - 1)
    got = bm.recognize_native(fb, e2, bl.Decoder(sc2, bl.DecoderConfig(**kw)), "m", 600, 800)
    assert [r.id for r in got] == [r.id for _, r in want]
    for g, (_, w) in zip(got, want):
        assert g.tokens == w.tokens and g.label_times == w.label_times
        assert g.steps_taken == w.steps_taken and abs(g.joint_logp - w.joint_logp) <= 1e-9
    with pytest.raises(RuntimeError, match="vocabulary"):
        bl.make_scorer("transformer:" + path, 99)


def test_native_chain_uniform_equals_python_chain():
    fb = _recording(5200, seed=14)
    e = enc.Encoder(ESPEC, enc.random_weights(ESPEC, seed=15))
    kw = dict(beam_width=5, margin_m2=15)
    from paper_2101_05600_b200 import model as bm
    want = recognize(fb, e, bl.Decoder(bl.UniformScorer(63), bl.DecoderConfig(**kw)), "t")
    got = bm.recognize_native(fb, e, bl.Decoder(bl.UniformScorer(63), bl.DecoderConfig(**kw)),
                              "t")
    assert [(r.id, r.tokens, r.joint_logp) for r in got] == \
        [(r.id, r.tokens, r.joint_logp) for _, r in want]
