"""Host-side pieces of the product path through the C ABI (no GPU needed):
segmentation, batching, config validation, scorer loading, file formats.
Mirrors test_segmentation.cpp, test_batched.cpp, test_beam_search.cpp,
test_scorer.cpp and test_grid.cpp of the reference."""
import io
import json
import os
import math
import random

import numpy as np
import pytest

import paper_2101_05600_b200 as bl


def test_hard_segments_fixtures():
    """test_segmentation.cpp:100-121."""
    segs = bl.hard_segments(4000, 1900, 2000, "u")
    assert [(s.start, s.end) for s in segs] == [(0, 2000), (2000, 4000)]
    assert segs[0].source == "hard" and segs[0].utterance_id == "u"
    assert all(s.end - s.start == 1625 for s in bl.hard_segments(6500, 1900, 2000))
    assert [(s.start, s.end) for s in bl.hard_segments(700, 1900, 2000)] == [(0, 700)]


def test_hard_segments_match_golden(golden):
    exp, _ = golden
    for key, want in exp["hard_segments"].items():
        T, lo, hi = map(int, key.split(","))
        assert [[s.start, s.end] for s in bl.hard_segments(T, lo, hi)] == want


def test_hard_segments_properties():
    """test_segmentation.cpp:123-139 / acceptance criterion 9 (hard part)."""
    rng = random.Random(61)
    for _ in range(200):
        t = rng.randint(1, 9000)
        segs = bl.hard_segments(t, 1500, 2000, "u")
        assert segs[0].start == 0 and segs[-1].end == t
        assert all(a.end == b.start for a, b in zip(segs, segs[1:]))
        lens = [s.end - s.start for s in segs]
        if t >= 1500:
            assert max(lens) <= 2000
        assert max(lens) - min(lens) <= 1


def test_hard_segments_errors():
    with pytest.raises(bl.InvalidArgument, match="T < 1"):
        bl.hard_segments(0, 1, 2)
    with pytest.raises(bl.InvalidArgument, match="min_len"):
        bl.hard_segments(10, 5, 4)


def _utts(lens):
    return [bl.Utterance(f"u{i}", bl.PosteriorGrid(np.zeros((t, 2), np.float32)))
            for i, t in enumerate(lens)]


def test_make_batches():
    """test_batched.cpp:35-54."""
    batches = bl.make_batches(_utts([100, 50, 200, 60]), 2)
    assert len(batches) == 2
    assert [u.true_frames for u in batches[0].utterances] == [50, 60]
    assert batches[0].padded_frames == 60
    assert [u.true_frames for u in batches[1].utterances] == [100, 200]
    assert batches[1].padded_frames == 200
    assert len(bl.make_batches(_utts([100, 50, 200, 60]), 16)) == 1
    assert bl.make_batches([], 4) == []
    with pytest.raises(bl.InvalidArgument):
        bl.make_batches(_utts([1]), 0)


def test_make_batches_stable():
    b = bl.make_batches(_utts([5, 3, 5, 3, 5]), 5)[0]
    assert [u.id for u in b.utterances] == ["u1", "u3", "u0", "u2", "u4"]


def test_config_validation_messages():
    """beam_search.cpp:36-46 / test_beam_search.cpp:193-204."""
    bl.DecoderConfig().validate()
    for kw, msg in [({"beam_width": 0}, "beam width"), ({"ctc_weight": 1.5}, "ctc weight"),
                    ({"eos_m": 0}, "eos M"), ({"eos_c": -1}, "eos C"),
                    ({"margin_m1": -1}, "margins"), ({"max_steps_ratio": 0.0}, "max steps")]:
        with pytest.raises(bl.InvalidArgument, match=msg):
            bl.DecoderConfig(**kw).validate()
    with pytest.raises(bl.InvalidArgument):
        bl.eos_mode_from_string("bogus")
    for m in ("baseline", "ctc", "both"):
        assert bl.eos_mode_from_string(m) == m


def test_scorers_host_side():
    """scorer.cpp:30-80 vectors (computed host-side, uploaded as-is)."""
    u = bl.UniformScorer(3)
    assert u.score("x", [1, 2]) == [-math.log(4.0)] * 4
    lp = bl.LoopScorer(2, 0, 0.9).score("x", [])
    assert lp[0] == math.log(0.9) and lp[1] == lp[2] == math.log((1.0 - 0.9) / 2)
    t = bl.TableScorer(2, 2)
    row = [math.log(0.5), math.log(0.25), math.log(0.25)]
    t.add_entry([1], row)
    assert t.score("x", [0, 1]) == row
    assert t.score("x", [1, 0]) == [-math.log(3.0)] * 3


def test_scorer_errors():
    """test_scorer.cpp: normalisation, ranges, spec parsing."""
    with pytest.raises(RuntimeError, match="not normalized"):
        bl.TableScorer(2, 2).add_entry([], [0.0, 0.0, 0.0])
    with pytest.raises(RuntimeError, match="wrong vector size"):
        bl.TableScorer(2, 2).add_entry([], [0.0])
    with pytest.raises(bl.InvalidArgument, match="loop token"):
        bl.LoopScorer(2, 5, 0.9)
    with pytest.raises(bl.InvalidArgument, match="p_loop"):
        bl.LoopScorer(2, 0, 0.3)
    with pytest.raises(RuntimeError, match="unknown scorer spec"):
        bl.make_scorer("bogus", 3)
    with pytest.raises(RuntimeError, match="loop:TOKEN:P"):
        bl.make_scorer("loop:3", 3)
    assert bl.make_scorer("loop:1:0.8", 3).score("x", [])[1] == math.log(0.8)
    with pytest.raises(RuntimeError, match="cannot open scorer file"):
        bl.make_scorer("table:/nonexistent.json", 3)


def test_table_scorer_file_roundtrip(tmp_path):
    t = bl.TableScorer(2, 2)
    row = [math.log(0.5), math.log(0.25), math.log(0.25)]
    t.add_entry([0], row)
    path = str(tmp_path / "t.json")
    bl.save_table_scorer(path, t)
    s = bl.make_scorer("table:" + path, 2)
    assert s.score("x", [1, 0]) == row
    with pytest.raises(RuntimeError, match="does not match grids"):
        bl.make_scorer("table:" + path, 3)


def test_grid_roundtrip(tmp_path):
    """CTCG v1 round trip is bit-identical (test_grid.cpp)."""
    g = bl.PosteriorGrid(np.random.default_rng(0).standard_normal((7, 5)).astype(np.float32), 40)
    path = str(tmp_path / "a.ctcg")
    bl.write_grid(path, g)
    h = bl.read_grid(path)
    assert h.frame_shift_ms == 40 and np.array_equal(h.logp, g.logp)
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(RuntimeError, match="bad magic"):
        bl.read_grid(path)


def test_results_jsonl_schema():
    """io.cpp:81-92: keys in nlohmann order, round-trip exact doubles."""
    r = bl.DecodeResult("a", [1, 2], -3.141592653589793, [4, 9], 12, "ctc")
    buf = io.StringIO()
    bl.write_results(buf, [r])
    line = buf.getvalue().strip()
    assert list(json.loads(line).keys()) == ["eos_trigger", "id", "joint_logp",
                                             "label_times", "steps", "tokens"]
    assert json.loads(line)["joint_logp"] == r.joint_logp


def test_decoder_needs_gpu_or_fails_loudly():
    """No CPU fallback: without a usable GPU the decoder raises CudaError."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bl.CudaError):
        bl.Decoder(bl.UniformScorer(3))


# ------------------------------------------------------------ VAD segmentation
def _vad_outputs(seed, T, nodes=4):
    rng = np.random.default_rng(seed)
    # slowly varying speech/noise evidence with bursts, some exact ties
    base = np.cumsum(rng.normal(0, 0.6, T))
    out = rng.normal(0, 0.3, (T, nodes)).astype(np.float32)
    out[:, 0] += base.astype(np.float32)
    out[:, 2] -= base.astype(np.float32)
    out[::17, 1] = out[::17, 3]
    return out


@pytest.mark.parametrize("seed", range(6))
def test_vad_segments_match_reference(ref, seed):
    """bl_vad_segments == reference frame_llr/smooth_and_decide/vad_segments."""
    import paper_2101_05600_b200 as bl
    rng = np.random.default_rng(100 + seed)
    T = int(rng.integers(50, 4000))
    outs = _vad_outputs(seed, T)
    for thr, win, mn, mx in ((0.0, 5, 150, 200), (0.5, 1, 1, 7), (-0.3, 12, 40, 40),
                             (0.0, 3, 1000, 2000)):
        want = ref.vad_segments(outs, [0, 1], [2, 3], thr, win, mn, mx)
        got = bl.vad_segments(outs, [0, 1], [2, 3], thr, win, mn, mx, "x")
        assert [(g.start, g.end) for g in got] == want
        assert all(g.source == "vad" for g in got)


def test_vad_segments_errors():
    import paper_2101_05600_b200 as bl
    o = np.zeros((10, 3), np.float32)
    with pytest.raises(ValueError):
        bl.vad_segments(o, [0], [0])           # overlapping node sets
    with pytest.raises(ValueError):
        bl.vad_segments(o, [0], [5])           # node out of range
    with pytest.raises(ValueError):
        bl.vad_segments(o, [0], [1], smooth_window=0)
    with pytest.raises(ValueError):
        bl.vad_segments(o, [0], [1], min_len=5, max_len=4)
    assert bl.vad_segments(np.zeros((0, 3), np.float32), [0], [1]) == []


def test_cpp_header_vad_matches_reference(ref, tmp_path):
    """The drop-in header's VAD functions (host C++) equal the reference."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "vad"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "vad_check.cpp"), "-o", str(exe)],
                   check=True)
    for seed in range(3):
        outs = _vad_outputs(seed, 1500 + 300 * seed).astype(np.float64)
        path = tmp_path / f"v{seed}.txt"
        with open(path, "w") as fh:
            fh.write(f"{outs.shape[0]} {outs.shape[1]}\n")
            for row in outs:
                fh.write(" ".join(repr(float(np.float32(x))) for x in row) + "\n")
        for thr, win, mn, mx in ((0.0, 5, 150, 200), (0.5, 1, 1, 7), (-0.3, 12, 40, 40)):
            got = subprocess.run([str(exe), str(path), repr(thr), str(win), str(mn), str(mx), "r"],
                                 capture_output=True, text=True, check=True).stdout.split()
            got = [(int(got[i]), int(got[i + 1])) for i in range(0, len(got), 2)]
            want = ref.vad_segments(outs.astype(np.float32), [0, 1], [2, 3], thr, win, mn, mx)
            assert got == want
