"""BLM1 model files (bl_model_save, include/bl_b200.h) on CPU: the byte
layout, and the loader's error paths through make_scorer("transformer:PATH")
(scorer.cpp:117-135 semantics: unreadable file / bad magic -> runtime_error)."""
import struct

import numpy as np
import pytest

import paper_2101_05600_b200 as bl
from paper_2101_05600_b200 import encoder as enc
from paper_2101_05600_b200 import model as bm
from paper_2101_05600_b200 import transformer as tr

ESPEC = enc.EncoderSpec(80, 128, 2, 256, 2, 64)
DSPEC = tr.DecoderSpec(128, 2, 256, 2, 64)


def test_model_file_layout(tmp_path):
    ew, dw = enc.random_weights(ESPEC, seed=1), tr.random_weights(DSPEC, seed=2)
    p = tmp_path / "m.blm"
    bm.save_model(str(p), ESPEC, ew, DSPEC, dw)
    b = p.read_bytes()
    assert b[:4] == b"BLM1" and struct.unpack("<II", b[4:12]) == (1, 2)
    o = 12
    kind, *spec = struct.unpack("<7I", b[o:o + 28])
    (cnt,) = struct.unpack("<Q", b[o + 28:o + 36])
    assert kind == 1 and spec == [80, 128, 2, 256, 2, 64] and cnt == ew.size
    np.testing.assert_array_equal(np.frombuffer(b[o + 36:o + 36 + 4 * cnt], "<f4"), ew)
    o += 36 + 4 * cnt
    kind, *spec = struct.unpack("<7I", b[o:o + 28])
    (cnt,) = struct.unpack("<Q", b[o + 28:o + 36])
    assert kind == 2 and spec == [128, 2, 256, 2, 64, 0] and cnt == dw.size
    np.testing.assert_array_equal(np.frombuffer(b[o + 36:], "<f4"), dw)


def test_model_file_errors(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open model file"):
        bl.make_scorer("transformer:" + str(tmp_path / "missing.blm"), 63)
    bad = tmp_path / "bad.blm"
    bad.write_bytes(b"XXXX" + b"\0" * 12)
    with pytest.raises(RuntimeError, match="bad magic"):
        bl.make_scorer("transformer:" + str(bad), 63)
    enc_only = tmp_path / "e.blm"
    bm.save_model(str(enc_only), ESPEC, enc.random_weights(ESPEC, seed=1))
    with pytest.raises(RuntimeError, match="no decoder section"):
        bl.make_scorer("transformer:" + str(enc_only), 63)
    with pytest.raises(bl.InvalidArgument, match="weight count"):
        bm.save_model(str(tmp_path / "x.blm"), ESPEC, np.zeros(5, np.float32))
