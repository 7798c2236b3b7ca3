"""bl_decode_into's two export paths (capi.cu, `direct`): page-locked output
arrays receive the token / label-time rows by 2D device-to-host copies, plain
(pageable) arrays by the host repacking loop. Both must give the same
results as each other and as the per-utterance result objects (bl_decode)."""
import ctypes as C

import numpy as np
import pytest

import paper_2101_05600_b200 as bl
from paper_2101_05600_b200.api import _check, lib

pytestmark = pytest.mark.gpu


def test_bulk_export_pageable_equals_pinned_and_objects():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    n, T, V = 300, 40, 30
    lens = [T - (i % 7) for i in range(n)]
    g = rng.standard_normal((n, T, V)).astype(np.float32) * 2.0
    g -= np.log(np.exp(g).sum(2, keepdims=True))
    dev = torch.from_numpy(g).cuda()
    dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=4, margin_m2=8))
    descs = [(f"u{i}", lens[i], V, dev[i].data_ptr()) for i in range(n)]
    torch.cuda.synchronize()
    pinned = list(dec.decode_raw(descs, on_device=True))  # pooled page-locked block
    rec = dec._desc_cache[2][0]
    cap = T
    nt, st, tr = (np.zeros(n, np.int32) for _ in range(3))
    jt = np.zeros(n, np.float64)
    tok, lt = np.full((n, cap), -7, np.int32), np.full((n, cap), -7, np.int32)
    h = C.c_void_p()
    _check(lib().bl_decode_into(dec._h, n, rec.ctypes.data_as(C.POINTER(bl.api._Utt)), 1, None,
                                0, cap, nt.ctypes.data, st.ctypes.data, tr.ctypes.data,
                                jt.ctypes.data, tok.ctypes.data, lt.ctypes.data, C.byref(h)))
    lib().bl_results_destroy(h)
    objs = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=4, margin_m2=8),
                      nbest=2).decode([bl.Utterance(f"u{i}", bl.PosteriorGrid(g[i, :lens[i]]))
                                       for i in range(n)])
    for i, (p, o) in enumerate(zip(pinned, objs)):
        k = int(nt[i])
        assert p.tokens == o.tokens == tok[i, :k].tolist()
        assert p.label_times == o.label_times == lt[i, :k].tolist()
        assert p.steps_taken == o.steps_taken == int(st[i])
        assert p.joint_logp == o.joint_logp == float(jt[i])
