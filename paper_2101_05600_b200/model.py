"""Model files and the native long-recording chain.

* ``save_model`` / ``load_encoder``: the BLM1 weight file (bl_model_save,
  include/bl_b200.h) holding the encoder and/or the Transformer decoder; the
  decoder is loaded through the reference's model-load hook,
  ``make_scorer("transformer:PATH")`` (scorer.hpp:84, scorer.cpp:117-135).
* ``recognize_native``: ``bl_recognize`` -- fbank of one long recording ->
  hard_segments -> encoder -> batched decode, the whole chain in the C ABI
  (the Python chain is recognize.recognize).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from .api import Decoder, DecodeCounters, _check, lib
from .encoder import Encoder, EncoderSpec
from .transformer import DecoderSpec


def save_model(path: str, enc_spec: Optional[EncoderSpec] = None,
               enc_weights: Optional[np.ndarray] = None,
               dec_spec: Optional[DecoderSpec] = None,
               dec_weights: Optional[np.ndarray] = None) -> None:
    ew = np.ascontiguousarray(enc_weights, np.float32) if enc_spec is not None else None
    dw = np.ascontiguousarray(dec_weights, np.float32) if dec_spec is not None else None
    _check(lib().bl_model_save(
        path.encode(), C.byref(enc_spec.c()) if enc_spec is not None else None,
        ew.ctypes.data if ew is not None else None, ew.size if ew is not None else 0,
        C.byref(dec_spec.c()) if dec_spec is not None else None,
        dw.ctypes.data if dw is not None else None, dw.size if dw is not None else 0))


class _FileEncoder(Encoder):
    """An Encoder whose weights come from a model file."""

    def __init__(self, path: str, device: int = 0, chunk: int = 148):
        h = C.c_void_p()
        _check(lib().bl_encoder_create_from_file(device, path.encode(), C.byref(h)))
        self._h = h
        self.spec = None
        _check(lib().bl_encoder_set_chunk(h, chunk))


def load_encoder(path: str, device: int = 0, chunk: int = 148) -> Encoder:
    return _FileEncoder(path, device, chunk)


def recognize_native(fbank: np.ndarray, encoder: Encoder, decoder: Decoder,
                     recording_id: str = "rec", min_len: int = 1000, max_len: int = 1000,
                     counters: Optional[DecodeCounters] = None) -> List:
    """bl_recognize: results in segment order, ids "<rec>:<start>-<end>"."""
    fb = np.ascontiguousarray(fbank, dtype=np.float32)
    h = C.c_void_p()
    _check(lib().bl_recognize(encoder._h, decoder._h, fb.ctypes.data, fb.shape[0], fb.shape[1],
                              recording_id.encode(), min_len, max_len, C.byref(h)))
    try:
        n = lib().bl_results_count(h)
        ids = []
        cid = C.c_char_p()
        ip = C.POINTER(C.c_int)
        t_, l_ = ip(), ip()
        nt, st, tr = C.c_int(), C.c_int(), C.c_int()
        jt = C.c_double()
        for i in range(n):
            _check(lib().bl_results_get(h, i, C.byref(cid), C.byref(t_), C.byref(nt),
                                        C.byref(jt), C.byref(l_), C.byref(st), C.byref(tr)))
            ids.append(cid.value.decode())
        return decoder._collect(h, counters, ids)
    finally:
        lib().bl_results_destroy(h)
