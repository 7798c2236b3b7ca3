"""Transformer attention decoder as a device scorer (SURVEY.md §8 a'2).

The reference's `Scorer` contract (`scorer.hpp:11-22`): a normalised
log-prob vector over C + {eos} (eos last) given the utterance and the token
prefix. The paper's scorer is the ESPnet Transformer decoder conditioned on
the utterance's encoder output. Here it runs on device for every live
hypothesis of every utterance at once, once per decode step, between
launches of the step-granular search kernel:

  embed(token) * sqrt(d) + PE(position)        (sos = eos = |C| at position 0)
  layers x [x + SelfAttn(LN1(x)) over the prefix (ancestor-indexed KV cache),
            x + SrcAttn(LN2(x), memory)       (memory K/V computed once),
            x + FFN(LN3(x))]
  LN, output linear, log_softmax (fp64 normaliser)  ->  att rows [U*B][|C|+1]

Weights are random-init (torch defaults: Embedding N(0,1), Linear fan-in
uniform, LayerNorm (1, 0)) in the flat order of ``include/bl_b200.h``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

from .api import Scorer, _check, lib


class _DSpec(C.Structure):
    _fields_ = [("d_model", C.c_int), ("heads", C.c_int), ("d_ff", C.c_int),
                ("layers", C.c_int), ("vocab", C.c_int)]


@dataclass(frozen=True)
class DecoderSpec:
    d_model: int = 256
    heads: int = 4
    d_ff: int = 2048
    layers: int = 3
    vocab: int = 500

    def c(self) -> _DSpec:
        return _DSpec(self.d_model, self.heads, self.d_ff, self.layers, self.vocab)

    def shapes(self) -> List[Tuple[str, Tuple[int, ...]]]:
        d, ff, V = self.d_model, self.d_ff, self.vocab
        out = [("embed.w", (V, d))]
        for i in range(self.layers):
            p = f"layers.{i}."
            for a in ("", "2"):   # self-attention, then source attention
                ln = "ln1" if a == "" else "ln2"
                out += [(p + ln + ".g", (d,)), (p + ln + ".b", (d,))]
                for m in ("q", "k", "v", "o"):
                    out += [(p + "w" + m + a, (d, d)), (p + "b" + m + a, (d,))]
            out += [(p + "ln3.g", (d,)), (p + "ln3.b", (d,)),
                    (p + "w1", (ff, d)), (p + "b1", (ff,)), (p + "w2", (d, ff)), (p + "b2", (d,))]
        out += [("after_norm.g", (d,)), ("after_norm.b", (d,)),
                ("out.w", (V, d)), ("out.b", (V,))]
        return out

    def num_weights(self) -> int:
        return int(sum(np.prod(s) for _, s in self.shapes()))


# BASELINE.json: cfg1/2 "6 enc/3 dec, d=256, 4 heads, vocab 500";
# cfg3/4 "12 enc/6 dec, d=512, 8 heads, vocab 5000"
SMALL = DecoderSpec(256, 4, 2048, 3, 500)
LARGE = DecoderSpec(512, 8, 2048, 6, 5000)


def random_weights(spec: DecoderSpec, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = spec.d_model
    parts = []
    for name, shape in spec.shapes():
        leaf = name.split(".")[-1]
        if name == "embed.w":
            parts.append(rng.standard_normal(shape).astype(np.float32))
            continue
        if "ln" in name or "norm" in name:
            parts.append((np.ones if leaf == "g" else np.zeros)(shape, np.float32))
            continue
        fi = spec.d_ff if leaf in ("w2", "b2") else d
        bound = 1.0 / np.sqrt(fi)
        parts.append(rng.uniform(-bound, bound, size=shape).astype(np.float32))
    w = np.concatenate([p.ravel() for p in parts])
    assert w.size == spec.num_weights()
    return w


def unflatten(spec: DecoderSpec, w: np.ndarray) -> Dict[str, np.ndarray]:
    out, o = {}, 0
    for name, shape in spec.shapes():
        n = int(np.prod(shape))
        out[name] = w[o:o + n].reshape(shape)
        o += n
    return out


class TransformerScorer(Scorer):
    """Device Transformer decoder behind the Scorer contract (`make_scorer`
    spec ``transformer``). Decoding with it needs each utterance's encoder
    output (``Decoder.decode_raw(..., memory=...)``)."""

    def __init__(self, spec: DecoderSpec, weights: np.ndarray, device: int = 0):
        w = np.ascontiguousarray(weights, dtype=np.float32)
        L = lib()
        if L.bl_transformer_num_weights(C.byref(spec.c())) != spec.num_weights():
            raise AssertionError("decoder weight layout disagrees with the library")
        h = C.c_void_p()
        _check(L.bl_scorer_create_transformer(device, C.byref(spec.c()), w.ctypes.data,
                                              w.size, C.byref(h)))
        self._h = h
        self._n = spec.vocab - 1
        self.spec = spec
        self.is_network = True

    def score(self, utterance_id, prefix):  # no host-side query for the network
        raise NotImplementedError("the Transformer scorer runs on device inside the decoder")
