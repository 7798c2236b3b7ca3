"""TEST INFRASTRUCTURE — torch-CPU fp32 reference of the Transformer
attention-decoder scorer (SURVEY.md §8 a'2).

Only tests/ and __graft_entry__.smoke() use this module, as the checker for
the device scorer (libbl_b200.so, `transformer` scorer). Parity is unpinned
by the reference (beamlattice has no network; its `Scorer::score(id, prefix)`
contract, scorer.hpp:11-22, is what the network implements). The model is the
ESPnet TransformerDecoder (eval mode):

  x = Embedding(ys) * sqrt(d) + PE,  ys = [sos] + prefix, sos = eos = |C|
  per layer: x += SelfAttn(LN1(x), causal); x += SrcAttn(LN2(x), memory);
             x += FFN(LN3(x))  (ReLU)
  log_softmax(out(LN(x)))[last position]

computed NON-incrementally over the whole prefix (the device path is
incremental with a KV cache; agreement checks the cache addressing).
``emulate_bf16`` rounds to bf16 where the device stores bf16.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


def _bf(x, on):
    return x.to(torch.bfloat16).to(torch.float32) if on else x


def pe_table(T: int, d: int) -> torch.Tensor:
    pos = torch.arange(T, dtype=torch.float32).unsqueeze(1)
    div = torch.exp(torch.arange(0, d, 2, dtype=torch.float32) * -(math.log(10000.0) / d))
    pe = torch.zeros(T, d)
    pe[:, 0::2] = torch.sin(pos * div)
    pe[:, 1::2] = torch.cos(pos * div)
    return pe


def decoder_scores(spec, weights: np.ndarray, memory: np.ndarray, prefixes,
                   emulate_bf16: bool = False) -> np.ndarray:
    """memory [T2, d] (one utterance); prefixes: list of token lists.
    Returns float64 [len(prefixes), vocab] log-probs of the next token."""
    from paper_2101_05600_b200.transformer import unflatten
    W = {k: torch.from_numpy(np.array(v, dtype=np.float32)) for k, v in
         unflatten(spec, weights).items()}
    e = emulate_bf16
    d, h = spec.d_model, spec.heads
    dk = d // h
    sos = spec.vocab - 1
    mem = torch.from_numpy(np.asarray(memory, dtype=np.float32))

    def lin(x, w, b):
        return _bf(x, e) @ _bf(w, e).T + b

    def heads(x):  # [t, d] -> [h, t, dk]
        return x.view(x.shape[0], h, dk).transpose(0, 1)

    out = []
    with torch.no_grad():
        for prefix in prefixes:
            ys = torch.tensor([sos] + list(prefix), dtype=torch.long)
            t = ys.shape[0]
            x = W["embed.w"][ys] * math.sqrt(d) + pe_table(t, d)
            causal = torch.triu(torch.ones(t, t, dtype=torch.bool), diagonal=1)
            for i in range(spec.layers):
                p = f"layers.{i}."
                y = _bf(F.layer_norm(x, (d,), W[p + "ln1.g"], W[p + "ln1.b"], eps=1e-12), e)
                q = heads(_bf(lin(y, W[p + "wq"], W[p + "bq"]), e))
                k = heads(_bf(lin(y, W[p + "wk"], W[p + "bk"]), e))
                v = heads(_bf(lin(y, W[p + "wv"], W[p + "bv"]), e))
                s = (q @ k.transpose(-2, -1)) / math.sqrt(dk)
                s = s.masked_fill(causal, float("-inf"))
                o = _bf((torch.softmax(s, -1) @ v).transpose(0, 1).reshape(t, d), e)
                x = x + lin(o, W[p + "wo"], W[p + "bo"])
                y = _bf(F.layer_norm(x, (d,), W[p + "ln2.g"], W[p + "ln2.b"], eps=1e-12), e)
                q = heads(_bf(lin(y, W[p + "wq2"], W[p + "bq2"]), e))
                k = heads(_bf(lin(mem, W[p + "wk2"], W[p + "bk2"]), e))
                v = heads(_bf(lin(mem, W[p + "wv2"], W[p + "bv2"]), e))
                s = (q @ k.transpose(-2, -1)) / math.sqrt(dk)
                o = _bf((torch.softmax(s, -1) @ v).transpose(0, 1).reshape(t, d), e)
                x = x + lin(o, W[p + "wo2"], W[p + "bo2"])
                y = _bf(F.layer_norm(x, (d,), W[p + "ln3.g"], W[p + "ln3.b"], eps=1e-12), e)
                hdn = _bf(torch.relu(lin(y, W[p + "w1"], W[p + "b1"])), e)
                x = x + lin(hdn, W[p + "w2"], W[p + "b2"])
            y = _bf(F.layer_norm(x[-1:], (d,), W["after_norm.g"], W["after_norm.b"],
                                 eps=1e-12), e)
            logits = lin(y, W["out.w"], W["out.b"])[0].double()
            out.append(torch.log_softmax(logits, -1).numpy())
    return np.stack(out)
