"""TEST INFRASTRUCTURE — torch-CPU fp32 reference of the CTC encoder forward.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this
module, as the checker for the device encoder (libbl_b200.so
``bl_encoder_forward``). It is never on the product path.

Parity is unpinned by the reference: beamlattice leaves the network out of
scope (SURVEY.md §8 a'1, "Network numerics (unpinned by the reference)") and
reads grids from files. The model restated here is the ESPnet Transformer
encoder the paper decodes with (eval mode, no dropout):

  Conv2dSubsampling  conv(1->d, 3x3/2) ReLU conv(d->d, 3x3/2) ReLU,
                     (b, c, t, f) -> (b, t, c*f), linear(d*F2 -> d),
                     x * sqrt(d) + sinusoidal PE
  layers x           x + MHA(LN1(x)), x + FFN(LN2(x))   (pre-LN, ReLU FFN)
  after_norm         LN (eps 1e-12)
  CTC head           log_softmax(linear(d -> vocab))

``emulate_bf16=True`` rounds the same tensors to bf16 that the device path
stores in bf16 (GEMM operands, conv outputs, LN outputs, Q/K/V, attention
output, FFN hidden) so the comparison isolates accumulation-order error.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


def _bf(x: torch.Tensor, on: bool) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32) if on else x


def pe_table(T: int, d: int) -> torch.Tensor:
    pos = torch.arange(T, dtype=torch.float32).unsqueeze(1)
    div = torch.exp(torch.arange(0, d, 2, dtype=torch.float32) * -(math.log(10000.0) / d))
    pe = torch.zeros(T, d)
    pe[:, 0::2] = torch.sin(pos * div)
    pe[:, 1::2] = torch.cos(pos * div)
    return pe


def encoder_forward(spec, weights: np.ndarray, fbank: np.ndarray,
                    emulate_bf16: bool = False) -> np.ndarray:
    """fbank [n, T, idim] -> log-posteriors [n, T2, vocab] (float32)."""
    from paper_2101_05600_b200.encoder import unflatten
    W = {k: torch.from_numpy(np.array(v, dtype=np.float32)) for k, v in
         unflatten(spec, weights).items()}
    e = emulate_bf16
    d, h = spec.d_model, spec.heads
    dk = d // h

    def lin(x, w, b):
        return _bf(x, e) @ _bf(w, e).T + b

    with torch.no_grad():
        x = torch.from_numpy(np.asarray(fbank, dtype=np.float32)).unsqueeze(1)  # b,1,t,f
        x = torch.relu(F.conv2d(x, W["conv1.w"], W["conv1.b"], stride=2))
        x = _bf(x, e)
        x = torch.relu(F.conv2d(x, _bf(W["conv2.w"], e), W["conv2.b"], stride=2))
        x = _bf(x, e)
        b, c, t, f = x.shape
        x = x.transpose(1, 2).contiguous().view(b, t, c * f)
        x = lin(x, W["out.w"], W["out.b"]) * math.sqrt(d) + pe_table(t, d)
        for i in range(spec.layers):
            p = f"layers.{i}."
            y = _bf(F.layer_norm(x, (d,), W[p + "ln1.g"], W[p + "ln1.b"], eps=1e-12), e)
            q = _bf(lin(y, W[p + "wq"], W[p + "bq"]), e).view(b, t, h, dk).transpose(1, 2)
            k = _bf(lin(y, W[p + "wk"], W[p + "bk"]), e).view(b, t, h, dk).transpose(1, 2)
            v = _bf(lin(y, W[p + "wv"], W[p + "bv"]), e).view(b, t, h, dk).transpose(1, 2)
            att = torch.softmax(q @ k.transpose(-2, -1) / math.sqrt(dk), dim=-1)
            o = _bf((att @ v).transpose(1, 2).reshape(b, t, d), e)
            x = x + lin(o, W[p + "wo"], W[p + "bo"])
            y = _bf(F.layer_norm(x, (d,), W[p + "ln2.g"], W[p + "ln2.b"], eps=1e-12), e)
            hdn = _bf(torch.relu(lin(y, W[p + "w1"], W[p + "b1"])), e)
            x = x + lin(hdn, W[p + "w2"], W[p + "b2"])
        y = _bf(F.layer_norm(x, (d,), W["after_norm.g"], W["after_norm.b"], eps=1e-12), e)
        logits = lin(y, W["ctc.w"], W["ctc.b"])
        return torch.log_softmax(logits, dim=-1).numpy()

