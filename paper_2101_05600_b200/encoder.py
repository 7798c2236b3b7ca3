"""CTC encoder forward on the B200 (SURVEY.md §8 a'1) — the producer of the
PosteriorGrid that the batched decoder consumes.

The reference reads grids from ``.ctcg`` files (``grid.cpp:108-127``) and
leaves the network out of scope; here the encoder writes the grid straight
into device memory, so ``Decoder.decode_raw(..., on_device=True)`` takes it
without a host round-trip. Model: ESPnet Transformer encoder (eval mode) —
Conv2dSubsampling, linear, x*sqrt(d) + PE, pre-LN self-attention/FFN layers,
final LayerNorm, CTC linear + log_softmax. The work runs in
``libbl_b200.so`` (``bl_encoder_*`` in ``include/bl_b200.h``): tcgen05 bf16
GEMMs with fp32 accumulation, fp32 LayerNorm/softmax.

Weights are random-init (there are no checkpoints offline): ``random_weights``
draws torch's default Linear/Conv init, U(-1/sqrt(fan_in), 1/sqrt(fan_in)),
LayerNorm gain 1 / bias 0, in the flat order of ``bl_b200.h``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

from . import api as _api
from .api import _check, lib


class _Spec(C.Structure):
    _fields_ = [("idim", C.c_int), ("d_model", C.c_int), ("heads", C.c_int),
                ("d_ff", C.c_int), ("layers", C.c_int), ("vocab", C.c_int)]


def frames_out(frames_in: int) -> int:
    """Encoder frames after two 3x3/2 convolutions (1000 -> 249)."""
    if frames_in < 7:
        return 0
    t1 = (frames_in - 3) // 2 + 1
    return (t1 - 3) // 2 + 1


@dataclass(frozen=True)
class EncoderSpec:
    idim: int = 80
    d_model: int = 256
    heads: int = 4
    d_ff: int = 2048
    layers: int = 6
    vocab: int = 500

    def c(self) -> _Spec:
        return _Spec(self.idim, self.d_model, self.heads, self.d_ff, self.layers, self.vocab)

    @property
    def f2(self) -> int:
        return frames_out(self.idim)

    def shapes(self) -> List[Tuple[str, Tuple[int, ...]]]:
        """(name, torch shape) in the flat weight order of bl_b200.h."""
        d, f2, ff, V = self.d_model, self.f2, self.d_ff, self.vocab
        out = [("conv1.w", (d, 1, 3, 3)), ("conv1.b", (d,)), ("conv2.w", (d, d, 3, 3)),
               ("conv2.b", (d,)), ("out.w", (d, d * f2)), ("out.b", (d,))]
        for i in range(self.layers):
            p = f"layers.{i}."
            out += [(p + "ln1.g", (d,)), (p + "ln1.b", (d,)),
                    (p + "wq", (d, d)), (p + "bq", (d,)), (p + "wk", (d, d)), (p + "bk", (d,)),
                    (p + "wv", (d, d)), (p + "bv", (d,)), (p + "wo", (d, d)), (p + "bo", (d,)),
                    (p + "ln2.g", (d,)), (p + "ln2.b", (d,)),
                    (p + "w1", (ff, d)), (p + "b1", (ff,)), (p + "w2", (d, ff)), (p + "b2", (d,))]
        out += [("after_norm.g", (d,)), ("after_norm.b", (d,)),
                ("ctc.w", (V, d)), ("ctc.b", (V,))]
        return out

    def num_weights(self) -> int:
        return int(sum(np.prod(s) for _, s in self.shapes()))


# BASELINE.json configs: cfg1/2 small (6 enc, d=256, 4 heads, vocab 500),
# cfg3/4 Librispeech-size (12 enc, d=512, 8 heads, vocab 5000); d_ff 2048.
SMALL = EncoderSpec(80, 256, 4, 2048, 6, 500)
LARGE = EncoderSpec(80, 512, 8, 2048, 12, 5000)


def random_weights(spec: EncoderSpec, seed: int = 0) -> np.ndarray:
    """Flat fp32 weights, torch default init (fan-in uniform), LN = (1, 0)."""
    rng = np.random.default_rng(seed)
    d = spec.d_model
    fan_in = {"conv1": 9, "conv2": 9 * d, "out": d * spec.f2, "ctc": d,
              "w2": spec.d_ff, "b2": spec.d_ff}
    parts = []
    for name, shape in spec.shapes():
        leaf = name.split(".")[-1]
        is_norm = "ln" in name or "norm" in name
        if is_norm:
            parts.append((np.ones if leaf == "g" else np.zeros)(shape, np.float32))
            continue
        fi = fan_in.get(name.split(".")[0], fan_in.get(leaf, d))
        bound = 1.0 / np.sqrt(fi)
        parts.append(rng.uniform(-bound, bound, size=shape).astype(np.float32))
    w = np.concatenate([p.ravel() for p in parts])
    assert w.size == spec.num_weights()
    return w


def unflatten(spec: EncoderSpec, w: np.ndarray) -> Dict[str, np.ndarray]:
    out, o = {}, 0
    for name, shape in spec.shapes():
        n = int(np.prod(shape))
        out[name] = w[o:o + n].reshape(shape)
        o += n
    return out


class Encoder:
    """Device encoder; ``forward`` writes log-posterior grids to device memory."""

    def __init__(self, spec: EncoderSpec, weights: np.ndarray, device: int = 0,
                 chunk: int = 148):
        self.spec = spec
        w = np.ascontiguousarray(weights, dtype=np.float32)
        L = lib()
        if L.bl_encoder_num_weights(C.byref(spec.c())) != spec.num_weights():
            raise AssertionError("encoder weight layout disagrees with the library")
        h = C.c_void_p()
        _check(L.bl_encoder_create(device, C.byref(spec.c()), w.ctypes.data, w.size,
                                   C.byref(h)))
        self._h = h
        _check(L.bl_encoder_set_chunk(h, chunk))

    def close(self) -> None:
        L = getattr(_api, "_lib", None) if _api is not None else None
        if getattr(self, "_h", None) and L is not None:
            L.bl_encoder_destroy(self._h)
        self._h = None

    __del__ = close

    def set_stream(self, stream_ptr: int) -> None:
        _check(lib().bl_encoder_set_stream(self._h, C.c_void_p(stream_ptr)))

    @property
    def launches(self) -> int:
        return lib().bl_encoder_launches(self._h)

    def forward_raw(self, n: int, frames_in: int, fbank_ptr: int, on_device: bool,
                    grid_ptr: int, sync: bool = True) -> None:
        """fbank [n][frames_in][idim] fp32 at fbank_ptr (host or device);
        grid [n][frames_out][vocab] fp32 device buffer at grid_ptr."""
        _check(lib().bl_encoder_forward(self._h, n, frames_in, C.c_void_p(fbank_ptr),
                                        1 if on_device else 0, C.c_void_p(grid_ptr),
                                        1 if sync else 0))

    def forward(self, fbank, memory: bool = False):
        """torch: fbank [n, frames, idim] float32 (CPU or CUDA) -> CUDA grid
        [n, frames_out, vocab] float32 (and, with memory=True, the encoder
        output bf16 [n, frames_out, d_model] for the attention decoder)."""
        import torch
        n, T, idim = fbank.shape
        if idim != self.spec.idim:
            raise ValueError(f"fbank has {idim} features, encoder expects {self.spec.idim}")
        fb = fbank.contiguous().float()
        T2 = frames_out(T)
        grid = torch.empty((n, T2, self.spec.vocab), dtype=torch.float32, device="cuda")
        self.set_stream(torch.cuda.current_stream().cuda_stream)
        if not memory:
            self.forward_raw(n, T, fb.data_ptr(), fb.is_cuda, grid.data_ptr(), sync=True)
            return grid
        mem = torch.empty((n, T2, self.spec.d_model), dtype=torch.bfloat16, device="cuda")
        _check(lib().bl_encoder_forward_mem(self._h, n, T, C.c_void_p(fb.data_ptr()),
                                            1 if fb.is_cuda else 0,
                                            C.c_void_p(grid.data_ptr()),
                                            C.c_void_p(mem.data_ptr()), 1))
        return grid, mem


def gemm_bf16(A, B, mode: int = 0, bias=None, out=None, out_bf16=None, scale: float = 1.0,
              pe=None):
    """Test/bench face of the tcgen05 GEMM: A [M,K], B [N,K] bf16 CUDA tensors.
    Returns fp32 [M,N] (or writes ``out``/``out_bf16``)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    if out is None and out_bf16 is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    ldo = (out if out is not None else out_bf16).stride(0)
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    _check(lib().bl_gemm_bf16(M, N, K, ptr(A), A.stride(0), ptr(B), B.stride(0), mode,
                              ptr(bias), ptr(out), ptr(out_bf16), ldo, scale, ptr(pe),
                              pe.shape[0] if pe is not None else 0,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out if out is not None else out_bf16


def synthetic_fbank(n: int, frames: int, idim: int = 80, seed: int = 0) -> np.ndarray:
    """Synthetic log-mel-like features [n, frames, idim]: per-segment spectral
    envelope, a slow spectro-temporal modulation and white noise."""
    rng = np.random.default_rng(seed)
    t = np.arange(frames)[None, :, None]
    f = np.arange(idim)[None, None, :]
    base = rng.normal(0, 1, (n, 1, idim)).astype(np.float32)
    mod = np.sin(2 * np.pi * (t / rng.uniform(20, 80, (n, 1, 1)) + f / idim))
    return (base + 0.8 * mod + 0.3 * rng.normal(0, 1, (n, frames, idim))).astype(np.float32)
