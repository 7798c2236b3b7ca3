"""CTC encoder (SURVEY.md §8 a'1): the tcgen05 GEMM and the device encoder
against torch-CPU fp32 (oracle/torch_encoder.py), and the encoder -> decoder
chain against the CPU decoder oracle on the grid the device produced.

Tolerances (network numerics are unpinned by the reference):
  * GEMM, bf16 operands: |dev - torch_fp32(bf16 operands)| <= 1e-3 * (1 + |ref|)
    (fp32 accumulation, order differs only).
  * encoder vs torch with the same bf16 rounding points: max |dlogp| <= 0.05,
    mean <= 2e-3 (a bf16 rounding flip upstream propagates).
  * encoder vs pure fp32 torch: max |dlogp| <= 0.25 (bf16 storage error).
  * decode of the device grid: identical to the CPU oracle decoding the same
    grid (tokens/label_times/steps/trigger identical, joint within 1e-9).
"""
import ctypes as C

import numpy as np
import pytest

from paper_2101_05600_b200 import encoder as enc
from paper_2101_05600_b200.api import lib

TINY = enc.EncoderSpec(80, 128, 2, 256, 2, 64)


def test_weight_count_matches_library():
    for spec in (enc.SMALL, enc.LARGE, TINY):
        assert lib().bl_encoder_num_weights(C.byref(spec.c())) == spec.num_weights()


def test_frames_out_matches_library():
    for t in (0, 6, 7, 8, 100, 500, 999, 1000, 2000):
        assert lib().bl_encoder_frames_out(t) == enc.frames_out(t)
    assert enc.frames_out(1000) == 249 and enc.frames_out(500) == 124
    assert enc.frames_out(2000) == 499


def test_invalid_spec_rejected_without_gpu():
    bad = enc.EncoderSpec(80, 200, 4, 2048, 6, 500)   # d not a multiple of 64
    assert lib().bl_encoder_num_weights(C.byref(bad.c())) == 0


def test_torch_reference_is_normalised():
    from torch_encoder import encoder_forward
    fb = enc.synthetic_fbank(1, 120, seed=3)
    w = enc.random_weights(TINY, seed=1)
    out = encoder_forward(TINY, w, fb)
    assert out.shape == (1, enc.frames_out(120), TINY.vocab)
    np.testing.assert_allclose(np.exp(out).sum(-1), 1.0, atol=1e-5)
    emu = encoder_forward(TINY, w, fb, emulate_bf16=True)
    assert np.abs(emu - out).max() < 0.25


# ---------------------------------------------------------------- GPU tests
def _torch():
    return pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 500, 264), (4731, 256, 2304),
                                   (1000, 768, 256), (77, 2048, 512), (249, 5000, 512),
                                   (513, 136, 4864)])
def test_gemm_plain_vs_torch(M, N, K):
    torch = _torch()
    g = torch.Generator().manual_seed(M * 7 + N)
    A = torch.randn(M, K, generator=g).bfloat16()
    B = torch.randn(N, K, generator=g).bfloat16()
    bias = torch.randn(N, generator=g)
    want = A.float() @ B.float().T + bias
    got = enc.gemm_bf16(A.cuda(), B.cuda(), bias=bias.cuda()).cpu()
    err = ((got - want).abs() / (1 + want.abs())).max().item()
    assert err <= 1e-3, err


@pytest.mark.gpu
def test_gemm_epilogues():
    torch = _torch()
    g = torch.Generator().manual_seed(5)
    M, N, K = 260, 384, 320
    A = torch.randn(M, K, generator=g).bfloat16().cuda()
    B = torch.randn(N, K, generator=g).bfloat16().cuda()
    bias = torch.randn(N, generator=g).cuda()
    acc = A.float() @ B.float().T + bias
    # ReLU, bf16 output
    ob = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    enc.gemm_bf16(A, B, mode=1, bias=bias, out_bf16=ob)
    assert (ob.float() - acc.relu().bfloat16().float()).abs().max().item() <= \
        2e-2 * (1 + acc.abs().max().item())
    # residual, in place fp32
    res = torch.randn(M, N, generator=g).cuda()
    out = res.clone()
    enc.gemm_bf16(A, B, mode=2, bias=bias, out=out)
    assert ((out - (res + acc)).abs() / (1 + acc.abs())).max().item() <= 1e-3
    # scale + positional table (row % pe_rows)
    pe = torch.randn(65, N, generator=g).cuda()
    out = torch.empty(M, N, device="cuda")
    enc.gemm_bf16(A, B, mode=3, bias=bias, out=out, scale=16.0, pe=pe)
    want = acc * 16.0 + pe[torch.arange(M, device="cuda") % 65]
    assert ((out - want).abs() / (1 + want.abs())).max().item() <= 1e-3
    # strided A (a column window of a wider matrix)
    wide = torch.randn(M, K + 64, generator=g).bfloat16().cuda()
    out = enc.gemm_bf16(wide[:, 64:], B)
    want = wide[:, 64:].float() @ B.float().T
    assert ((out - want).abs() / (1 + want.abs())).max().item() <= 1e-3


@pytest.mark.gpu
def test_gemm_rejects_bad_shapes():
    torch = _torch()
    A = torch.zeros(16, 12, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        enc.gemm_bf16(A, A)


def _run_encoder(spec, n, frames, seed):
    torch = _torch()
    w = enc.random_weights(spec, seed=seed)
    fb = enc.synthetic_fbank(n, frames, spec.idim, seed=seed + 1)
    e = enc.Encoder(spec, w, chunk=max(1, n // 2))
    grid = e.forward(torch.from_numpy(fb)).cpu().numpy()
    return w, fb, grid, e


@pytest.mark.gpu
@pytest.mark.parametrize("spec_name,n,frames", [("TINY", 3, 150), ("SMALL", 3, 1000),
                                                 ("LARGE", 1, 1000), ("TINY", 2, 1100),
                                                 ("SMALL", 2, 2000), ("TINY", 2, 1032),
                                                 ("LARGE", 1, 2000)])
def test_encoder_vs_torch(spec_name, n, frames):
    """T2 <= 256: one-tile tcgen05 attention; 256 < T2 <= 512 (frames 1032 ->
    257, 1100 -> 274, 2000 -> 499): the two-half tcgen05 attention."""
    from torch_encoder import encoder_forward
    spec = {"TINY": TINY, "SMALL": enc.SMALL, "LARGE": enc.LARGE}[spec_name]
    w, fb, grid, _ = _run_encoder(spec, n, frames, seed=11)
    assert grid.shape == (n, enc.frames_out(frames), spec.vocab)
    assert np.isfinite(grid).all()
    np.testing.assert_allclose(np.exp(grid.astype(np.float64)).sum(-1), 1.0, atol=1e-4)
    emu = encoder_forward(spec, w, fb, emulate_bf16=True)
    d = np.abs(grid - emu)
    assert d.max() <= 0.05 and d.mean() <= 2e-3, (d.max(), d.mean())
    f32 = encoder_forward(spec, w, fb)
    assert np.abs(grid - f32).max() <= 0.25


@pytest.mark.gpu
def test_encoder_host_and_device_fbank_identical():
    torch = _torch()
    spec = TINY
    w = enc.random_weights(spec, seed=2)
    fb = torch.from_numpy(enc.synthetic_fbank(5, 200, seed=9))
    e = enc.Encoder(spec, w, chunk=2)
    a = e.forward(fb)
    b = e.forward(fb.cuda())
    assert torch.equal(a, b)
    e1 = enc.Encoder(spec, w, chunk=5)   # chunking does not change the result
    assert torch.equal(a, e1.forward(fb))


@pytest.mark.gpu
def test_encoder_errors():
    torch = _torch()
    with pytest.raises(ValueError):
        enc.Encoder(TINY, np.zeros(10, np.float32))
    e = enc.Encoder(TINY, enc.random_weights(TINY))
    with pytest.raises(ValueError):
        e.forward(torch.zeros(1, 5, 80))


@pytest.mark.gpu
def test_encoder_grid_decodes_like_oracle(oracle):
    """Network in the loop: the device encoder's grid, decoded on device
    straight from HBM, equals the CPU oracle decoding the same grid."""
    torch = _torch()
    import paper_2101_05600_b200 as bl
    import pyoracle as po
    spec = enc.SMALL
    w = enc.random_weights(spec, seed=4)
    fb = torch.from_numpy(enc.synthetic_fbank(4, 1000, seed=5))
    e = enc.Encoder(spec, w)
    grid = e.forward(fb)                      # [4, 249, 500] in HBM
    kw = dict(beam_width=10, margin_m1=5, margin_m2=20)
    dec = bl.Decoder(bl.UniformScorer(spec.vocab - 1), bl.DecoderConfig(**kw))
    T, V = grid.shape[1], grid.shape[2]
    descs = [(f"s{i}", T, V, grid[i].data_ptr()) for i in range(grid.shape[0])]
    got = dec.decode_raw(descs, on_device=True)
    host = grid.cpu().numpy()
    want, _ = oracle.decode([host[i] for i in range(host.shape[0])],
                            po.ScorerSpec("uniform", spec.vocab - 1), po.config(**kw),
                            ids=[d[0] for d in descs])
    for g, r in zip(got, want):
        assert g.tokens == r.tokens and g.label_times == r.label_times
        assert g.steps_taken == r.steps and g.eos_trigger == r.eos_trigger
        assert abs(g.joint_logp - r.joint_logp) <= 1e-9
