"""Times the tcgen05 GEMM at the decoder-scorer step shapes (M = 2880
segments x beam 10 rows): TFLOP/s per (N, K, epilogue)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2101_05600_b200 import encoder as enc  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 28800
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256  # 512: the Librispeech-size decoder
V = 500 if d == 256 else 5000
for (N, K, mode, name) in [(3 * d, d, 0, "qkv"), (d, d, 2, "wo+res"), (d, d, 0, "q2"),
                           (2048, d, 1, "ff1+relu"), (d, 2048, 2, "ff2+res"),
                           (V, d, 0, "out")]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    res = torch.randn(M, N, device="cuda")
    ob = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kw = dict(mode=mode, bias=bias)
    if mode == 2 or N % 8:
        kw["out"] = res
    else:
        kw["out_bf16"] = ob
    for _ in range(3):
        enc.gemm_bf16(A, B, **kw)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        enc.gemm_bf16(A, B, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    # cuBLAS on the same shape (library reference point, bf16 out)
    for _ in range(3):
        torch.matmul(A, B.t())
    e0.record()
    for _ in range(20):
        torch.matmul(A, B.t())
    e1.record()
    torch.cuda.synchronize()
    cb = e0.elapsed_time(e1) / 20
    print(f"{name:9s} M={M} N={N} K={K}: {ms * 1e3:7.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s"
          f"   (cuBLAS {cb * 1e3:7.1f} us)")
