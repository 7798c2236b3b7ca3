"""Encoder forward time for 20 s segments (T2 = 499): tcgen05 two-half
attention vs the CUDA-core kernel (BL_ENC_ATTN_CUDA=1 in the environment)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_05600_b200 import encoder as enc
spec = enc.LARGE if (len(sys.argv) > 1 and sys.argv[1] == "large") else enc.SMALL
n = 148
e = enc.Encoder(spec, enc.random_weights(spec, seed=0), chunk=148)
fb = torch.from_numpy(enc.synthetic_fbank(n, 2000, spec.idim, seed=2)).cuda()
for _ in range(2):
    g = e.forward(fb)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    g = e.forward(fb)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 3 * 1e3
print(f"{'cuda-core' if os.environ.get('BL_ENC_ATTN_CUDA') else 'tcgen05'} attention, {n} x 20 s, "
      f"d={spec.d_model}: encoder {ms:.1f} ms ({n * 19.96 / (ms / 1e3):.0f} audio-s/s)")
