"""C3-shaped decode: vocab 5000 (|C|=4999), beam 10, default margins
(M1=5, M2=inf), flat posteriors, T_enc=249 (10 s)."""
import os
import sys
import time
sys.path.insert(0, ".")
import torch
import paper_2101_05600_b200 as bl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
V = 5000
gen = torch.Generator(device="cuda"); gen.manual_seed(3)
g = torch.empty((n, 249, V), dtype=torch.float32, device="cuda")
for s in range(0, n, 32):
    x = torch.empty((min(n, s + 32) - s, 249, V), dtype=torch.float64, device="cuda").exponential_(generator=gen)
    g[s:s + x.shape[0]] = torch.log(x / x.sum(-1, keepdim=True)).float()
torch.cuda.synchronize()
dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=10))
descs = [(f"c{i}", 249, V, g[i].data_ptr()) for i in range(n)]
for _ in range(2):
    dec.decode_raw(descs, on_device=True)
st = dec.last_stats
print({k: st[k] for k in ("kernel_ms", "k1_bytes", "fallback_steps", "contenders", "steps", "filter_keys")})
print("K1 GB/s %.1f  audio-s/s %.0f" % (st["k1_bytes"] / st["kernel_ms"] / 1e6, n * 9.96 / (st["kernel_ms"] / 1e3)))
if os.environ.get("BL_PROFILE"):
    names = ["init", "P1", "P2", "P3", "P4", "P5", "P6", "P7", "fb", "P8", "P9", "fin", "t0:P3fr", "t0:P3keys", "t0:P6ser", "t0:P6stg"]
    pc = st["profile_cycles"]; steps = st["steps"] / n
    print("  ".join(f"{a}={b / steps / 1e3:.1f}k" for a, b in zip(names, pc)))
