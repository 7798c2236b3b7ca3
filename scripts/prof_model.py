"""Per-phase cycles of the search kernel inside the full-model decode
(network scorer rows, step-granular), next to the same search with the
uniform scorer: python scripts/prof_model.py [N]"""
import os
import sys

os.environ["BL_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_2101_05600_b200 as bl  # noqa: E402
from paper_2101_05600_b200 import encoder as enc  # noqa: E402
from paper_2101_05600_b200 import transformer as tr  # noqa: E402
from paper_2101_05600_b200.api import _check, lib  # noqa: E402

names = ["init", "P1", "P2", "P3", "P4", "P5", "P6", "P7", "fallback", "P8", "P6-P9", "fin",
         "-", "-", "P6 serial", "P6 staging"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 296
espec, dspec = enc.LARGE, tr.LARGE
V, D, T = espec.vocab, espec.d_model, 249
e = enc.Encoder(espec, enc.random_weights(espec, seed=0), chunk=148)
fb = torch.from_numpy(enc.synthetic_fbank(n, 1000, seed=2)).pin_memory()
grid = torch.empty(n, T, V, device="cuda")
mem = torch.empty(n, T, D, device="cuda", dtype=torch.bfloat16)
_check(lib().bl_encoder_forward_mem(e._h, n, 1000, C.c_void_p(fb.data_ptr()), 0,
                                    C.c_void_p(grid.data_ptr()), C.c_void_p(mem.data_ptr()), 0))
torch.cuda.synchronize()
descs = [(f"s{i}", T, V, grid[i].data_ptr()) for i in range(n)]
for kind in ("uniform", "network"):
    if kind == "uniform":
        dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=10), step_mode=True)
        run = lambda: dec.decode_raw(descs, on_device=True)  # noqa: E731
    else:
        dec = bl.Decoder(tr.TransformerScorer(dspec, tr.random_weights(dspec, seed=1)),
                         bl.DecoderConfig(beam_width=10))
        run = lambda: dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(),  # noqa: E731
                                     mem_frames=T)
    run()
    run()
    st = dec.last_stats
    pc = st["profile_cycles"]
    steps = st["steps"] / n
    print(f"{kind}: search kernel {st['kernel_ms']:.1f} ms (incl. network for 'network'), "
          f"filter keys/step {st['filter_keys'] / st['steps']:.1f}, contenders/step "
          f"{st['contenders'] / st['steps']:.1f}")
    print("   " + "  ".join(f"{nm} {c / steps / 1e3:.1f}k" for nm, c in zip(names, pc)
                          if nm != "-" and c > 0))
