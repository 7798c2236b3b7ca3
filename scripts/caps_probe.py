"""Contender-cap probe: decode time and exact-fallback steps at beam 10/20
(vocab 5000, 10 s, 512 segments) for the cap multiplier in BL_CAPS_MULT."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_05600_b200 as bl
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
from c5_sweep import grids
for T, n in ((249, 512), (124, 512)):
    g = grids(n, T, 7000 + T)
    for beam in (10, 20):
        dec = bl.Decoder(bl.UniformScorer(4999), bl.DecoderConfig(beam_width=beam))
        descs = [(f"s{i}", T, 5000, g[i].data_ptr()) for i in range(n)]
        dec.decode_raw(descs, on_device=True)
        t0 = time.perf_counter(); dec.decode_raw(descs, on_device=True); ms = (time.perf_counter() - t0) * 1e3
        st = dec.last_stats
        print(f"caps_mult={os.environ.get('BL_CAPS_MULT', 3)} T={T} beam={beam} n={n}: {ms:.1f} ms kernel {st['kernel_ms']:.1f} fallback {st['fallback_steps']} contenders/step {st['contenders']/st['steps']:.1f}", flush=True)
