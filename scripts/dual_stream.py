"""Experiment: the full large model over N segments with the decode split
into G groups decoded concurrently (a host thread, decoder, scorer and
stream per group), so one group's network kernels fill the GPU while
another's search step runs. python scripts/dual_stream.py [N [G]]"""
import ctypes as C
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_05600_b200 as bl  # noqa: E402
from paper_2101_05600_b200 import encoder as enc  # noqa: E402
from paper_2101_05600_b200 import transformer as tr  # noqa: E402
from paper_2101_05600_b200.api import _check, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2880
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
espec, dspec = enc.LARGE, tr.LARGE
V, D, T = espec.vocab, espec.d_model, 249
e = enc.Encoder(espec, enc.random_weights(espec, seed=0), chunk=148)
w = tr.random_weights(dspec, seed=1)
fb = torch.from_numpy(enc.synthetic_fbank(n, 1000, seed=2)).pin_memory()
grid = torch.empty(n, T, V, device="cuda")
mem = torch.empty(n, T, D, device="cuda", dtype=torch.bfloat16)
st0 = torch.cuda.Stream()
e.set_stream(st0.cuda_stream)
_check(lib().bl_encoder_forward_mem(e._h, n, 1000, C.c_void_p(fb.data_ptr()), 0,
                                    C.c_void_p(grid.data_ptr()), C.c_void_p(mem.data_ptr()), 0))
st0.synchronize()
bounds = [n * g // G for g in range(G + 1)]
groups = []
for g in range(G):
    a, b = bounds[g], bounds[g + 1]
    sc = tr.TransformerScorer(dspec, w)
    dec = bl.Decoder(sc, bl.DecoderConfig(beam_width=10))
    s = torch.cuda.Stream()
    dec.set_stream(s.cuda_stream)
    descs = [(f"s{i}", T, V, grid[i].data_ptr()) for i in range(a, b)]
    groups.append((dec, descs, mem[a].data_ptr()))
out = [None] * G


def run(g):
    dec, descs, mp = groups[g]
    out[g] = dec.decode_raw(descs, on_device=True, memory=mp, mem_frames=T)


for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1000
    print(f"n {n} groups {G}: decode wall {wall:.1f} ms  ({n * 9.96 / (wall / 1000):.0f} audio-s/s "
          f"decode only); kernel_ms per group "
          f"{[round(gr[0].last_stats['kernel_ms'], 1) for gr in groups]}", flush=True)
