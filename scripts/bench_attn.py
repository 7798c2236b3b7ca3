"""Full-model pipeline timing: fbank (pinned host) -> encoder (grid + memory)
-> joint CTC/attention decode with the device Transformer scorer -> host
results. python scripts/bench_attn.py --n 2880 [--profile]"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_05600_b200 as bl  # noqa: E402
from paper_2101_05600_b200 import encoder as enc  # noqa: E402
from paper_2101_05600_b200 import transformer as tr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--beam", type=int, default=10)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--spec", default="small", choices=["small", "large"])
ap.add_argument("--m2", type=int, default=20, help="margin M2 (< 0: unbounded, the default knobs)")
ap.add_argument("--chunk", type=int, default=148, help="encoder segments per chunk")
a = ap.parse_args()
espec, dspec = (enc.SMALL, tr.SMALL) if a.spec == "small" else (enc.LARGE, tr.LARGE)
V, D = espec.vocab, espec.d_model
e = enc.Encoder(espec, enc.random_weights(espec, seed=0), chunk=a.chunk)
sc = tr.TransformerScorer(dspec, tr.random_weights(dspec, seed=1))
dec = bl.Decoder(sc, bl.DecoderConfig(beam_width=a.beam, margin_m1=5,
                                      margin_m2=bl.NO_MARGIN if a.m2 < 0 else a.m2))
fb = torch.from_numpy(enc.synthetic_fbank(a.n, 1000, seed=2)).pin_memory()
grid = torch.empty(a.n, 249, V, device="cuda")
mem = torch.empty(a.n, 249, D, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.Stream()
e.set_stream(st.cuda_stream)
dec.set_stream(st.cuda_stream)
descs = [(f"s{i}", 249, V, grid[i].data_ptr()) for i in range(a.n)]
from paper_2101_05600_b200.api import _check, lib  # noqa: E402
import ctypes as C  # noqa: E402


def step():
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(st)
    _check(lib().bl_encoder_forward_mem(e._h, a.n, 1000, C.c_void_p(fb.data_ptr()), 0,
                                        C.c_void_p(grid.data_ptr()), C.c_void_p(mem.data_ptr()), 0))
    ev[1].record(st)
    res = dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(), mem_frames=249)
    ev[2].record(st)
    st.synchronize()
    return res, ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])


res, _, _ = step()
t = [step() for _ in range(a.steps)]
enc_ms = statistics.mean(x[1] for x in t)
dec_ms = statistics.mean(x[2] for x in t)
lens = [len(r.tokens) for r in t[-1][0]]
out = {"spec": a.spec, "n": a.n, "encoder_ms": round(enc_ms, 2), "decode_ms": round(dec_ms, 2),
       "audio_s_per_s": round(a.n * 9.96 / ((enc_ms + dec_ms) / 1e3), 1),
       "steps_max": max(r.steps_taken for r in t[-1][0]),
       "mean_tokens": statistics.mean(lens), "stats": dec.last_stats}
if a.profile:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
    agg = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            nm = ev.name.replace("(anonymous namespace)::", "").replace("void ", "")
            k = nm.split("(")[0].split("<")[0]
            c = agg.setdefault(k, [0, 0.0])
            c[0] += 1
            c[1] += ev.device_time_total / 1e3
    out["kernels_ms"] = {k: [c, round(v, 2)] for k, (c, v) in
                         sorted(agg.items(), key=lambda x: -x[1][1])[:14]}
print(json.dumps(out, indent=1))
