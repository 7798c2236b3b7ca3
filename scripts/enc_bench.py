"""Encoder throughput and per-kernel breakdown on one B200.

python scripts/enc_bench.py [--spec small|large] [--n 256] [--chunk 64]
Prints GEMM TFLOP/s at the encoder's shapes, the whole-forward time, and a
torch.profiler kernel table (CUPTI) of one forward.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_05600_b200 import encoder as enc  # noqa: E402


def time_it(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def gemm_table(spec, seg):
    d, ff, V = spec.d_model, spec.d_ff, spec.vocab
    M = seg * 249
    shapes = {"conv2": (seg * 249 * 19, d, 9 * d), "out": (M, d, 19 * d), "qkv": (M, 3 * d, d),
              "oproj": (M, d, d), "ffn1": (M, ff, d), "ffn2": (M, d, ff), "ctc": (M, V, d)}
    rows = {}
    for k, (m, n, kk) in shapes.items():
        A = torch.randn(m, kk, device="cuda").bfloat16()
        B = torch.randn(n, kk, device="cuda").bfloat16()
        if n % 8 == 0:
            out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            ms = time_it(lambda: enc.gemm_bf16(A, B, out_bf16=out))
        else:
            out = torch.empty(m, n, device="cuda", dtype=torch.float32)
            ms = time_it(lambda: enc.gemm_bf16(A, B, out=out))
        ms_cublas = time_it(lambda: A @ B.T)
        fl = 2.0 * m * n * kk
        rows[k] = {"M": m, "N": n, "K": kk, "ms": round(ms, 4),
                   "tflops": round(fl / ms / 1e9, 1),
                   "cublas_tflops": round(fl / ms_cublas / 1e9, 1)}
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", default="small")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--no-table", action="store_true", help="skip the per-shape GEMM table")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = enc.SMALL if a.spec == "small" else enc.LARGE
    torch.cuda.init()
    out = {"spec": a.spec, "gemms": {} if a.no_table else gemm_table(spec, a.chunk)}
    w = enc.random_weights(spec)
    e = enc.Encoder(spec, w, chunk=a.chunk)
    fb = torch.from_numpy(enc.synthetic_fbank(a.n, 1000)).cuda()
    grid = torch.empty(a.n, 249, spec.vocab, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    e.set_stream(st)
    fwd = lambda: e.forward_raw(a.n, 1000, fb.data_ptr(), True, grid.data_ptr(), sync=False)  # noqa
    ms = time_it(fwd, reps=a.reps, warm=2)
    out["forward_ms"] = round(ms, 3)
    out["segments_per_s"] = round(a.n / ms * 1e3, 1)
    out["audio_s_per_s"] = round(a.n * 10 / ms * 1e3, 1)
    out["launches"] = e.launches
    if a.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fwd()
            torch.cuda.synchronize()
        agg = {}
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                nm = ev.name.replace("(anonymous namespace)::", "")
                key = nm.split("(")[0].split("<")[0].replace("void ", "")[:60]
                agg.setdefault(key, [0, 0.0])
                agg[key][0] += 1
                agg[key][1] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") \
                    else ev.cuda_time_total / 1e3
        out["kernels_ms"] = {k: [c, round(t, 3)] for k, (c, t) in
                             sorted(agg.items(), key=lambda x: -x[1][1])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
