#!/usr/bin/env python
"""Benchmark: offline batched joint CTC/attention beam search (BASELINE.json
metric: audio-seconds decoded per wall-second, i.e. inverse RTF).

Workload (configs[1], "C2"): an 8 h synthetic recording (2,880,000 fbank
frames at 10 ms) hard-segmented into 2880 x 10 s segments
(hard_segments(T, 1000, 1000)), each a CTC posterior grid of T_enc = 249
frames x vocab 500 (|C| = 499, blank = eos = 499) of flat random posteriors
(the random-init proxy), decoded with batch 64, beam 10, lambda 0.3, M1 = 5,
M2 = 20, CTC end detection on ("both"). One step decodes all 2880 segments
per GPU (batches in flight concurrently); under torchrun every
rank decodes its own 8 h recording (weak scaling) and the n-best records are
gathered to rank 0 with one NCCL all_gather.

  value  : grids resident in HBM, device-timed (CUDA events, max over ranks)
  e2e    : same call with pinned HOST grids through the C ABI, H2D + D2H inside
  --impl reference : the compiled reference CPU decoder on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "audio-sec decoded per wall-sec (inverse RTF) at 1/2/4/8 B200; prefix-score GB/s"
T_ENC, VOCAB, BEAM, M1, M2, LAMBDA = 249, 500, 10, 5, 20, 0.3
FRAME_SHIFT_MS = 40  # encoder frames (10 ms fbank, 4x subsampling)


def enc_frames(fbank):  # Conv2dSubsampling (3x3/2 twice), SURVEY §8 vocab note
    return ((fbank - 3) // 2 + 1 - 3) // 2 + 1


def workload_config(n_seg):
    return {"workload": "C2: 8 h synthetic recording -> hard_segments(2880000, 1000, 1000) "
                        "-> 2880 x 10 s segments per GPU; CTC grids T_enc=249 x vocab 500 "
                        "flat random posteriors (random-init proxy); batch 64, beam 10, "
                        "lambda 0.3, M1=5, M2=20, eos both; uniform attention scorer "
                        "(the Transformer decoder scorer is timed in pipeline_attn)",
            "segments_per_gpu": n_seg, "T_enc": T_ENC, "vocab": VOCAB, "batch": 64,
            "beam": BEAM, "margin_m1": M1, "margin_m2": M2, "ctc_weight": LAMBDA,
            "eos_mode": "both", "scorer": "uniform",
            "l2": "inputs larger than L2 (grids %.2f GB per GPU), no flush"
                  % (n_seg * T_ENC * VOCAB * 4 / 1e9)}


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.stop_ev = index, [], threading.Event()

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def flat_grids(torch, n, seed, device):
    """n x T_ENC x VOCAB float32 log-posteriors, rows ~ normalised Exp(1)
    (random_grid, synth.cpp:56-70), generated on the device in chunks."""
    g = torch.empty((n, T_ENC, VOCAB), dtype=torch.float32, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for s in range(0, n, 256):
        e = min(n, s + 256)
        x = torch.empty((e - s, T_ENC, VOCAB), dtype=torch.float64, device=device)
        x.exponential_(generator=gen)
        x = torch.log(x / x.sum(-1, keepdim=True))
        g[s:e] = x.float()
    return g


def cpu_reference_sample(grids_np, threads):
    """The compiled reference decoder (oracle/_ref) on host cores; falls back
    to the plain-C port when the reference could not be built."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    spec = po.ScorerSpec("uniform", VOCAB - 1)
    cfg = po.config(beam_width=BEAM, ctc_weight=LAMBDA, margin_m1=M1, margin_m2=M2)
    ids = [f"s{i}" for i in range(len(grids_np))]
    t0 = time.perf_counter()
    if po.Ref.available():
        po.Ref().decode(list(grids_np), spec, cfg, batch_size=64, ids=ids, threads=threads)
        kind, cores = "reference", threads
    else:
        po.Oracle().decode(list(grids_np), spec, cfg, ids=ids)
        kind, cores = "port", 1
    wall = time.perf_counter() - t0
    audio = len(grids_np) * T_ENC * FRAME_SHIFT_MS / 1000.0
    return audio / wall, kind, cores, wall


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np
    rng = np.random.default_rng(7)
    grids = []
    for _ in range(args.sample):
        p = rng.exponential(size=(T_ENC, VOCAB))
        grids.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_sample(grids[:2], threads)
    vals, walls = [], []
    for _ in range(args.steps):
        v, kind, cores, wall = cpu_reference_sample(grids, threads)
        vals.append(v)
        walls.append(wall)
    value = statistics.mean(vals)
    sample = (f"{args.sample} x 10 s segments (T_enc 249, vocab 500, beam 10, M2=20) per step, "
              f"same workload as the B200 arm")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "audio-s/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.mean(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.sample),
            "cpu_baseline": {"value": value, "unit": "audio-s/s", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": "audio-s/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_pipeline(args, torch, dist, bl, dec, ids, n, world, dev, local):
    """End to end through the public APIs: pinned host fbank (10 s, 80-dim,
    synthetic) -> device encoder (SMALL: 6 layers, d=256, 4 heads, ff 2048,
    vocab 500, random-init) -> grids in HBM -> device decode -> results on
    the host. Same segments, decoder and config as the headline."""
    from paper_2101_05600_b200 import encoder as benc
    spec = benc.SMALL
    enc = benc.Encoder(spec, benc.random_weights(spec, seed=0), device=local, chunk=148)
    fb = torch.from_numpy(benc.synthetic_fbank(n, 1000, spec.idim, seed=17 + local))
    fb = fb.pin_memory()
    grid = torch.empty((n, T_ENC, VOCAB), dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(device=dev)
    enc.set_stream(st.cuda_stream)
    dec.set_stream(st.cuda_stream)
    stride = T_ENC * VOCAB * 4
    descs = [(ids[i], T_ENC, VOCAB, grid.data_ptr() + i * stride) for i in range(n)]
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))

    def pstep():
        e0.record(st)
        enc.forward_raw(n, 1000, fb.data_ptr(), False, grid.data_ptr(), sync=False)
        e1.record(st)
        res = dec.decode_raw(descs, on_device=True)   # returns with results on the host
        e2.record(st)
        return res

    for _ in range(max(1, args.warmup - 1)):
        pstep()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_enc, t_all = [], []
    for _ in range(args.steps):
        pstep()
        st.synchronize()
        t_enc.append(e0.elapsed_time(e1))
        t_all.append(e0.elapsed_time(e2))
    ms = torch.tensor([statistics.mean(t_all)], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    dec.set_stream(0)
    enc_ms = statistics.mean(t_enc)
    d, ff, L, V, F2 = spec.d_model, spec.d_ff, spec.layers, spec.vocab, spec.f2
    flops_seg = 2.0 * (T_ENC * F2 * d * 9 * d + T_ENC * d * F2 * d
                       + L * T_ENC * (3 * d * d + d * d + 2 * d * ff) + T_ENC * V * d)
    audio = world * n * T_ENC * FRAME_SHIFT_MS / 1000.0
    return {"value": audio / (ms / 1000.0), "unit": "audio-s/s", "ms_per_step": ms,
            "encoder_ms": enc_ms, "decode_ms": ms - enc_ms,
            "encoder_tflops": n * flops_seg / (enc_ms / 1000.0) / 1e12,
            "encoder_flops_per_segment": flops_seg,
            "h2d_bytes_per_step": n * 1000 * spec.idim * 4,
            "d2h_bytes_per_step": dec.last_stats.get("d2h_bytes", 0),
            "model": "encoder 6 layers d=256 4 heads ff=2048 vocab 500 (random-init), "
                     "synthetic 80-dim fbank, 1000 frames per segment; decode as headline",
            "launches_per_step": enc.launches + dec.last_stats["launches"]}


def run_prefix_c3(torch, bl, dev, peak, n=592):
    """BASELINE's second metric ("prefix-score GB/s") where the prefix score
    dominates: the config-3 shape (vocab 5000, beam 10, M1 5, M2 unbounded,
    T_enc 249, flat posteriors) on 592 segments (4 per SM), K1 algorithmic
    bytes / kernel time against the measured HBM peak."""
    V = 5000
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)
    g = torch.empty((n, T_ENC, V), dtype=torch.float32, device=dev)
    for s0 in range(0, n, 64):
        x = torch.empty((min(n, s0 + 64) - s0, T_ENC, V), dtype=torch.float64, device=dev)
        x.exponential_(generator=gen)
        g[s0:s0 + x.shape[0]] = torch.log(x / x.sum(-1, keepdim=True)).float()
        del x
    dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=BEAM), device=dev.index)
    descs = [(f"c3_{i}", T_ENC, V, g[i].data_ptr()) for i in range(n)]
    torch.cuda.synchronize()
    dec.decode_raw(descs, on_device=True)
    dec.decode_raw(descs, on_device=True)
    st = dec.last_stats
    gbs = st["k1_bytes"] / (st["kernel_ms"] / 1000.0) / 1e9
    out = {"segments": n, "vocab": V, "kernel_ms": st["kernel_ms"], "k1_bytes": st["k1_bytes"],
           "k1_gbs": gbs, "peak_gbs": peak[0], "frac": gbs / peak[0],
           "audio_s_per_s": n * T_ENC * FRAME_SHIFT_MS / 1000.0 / (st["kernel_ms"] / 1000.0),
           "kernel": "decode_kernel<10, TMA> (K1 slab streamed by cp.async.bulk.tensor)"}
    del g, dec
    torch.cuda.empty_cache()
    return out


def run_pipeline_attn(args, torch, dist, bl, ids, n, world, dev, local):
    """The full model end to end: pinned host fbank -> device encoder (grid +
    memory) -> joint CTC/attention decode with the device Transformer decoder
    scorer (3 layers, d=256, 4 heads, ff 2048, vocab 500; BASELINE cfg 2's
    '6 enc/3 dec' model, random-init) -> results on the host."""
    from paper_2101_05600_b200 import encoder as benc
    from paper_2101_05600_b200 import transformer as btr
    from paper_2101_05600_b200.api import _check, lib
    import ctypes as C
    espec, dspec = benc.SMALL, btr.SMALL
    enc = benc.Encoder(espec, benc.random_weights(espec, seed=0), device=local, chunk=148)
    sc = btr.TransformerScorer(dspec, btr.random_weights(dspec, seed=1), device=local)
    cfg = bl.DecoderConfig(beam_width=BEAM, ctc_weight=LAMBDA, margin_m1=M1, margin_m2=M2,
                           eos_mode="both")
    dec = bl.Decoder(sc, cfg, device=local)
    fb = torch.from_numpy(benc.synthetic_fbank(n, 1000, espec.idim, seed=17 + local))
    fb = fb.pin_memory()
    grid = torch.empty((n, T_ENC, VOCAB), dtype=torch.float32, device=dev)
    mem = torch.empty((n, T_ENC, espec.d_model), dtype=torch.bfloat16, device=dev)
    st = torch.cuda.Stream(device=dev)
    enc.set_stream(st.cuda_stream)
    dec.set_stream(st.cuda_stream)
    stride = T_ENC * VOCAB * 4
    descs = [(ids[i], T_ENC, VOCAB, grid.data_ptr() + i * stride) for i in range(n)]
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))

    def pstep():
        e0.record(st)
        _check(lib().bl_encoder_forward_mem(enc._h, n, 1000, C.c_void_p(fb.data_ptr()), 0,
                                            C.c_void_p(grid.data_ptr()),
                                            C.c_void_p(mem.data_ptr()), 0))
        e1.record(st)
        res = dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(), mem_frames=T_ENC)
        e2.record(st)
        return res

    res = pstep()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_enc, t_all = [], []
    for _ in range(max(1, args.attn_steps)):
        res = pstep()
        st.synchronize()
        t_enc.append(e0.elapsed_time(e1))
        t_all.append(e0.elapsed_time(e2))
    ms = torch.tensor([statistics.mean(t_all)], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    enc_ms = statistics.mean(t_enc)
    lens = [len(r.tokens) for r in res]
    audio = world * n * T_ENC * FRAME_SHIFT_MS / 1000.0
    out = {"value": audio / (ms / 1000.0), "unit": "audio-s/s", "ms_per_step": ms,
           "steps": max(1, args.attn_steps), "encoder_ms": enc_ms, "decode_ms": ms - enc_ms,
           "decode_steps_max": max(r.steps_taken for r in res),
           "mean_hyp_tokens": statistics.mean(lens),
           "h2d_bytes_per_step": n * 1000 * espec.idim * 4,
           "d2h_bytes_per_step": dec.last_stats.get("d2h_bytes", 0),
           "launches_per_step": enc.launches + dec.last_stats["launches"],
           "model": "encoder 6 x d256 + Transformer decoder scorer 3 x d256 (4 heads, ff "
                    "2048, vocab 500), random-init; the near-uniform random decoder keeps "
                    "hypotheses ~T long (worst case for the per-step decoder)"}
    del dec, sc
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--segments", type=int, default=2880, help="segments per GPU")
    ap.add_argument("--sample", type=int, default=24, help="CPU baseline segments")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="skip the fbank -> encoder -> decoder legs")
    ap.add_argument("--attn-steps", type=int, default=2,
                    help="timed steps of the full-model (Transformer scorer) leg")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2101_05600_b200 as bl
    from paper_2101_05600_b200 import dist as bdist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.segments
    # hard segmentation of the 8 h recording (integer-exact, host C++)
    segs = bl.hard_segments(2_880_000 * n // 2880, 1000, 1000, f"rec{rank}")
    assert len(segs) == n and all(enc_frames(s.end - s.start) == T_ENC for s in segs)
    grids = flat_grids(torch, n, 1000 + rank, dev)
    torch.cuda.synchronize()
    cfg = bl.DecoderConfig(beam_width=BEAM, ctc_weight=LAMBDA, margin_m1=M1, margin_m2=M2,
                           eos_mode="both")
    dec = bl.Decoder(bl.UniformScorer(VOCAB - 1), cfg, device=local)
    stride = T_ENC * VOCAB * 4
    base = grids.data_ptr()
    ids = [f"{s.utterance_id}:{s.start}-{s.end}" for s in segs]
    descs = [(ids[i], T_ENC, VOCAB, base + i * stride) for i in range(n)]
    audio_per_step = n * T_ENC * FRAME_SHIFT_MS / 1000.0

    def step(on_device, d):
        res = dec.decode_raw(d, on_device=on_device)
        if world > 1:
            bdist.gather_results(res, T_ENC, n * world, device=dev)
        return res

    for _ in range(args.warmup):
        step(True, descs)
    kms, k1, launches = [], [], 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step(True, descs)
            kms.append(dec.last_stats["kernel_ms"])
            k1.append(dec.last_stats["k1_bytes"])
            launches += dec.last_stats["launches"]
        ev1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = world * audio_per_step / (ms / 1000.0)

    # e2e: pinned host grids through the C ABI (H2D + decode + D2H per step)
    e2e = None
    if not args.no_e2e:
        host = grids.cpu().pin_memory()
        del grids
        torch.cuda.empty_cache()
        hb = host.data_ptr()
        hdescs = [(ids[i], T_ENC, VOCAB, hb + i * stride) for i in range(n)]
        step(False, hdescs)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step(False, hdescs)
        ev1.record()
        torch.cuda.synchronize()
        ems = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        ems = float(ems.item())
        e2e = {"value": world * audio_per_step / (ems / 1000.0), "unit": "audio-s/s",
               "ms_per_step": ems, "h2d_bytes_per_step": n * stride,
               "d2h_bytes_per_step": dec.last_stats.get("d2h_bytes", 0)}

    prefix_c3 = None
    if not args.no_pipeline:
        prefix_c3 = run_prefix_c3(torch, bl, dev, peaks())
    pipeline = pipeline_attn = None
    if not args.no_pipeline:
        pipeline = run_pipeline(args, torch, dist, bl, dec, ids, n, world, dev, local)
        pipeline_attn = run_pipeline_attn(args, torch, dist, bl, ids, n, world, dev, local)

    peak, peak_kind = peaks()
    kernel_ms = statistics.mean(kms)
    achieved = statistics.mean(k1) / (kernel_ms / 1000.0) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "audio-s/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(n),
            "e2e": e2e, "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(),
                         "kernel": "decode_kernel (persistent: K1 bulk + search epilogue)",
                         "algorithmic_bytes_per_launch": statistics.mean(k1),
                         "kernel_ms": kernel_ms},
            "clocks": clk.summary(),
            "prefix_score_c3": prefix_c3,
            "pipeline": pipeline,
            "pipeline_attn": pipeline_attn,
            "counters": {k: dec.last_stats[k] for k in
                         ("steps", "scorer_queries", "ctc_frames_evaluated", "contenders",
                          "fallback_steps")}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import numpy as np
        sample = host[:args.sample].numpy() if e2e is not None else \
            grids[:args.sample].cpu().numpy()
        v, kind, cores, wall = cpu_reference_sample(list(np.ascontiguousarray(sample)),
                                                    os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": v, "unit": "audio-s/s", "cores": cores, "kind": kind,
                                "sample": f"first {args.sample} of the 2880 segments "
                                          f"({wall:.1f} s wall)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
