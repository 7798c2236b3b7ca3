"""BASELINE config 5: segment-length / batch / beam sweep of the device
decoder (vocab 5000, DecoderConfig defaults otherwise, flat random
posteriors, grids resident in HBM), one B200. Segments: 5 / 10 / 20 s
(T_enc 124 / 249 / 499 after the 4x subsampling); batch = segments per
decode call (all in flight at once); beam 4 / 10 / 20. A few points also run
the compiled reference CPU decoder (oracle/_ref, all host threads) on one
segment of the same shape, and its results are compared with the device's
(parity). Prints one JSON object per point.

python scripts/c5_sweep.py [--cpu] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_05600_b200 as bl  # noqa: E402

V = 5000
SEG = {5: 124, 10: 249, 20: 499}
BATCH = (16, 64, 128, 512)
BEAM = (4, 10, 20)
CPU_POINTS = {(5, 4), (5, 10), (10, 4), (10, 10)}


def grids(n, T, seed):
    g = torch.empty((n, T, V), dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cuda")
    x = torch.empty((T, V), dtype=torch.float64, device="cuda")
    for i in range(n):
        gen.manual_seed(seed + i)
        x.exponential_(generator=gen)
        g[i] = torch.log(x / x.sum(-1, keepdim=True)).float()
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true", help="also time the reference on CPU points")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else None
    for sec, T in SEG.items():
        g = grids(max(BATCH), T, 7000 + T)
        torch.cuda.synchronize()
        for beam in BEAM:
            dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=beam))
            for n in BATCH:
                descs = [(f"s{i}", T, V, g[i].data_ptr()) for i in range(n)]
                rec = {"segment_s": sec, "T_enc": T, "vocab": V, "beam": beam, "batch": n}
                try:
                    dec.decode_raw(descs, on_device=True)  # warm-up
                    kms = []
                    for _ in range(3):
                        t0 = time.perf_counter()
                        res = dec.decode_raw(descs, on_device=True)
                        kms.append((time.perf_counter() - t0) * 1000)
                    st = dec.last_stats
                    ms = min(kms)
                    audio = n * T * bench.FRAME_SHIFT_MS / 1000.0
                    rec.update(ms_per_call=ms, kernel_ms=st["kernel_ms"],
                               audio_s_per_s=audio / (ms / 1000.0),
                               k1_gbs=st["k1_bytes"] / (st["kernel_ms"] / 1000.0) / 1e9,
                               fallback_steps=st["fallback_steps"])
                    if args.cpu and n == BATCH[0] and (sec, beam) in CPU_POINTS:
                        # >= two OpenMP tasks (utterance x hypothesis) per host thread
                        k = max(1, min(8, -(-2 * (os.cpu_count() or 1) // beam)))
                        sample = [g[i].cpu().numpy() for i in range(k)]
                        sys.path.insert(0, os.path.join(bench.ROOT, "oracle"))
                        import pyoracle as po
                        cfg = po.config(beam_width=beam)
                        t0 = time.perf_counter()
                        want, _ = po.Ref().decode(sample, po.ScorerSpec("uniform", V - 1), cfg,
                                                  ids=[f"s{i}" for i in range(k)],
                                                  threads=os.cpu_count())
                        wall = time.perf_counter() - t0
                        rec["cpu_reference"] = {
                            "audio_s_per_s": k * T * bench.FRAME_SHIFT_MS / 1000.0 / wall,
                            "cores": os.cpu_count(), "sample": f"{k} segments",
                            "parity": all(r.tokens == w.tokens and r.label_times == w.label_times
                                          and abs(r.joint_logp - w.joint_logp) <= 1e-9
                                          for r, w in zip(res[:k], want))}
                except Exception as e:  # noqa: BLE001 - a refused shape is a result
                    rec["refused"] = str(e)[:200]
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
            del dec
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
