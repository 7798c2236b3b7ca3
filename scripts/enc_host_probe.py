"""Encoder timing with host (pinned) vs device fbank, plus memcpy/kernel
totals from torch.profiler, to locate host-input overheads."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_05600_b200 import encoder as enc  # noqa: E402


def main():
    spec = enc.SMALL
    e = enc.Encoder(spec, enc.random_weights(spec), chunk=64)
    for n in (256, 2880):
        fbh = torch.from_numpy(enc.synthetic_fbank(n, 1000)).pin_memory()
        fbd = fbh.cuda()
        grid = torch.empty(n, 249, spec.vocab, device="cuda")
        for sname, st in (("default", torch.cuda.current_stream()), ("side", torch.cuda.Stream())):
          e.set_stream(st.cuda_stream)
          for name, fb, ondev in (("device", fbd, True), ("host", fbh, False)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                e.forward_raw(n, 1000, fb.data_ptr(), ondev, grid.data_ptr(), sync=True)
            a.record(st)
            for _ in range(3):
                e.forward_raw(n, 1000, fb.data_ptr(), ondev, grid.data_ptr(), sync=False)
            b.record(st)
            st.synchronize()
            print(n, sname, name, "ms", round(a.elapsed_time(b) / 3, 2), flush=True)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            e.forward_raw(n, 1000, fbh.data_ptr(), False, grid.data_ptr(), sync=True)
        tot = {}
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                nm = ev.name.replace("(anonymous namespace)::", "").replace("void ", "")
                k = "memcpy" if "emcpy" in nm else nm.split("(")[0].split("<")[0]
                tot[k] = tot.get(k, 0) + ev.device_time_total / 1e3
        print(n, {k: round(v, 2) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]})


if __name__ == "__main__":
    main()
