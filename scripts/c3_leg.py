"""The C3 decode shape alone (vocab 5000, beam 10, M2 unbounded, T_enc 249,
flat posteriors, TMA slab variant): N segments (default 592) decoded from
HBM, prints kernel ms and K1 GB/s against the measured HBM peak.

python scripts/c3_leg.py [N [T_enc [beam]]]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_05600_b200 as bl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 592
if len(sys.argv) > 2:
    bench.T_ENC = int(sys.argv[2])
beam = int(sys.argv[3]) if len(sys.argv) > 3 else bench.BEAM
dev = torch.device("cuda", 0)
g = bench.segment_grids(torch, 0, n, dev, 100000)
# C3_STEP=1: step-granular search (one launch per step, state saved in HBM)
dec = bl.Decoder(bl.UniformScorer(bench.VOCAB - 1), bl.DecoderConfig(beam_width=beam),
                 step_mode=os.environ.get("C3_STEP") == "1")
stride = bench.T_ENC * bench.VOCAB * 4
descs = [(f"c3_{i}", bench.T_ENC, bench.VOCAB, g.data_ptr() + i * stride) for i in range(n)]
torch.cuda.synchronize()
for _ in range(2):
    dec.decode_raw(descs, on_device=True)
st = dec.last_stats
gbs = st["k1_bytes"] / (st["kernel_ms"] / 1000.0) / 1e9
print("c3 %d segments T %d B %d: kernel %.2f ms  %.0f GB/s  frac %.3f  filter_keys/step %.1f"
      "  fallback %d wide %s" % (
    n, bench.T_ENC, beam, st["kernel_ms"], gbs, gbs / bench.peaks()[0],
    st["filter_keys"] / max(1, st["steps"]), st["fallback_steps"], st.get("wide_steps", "-")))
