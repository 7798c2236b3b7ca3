"""Diagnostics for the Transformer scorer path: records, row error vs torch,
decode lengths, replay parity (small sizes)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2101_05600_b200 as bl  # noqa: E402
from paper_2101_05600_b200 import encoder as enc  # noqa: E402
from paper_2101_05600_b200 import transformer as tr  # noqa: E402
import pyoracle as po  # noqa: E402
from torch_decoder import decoder_scores  # noqa: E402

for espec, dspec, n, frames, beam in ((enc.SMALL, tr.SMALL, 2, 1000, 10),):
    e = enc.Encoder(espec, enc.random_weights(espec, seed=7))
    fb = torch.from_numpy(enc.synthetic_fbank(n, frames, espec.idim, seed=8))
    grid, mem = e.forward(fb, memory=True)
    w = tr.random_weights(dspec, seed=9)
    sc = tr.TransformerScorer(dspec, w)
    kw = dict(beam_width=beam, margin_m1=5, margin_m2=20)
    dec = bl.Decoder(sc, bl.DecoderConfig(**kw))
    dec.set_record(True)
    T, V = grid.shape[1], grid.shape[2]
    descs = [(f"s{i}", T, V, grid[i].data_ptr()) for i in range(n)]
    res = list(dec.decode_raw(descs, on_device=True, memory=mem.data_ptr(), mem_frames=T))
    recs = dec.records()
    print("records", len(recs), "max prefix", max(len(p) for _, p, _ in recs))
    for r in res:
        print(r.id, "len", len(r.tokens), "steps", r.steps_taken, r.eos_trigger,
              round(r.joint_logp, 3), r.tokens[:12])
    print("stats", dec.last_stats)
    memh = mem.float().cpu().numpy()
    pick = recs[::max(1, len(recs) // 40)]
    errs = []
    for u, p, row in pick:
        want = decoder_scores(dspec, w, memh[u], [p], emulate_bf16=True)[0]
        errs.append(np.abs(row - want).max())
    print("row err vs torch(bf16 emu): max %.4g mean %.4g over %d rows" %
          (max(errs), np.mean(errs), len(errs)))
    f32 = [np.abs(row - decoder_scores(dspec, w, memh[u], [p])[0]).max() for u, p, row in pick[:10]]
    print("row err vs torch fp32: max %.4g" % max(f32))
    print("row entropy-ish: max logp", float(np.max([r.max() for _, _, r in pick])))
    ref = po.Ref()
    host = grid.cpu().numpy()
    spec = po.ScorerSpec("replay", dspec.vocab - 1, replay_ids=[d[0] for d in descs],
                         entries=[(u, p, r) for u, p, r in recs])
    ref.replay_misses(reset=True)
    want, wc = ref.decode([host[i] for i in range(n)], spec, po.config(**kw),
                          ids=[d[0] for d in descs])
    print("replay misses", ref.replay_misses(), "ref counters", wc)
    print("identical:", all(g.tokens == r.tokens and g.steps_taken == r.steps for g, r in zip(res, want)))
