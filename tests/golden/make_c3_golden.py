"""Golden results at BASELINE config 3's decode shape (T=249, vocab 5000,
beam 10, DecoderConfig defaults: lambda 0.3, M1 5, M2 unbounded, eos both)
from the UNMODIFIED reference compiled here (oracle/_ref, batched
batched_beam_search, batch 16). ~1 min of CPU per segment, so the results
are committed (c3_expected.json) and the grids regenerated from seeds
(c3_grids.py) at test time. Run in the build container:
    python tests/golden/make_c3_golden.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402
from c3_grids import V, c3_grids, digest  # noqa: E402


def _oracle_nbest(i):
    uid, g = c3_grids()[i]
    r, _ = po.Oracle().decode([g], po.ScorerSpec("uniform", V - 1), po.config(beam_width=10),
                              ids=[uid], nbest=10)
    return r[0]


def main():
    items = c3_grids()
    t0 = time.time()
    res, cnt = po.Ref().decode([g for _, g in items], po.ScorerSpec("uniform", V - 1),
                               po.config(beam_width=10), batch_size=16,
                               ids=[u for u, _ in items], threads=os.cpu_count())
    # n-best: the plain-C restatement's sorted finished set (bit-identical
    # to the reference on the 1-best, checked below); one process per segment
    from multiprocessing import Pool
    with Pool(os.cpu_count()) as pool:
        onb = pool.map(_oracle_nbest, range(len(items)))
    for r, o in zip(res, onb):
        assert (r.tokens, r.label_times, r.steps, r.eos_trigger) == \
            (o.tokens, o.label_times, o.steps, o.eos_trigger) and r.joint_logp == o.joint_logp
    out = {"sha256": digest(items), "config": {"beam_width": 10, "vocab": V},
           "counters": {"steps": cnt[0], "scorer_queries": cnt[1],
                        "ctc_frames_evaluated": cnt[2]},
           "reference_wall_s": time.time() - t0,
           "results": [{"id": r.id, "tokens": r.tokens, "joint_logp": r.joint_logp,
                        "label_times": r.label_times, "steps": r.steps,
                        "eos_trigger": r.eos_trigger,
                        "nbest": [{"tokens": t, "joint_logp": j, "label_times": lt}
                                  for t, j, lt in o.nbest]}
                       for r, o in zip(res, onb)]}
    with open(os.path.join(HERE, "c3_expected.json"), "w") as f:
        json.dump(out, f)
    print("wrote c3_expected.json", out["counters"], "%.0f s" % out["reference_wall_s"])


if __name__ == "__main__":
    main()
