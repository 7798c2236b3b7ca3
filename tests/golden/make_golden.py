"""Generates the golden fixtures in tests/golden/ by RUNNING the compiled
reference (oracle/_ref/libblref.so, built from /root/reference/proj by
oracle/Makefile). Grids come from the reference's own generators
(random_grid / synth_corpus use libstdc++ distributions, so they are not
re-derived in Python) and expected results from its batched_beam_search /
beam_search. Run in the build container: python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402

NO = po.NO_MARGIN


def res_json(rs):
    return [{"id": r.id, "tokens": r.tokens, "joint_logp": r.joint_logp,
             "label_times": r.label_times, "steps": r.steps,
             "eos_trigger": r.eos_trigger} for r in rs]


def main():
    ref = po.Ref()
    corpora = {
        # acceptance.cpp:59-72 random_corpus(5, ., 10, 60, 3) (subset)
        "random3": ref.random_corpus(5, 24, 10, 60, 3),
        # test_batched.cpp:13-25 mixed_corpus(101, 20)
        "mixed": ref.random_corpus(101, 20, 10, 60, 3),
        # acceptance.cpp:202-234 planted T=500 (subset)
        "planted500": ref.synth_corpus(7, 6, 500, 500, 5, "planted"),
        # flat V=500 segments, bench-shaped but short
        "flat500": ref.random_corpus(17, 3, 60, 80, 499),
    }
    cases = [
        ("random3", "uniform3", {}, 16),
        ("random3", "uniform3", {"margin_m1": NO, "margin_m2": NO}, 4),
        ("random3", "uniform3", {"margin_m2": 3, "beam_width": 5}, 16),
        ("random3", "uniform3", {"ctc_weight": 1.0}, 16),
        ("random3", "uniform3", {"ctc_weight": 0.0}, 16),
        ("random3", "uniform3", {"eos_mode": "ctc", "beam_width": 4}, 16),
        ("random3", "uniform3", {"eos_mode": "baseline"}, 1),
        ("mixed", "uniform3", {}, 4),
        ("planted500", "uniform5", {"margin_m1": 5, "margin_m2": 20}, 16),
        ("flat500", "uniform499", {"beam_width": 10, "margin_m2": 20}, 8),
    ]
    scorers = {"uniform3": po.ScorerSpec("uniform", 3),
               "uniform5": po.ScorerSpec("uniform", 5),
               "uniform499": po.ScorerSpec("uniform", 499)}
    arrays = {}
    for name, corp in corpora.items():
        for i, (uid, g) in enumerate(corp):
            arrays[f"{name}/{uid}"] = g
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **arrays)
    out = {"corpora": {k: [u for u, _ in v] for k, v in corpora.items()}, "cases": []}
    for corp, sc, kw, bs in cases:
        ids = [u for u, _ in corpora[corp]]
        grids = [g for _, g in corpora[corp]]
        rs, cnt = ref.decode(grids, scorers[sc], po.config(**kw), batch_size=bs, ids=ids)
        out["cases"].append({"corpus": corp, "scorer": sc, "config": kw,
                             "batch_size": bs, "counters": list(cnt),
                             "results": res_json(rs)})
    # known-answer hard segmentation (test_segmentation.cpp:100-121) + the
    # 8 h recording at 10 ms frames into 10 s pieces
    segs = {}
    for T, lo, hi in [(4000, 1900, 2000), (6500, 1900, 2000), (700, 1900, 2000),
                      (2880000, 1000, 1000), (12345, 1500, 2000), (1, 1, 1)]:
        segs[f"{T},{lo},{hi}"] = ref.hard_segments(T, lo, hi)
    out["hard_segments"] = segs
    # chained prefix scores on the G1 fixture and random grids
    g1 = np.log(np.array([[0.6, 0.4], [0.5, 0.5]])).astype(np.float32)
    arrays_chain = {"g1": g1}
    chains = {"g1": ref.chain_prefix(g1, [0])}
    for k, (uid, g) in enumerate(corpora["random3"][:4]):
        pre = [int(x) for x in np.random.default_rng(k).integers(0, 3, size=4)]
        chains[f"random3/{uid}"] = ref.chain_prefix(g, pre) + (pre,)
    out["chains"] = {k: {"psi": v[0], "tau": v[1], "tau_tilde": v[2], "eos_ext": v[3],
                         "prefix": (v[4] if len(v) > 4 else [0])}
                     for k, v in chains.items()}
    np.savez_compressed(os.path.join(HERE, "chain_grids.npz"), **arrays_chain)
    with open(os.path.join(HERE, "expected.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
