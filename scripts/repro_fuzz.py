"""Re-run one tests/test_gpu_fuzz.py case by index (debugging aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import pyoracle as po
import paper_2101_05600_b200 as bl
import test_gpu_fuzz as f
ref = po.Ref()
for k in [int(x) for x in sys.argv[1:]]:
    items, kw, spec, sc, mode = f._case(k, ref)
    want, wc = ref.decode([g for _, g in items], spec, po.config(**kw), ids=[u for u, _ in items])
    dec = bl.Decoder(sc, bl.DecoderConfig(**kw), exact=mode == "exact", step_mode=mode == "step")
    try:
        got = dec.decode([bl.Utterance(u, bl.PosteriorGrid(g)) for u, g in items])
        ok = all(g.tokens == w.tokens and g.steps_taken == w.steps for g, w in zip(got, want))
        print(k, mode, kw["beam_width"], "ok" if ok else "MISMATCH", flush=True)
    except Exception as e:
        print(k, mode, kw["beam_width"], "ERROR", str(e)[:120], flush=True)
        break
