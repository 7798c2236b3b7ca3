import os, sys, time
os.environ["BL_PROFILE"] = "1"
sys.path.insert(0, ".")
import numpy as np
import paper_2101_05600_b200 as bl
names = ["init+Ftab", "P1 window/eos", "P2 phi/PhiF", "P3 bulk(+P4a)", "P4 theta", "P5 collect", "P6 contenders", "P7 rank (fb)", "fallback", "P8 walk (fb)", "P6-P9 overlap", "finalize", "t0:P3 frames", "t0:P3 keys", "t0:P6 serial", "t0:P6 staging"]
rng = np.random.default_rng(1)
CFGS = [(500, 10, 20, 64)]
TENC = 249
if len(sys.argv) > 1:  # V B M2 U [T_enc]  (M2 < 0: no margin)
    CFGS = [tuple(int(x) for x in sys.argv[1:5])]
    if len(sys.argv) > 5:
        TENC = int(sys.argv[5])
for (V, B, M2, U) in CFGS:
    M2 = bl.NO_MARGIN if M2 < 0 else M2
    G = []
    for i in range(U):
        p = rng.exponential(size=(TENC, V)); G.append(np.log(p / p.sum(1, keepdims=True)).astype(np.float32))
    utts = [bl.Utterance(f"b{i}", bl.PosteriorGrid(g)) for i, g in enumerate(G)]
    dec = bl.Decoder(bl.UniformScorer(V - 1), bl.DecoderConfig(beam_width=B, margin_m2=M2))
    for rep in range(2):
        dec.decode(utts)
    st = dec.last_stats
    pc = st["profile_cycles"]; tot = sum(pc[:12])
    print(f"V={V} B={B} M2={M2} U={U} W~{st['ctc_frames_evaluated'] / max(1, st['scorer_queries']) / (V - 1):.1f}: kernel {st['kernel_ms']:.2f} ms, steps/utt {st['steps']/U:.0f}, contenders/step {st['contenders']/st['steps']:.1f}, fallback {st['fallback_steps']}")
    for n, c in zip(names, pc):
        print(f"   {n:16s} {c/1e3:10.1f} kcyc {100*c/tot:5.1f}%  per-step {c/(st['steps']/U):8.0f} cyc")
