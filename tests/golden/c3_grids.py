"""Seeded CTC grids at BASELINE config 3's shape (T_enc = 249 frames of a
10 s segment, vocab 5000 = 4999 tokens + blank), shared by the golden
generator (make_c3_golden.py, runs oracle/_ref here) and the GPU parity test
(tests/test_c3_parity.py). numpy's Generator streams are platform-stable;
the generator script records a sha256 of the float32 bytes so drift fails
loudly instead of comparing different inputs."""
import hashlib

import numpy as np

T, V = 249, 5000


def _norm(logits):
    logits = logits - logits.max(1, keepdims=True)
    p = np.exp(logits)
    return np.log(p / p.sum(1, keepdims=True)).astype(np.float32)


def c3_grids():
    """[(id, grid)]: 8 flat random segments (the bench's posteriors), one
    sharpened x8 (peaky: plateau ties in gamma), one with 32 duplicated
    high-mass token columns (exact ties among hundreds of candidates: the
    contender set overflows and the exact fallback runs)."""
    out = []
    for i in range(8):
        p = np.random.default_rng(5000 + i).exponential(size=(T, V))
        out.append((f"flat{i}", np.log(p / p.sum(1, keepdims=True)).astype(np.float32)))
    z = np.random.default_rng(5100).standard_normal((T, V))
    out.append(("sharp8", _norm(8.0 * z)))
    p = np.random.default_rng(5200).exponential(size=(T, V))
    p[:, 0] *= 3.0
    p[:, 1:32] = p[:, :1]
    out.append(("dupcols", np.log(p / p.sum(1, keepdims=True)).astype(np.float32)))
    return out


def digest(grids):
    h = hashlib.sha256()
    for _, g in grids:
        h.update(np.ascontiguousarray(g, dtype=np.float32).tobytes())
    return h.hexdigest()
