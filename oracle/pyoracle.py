"""pyoracle.py — TEST INFRASTRUCTURE ONLY.

ctypes bindings to the two CPU checkers (see oracle/oracle.h):
  * ``Oracle``  -> oracle/liboracle.so, the plain-C restatement;
  * ``Ref``     -> oracle/_ref/libblref.so, the unmodified reference compiled
                   in place (absent when the reference could not be built).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NO_MARGIN = 1 << 29


class OrcConfig(C.Structure):
    _fields_ = [("beam_width", C.c_int), ("ctc_weight", C.c_double),
                ("eos_m", C.c_int), ("eos_dend", C.c_double), ("eos_c", C.c_int),
                ("margin_m1", C.c_int), ("margin_m2", C.c_int),
                ("eos_mode", C.c_int), ("max_steps_ratio", C.c_double)]


class OrcScorer(C.Structure):
    _fields_ = [("kind", C.c_int), ("num_tokens", C.c_int), ("order", C.c_int),
                ("n_entries", C.c_int), ("ctx_len", C.POINTER(C.c_int)),
                ("ctx", C.POINTER(C.c_int)), ("logp", C.POINTER(C.c_double)),
                ("loop_token", C.c_int), ("p_loop", C.c_double),
                ("ent_utt", C.POINTER(C.c_int)), ("replay_ids", C.POINTER(C.c_char_p))]


class OrcCounters(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("scorer_queries", C.c_uint64),
                ("ctc_frames_evaluated", C.c_uint64)]


class OrcResult(C.Structure):
    _fields_ = [("n_tokens", C.c_int), ("tokens", C.POINTER(C.c_int)),
                ("label_times", C.POINTER(C.c_int)), ("joint_logp", C.c_double),
                ("steps", C.c_int), ("eos_trigger", C.c_int)]


TRIGGERS = ("baseline", "ctc", "max_len")
EOS_MODES = {"baseline": 0, "ctc": 1, "both": 2}


@dataclass
class Result:
    id: str
    tokens: List[int]
    joint_logp: float
    label_times: List[int]
    steps: int
    eos_trigger: str
    nbest: list = field(default_factory=list)


@dataclass
class ScorerSpec:
    """kind: 'uniform' | 'table' | 'loop' (scorer.hpp:24-70)."""
    kind: str
    num_tokens: int
    order: int = 1
    entries: list = field(default_factory=list)  # [(ctx tuple, logp list)]
    loop_token: int = 0
    p_loop: float = 0.9
    replay_ids: list = field(default_factory=list)  # replay: entries are (utt, ctx, logp)


def config(beam_width=3, ctc_weight=0.3, eos_m=3, eos_dend=-10.0, eos_c=2,
           margin_m1=5, margin_m2=NO_MARGIN, eos_mode="both",
           max_steps_ratio=1.0) -> OrcConfig:
    """DecoderConfig defaults (beam_search.hpp:21-33)."""
    return OrcConfig(beam_width, ctc_weight, eos_m, eos_dend, eos_c, margin_m1,
                     margin_m2, EOS_MODES[eos_mode] if isinstance(eos_mode, str)
                     else eos_mode, max_steps_ratio)


class _ScorerC:
    def __init__(self, spec: ScorerSpec):
        kind = {"uniform": 0, "table": 1, "loop": 2, "replay": 3}[spec.kind]
        replay = kind == 3
        ents = spec.entries
        order = spec.order
        if replay:   # (utt index, full prefix, row): order covers the longest prefix
            order = max([len(c) for _, c, _ in ents] + [0]) + 1
        w = max(order - 1, 1)
        n = len(ents)
        V = spec.num_tokens + 1
        self.ctx_len = (C.c_int * max(n, 1))()
        self.ctx = (C.c_int * max(n * w, 1))()
        self.logp = np.zeros(max(n * V, 1), np.float64)
        self.ent_utt = (C.c_int * max(n, 1))()
        for k, e in enumerate(ents):
            if replay:
                self.ent_utt[k] = int(e[0])
                ctx, lp = e[1], e[2]
            else:
                ctx, lp = e
            self.ctx_len[k] = len(ctx)
            for i, t in enumerate(ctx):
                self.ctx[k * w + i] = int(t)
            self.logp[k * V:(k + 1) * V] = np.asarray(lp, np.float64)
        self.ids = (C.c_char_p * max(len(spec.replay_ids), 1))(
            *[i.encode() for i in spec.replay_ids])
        self.s = OrcScorer(kind, spec.num_tokens, order, n, self.ctx_len, self.ctx,
                           self.logp.ctypes.data_as(C.POINTER(C.c_double)), spec.loop_token,
                           spec.p_loop, self.ent_utt, self.ids)


def _grid_ptrs(grids: Sequence[np.ndarray]):
    arrs = [np.ascontiguousarray(g, dtype=np.float32) for g in grids]
    ptrs = (C.POINTER(C.c_float) * max(len(arrs), 1))()
    for i, a in enumerate(arrs):
        ptrs[i] = a.ctypes.data_as(C.POINTER(C.c_float))
    frames = (C.c_int * max(len(arrs), 1))(*[a.shape[0] for a in arrs])
    return arrs, ptrs, frames


def _collect(lib, prefix, h, ids, nbest=0):
    out = []
    n = getattr(lib, prefix + "results_count")(h)
    for i in range(n):
        r = OrcResult()
        getattr(lib, prefix + "results_get")(h, i, C.byref(r))
        res = Result(ids[i], [r.tokens[k] for k in range(r.n_tokens)],
                     r.joint_logp,
                     [r.label_times[k] for k in range(r.n_tokens)],
                     r.steps, TRIGGERS[r.eos_trigger])
        if nbest:
            # the finished set, (joint desc, insertion asc): [(tokens, joint, label_times)]
            res.nbest = []
            nf = lib.orc_results_nbest(h, i, -1, C.byref(r))
            for k in range(min(nf, nbest)):
                lib.orc_results_nbest(h, i, k, C.byref(r))
                res.nbest.append(([r.tokens[q] for q in range(r.n_tokens)], r.joint_logp,
                                  [r.label_times[q] for q in range(r.n_tokens)]))
        out.append(res)
    getattr(lib, prefix + "results_free")(h)
    return out


def build(quiet: bool = True) -> None:
    """Build liboracle.so always and _ref/ when the reference tree exists."""
    targets = ["liboracle.so"]
    if os.path.isdir(os.environ.get("REF", "/root/reference/proj")):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class Oracle:
    """The plain-C restatement (oracle/ctc_oracle.c)."""

    def __init__(self, path: Optional[str] = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_decode.restype = C.c_void_p
        L.orc_decode.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int,
                                 C.POINTER(C.POINTER(C.c_float)),
                                 C.POINTER(OrcScorer), C.POINTER(OrcConfig),
                                 C.c_int, C.POINTER(OrcCounters), C.c_char_p,
                                 C.c_int]
        for n in ("orc_results_count", "orc_results_free"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.orc_results_get.argtypes = [C.c_void_p, C.c_int, C.POINTER(OrcResult)]
        L.orc_log_add.restype = C.c_double
        L.orc_log_add.argtypes = [C.c_double, C.c_double]
        L.orc_mix_joint.restype = C.c_double
        L.orc_mix_joint.argtypes = [C.c_double, C.c_double, C.c_double]
        L.orc_hard_segments.argtypes = [C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.c_int]
        L.orc_make_batches.argtypes = [C.c_int, C.POINTER(C.c_uint32), C.c_int,
                                       C.POINTER(C.c_int)]
        L.orc_results_nbest.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(OrcResult)]

    def decode(self, grids, scorer: ScorerSpec, cfg: OrcConfig, batched=True,
               ids=None, nbest=0):
        """nbest > 0: each Result also carries the first `nbest` entries of
        the finished set in (joint desc, insertion asc) order."""
        ids = ids or [f"u{i}" for i in range(len(grids))]
        arrs, ptrs, frames = _grid_ptrs(grids)
        V = arrs[0].shape[1]
        sc = _ScorerC(scorer)
        cnt = OrcCounters()
        err = C.create_string_buffer(512)
        h = self.lib.orc_decode(len(arrs), frames, V, ptrs, C.byref(sc.s),
                                C.byref(cfg), 1 if batched else 0,
                                C.byref(cnt), err, 512)
        if not h:
            raise ValueError(err.value.decode())
        return _collect(self.lib, "orc_", h, ids, nbest), (cnt.steps, cnt.scorer_queries,
                                                     cnt.ctc_frames_evaluated)

    def hard_segments(self, T, min_len, max_len):
        cap = max(1, T // max(1, max_len) + 2)
        s = (C.c_int * cap)()
        e = (C.c_int * cap)()
        n = self.lib.orc_hard_segments(T, min_len, max_len, s, e, cap)
        if n < 0:
            raise ValueError("hard_segments: invalid arguments")
        return [(s[k], e[k]) for k in range(n)]

    def make_batches(self, frames, batch_size):
        n = len(frames)
        fr = (C.c_uint32 * max(n, 1))(*frames)
        order = (C.c_int * max(n, 1))()
        nb = self.lib.orc_make_batches(n, fr, batch_size, order)
        if nb < 0:
            raise ValueError("batch size must be >= 1")
        o = [order[i] for i in range(n)]
        return [o[k:k + batch_size] for k in range(0, n, batch_size)]


class Ref:
    """The unmodified reference compiled in place (oracle/_ref/libblref.so)."""

    PATH = os.path.join(HERE, "_ref", "libblref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(self.PATH)
        self.lib = C.CDLL(self.PATH)
        L = self.lib
        L.ref_synth_corpus.restype = C.c_void_p
        L.ref_synth_corpus.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_char_p, C.c_double,
                                       C.c_uint32]
        L.ref_random_corpus.restype = C.c_void_p
        L.ref_random_corpus.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int,
                                        C.c_int]
        for n in ("ref_corpus_count", "ref_corpus_free"):
            getattr(L, n).argtypes = [C.c_void_p]
        for n in ("ref_corpus_frames", "ref_corpus_vocab"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_int]
        L.ref_corpus_logp.restype = C.POINTER(C.c_float)
        L.ref_corpus_logp.argtypes = [C.c_void_p, C.c_int]
        L.ref_corpus_id.restype = C.c_char_p
        L.ref_corpus_id.argtypes = [C.c_void_p, C.c_int]
        L.ref_decode.restype = C.c_void_p
        L.ref_decode.argtypes = [C.c_int, C.POINTER(C.c_char_p),
                                 C.POINTER(C.c_int), C.c_int,
                                 C.POINTER(C.POINTER(C.c_float)),
                                 C.POINTER(OrcScorer), C.POINTER(OrcConfig),
                                 C.c_int, C.c_int, C.POINTER(OrcCounters),
                                 C.c_char_p, C.c_int]
        for n in ("ref_results_count", "ref_results_free"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.ref_results_get.argtypes = [C.c_void_p, C.c_int, C.POINTER(OrcResult)]
        L.ref_hard_segments.argtypes = [C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.c_int]
        L.ref_chain_prefix.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_float),
                                       C.c_int, C.POINTER(C.c_int), C.c_int,
                                       C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_double)]
        L.ref_verify.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int,
                                 C.c_uint64]
        L.ref_vad_segments.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int,
                                       C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_char_p,
                                       C.c_int]
        L.ref_replay_misses.restype = C.c_longlong
        L.ref_replay_misses.argtypes = [C.c_int]
        L.ref_result_json.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_int, C.c_double,
                                      C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                                      C.c_char_p, C.c_int]

    def result_json(self, id, tokens, joint, label_times, steps, trigger) -> str:
        """One line of the reference's write_results (io.cpp:81-92), no newline."""
        tok = (C.c_int * max(1, len(tokens)))(*tokens)
        lt = (C.c_int * max(1, len(label_times)))(*label_times)
        buf = C.create_string_buffer(1 << 16)
        n = self.lib.ref_result_json(id.encode(), tok, len(tokens), joint, lt,
                                     len(label_times), steps, TRIGGERS.index(trigger), buf,
                                     len(buf))
        assert n >= 0
        return buf.raw[:n].decode().rstrip("\n")

    def _corpus(self, h):
        out = []
        for i in range(self.lib.ref_corpus_count(h)):
            T = self.lib.ref_corpus_frames(h, i)
            V = self.lib.ref_corpus_vocab(h, i)
            p = self.lib.ref_corpus_logp(h, i)
            g = np.ctypeslib.as_array(p, shape=(T * V,)).reshape(T, V).copy()
            out.append((self.lib.ref_corpus_id(h, i).decode(), g))
        self.lib.ref_corpus_free(h)
        return out

    def synth_corpus(self, seed, num_utts, t_min, t_max, num_tokens,
                     style="random", blank_mass=0.9, frame_shift_ms=10):
        """synth_corpus (synth.cpp:151-157) -> [(id, grid[T,V])]."""
        return self._corpus(self.lib.ref_synth_corpus(
            seed, num_utts, t_min, t_max, num_tokens, style.encode(),
            blank_mass, frame_shift_ms))

    def random_corpus(self, seed, n, t_lo, t_hi, num_tokens):
        """acceptance.cpp:59-72 corpus -> [(id, grid[T,V])]."""
        return self._corpus(self.lib.ref_random_corpus(seed, n, t_lo, t_hi,
                                                       num_tokens))

    def decode(self, grids, scorer: ScorerSpec, cfg: OrcConfig, batch_size=16,
               ids=None, threads=0):
        ids = ids or [f"u{i}" for i in range(len(grids))]
        arrs, ptrs, frames = _grid_ptrs(grids)
        V = arrs[0].shape[1]
        sc = _ScorerC(scorer)
        cids = (C.c_char_p * max(len(ids), 1))(*[i.encode() for i in ids])
        cnt = OrcCounters()
        err = C.create_string_buffer(512)
        h = self.lib.ref_decode(len(arrs), cids, frames, V, ptrs, C.byref(sc.s),
                                C.byref(cfg), batch_size, threads, C.byref(cnt),
                                err, 512)
        if not h:
            raise ValueError(err.value.decode())
        return _collect(self.lib, "ref_", h, ids), (cnt.steps, cnt.scorer_queries,
                                                     cnt.ctc_frames_evaluated)

    def vad_segments(self, outputs, speech, noise, threshold, smooth_window, min_len,
                     max_len):
        """segmentation.cpp frame_llr -> smooth_and_decide -> vad_segments."""
        o = np.ascontiguousarray(outputs, np.float32)
        sp = np.asarray(speech, np.int32)
        no = np.asarray(noise, np.int32)
        cap = o.shape[0] + 1
        st = np.zeros(cap, np.int32)
        en = np.zeros(cap, np.int32)
        err = C.create_string_buffer(512)
        n = self.lib.ref_vad_segments(o.ctypes.data, o.shape[0], o.shape[1], sp.ctypes.data,
                                      len(sp), no.ctypes.data, len(no), threshold,
                                      smooth_window, min_len, max_len, st.ctypes.data,
                                      en.ctypes.data, cap, err, 512)
        if n < 0:
            raise ValueError(err.value.decode())
        return list(zip(st[:n].tolist(), en[:n].tolist()))

    def replay_misses(self, reset=True) -> int:
        """Queries the replay scorer could not answer since the last reset."""
        return int(self.lib.ref_replay_misses(1 if reset else 0))

    def hard_segments(self, T, min_len, max_len):
        cap = max(1, T // max(1, max_len) + 2)
        s = (C.c_int * cap)()
        e = (C.c_int * cap)()
        n = self.lib.ref_hard_segments(T, min_len, max_len, s, e, cap)
        if n < 0:
            raise ValueError("hard_segments: invalid arguments")
        return [(s[k], e[k]) for k in range(n)]

    def chain_prefix(self, grid, prefix, s=0, e=0):
        g = np.ascontiguousarray(grid, dtype=np.float32)
        T, V = g.shape
        n = len(prefix)
        pre = (C.c_int * max(n, 1))(*prefix)
        psi = (C.c_double * max(n, 1))()
        tau = (C.c_int * max(n, 1))()
        taut = (C.c_int * max(n, 1))()
        eos = (C.c_double * (n + 1))()
        rc = self.lib.ref_chain_prefix(T, V, g.ctypes.data_as(C.POINTER(C.c_float)),
                                       n, pre, s, e, psi, tau, taut, eos)
        if rc != 0:
            raise ValueError("ref_chain_prefix failed")
        return list(psi), list(tau), list(taut), list(eos)

    def verify(self, suite, trials, max_frames=6, max_vocab=3, seed=1):
        return self.lib.ref_verify(suite.encode(), trials, max_frames, max_vocab,
                                   seed)
