"""Python mirror of the beamlattice decoder API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/beamlattice/*.hpp), so code and tests written
against the reference read the same here. Every call goes through
``libbl_b200.so`` (include/bl_b200.h); decoding runs only on the GPU and the
module raises if the CUDA library is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import struct
from collections.abc import Sequence as _Seq
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BL_LIB", os.path.join(_HERE, "libbl_b200.so"))

NO_MARGIN = 1 << 29  # kNoMargin, ctc_prefix.hpp:12
K_LOG_ZERO = -1e30   # logmath.hpp:11

BL_OK, BL_INVALID_ARGUMENT, BL_RUNTIME_ERROR, BL_LOGIC_ERROR, BL_CUDA_ERROR = range(5)
EOS_MODES = ("baseline", "ctc", "both")
TRIGGERS = ("baseline", "ctc", "max_len")


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class LogicError(RuntimeError):
    """std::logic_error."""


class CudaError(RuntimeError):
    """CUDA failure in the device decoder (no CPU fallback exists)."""


class _Config(C.Structure):
    _fields_ = [("beam_width", C.c_int), ("ctc_weight", C.c_double),
                ("eos_m", C.c_int), ("eos_dend", C.c_double), ("eos_c", C.c_int),
                ("margin_m1", C.c_int), ("margin_m2", C.c_int),
                ("eos_mode", C.c_int), ("max_steps_ratio", C.c_double)]


class _Utt(C.Structure):
    _fields_ = [("id", C.c_char_p), ("num_frames", C.c_uint32),
                ("vocab", C.c_uint32), ("frame_shift_ms", C.c_uint32),
                ("logp", C.c_void_p)]


_lib = None
_UTT_DTYPE = np.dtype([("id", np.uint64), ("num_frames", np.uint32), ("vocab", np.uint32),
                       ("frame_shift_ms", np.uint32), ("pad", np.uint32), ("logp", np.uint64)])
assert _UTT_DTYPE.itemsize == C.sizeof(_Utt)


def lib() -> C.CDLL:
    """Load libbl_b200.so (built by __graft_entry__.build()); fail loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a extension with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.bl_last_error.restype = C.c_char_p
    L.bl_config_default.argtypes = [C.POINTER(_Config)]
    L.bl_config_validate.argtypes = [C.POINTER(_Config)]
    L.bl_hard_segments.argtypes = [C.c_int, C.c_int, C.c_int, ip, ip, C.c_int, ip]
    L.bl_vad_segments.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, C.c_double,
                                  C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, ip]
    L.bl_make_batches.argtypes = [C.c_int, C.POINTER(C.c_uint32), C.c_int, ip, ip]
    L.bl_scorer_create.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
    L.bl_scorer_create_table.argtypes = [C.c_int, C.c_int, C.c_int, ip, ip, dp,
                                         C.POINTER(vp)]
    L.bl_scorer_create_loop.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(vp)]
    L.bl_scorer_num_tokens.argtypes = [vp]
    L.bl_scorer_score.argtypes = [vp, ip, C.c_int, dp]
    L.bl_scorer_destroy.argtypes = [vp]
    L.bl_decoder_create.argtypes = [C.c_int, C.POINTER(_Config), vp, C.POINTER(vp)]
    L.bl_decoder_set_options.argtypes = [vp, C.c_int, C.c_int, C.c_double]
    L.bl_decoder_set_stream.argtypes = [vp, vp]
    L.bl_decoder_set_step_mode.argtypes = [vp, C.c_int]
    L.bl_decoder_set_record.argtypes = [vp, C.c_int]
    L.bl_decoder_record_count.argtypes = [vp]
    L.bl_decoder_record_get.argtypes = [vp, C.c_int, ip, ip, C.POINTER(ip), C.POINTER(dp)]
    L.bl_decoder_destroy.argtypes = [vp]
    L.bl_decode.argtypes = [vp, C.c_int, C.POINTER(_Utt), C.c_int, C.POINTER(vp)]
    L.bl_results_count.argtypes = [vp]
    L.bl_results_get.argtypes = [vp, C.c_int, C.POINTER(C.c_char_p), C.POINTER(ip),
                                 ip, dp, C.POINTER(ip), ip, ip]
    L.bl_results_nbest_count.argtypes = [vp, C.c_int]
    L.bl_results_nbest.argtypes = [vp, C.c_int, C.c_int, C.POINTER(ip), ip, dp,
                                   C.POINTER(ip)]
    u64p = C.POINTER(C.c_uint64)
    L.bl_results_counters.argtypes = [vp, u64p, u64p, u64p]
    L.bl_results_stats.argtypes = [vp, dp, u64p, ip, u64p, u64p]
    L.bl_results_profile.argtypes = [vp, dp]
    L.bl_results_filter_keys.argtypes = [vp, u64p]
    if hasattr(L, "bl_results_wide_steps"):  # (absent in pre-round-2 A/B builds)
        L.bl_results_wide_steps.argtypes = [vp, u64p]
    L.bl_results_transfer.argtypes = [vp, u64p, u64p]
    L.bl_results_max_tokens.argtypes = [vp]
    L.bl_results_export.argtypes = [vp, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]
    L.bl_results_destroy.argtypes = [vp]
    L.bl_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.bl_host_free.argtypes = [vp]
    L.bl_host_free.restype = None
    L.bl_encoder_frames_out.argtypes = [C.c_int]
    L.bl_encoder_num_weights.argtypes = [vp]
    L.bl_encoder_num_weights.restype = C.c_size_t
    L.bl_encoder_create.argtypes = [C.c_int, vp, vp, C.c_size_t, C.POINTER(vp)]
    L.bl_encoder_set_stream.argtypes = [vp, vp]
    L.bl_encoder_set_chunk.argtypes = [vp, C.c_int]
    L.bl_encoder_forward.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int]
    L.bl_encoder_launches.argtypes = [vp]
    L.bl_encoder_destroy.argtypes = [vp]
    L.bl_transformer_num_weights.argtypes = [vp]
    L.bl_transformer_num_weights.restype = C.c_size_t
    L.bl_scorer_create_transformer.argtypes = [C.c_int, vp, vp, C.c_size_t, C.POINTER(vp)]
    L.bl_decode_memory.argtypes = [vp, C.c_int, C.POINTER(_Utt), C.c_int, vp, C.c_int,
                                   C.POINTER(vp)]
    L.bl_decode_into.argtypes = [vp, C.c_int, C.POINTER(_Utt), C.c_int, vp, C.c_int, C.c_int,
                                 vp, vp, vp, vp, vp, vp, C.POINTER(vp)]
    L.bl_encoder_forward_mem.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, C.c_int]
    L.bl_model_save.argtypes = [C.c_char_p, vp, vp, C.c_size_t, vp, vp, C.c_size_t]
    L.bl_encoder_create_from_file.argtypes = [C.c_int, C.c_char_p, C.POINTER(vp)]
    L.bl_recognize.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_int,
                               C.POINTER(vp)]
    L.bl_group_create.argtypes = [C.c_int, ip, C.POINTER(_Config), vp, C.POINTER(vp)]
    L.bl_group_size.argtypes = [vp]
    L.bl_group_set_options.argtypes = [vp, C.c_int, C.c_int, C.c_double]
    L.bl_group_decode.argtypes = [vp, C.c_int, C.POINTER(_Utt), C.POINTER(vp)]
    L.bl_group_destroy.argtypes = [vp]
    L.bl_group_destroy.restype = None
    L.bl_gemm_bf16.argtypes = [C.c_int, C.c_int, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
                               vp, vp, vp, C.c_int, C.c_float, vp, C.c_int, vp]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == BL_OK:
        return
    msg = lib().bl_last_error().decode()
    if rc == BL_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == BL_LOGIC_ERROR:
        raise LogicError(msg)
    if rc == BL_CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(msg)


# ------------------------------------------------------------------ config
@dataclass
class DecoderConfig:
    """beam_search.hpp:21-33 (same defaults)."""
    beam_width: int = 3
    ctc_weight: float = 0.3
    eos_m: int = 3
    eos_dend: float = -10.0
    eos_c: int = 2
    margin_m1: int = 5
    margin_m2: int = NO_MARGIN
    eos_mode: str = "both"
    max_steps_ratio: float = 1.0

    def _c(self) -> _Config:
        if self.eos_mode not in EOS_MODES:
            raise InvalidArgument("unknown eos mode: " + str(self.eos_mode))
        return _Config(self.beam_width, self.ctc_weight, self.eos_m, self.eos_dend,
                       self.eos_c, self.margin_m1, self.margin_m2,
                       EOS_MODES.index(self.eos_mode), self.max_steps_ratio)

    def validate(self) -> None:
        """DecoderConfig::validate (beam_search.cpp:36-46)."""
        c = self._c()
        _check(lib().bl_config_validate(C.byref(c)))


def eos_mode_from_string(s: str) -> str:
    """beam_search.cpp:29-34."""
    if s not in EOS_MODES:
        raise InvalidArgument("unknown eos mode: " + s)
    return s


# -------------------------------------------------------------- data model
@dataclass
class PosteriorGrid:
    """grid.hpp:24-43: T x (|C|+1) float32 log-posteriors, blank last."""
    logp: np.ndarray
    frame_shift_ms: int = 10

    def __post_init__(self):
        self.logp = np.ascontiguousarray(self.logp, dtype=np.float32)
        if self.logp.ndim != 2:
            raise InvalidArgument("grid must be 2-D [T, vocab]")

    @property
    def num_frames(self) -> int:
        return int(self.logp.shape[0])

    @property
    def vocab(self) -> int:
        return int(self.logp.shape[1])

    def num_tokens(self) -> int:
        return self.vocab - 1

    def blank_id(self) -> int:
        return self.vocab - 1

    def at(self, frame: int, symbol: int) -> float:
        """1-based frame, promoted to double (grid.hpp:36-38)."""
        return float(self.logp[frame - 1, symbol])

    def audio_seconds(self) -> float:
        return self.num_frames * self.frame_shift_ms / 1000.0


@dataclass
class Utterance:
    """grid.hpp:50-54."""
    id: str
    grid: PosteriorGrid
    true_frames: int = 0

    def __post_init__(self):
        if not self.true_frames:
            self.true_frames = self.grid.num_frames


@dataclass
class Batch:
    """batched.hpp:13-16."""
    utterances: List[Utterance]
    padded_frames: int = 0


@dataclass
class DecodeResult:
    """beam_search.hpp:35-42, plus the n-best list (new)."""
    id: str
    tokens: List[int]
    joint_logp: float
    label_times: List[int]
    steps_taken: int
    eos_trigger: str
    nbest: List[Tuple[List[int], float, List[int]]] = field(default_factory=list)


@dataclass
class DecodeCounters:
    """beam_search.hpp:68-79."""
    steps: int = 0
    scorer_queries: int = 0
    ctc_frames_evaluated: int = 0

    def __iadd__(self, o: "DecodeCounters") -> "DecodeCounters":
        self.steps += o.steps
        self.scorer_queries += o.scorer_queries
        self.ctc_frames_evaluated += o.ctc_frames_evaluated
        return self


@dataclass
class Segment:
    """segmentation.hpp:45-50."""
    utterance_id: str
    start: int
    end: int
    source: str = "hard"


# -------------------------------------------------------- host path pieces
def make_batches(utterances: Sequence[Utterance], batch_size: int) -> List[Batch]:
    """batched.cpp:12-30 (stable length sort, then chunk)."""
    n = len(utterances)
    frames = (C.c_uint32 * max(n, 1))(*[u.true_frames for u in utterances])
    order = (C.c_int * max(n, 1))()
    nb = C.c_int()
    _check(lib().bl_make_batches(n, frames, batch_size, order, C.byref(nb)))
    out = []
    for k in range(0, n, batch_size):
        us = [utterances[order[i]] for i in range(k, min(n, k + batch_size))]
        out.append(Batch(us, max(u.true_frames for u in us)))
    return out


def hard_segments(num_frames: int, min_len: int, max_len: int,
                  utterance_id: str = "") -> List[Segment]:
    """segmentation.cpp:121-133 (integer-exact)."""
    cap = max(1, num_frames // max(1, max_len) + 2)
    s = (C.c_int * cap)()
    e = (C.c_int * cap)()
    n = C.c_int()
    _check(lib().bl_hard_segments(num_frames, min_len, max_len, s, e, cap,
                                  C.byref(n)))
    return [Segment(utterance_id, s[k], e[k], "hard") for k in range(n.value)]


def vad_segments(outputs, speech_nodes: Sequence[int], noise_nodes: Sequence[int],
                 threshold: float = 0.0, smooth_window: int = 5, min_len: int = 1500,
                 max_len: int = 2000, utterance_id: str = "") -> List[Segment]:
    """VAD segmentation (segmentation.hpp:49-60, VadConfig defaults): raw VAD
    model outputs [T][num_nodes] -> speech segments (source "vad")."""
    o = np.ascontiguousarray(outputs, np.float32)
    if o.ndim != 2:
        raise InvalidArgument("VAD outputs must be [frames, nodes]")
    sp = np.ascontiguousarray(speech_nodes, np.int32)
    no = np.ascontiguousarray(noise_nodes, np.int32)
    cap = o.shape[0] + 1
    st = np.zeros(cap, np.int32)
    en = np.zeros(cap, np.int32)
    n = C.c_int()
    _check(lib().bl_vad_segments(o.ctypes.data, o.shape[0], o.shape[1], sp.ctypes.data, len(sp),
                                 no.ctypes.data, len(no), threshold, smooth_window, min_len,
                                 max_len, st.ctypes.data, en.ctypes.data, cap, C.byref(n)))
    return [Segment(utterance_id, int(st[k]), int(en[k]), "vad") for k in range(n.value)]


# ------------------------------------------------------------------ scorers
class Scorer:
    """Scorer contract (scorer.hpp:16-22), realised as a device scorer."""

    _h: Optional[C.c_void_p] = None

    def num_tokens(self) -> int:
        return lib().bl_scorer_num_tokens(self._h)

    def score(self, utterance_id: str, prefix: Sequence[int]) -> List[float]:
        n = len(prefix)
        arr = (C.c_int * max(n, 1))(*prefix)
        out = (C.c_double * (self.num_tokens() + 1))()
        _check(lib().bl_scorer_score(self._h, arr, n, out))
        return list(out)

    def _key(self):
        return id(self)

    def __del__(self):
        if self._h is not None and _lib is not None:
            _lib.bl_scorer_destroy(self._h)
            self._h = None


class UniformScorer(Scorer):
    def __init__(self, num_tokens: int):
        h = C.c_void_p()
        _check(lib().bl_scorer_create(b"uniform", num_tokens, C.byref(h)))
        self._h = h


class LoopScorer(Scorer):
    def __init__(self, num_tokens: int, loop_token: int, p_loop: float):
        h = C.c_void_p()
        _check(lib().bl_scorer_create_loop(num_tokens, loop_token, p_loop, C.byref(h)))
        self._h = h


class TableScorer(Scorer):
    """n-gram table keyed by the last order-1 tokens (scorer.hpp:38-55)."""

    def __init__(self, num_tokens: int, order: int):
        self._n, self._order = num_tokens, order
        self._entries: Dict[Tuple[int, ...], List[float]] = {}
        self._rebuild()

    def order(self) -> int:
        return self._order

    def add_entry(self, context: Sequence[int], logp: Sequence[float]) -> None:
        new = dict(self._entries)
        new[tuple(int(x) for x in context)] = [float(v) for v in logp]
        old = self._entries
        self._entries = new
        try:
            self._rebuild()
        except Exception:
            self._entries = old
            raise

    def entries(self):
        return dict(self._entries)

    def _rebuild(self):
        ents = list(self._entries.items())
        w = max(self._order - 1, 1)
        n = len(ents)
        V = self._n + 1
        clen = (C.c_int * max(n, 1))()
        ctx = (C.c_int * max(n * w, 1))()
        lp = (C.c_double * max(n * V, 1))()
        for k, (c, v) in enumerate(ents):
            clen[k] = len(c)
            for i, t in enumerate(c[:w]):
                ctx[k * w + i] = t
            if len(v) != V:
                raise RuntimeError("TableScorer entry: wrong vector size")
            for i, x in enumerate(v):
                lp[k * V + i] = x
        h = C.c_void_p()
        _check(lib().bl_scorer_create_table(self._n, self._order, n, clen, ctx, lp,
                                            C.byref(h)))
        if self._h is not None:
            lib().bl_scorer_destroy(self._h)
        self._h = h


class _SpecScorer(Scorer):
    def __init__(self, spec: str, num_tokens: int):
        h = C.c_void_p()
        _check(lib().bl_scorer_create(spec.encode(), num_tokens, C.byref(h)))
        self._h = h
        self.spec_string = spec
        # a network scorer: decoding needs the encoder memory
        self.is_network = spec.startswith("transformer:")


def make_scorer(spec: str, num_tokens: int) -> Scorer:
    """scorer.cpp:117-135: "uniform" | "table:PATH" | "loop:TOKEN:P", plus
    "transformer:PATH[@DEVICE]" (the decoder network of a model file written
    by paper_2101_05600_b200.model.save_model / bl_model_save)."""
    return _SpecScorer(spec, num_tokens)


def save_table_scorer(path: str, scorer: TableScorer) -> None:
    """scorer.cpp:105-115 file schema."""
    j = {"order": scorer.order(), "num_tokens": scorer._n,
         "entries": [{"ctx": list(c), "logp": v}
                     for c, v in sorted(scorer.entries().items())]}
    with open(path, "w") as f:
        f.write(json.dumps(j) + "\n")


class _HostBlock:
    """A page-locked host buffer leased from _HostPool; returns to the pool
    when the last numpy view of it (and the block) is gone."""

    def __init__(self, pool, ptr, nbytes):
        self.pool, self.ptr, self.nbytes = pool, ptr, nbytes

    def array(self, offset, shape, dtype):
        dt = np.dtype(dtype)
        view = _BlockView(self, self.ptr + offset, shape, dt.str)
        return np.asarray(view)

    def __del__(self):
        try:
            self.pool.give(self.ptr, self.nbytes)
        except Exception:  # interpreter shutdown
            pass


class _BlockView:
    def __init__(self, block, addr, shape, typestr):
        self.block = block  # keeps the lease alive while a view exists
        self.__array_interface__ = {"data": (addr, False), "shape": tuple(shape),
                                    "typestr": typestr, "version": 3}


class _HostPool:
    """Page-locked result blocks (bl_host_alloc), reused across decode calls
    by size."""

    def __init__(self):
        self.free = {}

    def take(self, nbytes):
        lst = self.free.get(nbytes)
        if lst:
            return _HostBlock(self, lst.pop(), nbytes)
        p = C.c_void_p()
        _check(lib().bl_host_alloc(nbytes, C.byref(p)))
        return _HostBlock(self, p.value, nbytes)

    def give(self, ptr, nbytes):
        lst = self.free.setdefault(nbytes, [])
        if len(lst) < 4:
            lst.append(ptr)
        else:
            lib().bl_host_free(ptr)


_HOST_POOL = _HostPool()


class ResultSet(_Seq):
    """Results of one decode call as flat arrays (one bulk export from the
    C ABI); indexing materialises DecodeResult objects lazily."""

    def __init__(self, ids, n_tokens, steps, trigger, joint, tokens, label_times, nbest=None):
        self.ids, self.n_tokens, self.steps, self.trigger = ids, n_tokens, steps, trigger
        self.joint, self.tokens, self.label_times = joint, tokens, label_times
        self.nbest = nbest

    def __len__(self):
        return len(self.ids)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        n = int(self.n_tokens[i])
        return DecodeResult(self.ids[i], self.tokens[i, :n].tolist(), float(self.joint[i]),
                            self.label_times[i, :n].tolist(), int(self.steps[i]),
                            TRIGGERS[int(self.trigger[i])],
                            self.nbest[i] if self.nbest is not None else [])

    def __eq__(self, other):
        return list(self) == list(other)


# ------------------------------------------------------------------ decoder
class Decoder:
    """One device decoder (one GPU, one CUDA stream)."""

    def __init__(self, scorer: Scorer, cfg: Optional[DecoderConfig] = None,
                 device: int = 0, nbest: int = 1, exact: bool = False,
                 slack: float = 1.0, step_mode: bool = False):
        self.nbest = nbest
        self._desc_cache = None
        self.cfg = cfg or DecoderConfig()
        self.scorer = scorer
        self.device = device
        c = self.cfg._c()
        h = C.c_void_p()
        _check(lib().bl_decoder_create(device, C.byref(c), scorer._h, C.byref(h)))
        self._h = h
        _check(lib().bl_decoder_set_options(h, nbest, 1 if exact else 0, slack))
        if step_mode:
            _check(lib().bl_decoder_set_step_mode(h, 1))
        self.last_stats: Dict[str, float] = {}

    def set_stream(self, stream_ptr: int) -> None:
        lib().bl_decoder_set_stream(self._h, C.c_void_p(stream_ptr or None))

    def set_record(self, on: bool) -> None:
        """Record the network scorer's rows of every live hypothesis (tests)."""
        _check(lib().bl_decoder_set_record(self._h, 1 if on else 0))

    def records(self):
        """[(utterance index, prefix tuple, float64 row)] of the last decode."""
        L = lib()
        out = []
        u, n = C.c_int(), C.c_int()
        pp, rp = C.POINTER(C.c_int)(), C.POINTER(C.c_double)()
        V = self.scorer.num_tokens() + 1
        for i in range(L.bl_decoder_record_count(self._h)):
            _check(L.bl_decoder_record_get(self._h, i, C.byref(u), C.byref(n), C.byref(pp),
                                           C.byref(rp)))
            pre = tuple(pp[k] for k in range(n.value))
            out.append((u.value, pre, np.ctypeslib.as_array(rp, shape=(V,)).copy()))
        return out

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.bl_decoder_destroy(self._h)
            self._h = None

    def decode_raw(self, descs: Sequence[Tuple[str, int, int, int]],
                   on_device: bool, counters: Optional[DecodeCounters] = None,
                   frame_shift_ms: int = 10, memory: Optional[int] = None,
                   mem_frames: int = 0) -> "ResultSet":
        """descs: (id, num_frames, vocab, data pointer). The bl_utt array is
        built vectorised (one ids buffer, numpy structured records).
        memory: device pointer to the encoder output bf16 [n][mem_frames][d]
        (required by the Transformer scorer)."""
        n = len(descs)
        ids = [d[0] for d in descs]
        # the packed records are reused only when the descriptors are equal in
        # content (ids, frames, vocab, pointers), not merely the same list
        snap = tuple(tuple(d) for d in descs)
        key = (n, frame_shift_ms)
        cached = self._desc_cache
        if cached is not None and cached[0] == key and cached[1] == snap:
            arr = cached[2]
        else:
            blob = b"".join(i.encode() + b"\0" for i in ids)
            buf = C.create_string_buffer(blob, len(blob))
            offs = np.zeros(n, np.int64)
            if n:
                lens = np.fromiter((len(i.encode()) + 1 for i in ids), np.int64, n)
                offs[1:] = np.cumsum(lens)[:-1]
            rec = np.zeros(max(n, 1), dtype=_UTT_DTYPE)
            if n:
                rec["id"][:n] = C.addressof(buf) + offs
                rec["num_frames"][:n] = [d[1] for d in descs]
                rec["vocab"][:n] = [d[2] for d in descs]
                rec["frame_shift_ms"][:n] = frame_shift_ms
                rec["logp"][:n] = [d[3] for d in descs]
            arr = (rec, buf)
            self._desc_cache = (key, snap, arr)
        rec = arr[0]
        h = C.c_void_p()
        if self.nbest == 1 and n > 0:
            # bulk path: 1-best results written straight into numpy arrays
            cap = max(1, int(rec["num_frames"][:n].max()))
            # page-locked, reused result block: the library copies token and
            # label-time rows straight into it (no first-touch page faults)
            blk = _HOST_POOL.take(n * (24 + 8 * cap))
            jt = blk.array(0, (n,), np.float64)
            nt = blk.array(8 * n, (n,), np.int32)
            st = blk.array(12 * n, (n,), np.int32)
            tr = blk.array(16 * n, (n,), np.int32)
            tok = blk.array(24 * n, (n, cap), np.int32)
            lt = blk.array(24 * n + 4 * n * cap, (n, cap), np.int32)
            _check(lib().bl_decode_into(
                self._h, n, rec.ctypes.data_as(C.POINTER(_Utt)), 1 if on_device else 0,
                C.c_void_p(memory) if memory is not None else None, mem_frames, cap,
                nt.ctypes.data, st.ctypes.data, tr.ctypes.data, jt.ctypes.data,
                tok.ctypes.data, lt.ctypes.data, C.byref(h)))
            try:
                self._stats(h, counters)
            finally:
                lib().bl_results_destroy(h)
            return ResultSet(ids, nt, st, tr, jt, tok, lt, None)
        if memory is not None:
            _check(lib().bl_decode_memory(self._h, n, rec.ctypes.data_as(C.POINTER(_Utt)),
                                          1 if on_device else 0, C.c_void_p(memory),
                                          mem_frames, C.byref(h)))
        else:
            _check(lib().bl_decode(self._h, n, rec.ctypes.data_as(C.POINTER(_Utt)),
                                   1 if on_device else 0, C.byref(h)))
        try:
            return self._collect(h, counters, ids)
        finally:
            lib().bl_results_destroy(h)

    def decode(self, utterances: Sequence[Utterance],
               counters: Optional[DecodeCounters] = None) -> List[DecodeResult]:
        keep = [u.grid.logp for u in utterances]
        return self.decode_raw([(u.id, u.grid.num_frames, u.grid.vocab,
                                 g.ctypes.data) for u, g in zip(utterances, keep)],
                               on_device=False, counters=counters)

    def _collect(self, h, counters, ids) -> "ResultSet":
        L = lib()
        n = L.bl_results_count(h)
        cap = max(1, L.bl_results_max_tokens(h))
        nt = np.zeros(n, np.int32)
        st = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        jt = np.zeros(n, np.float64)
        tok = np.zeros((n, cap), np.int32)
        lt = np.zeros((n, cap), np.int32)
        if n:
            _check(L.bl_results_export(h, cap, nt.ctypes.data, st.ctypes.data, tr.ctypes.data,
                                       jt.ctypes.data, tok.ctypes.data, lt.ctypes.data))
        nbest = [] if self.nbest > 1 else None
        ip = C.POINTER(C.c_int)
        for i in range(n if nbest is not None else 0):
            if nbest is not None:
                lst = []
                t_, l_ = ip(), ip()
                m_, j_ = C.c_int(), C.c_double()
                for k in range(L.bl_results_nbest_count(h, i)):
                    _check(L.bl_results_nbest(h, i, k, C.byref(t_), C.byref(m_), C.byref(j_),
                                              C.byref(l_)))
                    lst.append(([t_[q] for q in range(m_.value)], j_.value,
                                [l_[q] for q in range(m_.value)]))
                nbest.append(lst)
        out = ResultSet(ids, nt, st, tr, jt, tok, lt, nbest)
        self._stats(h, counters)
        return out

    def _stats(self, h, counters) -> None:
        L = lib()
        s, q, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        L.bl_results_counters(h, C.byref(s), C.byref(q), C.byref(f))
        if counters is not None:
            counters += DecodeCounters(s.value, q.value, f.value)
        ms, k1, fb, nc = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        nl = C.c_int()
        L.bl_results_stats(h, C.byref(ms), C.byref(k1), C.byref(nl), C.byref(fb),
                           C.byref(nc))
        self.last_stats = {"kernel_ms": ms.value, "k1_bytes": k1.value,
                           "launches": nl.value, "fallback_steps": fb.value,
                           "contenders": nc.value, "steps": s.value,
                           "scorer_queries": q.value, "ctc_frames_evaluated": f.value}
        h2d, d2h = C.c_uint64(), C.c_uint64()
        L.bl_results_transfer(h, C.byref(h2d), C.byref(d2h))
        self.last_stats["h2d_bytes"] = h2d.value
        self.last_stats["d2h_bytes"] = d2h.value
        rk = C.c_uint64()
        L.bl_results_filter_keys(h, C.byref(rk))
        self.last_stats["filter_keys"] = rk.value
        if hasattr(L, "bl_results_wide_steps"):
            L.bl_results_wide_steps(h, C.byref(rk))
            self.last_stats["wide_steps"] = rk.value
        if os.environ.get("BL_PROFILE"):
            prof = (C.c_double * 16)()
            L.bl_results_profile(h, prof)
            self.last_stats["profile_cycles"] = [round(x) for x in prof]


class Group:
    """Several GPUs of one process (bl_group_*): segments sharded
    contiguously over `devices`, decoded concurrently with no per-step
    exchange, result records (1-best + n-best) gathered to the first device
    by one NCCL group, results in input order."""

    _collect = Decoder._collect
    _stats = Decoder._stats

    def __init__(self, scorer: Scorer, cfg: Optional[DecoderConfig] = None,
                 devices: Sequence[int] = (0,), nbest: int = 1, exact: bool = False,
                 slack: float = 1.0):
        self.nbest = nbest
        self.cfg = cfg or DecoderConfig()
        self.scorer = scorer
        self.devices = list(devices)
        dv = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _check(lib().bl_group_create(len(self.devices), dv, C.byref(self.cfg._c()),
                                     scorer._h, C.byref(h)))
        self._h = h
        _check(lib().bl_group_set_options(h, nbest, 1 if exact else 0, slack))
        self.last_stats: Dict[str, float] = {}

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.bl_group_destroy(self._h)
            self._h = None

    def decode(self, utterances: Sequence[Utterance],
               counters: Optional[DecodeCounters] = None) -> "ResultSet":
        keep = [u.grid.logp for u in utterances]
        n = len(utterances)
        ids = [u.id for u in utterances]
        arr = (_Utt * max(n, 1))()
        for i, (u, g) in enumerate(zip(utterances, keep)):
            arr[i] = _Utt(ids[i].encode(), u.grid.num_frames, u.grid.vocab,
                          u.grid.frame_shift_ms, g.ctypes.data)
        h = C.c_void_p()
        _check(lib().bl_group_decode(self._h, n, arr, C.byref(h)))
        try:
            return self._collect(h, counters, ids)
        finally:
            lib().bl_results_destroy(h)


_decoders: Dict[tuple, Decoder] = {}


def _decoder_for(scorer: Scorer, cfg: DecoderConfig, device: int = 0) -> Decoder:
    key = (scorer._key(), tuple(vars(cfg).values()), device)
    d = _decoders.get(key)
    if d is None or d.scorer is not scorer:
        d = Decoder(scorer, cfg, device)
        _decoders[key] = d
    return d


def batched_beam_search(batch: Batch, scorer: Scorer, cfg: DecoderConfig,
                        counters: Optional[DecodeCounters] = None,
                        device: int = 0) -> List[DecodeResult]:
    """batched.hpp:34-38: results in batch order."""
    cfg.validate()
    if not batch.utterances:
        return []
    return _decoder_for(scorer, cfg, device).decode(batch.utterances, counters)


def beam_search(utt: Utterance, scorer: Scorer, cfg: DecoderConfig,
                counters: Optional[DecodeCounters] = None,
                device: int = 0) -> DecodeResult:
    """beam_search.hpp:109-111 (a one-utterance batch is exactly Alg. 1)."""
    return batched_beam_search(Batch([utt], utt.true_frames), scorer, cfg,
                               counters, device)[0]


# ---------------------------------------------------------------------- I/O
def write_grid(path: str, grid: PosteriorGrid) -> None:
    """CTCG v1 (grid.cpp:94-106)."""
    with open(path, "wb") as f:
        f.write(b"CTCG" + struct.pack("<IIII", 1, grid.num_frames, grid.vocab,
                                      grid.frame_shift_ms))
        f.write(grid.logp.astype("<f4").tobytes())


def read_grid(path: str) -> PosteriorGrid:
    """CTCG v1 (grid.cpp:108-127), same error messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError("cannot open grid file: " + path)
    with f:
        magic = f.read(4)
        if magic != b"CTCG":
            raise RuntimeError("bad magic in grid file: " + path)
        hdr = f.read(16)
        if len(hdr) < 4 or struct.unpack("<I", hdr[:4])[0] != 1:
            raise RuntimeError("unsupported grid version in " + path)
        _, T, V, fs = struct.unpack("<IIII", hdr)
        data = f.read(4 * T * V)
        if len(data) != 4 * T * V:
            raise RuntimeError("truncated grid file: " + path)
    return PosteriorGrid(np.frombuffer(data, "<f4").reshape(T, V).copy(), fs)


def _grisu_cached_powers():
    """10^k, k = -300, -292, ..., 324: round-to-nearest 64-bit significands
    (the cached-power table of Grisu2 as nlohmann::json uses it)."""
    from fractions import Fraction
    out = []
    for k in range(-300, 325, 8):
        x = Fraction(10) ** k
        e = x.numerator.bit_length() - x.denominator.bit_length() - 64
        while x / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while x / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = x / Fraction(2) ** e
        f = int(q) + (1 if q - int(q) >= Fraction(1, 2) else 0)
        out.append((f, e, k))
    return out


_GRISU_POW = None
_M64 = (1 << 64) - 1


def _grisu_mul(xf, xe, yf, ye):
    ul, uh, vl, vh = xf & 0xFFFFFFFF, xf >> 32, yf & 0xFFFFFFFF, yf >> 32
    p0, p1, p2, p3 = ul * vl, ul * vh, uh * vl, uh * vh
    q = (p0 >> 32) + (p1 & 0xFFFFFFFF) + (p2 & 0xFFFFFFFF) + (1 << 31)
    return (p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32)) & _M64, xe + ye + 64


def _grisu_digits(v: float):
    """Grisu2 digits of v > 0 (Loitsch 2010) with nlohmann::json's boundary,
    cached-power and rounding choices: v = int(digits) * 10**dec. Mirrors
    include/beamlattice/b200.hpp grisu::digits."""
    global _GRISU_POW
    if _GRISU_POW is None:
        _GRISU_POW = _grisu_cached_powers()
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52 & 0x7FF, bits & ((1 << 52) - 1)
    vf, ve = (F, 1 - 1075) if E == 0 else (F + (1 << 52), E - 1075)
    mpf, mpe = 2 * vf + 1, ve - 1
    mmf, mme = (4 * vf - 1, ve - 2) if (F == 0 and E > 1) else (2 * vf - 1, ve - 1)
    sh = 64 - mpf.bit_length()
    wpf, wpe = mpf << sh, mpe - sh
    wmf, wme = mmf << (mme - wpe), wpe
    sh = 64 - vf.bit_length()
    wf, we = vf << sh, ve - sh
    f = -60 - wpe - 1
    k = abs(f * 78913) >> 18
    k = (-k if f < 0 else k) + (1 if f > 0 else 0)
    cf, ce, ck = _GRISU_POW[(300 + k + 7) // 8]
    w = _grisu_mul(wf, we, cf, ce)
    mm = _grisu_mul(wmf, wme, cf, ce)
    mp = _grisu_mul(wpf, wpe, cf, ce)
    mmf_, mpf_, sh = mm[0] + 1, mp[0] - 1, -mp[1]
    dec = -ck
    delta, dist = (mpf_ - mmf_) & _M64, (mpf_ - w[0]) & _M64
    one = 1 << sh
    p1, p2 = mpf_ >> sh, mpf_ & (one - 1)
    n = max(1, len(str(p1)))
    pow10 = 10 ** (n - 1)
    buf = []

    def rnd(dist, delta, rest, ten):
        while rest < dist and delta - rest >= ten and \
                (rest + ten < dist or dist - rest > rest + ten - dist):
            buf[-1] -= 1
            rest += ten

    while n > 0:
        d, p1 = divmod(p1, pow10)
        buf.append(d)
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            rnd(dist, delta, rest, pow10 << sh)
            return "".join(map(str, buf)), dec + n
        pow10 //= 10
    m = 0
    while True:
        p2 = (p2 * 10) & _M64
        buf.append(p2 >> sh)
        p2 &= one - 1
        m += 1
        delta, dist = (delta * 10) & _M64, (dist * 10) & _M64
        if p2 <= delta:
            break
    rnd(dist, delta, p2, one)
    return "".join(map(str, buf)), dec - m


def json_double(v: float) -> str:
    """nlohmann::json's number format (the reference writer, io.cpp:81-92):
    Grisu2 digits, fixed notation while the decimal point falls in (-4, 15],
    else d.ddde+XX with at least two exponent digits; non-finite -> null."""
    v = float(v)
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    digits, dec = _grisu_digits(abs(v))
    k = len(digits)
    n = k + dec
    if k <= n <= 15:
        o = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        o = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        o = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        o = digits[0] + ("." + digits[1:] if k > 1 else "") + ("e-" if e < 0 else "e+") \
            + "%02d" % abs(e)
    return ("-" if v < 0 else "") + o


def _json_ints(v) -> str:
    return "[" + ",".join(str(int(x)) for x in v) + "]"


def result_json(r: DecodeResult) -> str:
    """io.cpp:81-92 line as nlohmann::json dumps it: keys sorted, raw UTF-8
    strings, nlohmann's number format (json_double)."""
    parts = ['"eos_trigger":' + json.dumps(r.eos_trigger, ensure_ascii=False),
             '"id":' + json.dumps(r.id, ensure_ascii=False),
             '"joint_logp":' + json_double(r.joint_logp),
             '"label_times":' + _json_ints(r.label_times)]
    if r.nbest and len(r.nbest) > 1:
        parts.append('"nbest":[' + ",".join(
            '{"joint_logp":%s,"label_times":%s,"tokens":%s}'
            % (json_double(j), _json_ints(lt), _json_ints(t)) for t, j, lt in r.nbest) + "]")
    parts += ['"steps":%d' % int(r.steps_taken), '"tokens":' + _json_ints(r.tokens)]
    return "{" + ",".join(parts) + "}"


def write_results(fp, results: Iterable[DecodeResult]) -> None:
    for r in results:
        fp.write(result_json(r) + "\n")
