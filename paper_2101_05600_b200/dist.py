"""Multi-GPU plumbing: segments shard across ranks with no per-step
collective; the only exchange is the final gather of fixed-size result
records to rank 0 (NCCL over NVLink on GPUs, gloo in the CPU tests).

The reference has no distributed execution; this is the
B200 build's data-parallel layer over independent segments.
"""
from __future__ import annotations

import struct
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .api import TRIGGERS, DecodeResult, ResultSet

HDR = 6  # n_tokens, steps, trigger, joint (2 x int32 bit pattern), n-best count
NB_HDR = 3  # per n-best entry: n_tokens, joint (2 x int32)


def shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced shard [start, end) of n segments for `rank`."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def record_width(max_tokens: int, nbest: int = 1) -> int:
    """int32 words per segment record: the 1-best, then `nbest` n-best
    entries (the finished set in (joint desc, insertion asc) order) when
    nbest > 1."""
    k = nbest if nbest > 1 else 0
    return HDR + 2 * max_tokens + k * (NB_HDR + 2 * max_tokens)


def _joint_words(x: float):
    return struct.unpack("<ii", struct.pack("<d", x))


def pack_results(results: Sequence[DecodeResult], max_tokens: int,
                 rows: Optional[int] = None, nbest: int = 1) -> np.ndarray:
    """Fixed-size int32 records (padded to `rows`): the gather payload."""
    rows = len(results) if rows is None else rows
    L, K = max_tokens, (nbest if nbest > 1 else 0)
    out = np.full((rows, record_width(max_tokens, nbest)), -1, dtype=np.int32)
    if isinstance(results, ResultSet):  # vectorised 1-best (bulk-exported arrays)
        n = len(results)
        w = min(L, results.tokens.shape[1])
        if n and int(results.n_tokens.max()) > L:
            raise ValueError("result longer than the record capacity")
        out[:n, 0] = results.n_tokens
        out[:n, 1] = results.steps
        out[:n, 2] = results.trigger
        out[:n, 3:5] = results.joint.astype("<f8").view("<i4").reshape(n, 2)
        out[:n, 5] = 0
        mask = np.arange(w)[None, :] < results.n_tokens[:, None]
        out[:n, HDR:HDR + w] = np.where(mask, results.tokens[:, :w], -1)
        out[:n, HDR + L:HDR + L + w] = np.where(mask, results.label_times[:, :w], -1)
        nbl = results.nbest if results.nbest is not None else [[]] * n
    else:
        nbl = []
        for i, r in enumerate(results):
            k = len(r.tokens)
            if k > L:
                raise ValueError("result longer than the record capacity")
            lo, hi = _joint_words(r.joint_logp)
            out[i, :HDR] = (k, r.steps_taken, TRIGGERS.index(r.eos_trigger), lo, hi, 0)
            out[i, HDR:HDR + k] = r.tokens
            out[i, HDR + L:HDR + L + k] = r.label_times
            nbl.append(r.nbest or [])
    if K:
        for i, lst in enumerate(nbl):
            lst = lst[:K]
            out[i, 5] = len(lst)
            for e, (toks, joint, lts) in enumerate(lst):
                k = len(toks)
                if k > L:
                    raise ValueError("n-best entry longer than the record capacity")
                o = HDR + 2 * L + e * (NB_HDR + 2 * L)
                out[i, o] = k
                out[i, o + 1:o + 3] = _joint_words(joint)
                out[i, o + NB_HDR:o + NB_HDR + k] = toks
                out[i, o + NB_HDR + L:o + NB_HDR + L + k] = lts
    return out


def unpack_results(arr: np.ndarray, ids: Sequence[str], max_tokens: int,
                   nbest: int = 1) -> List[DecodeResult]:
    L, K = max_tokens, (nbest if nbest > 1 else 0)
    out = []
    for i, uid in enumerate(ids):
        n, steps, trig, lo, hi, nn = (int(x) for x in arr[i, :HDR])
        joint = struct.unpack("<d", struct.pack("<ii", lo, hi))[0]
        nb = []
        for e in range(min(nn, K)):
            o = HDR + 2 * L + e * (NB_HDR + 2 * L)
            k = int(arr[i, o])
            j = struct.unpack("<d", struct.pack("<ii", int(arr[i, o + 1]), int(arr[i, o + 2])))[0]
            nb.append((arr[i, o + NB_HDR:o + NB_HDR + k].tolist(), j,
                       arr[i, o + NB_HDR + L:o + NB_HDR + L + k].tolist()))
        out.append(DecodeResult(uid, arr[i, HDR:HDR + n].tolist(), joint,
                                arr[i, HDR + L:HDR + L + n].tolist(), steps, TRIGGERS[trig], nb))
    return out


def gather_results(results: Sequence[DecodeResult], max_tokens: int, n_total: int,
                   device=None, nbest: int = 1) -> Optional[np.ndarray]:
    """All ranks contribute their shard's records; rank 0 receives the
    [n_total, width] array in global segment order (None elsewhere). Uses
    all_gather_into_tensor (one NCCL collective) on CUDA, all_gather on gloo."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    rows = max(shard(n_total, world, r)[1] - shard(n_total, world, r)[0] for r in range(world))
    local = torch.from_numpy(pack_results(results, max_tokens, rows, nbest))
    if device is not None:
        local = local.to(device)
        full = torch.empty((world * rows, local.shape[1]), dtype=local.dtype, device=device)
        dist.all_gather_into_tensor(full, local)
        if rank != 0:
            return None
        parts = list(full.view(world, rows, -1).cpu().numpy())
    else:
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(bufs, local)
        if rank != 0:
            return None
        parts = [b.numpy() for b in bufs]
    out = []
    for r in range(world):
        s, e = shard(n_total, world, r)
        out.append(parts[r][:e - s])
    return np.concatenate(out, axis=0)
