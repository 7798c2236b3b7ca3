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

HDR = 5  # n_tokens, steps, trigger, joint (2 x int32 bit pattern)


def shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced shard [start, end) of n segments for `rank`."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def record_width(max_tokens: int) -> int:
    return HDR + 2 * max_tokens


def pack_results(results: Sequence[DecodeResult], max_tokens: int,
                 rows: Optional[int] = None) -> np.ndarray:
    """Fixed-size int32 records (padded to `rows`): the gather payload."""
    rows = len(results) if rows is None else rows
    out = np.full((rows, record_width(max_tokens)), -1, dtype=np.int32)
    if isinstance(results, ResultSet):  # vectorised path (bulk-exported arrays)
        n = len(results)
        w = min(max_tokens, results.tokens.shape[1])
        if n and int(results.n_tokens.max()) > max_tokens:
            raise ValueError("result longer than the record capacity")
        out[:n, 0] = results.n_tokens
        out[:n, 1] = results.steps
        out[:n, 2] = results.trigger
        out[:n, 3:5] = results.joint.astype("<f8").view("<i4").reshape(n, 2)
        mask = np.arange(w)[None, :] < results.n_tokens[:, None]
        out[:n, HDR:HDR + w] = np.where(mask, results.tokens[:, :w], -1)
        out[:n, HDR + max_tokens:HDR + max_tokens + w] = np.where(mask, results.label_times[:, :w], -1)
        return out
    for i, r in enumerate(results):
        n = len(r.tokens)
        if n > max_tokens:
            raise ValueError("result longer than the record capacity")
        lo, hi = struct.unpack("<ii", struct.pack("<d", r.joint_logp))
        out[i, :HDR] = (n, r.steps_taken, TRIGGERS.index(r.eos_trigger), lo, hi)
        out[i, HDR:HDR + n] = r.tokens
        out[i, HDR + max_tokens:HDR + max_tokens + n] = r.label_times
    return out


def unpack_results(arr: np.ndarray, ids: Sequence[str], max_tokens: int) -> List[DecodeResult]:
    out = []
    for i, uid in enumerate(ids):
        n, steps, trig, lo, hi = (int(x) for x in arr[i, :HDR])
        joint = struct.unpack("<d", struct.pack("<ii", lo, hi))[0]
        out.append(DecodeResult(uid, arr[i, HDR:HDR + n].tolist(), joint,
                                arr[i, HDR + max_tokens:HDR + max_tokens + n].tolist(),
                                steps, TRIGGERS[trig]))
    return out


def gather_results(results: Sequence[DecodeResult], max_tokens: int, n_total: int,
                   device=None) -> Optional[np.ndarray]:
    """All ranks contribute their shard's records; rank 0 receives the
    [n_total, width] array in global segment order (None elsewhere). Uses
    all_gather_into_tensor (one NCCL collective) on CUDA, all_gather on gloo."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    rows = max(shard(n_total, world, r)[1] - shard(n_total, world, r)[0] for r in range(world))
    local = torch.from_numpy(pack_results(results, max_tokens, rows))
    if device is not None:
        local = local.to(device)
        full = torch.empty((world * rows, local.shape[1]), dtype=local.dtype, device=device)
        dist.all_gather_into_tensor(full, local)
        parts = list(full.view(world, rows, -1).cpu().numpy())
    else:
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(bufs, local)
        parts = [b.numpy() for b in bufs]
    if rank != 0:
        return None
    out = []
    for r in range(world):
        s, e = shard(n_total, world, r)
        out.append(parts[r][:e - s])
    return np.concatenate(out, axis=0)
