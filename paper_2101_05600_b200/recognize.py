"""Long-recording recognition: segment -> slice -> encode -> batched decode
(the chaining the reference leaves to its CLI).

The reference decodes pre-cut utterances (`tools/beamlattice.cpp:117-146`
reads grids, `hard_segments` / `vad_segments` cut long inputs,
`make_batches` groups them). Here one call takes a long fbank recording and
returns one result per segment, ids ``"<rec>:<start>-<end>"`` in segment
order:

  1. segments: `hard_segments(T, min_len, max_len)` (or caller-supplied, e.g.
     from `vad_segments`);
  2. equal-length groups: the encoder runs per group (hard segmentation
     gives at most two lengths, differing by one frame);
  3. the grids (and, for the Transformer scorer, the encoder memory) stay in
     HBM; each group is decoded by one `bl_decode` / `bl_decode_memory` call.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .api import Decoder, DecodeResult, Segment, hard_segments
from .encoder import Encoder, frames_out


def recognize(fbank: np.ndarray, encoder: Encoder, decoder: Decoder,
              recording_id: str = "rec", min_len: int = 1000, max_len: int = 1000,
              segments: Optional[Sequence[Segment]] = None,
              frame_shift_ms: int = 40) -> List[Tuple[Segment, DecodeResult]]:
    """fbank [T, idim] float32 (host) -> [(segment, result)] in segment order."""
    import torch
    fb = np.ascontiguousarray(fbank, dtype=np.float32)
    T = fb.shape[0]
    segs = list(segments) if segments is not None else \
        hard_segments(T, min_len, max_len, recording_id)
    attn = getattr(decoder.scorer, "is_network", False)
    groups: dict = {}
    for i, s in enumerate(segs):
        groups.setdefault(s.end - s.start, []).append(i)
    out: List[Optional[Tuple[Segment, DecodeResult]]] = [None] * len(segs)
    for length, idx in groups.items():
        T2 = frames_out(length)
        if T2 < 1:
            raise ValueError(f"segment of {length} frames is too short for the encoder")
        # slice: one pinned host block per group, segments back to back
        blk = torch.empty((len(idx), length, fb.shape[1]), dtype=torch.float32).pin_memory()
        npb = blk.numpy()
        for r, i in enumerate(idx):
            npb[r] = fb[segs[i].start:segs[i].end]
        if attn:
            grid, mem = encoder.forward(blk, memory=True)
        else:
            grid, mem = encoder.forward(blk), None
        V = grid.shape[2]
        descs = [(f"{segs[i].utterance_id}:{segs[i].start}-{segs[i].end}", T2, V,
                  grid[r].data_ptr()) for r, i in enumerate(idx)]
        torch.cuda.synchronize()
        if attn:
            res = decoder.decode_raw(descs, on_device=True, frame_shift_ms=frame_shift_ms,
                                     memory=mem.data_ptr(), mem_frames=T2)
        else:
            res = decoder.decode_raw(descs, on_device=True, frame_shift_ms=frame_shift_ms)
        for r, i in enumerate(idx):
            out[i] = (segs[i], res[r])
        del grid, mem
    return out  # type: ignore[return-value]
