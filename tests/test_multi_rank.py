"""N>1 host path on CPU: world_size-2 gloo ranks shard the segment list and
gather fixed-size result records to rank 0 (the only collective)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2101_05600_b200 as bl
from paper_2101_05600_b200 import dist as bdist


def test_shard_partition():
    for n in (0, 1, 7, 2880, 2881):
        for w in (1, 2, 3, 8):
            spans = [bdist.shard(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_pack_roundtrip():
    rs = [bl.DecodeResult("a", [1, 2, 3], -12.345678901234567, [2, 5, 9], 40, "ctc"),
          bl.DecodeResult("b", [], -1e30, [], 3, "max_len")]
    arr = bdist.pack_results(rs, 8, rows=4)
    assert arr.shape == (4, bdist.record_width(8))
    back = bdist.unpack_results(arr, ["a", "b"], 8)
    assert back == rs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = bdist.shard(n_total, world, rank)
    mine = [bl.DecodeResult(f"seg{i}", [i % 7, (i * 3) % 11], -float(i) - 0.25, [1, i + 2],
                            i + 1, "baseline") for i in range(s, e)]
    full = bdist.gather_results(mine, 4, n_total)
    if rank == 0:
        q.put(bdist.unpack_results(full, [f"seg{i}" for i in range(n_total)], 4))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_gloo_two_rank_gather(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r.id for r in got] == [f"seg{i}" for i in range(n_total)]
    for i, r in enumerate(got):
        assert r.tokens == [i % 7, (i * 3) % 11] and r.joint_logp == -float(i) - 0.25
        assert r.label_times == [1, i + 2] and r.steps_taken == i + 1


def _rec_grids(n_frames, seed=3, V=6):
    """An 'encoded' synthetic recording: hard_segments(n_frames, 100, 100)
    pieces, each a seeded CTC grid of enc_frames(piece) rows (the encoder's
    4x subsampling) -- what every rank derives identically."""
    segs = bl.hard_segments(n_frames, 100, 100, "rec")
    out = []
    for k, s in enumerate(segs):
        T = ((s.end - s.start - 3) // 2 + 1 - 3) // 2 + 1
        p = np.random.default_rng(seed * 1000 + k).exponential(size=(T, V))
        p[:, -1] *= 4.0  # blank-heavy: eos entries appear, so the n-best lists are non-empty
        out.append((f"{s.utterance_id}:{s.start}-{s.end}",
                    np.log(p / p.sum(1, keepdims=True)).astype(np.float32)))
    return out


def _decode_nbest(items, V=6):
    import pyoracle as po
    res, _ = po.Oracle().decode([g for _, g in items], po.ScorerSpec("uniform", V - 1),
                                po.config(beam_width=4, margin_m2=10), ids=[u for u, _ in items],
                                nbest=5)
    return [bl.DecodeResult(r.id, r.tokens, r.joint_logp, r.label_times, r.steps, r.eos_trigger,
                            list(r.nbest)) for r in res]


def _rec_worker(rank, world, port, n_frames, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = _rec_grids(n_frames)
    s, e = bdist.shard(len(items), world, rank)
    mine = _decode_nbest(items[s:e])  # this rank's contiguous block only
    full = bdist.gather_results(mine, 64, len(items), nbest=5)
    if rank == 0:
        q.put(bdist.unpack_results(full, [u for u, _ in items], 64, nbest=5))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [1000, 1230])
def test_gloo_two_rank_recording_nbest(n_frames):
    """One recording hard-segmented, sharded contiguously over 2 gloo ranks,
    each rank decoding only its block (CPU oracle standing in for the device
    decoder), n-best records gathered to rank 0 by one collective: equal to
    the single-rank decode of the whole recording, n-best lists included."""
    items = _rec_grids(n_frames)
    want = _decode_nbest(items)
    assert sum(len(r.nbest) for r in want) > 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rec_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want


def test_pack_roundtrip_nbest():
    rs = [bl.DecodeResult("a", [1, 2], -3.5, [4, 9], 12, "baseline",
                          [([1, 2], -3.5, [4, 9]), ([1], -7.25, [4])]),
          bl.DecodeResult("b", [5], -1e30, [2], 3, "max_len", [])]
    arr = bdist.pack_results(rs, 6, rows=3, nbest=5)
    assert arr.shape == (3, bdist.record_width(6, 5))
    assert bdist.unpack_results(arr, ["a", "b"], 6, nbest=5) == rs
