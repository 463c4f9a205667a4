"""Multi-rank logic on CPU (gloo, world size 2): codeword shards cover the
batch exactly once, per-rank counters sum to the single-process counters, and
the per-shard work is independent of the rank count."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_12063_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition_the_batch():
    for w in (0, 1, 7, 65536, 1 << 22):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.shard_range(w, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == w
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _worker(rank, world, port, w, k, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(1234)           # identical global batch on every rank
    hard = torch.randint(0, 2, (w, n), dtype=torch.uint8, generator=g)
    info = torch.randint(0, 2, (w, k), dtype=torch.uint8, generator=g)
    iters = torch.randint(1, 11, (w,), dtype=torch.int32, generator=g)
    conv = torch.randint(0, 2, (w,), dtype=torch.uint8, generator=g)
    a, b = shard.shard_range(w, rank, world)
    cnt = shard.decode_counters(hard[a:b], iters[a:b], conv[a:b], info[a:b], k)
    shard.all_reduce_counters(cnt)
    if rank == 0:
        q.put(cnt.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_counters_all_reduce_over_two_gloo_ranks():
    w, k, n = 1001, 48, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, w, k, n, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = torch.Generator().manual_seed(1234)
    hard = torch.randint(0, 2, (w, n), dtype=torch.uint8, generator=g)
    info = torch.randint(0, 2, (w, k), dtype=torch.uint8, generator=g)
    iters = torch.randint(1, 11, (w,), dtype=torch.int32, generator=g)
    conv = torch.randint(0, 2, (w,), dtype=torch.uint8, generator=g)
    want = shard.decode_counters(hard, iters, conv, info, k).tolist()
    assert got == want and got[4] == w


def test_strong_scaling_workload_shards_cover_the_job():
    from paper_2306_12063_b200.workloads import WORKLOADS
    c5 = WORKLOADS["C5"]
    assert c5.strong
    for world in (1, 2, 3, 4, 8):
        parts = [c5.for_rank(r, world).w_per_code for r in range(world)]
        assert sum(parts) == c5.w_per_code and max(parts) - min(parts) <= 1
    c2 = WORKLOADS["C2"]
    assert not c2.strong and c2.for_rank(3, 8).w_per_code == c2.w_per_code


def _fake_chunk_sums(seed):
    """Deterministic per-batch counters of frames [f0, f0+count): stands in for
    the device pipeline so the distributed frame loop can run on CPU ranks."""
    from paper_2306_12063_b200.channel import BATCH_FRAMES

    def fn(f0, count):
        nb = (count + BATCH_FRAMES - 1) // BATCH_FRAMES
        out = torch.zeros((nb, 3), dtype=torch.int64)
        for b in range(nb):
            g = torch.Generator().manual_seed(seed * 1_000_003 + f0 + b * BATCH_FRAMES)
            frames = min(BATCH_FRAMES, count - b * BATCH_FRAMES)
            fe = int(torch.randint(0, frames + 1, (1,), generator=g))
            out[b] = torch.tensor([fe * int(torch.randint(1, 30, (1,), generator=g)), fe,
                                   frames * int(torch.randint(1, 9, (1,), generator=g))])
        return out
    return fn


_WF_CASES = [(7, 4096, 800, 300, 512), (8, 5000, 100000, 1, 1024), (9, 3000, 50, 2500, 256)]


def _wf_worker(rank, world, port, q):
    from paper_2306_12063_b200.channel import _point_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = [_point_distributed(_fake_chunk_sums(s), chunk, mf, me, mfr, group=dist.group.WORLD, device="cpu")
           for s, mf, me, mfr, chunk in _WF_CASES]
    if rank == 0:
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_waterfall_frame_loop_identical_on_two_gloo_ranks():
    """run_waterfall's distributed frame loop (chunks spread over ranks, one
    all_gather per round, the reference's 256-frame stop rule walked in frame
    order) gives the single-process result."""
    from paper_2306_12063_b200.channel import _point_distributed
    single = [_point_distributed(_fake_chunk_sums(s), chunk, mf, me, mfr, device="cpu")
              for s, mf, me, mfr, chunk in _WF_CASES]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_wf_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert got == single
