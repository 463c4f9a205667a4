"""Decode on codeword shards: 2 ranks (one process each, gloo for the counter
all_reduce) produce byte-identical hard bits / iterations / converged flags
to one process decoding the whole job -- the GPU-count analogue of the
reference's worker/pool invariance (/root/reference/pkg/tests/test_decoder.py:228-242,
contiguous chunks as in decoder.py:240-256).  Both ranks use cuda:0 (the
GPU box has one GPU); their kernels never wait on each other, only the host
all_reduce joins them.  Inputs are keyed by global frame index
(workloads.shard_llrs), exactly as bench.py generates them at N GPUs.
"""

import os
import socket
from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, key, w, out_dir):
    import torch.distributed as dist
    import paper_2306_12063_b200 as P
    from paper_2306_12063_b200 import shard
    from paper_2306_12063_b200.workloads import WORKLOADS, frame_range, shard_info, shard_llrs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    wl = replace(WORKLOADS[key], w_per_code=w)
    lo, hi = frame_range(wl, rank, world)
    mm = wl.model_matrices()[0]
    t = shard_llrs(wl, 0, lo, hi, "cuda")
    hard, it, conv = P.decode_batch(mm, t, wl.config())
    cnt = shard.decode_counters(hard, it, conv, shard_info(wl, 0, lo, hi, "cuda"), mm.k).cpu()
    shard.all_reduce_counters(cnt)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi, hard=hard.cpu().numpy(),
             iters=it.cpu().numpy(), conv=conv.cpu().numpy(), cnt=cnt.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("key,w", [("C5", 6000 + 77), ("C2", 3000)])
def test_two_rank_shards_equal_one_rank(tmp_path, key, w):
    """C5 (strong: the job's frames split into two contiguous shards) and C2
    (weak: rank r decodes frames [r W, (r+1) W)); world 2 vs world 1."""
    import torch.multiprocessing as mp
    import paper_2306_12063_b200 as P
    from paper_2306_12063_b200 import shard
    from paper_2306_12063_b200.workloads import WORKLOADS, shard_info, shard_llrs
    world = 2
    mp.spawn(_rank, args=(world, _free_port(), key, w, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    wl = replace(WORKLOADS[key], w_per_code=w)
    total = w if wl.strong else w * world
    assert parts[0]["lo"] == 0 and parts[-1]["hi"] == total
    assert all(parts[r]["hi"] == parts[r + 1]["lo"] for r in range(world - 1))
    mm = wl.model_matrices()[0]
    t = shard_llrs(wl, 0, 0, total, "cuda")
    hard, it, conv = P.decode_batch(mm, t, wl.config())
    for name, ref in (("hard", hard), ("iters", it), ("conv", conv)):
        got = np.concatenate([p[name] for p in parts])
        assert np.array_equal(got, ref.cpu().numpy()), name
    cnt = shard.decode_counters(hard, it, conv, shard_info(wl, 0, 0, total, "cuda"), mm.k).cpu().numpy()
    assert all(np.array_equal(p["cnt"], cnt) for p in parts)


def test_bench_two_ranks_match_one_rank():
    """bench.py end to end at --gpus 1 and --gpus 2 (self-launched torchrun;
    gloo so that both ranks can share the one GPU of the test box): the job's
    hard-decision digest, counters and oracle check are the same -- the
    scaling run decodes the same 2^22-codeword job whatever N is."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lines = []
    for n in (1, 2):
        env = dict(os.environ, QCB_BENCH_BACKEND="gloo")
        out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(n), "--config", "C5",
                              "--codewords", "20001", "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu",
                              "--no-encode"], env=env, capture_output=True, text=True, timeout=600, cwd=root)
        assert out.returncode == 0, out.stderr[-3000:]
        lines.append(json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1]))
    one, two = lines
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["digest"] == two["digest"]
    assert one["counters"] == two["counters"] and one["counters"]["frames"] == 20001
    assert one["check"]["result"] == two["check"]["result"] == "bit-exact"
    assert two["config"]["codewords_total"] == 20001
