#!/usr/bin/env python
"""Benchmark: decoded coded Gbit/s of batched layered min-sum on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

BASELINE.json metric: "decoded coded Gbit/s per GPU and at 1/2/4/8 B200 (fixed
iters); % of roofline", quoted on configs[4] = C5, the default here: WiMAX
N=2304 R=3/4A, the reference's int16 fixed point, 10 fixed iterations, 2^22
codewords sharded across the GPUs (strong scaling), plus bit-packed direct
encoding of 2^22 info words (K=1728).  `--config C1..C4` measure the other
BASELINE configs (per-GPU batches, weak scaling).  A step = one decode pass over
the whole (per-rank) batch.

Launch: `python bench.py --gpus N` with N > 1 re-executes itself under
`torch.distributed.run` (one rank per GPU, NCCL, 127.0.0.1); under torchrun
the world size must equal --gpus.

Inputs: generated on the device from counter-based Philox streams keyed by the
GLOBAL frame index (workloads.shard_llrs), so rank r of N holds exactly rows
[lo, hi) of the one-GPU batch; `digest` (a position-weighted hash of all hard
decisions of the job, summed over ranks) is therefore identical at every N.

`value`  device-resident decode throughput: inputs already in HBM, one
         libqcb200 launch per step (replayed from a CUDA graph); after a common
         barrier each rank records start / end events around its K steps on the
         launching stream; time = max over ranks of that span (the last rank's
         completion); Gbit/s = coded bits of the whole job per step / time.
         C5's 19.3 GB of LLRs exceed the 126 MB L2 (no flush needed).  A batch
         smaller than L2 (C1: 2.7 MB) steps through a ring of distinct batches
         totalling > 2 x L2 (so no step finds its LLRs in L2; L2 flushed once
         before the timed steps); its K steps are one CUDA graph with the start
         / end events recorded inside it (in-graph event timestamps tick at
         ~2 us, which a per-step pair would add to a 17 us launch).
`e2e`    the same decode through the reference's kernel boundary
         (`_kernels.decode_batch_i16` -> `qc_decode_batch_i16_host`) with HOST
         numpy buffers, every step including the H2D of the LLRs and the D2H of
         hard bits / iterations / converged flags: `value` = pageable numpy (the
         way decode_block calls it, decoder.py:235-246), `pinned` = the same
         with page-locked buffers.
`roofline` ALU-issue bound: 12 lane-ops per edge-update, peak =
         SMs x 128 lanes x sm_max_mhz (MEASURED_PEAKS.json); int16 carries two
         codewords per 32-bit lane-op, so its peak counts 2x.
`check`  a sample of the timed batch (uniform rows + the last 4096 rows of the
         shard, past the 2^31-byte mark for C5) decoded by the CPU oracle
         (oracle/qc_oracle.c) and compared bit for bit.
`cpu_baseline` the reference's own CPU decoder -- `qcldpc.decode_block(...,
         workers=os.cpu_count(), pool="mtx")` from baseline/_ref (numba) -- on a
         bounded sample of the workload, rank 0, N=1; the C port of its loops
         (oracle/qc_oracle.c, `kind: "port"`) if the reference cannot load.

`--impl reference` times that same reference decoder on the same config /
metric (rank 0 only; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

OPS_PER_EDGE_UPDATE = 12   # SURVEY.md §8d algorithmic ALU ops per edge-update
L2_BYTES = 126e6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the sampled oracle check")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu/check)")
    ap.add_argument("--no-encode", action="store_true", help="C5: skip the packed-encoder measurement")
    ap.add_argument("--no-graph", action="store_true", help="launch each step directly (no CUDA graph)")
    ap.add_argument("--codewords", type=int, default=None,
                    help="tests only: override the config's codewords per code (job total for C5)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def self_launch(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(config: str):
    """Per-launch DRAM bytes from the newest committed ncu --set full summary, if any."""
    for f in sorted((ROOT / "profiles").glob("*ncu_summary*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
            if config in d and d[config].get("dram_bytes_per_launch"):
                return d[config]["dram_bytes_per_launch"], f.name
        except Exception:
            continue
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7
                          for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def code_name(c):
    return f"{c[0]}-{c[1]}-r{c[2].replace('/', '')}"


def coded_bits(wl, frames_per_code=None):
    f = wl.w_per_code if frames_per_code is None else frames_per_code
    return sum(mm.n for mm in wl.model_matrices()) * f


def edge_updates(wl, frames_per_code):
    return sum(mm.edges for mm in wl.model_matrices()) * frames_per_code * wl.iters


def hbm_bytes(wl, frames_per_code):
    """Algorithmic HBM bytes per step: LLR in + unpacked hard bits out + iters/conv."""
    b = 2 if wl.fixed else 4
    return sum(mm.n * (b + 1) + 5 for mm in wl.model_matrices()) * frames_per_code


def ring_slots(batch_bytes, warmup, steps, cap=256):
    """Distinct batches a workload smaller than L2 steps through: enough that no batch
    is reused inside warm-up + timed steps, and never fewer than 2 x L2 worth of bytes
    (so a reused slot has left L2 long before); capped (a reuse then happens only after
    `cap` other batches, still > 2 x L2 for any batch the cap matters for)."""
    need_l2 = int(2 * L2_BYTES // max(1, batch_bytes)) + 1
    return min(max(cap, need_l2), max(warmup + steps, need_l2))


def config_dict(wl, args, world, lo_hi=None):
    names = [code_name(c) for c in wl.codes]
    per_gpu = (wl.w_per_code // world if wl.strong else wl.w_per_code) * len(wl.codes)
    d = {"workload": f"{wl.key}: " + (names[0] if len(names) == 1 else f"{len(names)} codes mixed"),
         "codewords_total": wl.w_total * (1 if wl.strong else world),
         "codewords_per_gpu": per_gpu,
         "n_bits": wl.model_matrices()[0].n,
         "iterations": wl.iters, "early_termination": False, "ebn0_db": wl.ebn0_db,
         "arithmetic": wl.arithmetic.value,
         "parallelism": f"dp{world} (contiguous codeword shards, no data-path collective)",
         "launch": "direct" if args.no_graph else "CUDA graph replay of the step",
         "l2": "inputs larger than L2 (no flush needed)" if hbm_bytes(wl, per_gpu // len(wl.codes)) > L2_BYTES
               else "one batch is smaller than L2: every step decodes a different batch of a ring of distinct "
                    "batches totalling > 2 x L2 (inputs larger than L2), L2 flushed before the timed steps"}
    return d


# --- the reference's CPU decoder (baseline/_ref), or the C port of its loops -----------

class CpuDecoder:
    """`qcldpc.decode_block(h, LlrBlock, DecoderConfig(..., early_termination=False),
    workers=os.cpu_count(), pool="mtx")` from the pip-installed reference
    (baseline/_ref, numba); `kind: "port"` = oracle/qc_oracle.c (the same
    loops in C, one pthread per core) when the reference cannot be imported."""

    def __init__(self, threads: int):
        self.threads = threads
        self.ref = None
        ref_dir = ROOT / "baseline" / "_ref"
        if (ref_dir / "qcldpc").is_dir():
            try:
                sys.path.insert(0, str(ref_dir))
                import numba  # noqa: F401
                import qcldpc
                self.ref = qcldpc
            except Exception as exc:  # pragma: no cover - depends on the box
                self.why = f"reference import failed: {exc}"
        else:
            self.why = "baseline/_ref not installed"
        self.kind = "reference" if self.ref else "port"
        self._h = {}

    def describe(self):
        if self.ref:
            return (f"qcldpc.decode_block (baseline/_ref, numba {sys.modules['numba'].__version__}), "
                    f"workers={self.threads}, pool='mtx', early_termination=False")
        return f"oracle/qc_oracle.c (reference _kernels.py loops in C), {self.threads} pthreads ({self.why})"

    def decode(self, code, llr, iters, fixed):
        if self.ref:
            R = self.ref
            h = self._h.get(code)
            if h is None:
                h = self._h[code] = R.expand(R.get_model_matrix(*code))
            arith = R.Arithmetic.Fixed16 if fixed else R.Arithmetic.Float32
            R.decode_block(h, R.LlrBlock(llr, arith),
                           R.DecoderConfig(max_iterations=iters, arithmetic=arith, early_termination=False),
                           workers=self.threads, pool="mtx")
            return
        from oracle import oracle as O
        from paper_2306_12063_b200 import codebook as CB
        h = self._h.get(code)
        if h is None:
            h = self._h[code] = CB.expand(CB.get_model_matrix(*code))
        O.decode_batch(h, llr, iters, False, workers=self.threads)


def cpu_inputs(wl, ci, w, pool=4096):
    """Host LLRs of code ci (reference recipe, numpy): a seeded pool tiled to w rows."""
    from paper_2306_12063_b200.workloads import host_llrs
    mm = wl.model_matrices()[ci]
    p = min(pool, w)
    llr, _ = host_llrs(mm, p, wl.ebn0_db, [wl.seed, ci, 99], wl.fixed)
    return np.ascontiguousarray(np.resize(llr, (w, mm.n)))


def cpu_plan(dec, wl, seconds_per_call):
    """Per code: (code, llr sample) sized so one decode of all codes takes about
    `seconds_per_call`; capped at the workload's own batch."""
    plan = []
    per_code = seconds_per_call / len(wl.codes)
    for ci, code in enumerate(wl.codes):
        probe = cpu_inputs(wl, ci, max(16 * dec.threads, 256))
        dec.decode(code, probe[: dec.threads], wl.iters, wl.fixed)     # JIT / pool warm-up
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            dec.decode(code, probe, wl.iters, wl.fixed)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        rate = probe.shape[0] / max(best, 1e-6)
        w = int(min(wl.w_per_code, max(dec.threads, rate * per_code)))
        w = max(1, (w // dec.threads) * dec.threads) if w >= dec.threads else w
        plan.append((code, cpu_inputs(wl, ci, w)))
    return plan


def physical_cores():
    try:
        import psutil
        return psutil.cpu_count(logical=False)
    except Exception:  # pragma: no cover - psutil is in the image
        return None


def cpu_baseline(wl, seconds):
    """Best of 3 timed decodes of a bounded sample (rank 0, N=1)."""
    threads = os.cpu_count() or 1
    dec = CpuDecoder(threads)
    plan = cpu_plan(dec, wl, seconds / 3)
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        for code, llr in plan:
            dec.decode(code, llr, wl.iters, wl.fixed)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    bits = sum(llr.shape[0] * llr.shape[1] for _, llr in plan)
    sample = "; ".join(f"{code_name(c)}: {llr.shape[0]} codewords" for c, llr in plan)
    return {"value": round(bits / best / 1e9, 6), "unit": "Gbit/s", "cores": threads,
            "physical_cores": physical_cores(), "kind": dec.kind,
            "sample": f"{sample}; best of 3 in {best:.2f} s; {dec.describe()}"}


def run_reference(args, wl):
    rank, _, world = dist_env()
    if rank != 0:
        return                       # rank 0 alone runs the CPU reference
    threads = os.cpu_count() or 1
    dec = CpuDecoder(threads)
    step_s = min(4.0, max(0.5, 100.0 / max(1, args.steps + args.warmup)))
    plan = cpu_plan(dec, wl, step_s)

    def step():
        for code, llr in plan:
            dec.decode(code, llr, wl.iters, wl.fixed)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    bits = sum(llr.shape[0] * llr.shape[1] for _, llr in plan)
    t = sum(times)
    value = bits * args.steps / t / 1e9
    sample = "; ".join(f"{code_name(c)}: {llr.shape[0]} codewords" for c, llr in plan)
    cfg = config_dict(wl, args, world)
    cfg["launch"] = "host"
    cfg["reference_sample"] = f"each step decodes {sample} (a bounded sample of the workload)"
    line = {
        "impl": "reference", "metric": f"decoded coded Gbit/s ({wl.key}, fixed {wl.iters} iters)",
        "value": round(value, 6), "unit": "Gbit/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if wl.strong else "weak", "vs_baseline": None,
        "dtype": "int16" if wl.fixed else "f32", "data": "synthetic (seeded BPSK/AWGN, reference recipe)",
        "config": cfg,
        "cpu_baseline": {"value": round(value, 6), "unit": "Gbit/s", "cores": threads,
                         "physical_cores": physical_cores(), "kind": dec.kind,
                         "sample": f"{sample} per step; {dec.describe()}"},
        "e2e": {"value": round(value, 6), "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --- GPU arm -----------------------------------------------------------------------

_DIGEST_MUL = None


def hard_digest(hard, first_frame: int):
    """Position-weighted 64-bit hash of hard decisions (row f = global frame
    first_frame + i): sum_i (2 f_i + 1) * sum_c hard_i[c] * M_c  (mod 2^64),
    additive over shards, so the job digest is the same for every GPU count."""
    import torch
    global _DIGEST_MUL
    w, n = hard.shape
    words = n // 8
    if _DIGEST_MUL is None or _DIGEST_MUL.shape[0] < words or _DIGEST_MUL.device != hard.device:
        g = np.random.default_rng(0xD16E57).integers(0, 2**63 - 1, size=max(words, 512), dtype=np.int64) | 1
        _DIGEST_MUL = torch.from_numpy(g).to(hard.device)
    mul = _DIGEST_MUL[:words]
    tot = torch.zeros((), dtype=torch.int64, device=hard.device)
    for r0 in range(0, w, 1 << 15):
        r1 = min(w, r0 + (1 << 15))
        rows = (hard[r0:r1].contiguous().view(torch.int64) * mul).sum(dim=1)
        pos = torch.arange(first_frame + r0, first_frame + r1, device=hard.device, dtype=torch.int64) * 2 + 1
        tot += (rows * pos).sum()
    return tot


def oracle_check(wl, llrs, outs, threads, rows_uniform=512, rows_tail=512):
    """Sampled rows of the timed batch decoded by the CPU oracle; bit-exact compare."""
    import torch
    from oracle import oracle as O
    from paper_2306_12063_b200 import codebook as CB
    rng = np.random.default_rng(1234)
    total = bad = 0
    desc = []
    for ci, (mm, t, (hard, iters, conv)) in enumerate(zip(wl.model_matrices(), llrs, outs)):
        w = t.shape[0]
        if w == 0:
            continue
        per = max(1, (rows_uniform + rows_tail) // len(llrs))
        nu, nt = (rows_uniform, rows_tail) if len(llrs) == 1 else (per // 2, per - per // 2)
        tail0 = max(0, w - 4096)
        idx = np.unique(np.concatenate([rng.integers(0, w, nu), rng.integers(tail0, w, nt)]))
        ti = torch.from_numpy(idx).to(t.device)
        llr = t[ti].cpu().numpy()
        oh, oi, oc = O.decode_batch(CB.expand(mm), llr, wl.iters, False, workers=threads)
        ok = (np.array_equal(hard[ti].cpu().numpy(), oh) and np.array_equal(iters[ti].cpu().numpy(), oi)
              and np.array_equal(conv[ti].cpu().numpy(), oc))
        total += len(idx)
        bad += 0 if ok else 1
        if ci == 0:
            desc.append(f"{len(idx)} rows ({nu} uniform + {nt} of the last 4096, max row {int(idx.max())}, "
                        f"max LLR byte offset {int(idx.max()) * mm.n * t.element_size()})")
    return total, bad, "; ".join(desc)


def run_ours(args, wl):
    import torch
    rank, local, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    # QCB_BENCH_BACKEND=gloo: test hook that runs N ranks on fewer GPUs (ranks
    # share a device round-robin; the decode kernels never wait on each other)
    backend = os.environ.get("QCB_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=dev)
        else:
            dist.init_process_group(backend, init_method="env://")
    import paper_2306_12063_b200 as P
    from paper_2306_12063_b200 import _lib, shard
    from paper_2306_12063_b200.workloads import frame_range, shard_info, shard_llrs
    _lib.lib()
    cfg = wl.config()
    mms = wl.model_matrices()
    codes = [P.code_handle(mm) for mm in mms]
    assert all(c.specialised for c in codes)
    lo, hi = frame_range(wl, rank, world)
    w = hi - lo                                   # frames of each code on this rank
    llrs = [shard_llrs(wl, ci, lo, hi, dev) for ci in range(len(mms))]
    outs = [(torch.empty((w, mm.n), dtype=torch.uint8, device=dev), torch.empty(w, dtype=torch.int32, device=dev),
             torch.empty(w, dtype=torch.uint8, device=dev)) for mm in mms]
    # A batch smaller than L2 (C1) would be re-read from L2 by back-to-back steps:
    # such a workload steps through a RING of distinct batches (global frames beyond
    # the job's own, same channel recipe) whose total is > 2 x L2, every slot with its
    # own outputs, so each timed step reads LLRs that are not L2-resident.  The K
    # timed steps are one CUDA graph; L2 is flushed once before it.
    small = hbm_bytes(wl, w) <= L2_BYTES
    ring_n = 1
    if small:
        assert len(codes) == 1
        ring_n = ring_slots(hbm_bytes(wl, w), args.warmup, args.steps)
        span_w = wl.w_per_code * world            # slot s: the job's frames shifted by s spans
        llr_ring = [llrs[0]] + [shard_llrs(wl, 0, lo + s * span_w, hi + s * span_w, dev) for s in range(1, ring_n)]
        out_ring = [outs[0]] + [tuple(torch.empty_like(t) for t in outs[0]) for _ in range(1, ring_n)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None
    stream = torch.cuda.Stream(dev)

    def step(i=0):
        if len(codes) > 1:                     # C4: one grouped call, the codes decode concurrently
            P.decode_grouped(list(zip(codes, llrs)), cfg, out=outs, stream=stream)
            return
        if small:
            P.decode_batch(codes[0], llr_ring[i % ring_n], cfg, out=out_ring[i % ring_n], stream=stream)
            return
        P.decode_batch(codes[0], llrs[0], cfg, out=outs[0], stream=stream)

    clocks = ClockSampler(local).__enter__()   # nvidia-smi needs ~0.5 s to start sampling
    time.sleep(0.5)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize(dev)
    graph, gev = None, None
    if small:
        # the whole timed region (K steps on ring slots W .. W+K-1) is ONE graph with
        # events recorded inside it around the K launches: no host launch gaps, and the
        # 2 us granularity of in-graph event timestamps is spread over K steps
        graph = torch.cuda.CUDAGraph()
        gev = (torch.cuda.Event(enable_timing=True, external=True),
               torch.cuda.Event(enable_timing=True, external=True))
        with torch.cuda.graph(graph, stream=stream):
            gev[0].record(stream)
            for i in range(args.steps):
                step(args.warmup + i)
            gev[1].record(stream)
        torch.cuda.synchronize(dev)
    elif not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        torch.cuda.synchronize(dev)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    span = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()                         # common start
    clocks.rows.clear()                        # keep only samples taken during the timed steps
    with torch.cuda.stream(stream):
        if small:
            flush.zero_()
            span[0].record(stream)
            graph.replay()
            span[1].record(stream)
        else:
            span[0].record(stream)
            for i in range(args.steps):
                kev[i][0].record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step()
                kev[i][1].record(stream)
            span[1].record(stream)
    torch.cuda.synchronize(dev)
    time.sleep(0.25)
    clocks.__exit__(None, None, None)
    span_ms = span[0].elapsed_time(span[1])
    if small:
        # device time of the K launches (events inside the graph); span_ms adds the graph launch
        mine = gev[0].elapsed_time(gev[1])
        kmean = mine / args.steps
        with torch.cuda.stream(stream):        # slot 0 = the job's own frames, for the counters / check below
            step(0)
        torch.cuda.synchronize(dev)
    else:
        mine = span_ms
        kmean = statistics.mean(a.elapsed_time(b) for a, b in kev)
    t = torch.tensor([mine, kmean], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t[0]) / args.steps
    kavg = float(t[1]) * 1e-3                  # slowest rank's average launch
    job_bits = coded_bits(wl) if wl.strong else coded_bits(wl) * world
    value = job_bits / (ms_per_step * 1e-3) / 1e9

    # counters vs the transmitted info bits + hard-decision digest -> one NCCL all_reduce
    cnt = torch.zeros(6, dtype=torch.int64, device=dev)
    for ci, ((hard, iters, conv), mm) in enumerate(zip(outs, mms)):
        for c0 in range(0, w, 1 << 16):
            c1 = min(w, c0 + (1 << 16))
            info = shard_info(wl, ci, lo + c0, lo + c1, dev)
            cnt[:5] += shard.decode_counters(hard[c0:c1], iters[c0:c1], conv[c0:c1], info, mm.k)
        cnt[5] += hard_digest(hard, lo) * (2 * ci + 1)
    shard.all_reduce_counters(cnt)
    cnt = cnt.cpu().tolist()

    check = None
    if not args.no_check and not args.profile:
        threads = max(1, (os.cpu_count() or 1) // world)
        n_rows, n_bad, desc = oracle_check(wl, llrs, outs, threads)
        c = torch.tensor([n_rows, n_bad], dtype=torch.int64, device=dev)
        if dist:
            dist.all_reduce(c)
        check = {"rows": int(c[0]), "mismatching_codes": int(c[1]),
                 "result": "bit-exact" if int(c[1]) == 0 else "MISMATCH",
                 "what": "hard bits, iterations, converged flags vs oracle/qc_oracle.c on sampled rows of every "
                         "rank's timed batch; rank 0: " + desc}

    peaks, peak_kind = measured_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    simd = 2 if wl.fixed else 1               # int16: two codewords per 32-bit lane-op (16x2 SIMD)
    alu_peak *= simd
    eu = edge_updates(wl, w)
    achieved = eu * OPS_PER_EDGE_UPDATE / kavg / 1e12
    traffic, traffic_src = ncu_traffic(wl.key)
    hbm_ach = hbm_bytes(wl, w) / kavg / 1e9

    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = run_e2e(args, wl, mms, llrs, world, dist, dev)

    enc = None
    if wl.key == "C5" and not args.no_encode:
        del llrs, outs
        torch.cuda.empty_cache()
        enc = run_encode(args, wl, mms[0], dev, dist, lo, hi)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = cpu_baseline(wl, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": f"decoded coded Gbit/s ({wl.key}, fixed {wl.iters} iters)",
            "value": round(value, 4), "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if wl.strong else "weak", "vs_baseline": None,
            "dtype": "int16" if wl.fixed else "f32",
            "data": "synthetic (device Philox info bits + AWGN keyed by global frame index; reference "
                    "channel recipe: BPSK, LLR = 2y/sigma^2, quantize_llr q_b=10)",
            "config": config_dict(wl, args, world),
            "timing": ((f"events recorded inside one CUDA graph around the {args.steps} launches, each on a "
                        f"different batch of a ring of {ring_n} (ring > 2 x L2, L2 flushed once before the "
                        f"graph); with the graph launch: {span_ms / args.steps:.4f} ms per step") if small else
                       "common barrier, then start/end events around the K steps on each rank; max over ranks"),
            "roofline": {"bound": "alu", "achieved": round(achieved, 4), "peak": round(alu_peak, 3),
                         "unit": "Tops/s", "frac": round(achieved / alu_peak, 4),
                         "traffic": traffic,
                         "note": f"{OPS_PER_EDGE_UPDATE} lane-ops per edge-update x {eu} edge-updates per launch "
                                 f"/ avg launch {kavg * 1e3:.3f} ms; peak = {sms} SMs x 128 lanes x "
                                 f"{peaks.get('sm_max_mhz', 1965.0):.0f} MHz ({peak_kind} sm_max_mhz)"
                                 + (" x 2 (int16 16x2 SIMD: two codewords per lane-op)" if simd == 2 else "")
                                 + (f"; traffic (DRAM bytes per launch) from {traffic_src}" if traffic_src else ""),
                         "hbm": {"achieved": round(hbm_ach, 1), "peak": peaks.get("hbm_gbs"),
                                 "unit": "GB/s", "frac": round(hbm_ach / peaks.get("hbm_gbs", 6650.0), 4)}},
            "gpu_launches": args.steps * len(codes),
            "info_gbit_s": round(value * sum(m.k for m in mms) / sum(m.n for m in mms), 4),
            "clocks": clocks.summary(),
            "counters": {"bit_errors": cnt[0], "frame_errors": cnt[1], "iter_sum": cnt[2],
                         "converged": cnt[3], "frames": cnt[4],
                         "ber": cnt[0] / max(1, cnt[4] * mms[0].k)},
            "digest": f"{cnt[5] & (2**64 - 1):016x}",
        }
        if check:
            line["check"] = check
        if e2e:
            line["e2e"] = e2e
        if enc:
            line["encode"] = enc
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_encode(args, wl, mm, dev, dist, lo, hi):
    """BASELINE config 5, second half: bit-packed direct encoding of 2^22 seeded
    info words (K = 1728 bits), sharded like the decode; HBM-bound (216 B in +
    288 B out per codeword).  A sample is checked against the CPU oracle."""
    import torch
    import paper_2306_12063_b200 as P
    plan = P.make_plan(mm, P.EncoderVariant.Packed)
    w = hi - lo
    info = torch.empty((w, mm.k // 8), dtype=torch.uint8, device=dev)
    for f0 in range(lo, hi, 1 << 18):        # info words keyed by global index: rows independent of N
        f1 = min(hi, f0 + (1 << 18))
        g = torch.Generator(device=dev).manual_seed(wl.seed * 7919 + f0)
        info[f0 - lo:f1 - lo] = torch.randint(0, 256, (f1 - f0, mm.k // 8), dtype=torch.uint8, device=dev,
                                              generator=g)
    stream = torch.cuda.Stream(dev)
    out = None
    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            out = P.encode_packed(plan, info, stream=stream)
    torch.cuda.synchronize(dev)
    steps = max(20, args.steps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(steps):
            out = P.encode_packed(plan, info, stream=stream)
        b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes = w * (mm.k // 8 + mm.n // 8)
    peaks, kind = measured_peaks()
    gbs = nbytes / (ms * 1e-3) / 1e9
    from oracle import oracle as O
    idx = torch.cat([torch.randint(0, w, (512,), device=dev), torch.arange(max(0, w - 512), w, device=dev)])
    ok = bool(np.array_equal(out[idx].cpu().numpy(), O.encode_packed(mm, info[idx].cpu().numpy())))
    return {"metric": "encoded coded Gbit/s (C5, 2^22 x K=1728 info words)",
            "value": round(wl.w_per_code * mm.n / (ms * 1e-3) / 1e9, 2), "unit": "Gbit/s",
            "ms_per_step": round(ms, 4), "codewords_per_gpu": w, "gpu_launches": steps,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks.get("hbm_gbs"),
                         "unit": "GB/s", "frac": round(gbs / peaks.get("hbm_gbs", 6650.0), 4),
                         "note": f"{mm.k // 8} B in + {mm.n // 8} B out per codeword ({kind} peak)"},
            "sample_vs_oracle": "bit-exact" if ok else "MISMATCH"}


def run_e2e(args, wl, mms, llrs, world, dist, dev):
    """The reference-facing drop-in (_kernels.decode_batch_*) with host buffers:
    pageable numpy (as decode_block passes them) and page-locked, side by side."""
    import torch
    from paper_2306_12063_b200 import _kernels
    from paper_2306_12063_b200 import codebook as CB
    steps = args.e2e_steps or 3
    fn = _kernels.decode_batch_i16 if wl.fixed else _kernels.decode_batch_f32
    hs = [CB.expand(mm) for mm in mms]
    w = llrs[0].shape[0]

    def timed(bufs):
        def step():
            for h, (src, hard, iters, conv) in zip(hs, bufs):
                fn(h.row_ptr, h.row_cols, h.m // h.z, h.z, src, wl.iters, 0, hard, iters, conv)
        step()                                   # warm-up (first-touch of the outputs, staging slots)
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        # host calls are blocking: events on the idle default stream bracket them
        # (device clock); max over ranks
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.default_stream(dev))
        for _ in range(steps):
            step()
        e1.record(torch.cuda.default_stream(dev))
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # host memory: both copies of the shard (LLRs + outputs) must fit comfortably
    need = sum(t.numel() * t.element_size() + w * (mm.n + 5) for mm, t in zip(mms, llrs))
    note = ""
    try:
        import psutil
        avail = psutil.virtual_memory().available / max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        if need * 1.5 > avail:
            w2 = max(1, int(w * avail / (need * 1.5)))
            note = f"; host RAM: e2e on the first {w2} of {w} codewords per code"
            llrs = [t[:w2] for t in llrs]
            w = w2
    except ImportError:
        pass
    job_bits = coded_bits(wl, w) * world          # every rank decodes w codewords of each code
    res = {}
    for kind in ("pinned", "pageable"):
        bufs = []
        for mm, t in zip(mms, llrs):
            if kind == "pinned":
                src = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                src.copy_(t)
                keep = (src, torch.empty((w, mm.n), dtype=torch.uint8, pin_memory=True),
                        torch.empty(w, dtype=torch.int32, pin_memory=True),
                        torch.empty(w, dtype=torch.uint8, pin_memory=True))
                bufs.append(tuple(x.numpy() for x in keep) + (keep,))
            else:
                bufs.append((t.cpu().numpy(), np.empty((w, mm.n), np.uint8), np.empty(w, np.int32),
                             np.empty(w, np.uint8)))
        dt = timed([b[:4] for b in bufs])
        res[kind] = {"value": round(job_bits * steps / dt / 1e9, 4), "ms_per_step": round(dt * 1e3 / steps, 3)}
        del bufs
    b = 2 if wl.fixed else 4
    h2d = sum(mm.n * b for mm in mms) * w
    d2h = sum(mm.n + 5 for mm in mms) * w
    name = "i16" if wl.fixed else "f32"
    return {"value": res["pageable"]["value"], "unit": "Gbit/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "ms_per_step": res["pageable"]["ms_per_step"],
            "pinned": res["pinned"],
            "path": f"_kernels.decode_batch_{name} -> qc_decode_batch_{name}_host with pageable numpy arrays "
                    f"(pinned staging ring + host copy pool); 'pinned' = page-locked caller buffers (direct DMA)" + note}


def main():
    args = parse()
    if args.steps < 1 or args.warmup < 0:
        raise SystemExit("steps >= 1, warmup >= 0")
    rc = self_launch(args)
    if rc is not None:
        raise SystemExit(rc)
    from paper_2306_12063_b200.workloads import WORKLOADS
    wl = WORKLOADS[args.config]
    if args.codewords is not None:
        from dataclasses import replace
        wl = replace(wl, w_per_code=args.codewords)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
