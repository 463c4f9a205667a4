"""Summarise ncu captures into profiles/*.json (run here, on the CPU box).

    python tools/profile_summary.py gpurun_out/prof_c2.ncu-rep C2 profiles/r01_ncu_summary.json
    python tools/profile_summary.py --launches gpurun_out/launches_c2.csv C2 profiles/r01_launches_c2.json
    python tools/profile_summary.py --phases gpurun_out/prof_c2.ncu-rep C2 profiles/r01_ncu_summary.json

For a `--set full` report: per-launch duration, DRAM bytes (the `traffic`
figure bench.py reports), issue utilisation, pipe utilisation, occupancy,
registers and the top stall reasons.  For a launch list (`--metrics
gpu__time_duration.sum --csv`): every kernel launch with its duration and the
share of the decoder kernel in the step.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "inst_executed_warp": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "block_size": "launch__block_size",
    "grid_size": "launch__grid_size",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
}

SCALE = {"dram_read_bytes": None, "dram_write_bytes": None}


def _num(v: str):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return v


def full(rep: str, config: str, out: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    recs = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        rec = {"kernel": d.get("Kernel Name", "")[:160]}
        for k, m in KEYS.items():
            v = _num(d.get(m, ""))
            u = unit.get(m, "")
            if k.startswith("dram") and isinstance(v, float):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            if k == "duration_ms" and isinstance(v, float):
                v *= {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}.get(u, 1.0)
            rec[k] = v
        stalls = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): _num(v) for m, v in d.items()
                  if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued")}
        tot = sum(x for x in stalls.values() if isinstance(x, float)) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in
                                 sorted(stalls.items(), key=lambda kv: -kv[1] if isinstance(kv[1], float) else 0)[:6]}
        if isinstance(rec["dram_read_bytes"], float) and isinstance(rec["dram_write_bytes"], float):
            rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        recs.append(rec)
    p = Path(out)
    data = json.loads(p.read_text()) if p.exists() else {}
    main = max(recs, key=lambda r: r["duration_ms"] if isinstance(r["duration_ms"], float) else 0)
    data[config] = dict(main, source=Path(rep).name, launches_captured=len(recs))
    if "--sum" in sys.argv and len(recs) > 1:
        # one step = several kernels (C4: one grouped call, 18 codes): traffic and time summed
        data[config]["dram_bytes_per_launch"] = sum(r.get("dram_bytes_per_launch", 0.0) for r in recs)
        data[config]["duration_ms_sum"] = sum(r["duration_ms"] for r in recs if isinstance(r["duration_ms"], float))
        data[config]["note"] = f"dram bytes summed over the {len(recs)} kernels of one step; stats of the longest"
    p.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data[config], indent=1))


def phases(rep: str, config: str, out: str) -> None:
    """Warp-sample share of the code between consecutive barriers (SASS
    source view): prologue (LLR load), the tier segments, syndrome /
    bookkeeping, epilogue (outputs)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[1], rows[2:]
    i_src, i_all = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    tot = sum(int(r[i_all]) for r in data if r[i_all].isdigit()) or 1
    segs, cum, last = [], 0, 0
    for r in data:
        cum += int(r[i_all]) if r[i_all].isdigit() else 0
        if "BAR.SYNC" in r[i_src] or "EXIT" in r[i_src]:
            segs.append({"ends_at": r[i_src].strip()[:24], "executed": _num(r[i_ex]),
                         "sample_pct": round(100 * (cum - last) / tot, 1)})
            last = cum
    p = Path(out)
    data_out = json.loads(p.read_text()) if p.exists() else {}
    data_out[config + "_phases"] = {"source": Path(rep).name, "segments": segs}
    p.write_text(json.dumps(data_out, indent=1) + "\n")
    print(json.dumps(segs, indent=1))


def launches(csvfile: str, config: str, out: str) -> None:
    text = Path(csvfile).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    ks = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = _num(r["Metric Value"])
        u = r.get("Metric Unit", "")
        ms = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1.0)
        ks.append({"id": int(r["ID"]), "kernel": r["Kernel Name"][:120], "ms": ms})
    tot = sum(k["ms"] for k in ks) or 1.0
    by = {}
    for k in ks:
        name = k["kernel"].split("(")[0].split("<")[0]
        by.setdefault(name, [0, 0.0])
        by[name][0] += 1
        by[name][1] += k["ms"]
    step = [k for k in ks if "decode" in k["kernel"] or "encode" in k["kernel"]]
    step_ms = sum(k["ms"] for k in step) or 1.0
    summary = {"launches": len(ks), "total_ms": tot,
               "by_kernel": {n: {"count": c, "ms": round(t, 4), "share": round(t / tot, 4)} for n, (c, t) in by.items()},
               "note": "whole bench process; at:: kernels are input generation and error counters outside "
                       "the timed region, whose step is the codec kernel alone",
               "codec_kernels": {"count": len(step), "ms": round(step_ms, 4),
                                 "share_of_all_launches": round(step_ms / tot, 4)},
               "list": ks}
    Path(out).write_text(json.dumps({config: summary}, indent=1) + "\n")
    print(json.dumps({k: v for k, v in summary.items() if k != "list"}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(*sys.argv[2:5])
    elif sys.argv[1] == "--phases":
        phases(*sys.argv[2:5])
    else:
        full(*sys.argv[1:4])
