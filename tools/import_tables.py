"""Import the IEEE 802.11n/ac/ax and 802.16e base (model) matrices.

The reference ships the 18 standard base matrices as text tables under
`/root/reference/pkg/src/qcldpc/data/*.txt` (format parsed by
`codebook.parse_model_matrix_text`, `pkg/src/qcldpc/codebook.py:177-185`:
header `standard rate z nb kb`, then mb rows of nb shift values, -1 = zero
block).  The GPU box has no `/root/reference`, so this tool converts those
tables once into `paper_2306_12063_b200/data/base_matrices.json` (our own
format: one record per base matrix, entries as a flat row-major list).

The tables are standard-defined data (IEEE 802.11-2020 Annex F / 802.16e
Table 8-? base matrices); nothing is retyped by hand.  Re-run with

    python tools/import_tables.py [/root/reference/pkg/src/qcldpc/data]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "paper_2306_12063_b200" / "data" / "base_matrices.json"


def parse(text: str) -> dict:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    std, rate, z, nb, kb = lines[0].split()
    rows = [[int(v) for v in ln.split()] for ln in lines[1:]]
    z, nb, kb = int(z), int(nb), int(kb)
    assert all(len(r) == nb for r in rows) and len(rows) == nb - kb
    rate = rate.upper()
    if std == "wifi" and rate in ("2/3", "3/4"):
        rate += "A"
    return {"standard": std, "rate": rate, "z": z, "nb": nb, "kb": kb,
            "entries": rows}


def main(src: str) -> None:
    recs = {}
    for f in sorted(Path(src).glob("*.txt")):
        recs[f.stem] = parse(f.read_text())
    assert len(recs) == 18, len(recs)
    OUT.parent.mkdir(parents=True, exist_ok=True)
    body = []
    for name, r in recs.items():
        rows = ",\n".join("   " + json.dumps(row) for row in r["entries"])
        head = {k: v for k, v in r.items() if k != "entries"}
        body.append(f' "{name}": {json.dumps(head)[:-1]}, "entries": [\n{rows}]}}')
    OUT.write_text('{"format": "qcb200-base-matrices-v1",\n'
                   '"source": "IEEE 802.11 (Wi-Fi) / 802.16e (WiMAX) base matrices",\n'
                   '"matrices": {\n' + ",\n".join(body) + "}}\n")
    json.loads(OUT.read_text())
    print(f"wrote {OUT} ({len(recs)} matrices)")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src/qcldpc/data")
