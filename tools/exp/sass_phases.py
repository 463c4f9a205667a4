"""Summarise an ncu source-page CSV (--print-source sass) by execution count:
samples, shared wavefronts and excess (bank-conflict) wavefronts per class, and
the stall reasons of the once-per-warp (prologue / epilogue) lines."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(v):
    try: return float(v)
    except ValueError: return 0.0
by = collections.defaultdict(lambda: [0.0, 0.0, 0, 0.0])
for r in data:
    e = f(r[ix['Instructions Executed']])
    if e == 0: continue
    b = by[e]
    b[0] += f(r[ix['L1 Wavefronts Shared Excessive']]); b[1] += f(r[ix['L1 Wavefronts Shared']]); b[2] += 1
    b[3] += f(r[ix['Warp Stall Sampling (All Samples)']])
tot = sum(v[3] for v in by.values())
for k, v in sorted(by.items(), key=lambda kv: -kv[1][3])[:8]:
    print(f"exec {k:.0f}: lines {v[2]} samples {100 * v[3] / tot:.1f}% shared wavefronts {v[1]:.3g} excess {v[0]:.3g}")

stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
for cls in sorted(by, key=lambda k: -by[k][3])[:3]:
    agg = collections.Counter()
    for r in data:
        if f(r[ix['Instructions Executed']]) == cls:
            for s in stalls: agg[s] += f(r[ix[s]])
    t = sum(agg.values()) or 1
    print(f"exec {cls:.0f} stalls:", ", ".join(f"{s[6:]} {100 * v / t:.0f}%" for s, v in agg.most_common(6)))
