"""Render a scripts/sweep.py JSONL file as markdown tables (GB/s and % of the measured HBM peak).
Variants absent from the file are omitted; B_r is taken from the records (fixed 32 or tuned)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
variants = [v for v in ("sparse", "tc", "auto") if any(r["variant"] == v for r in rows)]
out = []
for dt in ("bf16", "f32"):
    sel = [r for r in rows if r["dtype"] == dt]
    if not sel:
        continue
    brs = sorted({r.get("B_r", 32) for r in sel})
    br_txt = f"B_r={brs[0]}" if len(brs) == 1 else "B_r tuned per κ (clamp(128/κ, max(s,8), 64))"
    out.append(f"\n### {dt} input (d=2^22, k=4096, n=1024, {br_txt}) — GB/s (% of 6545 GB/s measured copy peak)\n")
    out.append("| κ \\\\ s | " + " | ".join(f"s={s} {v}" for s in (1, 2, 4, 8) for v in variants) + " |")
    out.append("|---|" + "---|" * (4 * len(variants)))
    for k in (1, 2, 4, 8, 16):
        cells = []
        for s in (1, 2, 4, 8):
            for v in variants:
                r = next((x for x in sel if x["kappa"] == k and x["s"] == s and x["variant"] == v), None)
                if r is None:
                    cells.append("—")
                elif "gbs" in r:
                    hbm = r["gbs"] / 6545.0
                    # bench.py reports the tensor roofline where the dense band MMA outweighs the bytes
                    tensor = f", tensor {100*r['frac']:.0f}%" if r.get("frac", 0) > hbm + 0.08 else ""
                    cells.append(f"{r['gbs']:.0f} ({100*hbm:.0f}%{tensor})" + (f" B_r={r['B_r']}" if len(brs) > 1 and v == variants[-1] else ""))
                else:
                    cells.append("n/a")
        out.append(f"| κ={k} | " + " | ".join(cells) + " |")
print("\n".join(out))
