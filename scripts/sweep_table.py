"""Render gpurun_out/sweep.jsonl (scripts/sweep.py) as a markdown table of % of measured HBM peak."""
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
out = []
for dt in ("bf16", "f32"):
    out.append(f"\n### {dt} input (d=2^22, k=4096, n=1024, B_r=32) — GB/s (% of 6545 GB/s measured copy peak)\n")
    out.append("| κ \\\\ s | " + " | ".join(f"s={s} sparse | s={s} tc" for s in (1, 2, 4, 8)) + " |")
    out.append("|---|" + "---|" * 8)
    for k in (1, 2, 4, 8, 16):
        cells = []
        for s in (1, 2, 4, 8):
            for v in ("sparse", "tc"):
                r = next((x for x in rows if x["dtype"] == dt and x["kappa"] == k and x["s"] == s and x["variant"] == v), None)
                if r is None:
                    cells.append("—")
                elif "gbs" in r:
                    cells.append(f"{r['gbs']:.0f} ({100*r['frac']:.0f}%)")
                else:
                    cells.append("n/a")
        out.append(f"| κ={k} | " + " | ".join(cells) + " |")
print("\n".join(out))
