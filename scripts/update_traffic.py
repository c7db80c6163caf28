"""Write profiles/traffic.json (bench.py's roofline.traffic) from ncu --set full summaries:
dram__bytes_read.sum + dram__bytes_write.sum of one launch of the main kernel.
usage: python scripts/update_traffic.py TAG   (reads profiles/TAG_ncu_{ls,grad,smalln,gradt,lst}.txt)"""
import json, os, re, sys

tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out = {}
for key, name in [("ls", "ls"), ("grad", "grad"), ("smalln", "smalln"), ("grad:t", "gradt"), ("ls:t", "lst")]:
    p = os.path.join(root, "profiles", f"{tag}_ncu_{name}.txt")
    if not os.path.exists(p):
        continue
    tot = 0.0
    for line in open(p):
        m = re.match(r"\s*dram__bytes_(read|write)\.sum\s+([\d.]+)\s+(\w+)", line)
        if m:
            tot += float(m.group(2)) * units[m.group(3)]
    out[key] = {"auto": tot, "tc": tot, "_source": f"profiles/{tag}_ncu_{name}.txt (ncu --set full, one launch of the main kernel)"}
json.dump(out, open(os.path.join(root, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
