"""Record the DRAM traffic per launch of each kernel of an ncu --set full capture into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic):
python tools/ncu_traffic.py <rep.ncu-rep> <config/Dk> <commit>"""
import csv
import json
import os
import subprocess
import sys

rep, key, commit = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("vr::", "").replace("(int)", "")
    if "<" in short:  # the first template argument (the dimension) names the launch: k<3, 4> -> k<3>
        head, args = short.split("<", 1)
        short = head + "<" + args.split(",")[0].rstrip(">").strip() + ">"
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        b += float(r[i]) * scale[u[i]]
    e = res.setdefault(short, {"dram_bytes": 0.0, "launches": 0})
    e["dram_bytes"] = (e["dram_bytes"] * e["launches"] + b) / (e["launches"] + 1)
    e["launches"] += 1
    e["source"] = f"{os.path.basename(rep)} (ncu --set full, cold L2) at commit {commit}"
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = {}
if os.path.exists(path):
    db = json.load(open(path))
    if not isinstance(next(iter(db.values()), {}), dict) or any("/" not in k for k in db):
        db = {}
db[key] = res
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(res, indent=1))
