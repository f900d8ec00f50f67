"""SASS opcode mix (executed warp instructions) of one kernel in an ncu report:
python tools/ncu_sass_ops.py rep.ncu-rep 'k_enum_sparse2<(int)3>'"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, ops, tot = None, None, {}, 0.0
for r in rows:
    if not r:
        continue
    if r[0] == "Kernel Name":
        cur = r[1]
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if cur is None or sys.argv[2] not in cur or hdr is None:
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    src = r[hdr.index("Source")].strip()
    toks = src.split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    ops[op] = ops.get(op, 0.0) + ie
    tot += ie
print(f"total warp instructions {tot:.4g}")
for k, v in sorted(ops.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{k:12s} {100 * v / tot:5.1f}%")
