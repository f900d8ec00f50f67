"""Per-CUDA-line instruction / stall-sample table from an ncu report (diagnostics):
python tools/ncu_lines.py report.ncu-rep 'k_enumerate<(int)3>' [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, lines, fname = None, None, {}, "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Function Name":
        cur = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if cur is None or kern not in cur or hdr is None or not r[0].isdigit():
        continue
    def f(k):
        try:
            return float(r[hdr.index(k)])
        except (ValueError, IndexError):
            return 0.0
    d = lines.setdefault((fname, int(r[0])), [r[1][:80], 0.0, 0.0, 0.0])
    d[1] += f("Instructions Executed")
    d[2] += f("Warp Stall Sampling (All Samples)")
    d[3] += f("Thread Instructions Executed")
ti = sum(v[1] for v in lines.values()) or 1
ts = sum(v[2] for v in lines.values()) or 1
print(f"kernel {kern}: warp instructions {ti:.4g}, samples {ts:.4g}")
for ln, (src, ie, sm, te) in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln[0][:14]:>14s}:{ln[1]:<4d} {ie / ti * 100:5.1f}% inst {sm / ts * 100:5.1f}% smp lanes {te / max(ie, 1):4.1f}  {src}")
