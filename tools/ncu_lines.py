"""Per-CUDA-line hot spots of an ncu report (cuda,sass source view):
   python tools/ncu_lines.py report.ncu-rep [TOP]
Columns: warp-stall samples, executed warp instructions, and top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], text=True)
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows:
    if r and r[0] not in ("", "Line No") and r[0].isdigit() and len(r) > 6:
        try:
            samp = int(r[4]); inst = int(r[7])
        except ValueError:
            continue
        st = sorted(((int(r[i]) if r[i].isdigit() else 0, h[6:]) for i, h in stall_cols), reverse=True)[:3]
        lines.append((samp, inst, int(r[0]), r[1].strip()[:70], st))
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"| line | samples % | warp insts % | top stalls | source |\n|---|---|---|---|---|")
for samp, inst, ln, src, st in sorted(lines, reverse=True)[:top]:
    s = ", ".join(f"{n} {100 * v / max(samp, 1):.0f}%" for v, n in st if v)
    print(f"| {ln} | {100 * samp / tot_s:.1f} | {100 * inst / tot_i:.1f} | {s} | `{src}` |")
