"""Summarise an ncu source page (cuda,sass csv) per CUDA source line:
stall samples and instructions executed, top N lines.
usage: ncu -i rep --page source --csv --kernel-name regex:K --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
out = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0]:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        out.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]),
                    float(d["Avg. Threads Executed"]), r[0], r[1][:90]))
    except (ValueError, KeyError):
        pass
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}  warp-instr {tot_i:.3e}")
for s, i, th, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins thr{th:5.1f} L{ln:>5} {src}")
