"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per CUDA source line:
instructions executed and warp-stall samples.   python tools/ncu_lines.py export.csv [top]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = None
with open(path) as f:
    for rec in csv.reader(f):
        if len(rec) >= 2 and rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if len(rec) < 9 or rec[0] in ("Line No", "Function Name"):
            continue
        if rec[2] != "-":  # sass rows carry an address; cuda rows have '-'
            continue
        try:
            samples = int(rec[4])
            inst = int(rec[7])
        except ValueError:
            continue
        rows.append((samples, inst, fname, rec[0], rec[1][:110]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, fn, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {fn}:{ln}  {src}")
