"""Summarise an ncu report's source page: top source lines by instructions / stall samples.

    python tools/ncu_lines.py report.ncu-rep [function-substring] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
funcs, cur, hdr = {}, None, None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        cur = r[1]
        funcs.setdefault(cur, [])
        continue
    if "Line No" in r and "Instructions Executed" in r:
        hdr = r
        continue
    if cur is None or hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ws = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    funcs[cur].append((ie, ws, r[0], r[1][:100]))
for f, lines in funcs.items():
    if want not in f:
        continue
    tot = sum(x[0] for x in lines) or 1
    totw = sum(x[1] for x in lines) or 1
    print(f"== {f}: warp-instructions {tot:.3e}, stall samples {totw}")
    for ie, ws, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100*ie/tot:5.1f}% inst {100*ws/totw:5.1f}% stall  L{ln:>5} {src}")
