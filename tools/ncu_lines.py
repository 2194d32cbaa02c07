"""Summarise an ncu report's source page: top source lines by instructions,
stall samples and shared-memory wavefronts (total / excessive = bank conflicts).

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
STALLS = ["stall_long_sb", "stall_short_sb", "stall_mio", "stall_wait", "stall_math", "stall_lg", "stall_barrier",
          "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_dispatch", "stall_no_inst"]
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

    def g(name):
        try:
            return int(float(r[hdr.index(name)] or 0))
        except (ValueError, IndexError):
            return 0

    st = {k: g(k) for k in STALLS}
    funcs[cur].append((g("Instructions Executed"), g("Warp Stall Sampling (All Samples)"),
                       g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Excessive"), st, r[0], r[1][:90]))
for f, lines in funcs.items():
    if want not in f:
        continue
    tot = sum(x[0] for x in lines) or 1
    totw = sum(x[1] for x in lines) or 1
    totf = sum(x[2] for x in lines) or 1
    tote = sum(x[3] for x in lines)
    agg = {k: sum(x[4][k] for x in lines) for k in STALLS}
    print(f"== {f}: warp-instructions {tot:.3e}, stall samples {totw}, smem wavefronts {totf:.3e} "
          f"(excessive {tote:.3e})")
    print("   stalls: " + ", ".join(f"{k[6:]} {100*v/totw:.1f}%" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:7]))
    for ie, ws, wf, wx, st, ln, src in sorted(lines, key=lambda t: -t[0])[:top]:
        print(f"{100*ie/tot:5.1f}% inst {100*ws/totw:5.1f}% stall {100*wf/totf:5.1f}% smem"
              f"{'(x%.0f%%)' % (100*wx/max(wf,1)) if wx else '':>7}  L{ln:>5} {src}")
