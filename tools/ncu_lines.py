"""Per-source-line instructions executed and stall samples from an ncu report (cuda,sass view).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or r[2] != "-":
        continue  # cuda-level rows have '-' in the Address column
    d = dict(zip(hdr, r))
    try:
        ie = float(d["Instructions Executed"])
        ss = float(d["Warp Stall Sampling (All Samples)"])
    except Exception:
        continue
    rows.append((ie, ss, fname, r[0], r[1][:90]))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total instructions {ti:.3e}, samples {ts:.0f}")
for ie, ss, f, ln, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{ie / ti:6.1%} inst {ss / ts:6.1%} smp  {f}:{ln}  {src}")
