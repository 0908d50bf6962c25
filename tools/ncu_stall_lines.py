"""Top source lines per stall reason from an ncu report (cuda,sass source view).
usage: python tools/ncu_stall_lines.py report.ncu-rep reason [top]   (reason e.g. wait, no_inst, short_sb)"""
import csv, subprocess, sys, collections
rep, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, tot = None, None, collections.Counter()
src = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name" or len(r) < 3 or r[2] != "-":
        continue
    d = dict(zip(hdr, r))
    try:
        v = float(d["stall_" + reason])
    except Exception:
        continue
    k = f"{cur}:{r[0]}"
    tot[k] += v
    src[k] = r[1][:80]
T = sum(tot.values()) or 1
print(f"stall_{reason}: {T:.0f} samples")
for k, v in tot.most_common(top):
    print(f"{v / T:6.1%}  {k}  {src[k]}")
