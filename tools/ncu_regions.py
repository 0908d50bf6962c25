"""Group ncu per-line instruction counts and stall samples into named source-line regions.
usage: python tools/ncu_regions.py report.ncu-rep file.cuh name:lo-hi [name:lo-hi ...]
(lines of other files, e.g. inlined closures or intrinsics, are attributed to the caller region
 only when the call line falls in a region; otherwise listed under their file name)"""
import csv, subprocess, sys, collections
rep, fname = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    nm, rng = a.split(":")
    lo, hi = map(int, rng.split("-"))
    regions.append((nm, lo, hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
inst, smp = collections.Counter(), collections.Counter()
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
        ie, ss = float(d["Instructions Executed"]), float(d["Warp Stall Sampling (All Samples)"])
        ln = int(r[0])
    except Exception:
        continue
    key = cur
    if cur == fname:
        key = next((nm for nm, lo, hi in regions if lo <= ln <= hi), f"{fname}:other")
    inst[key] += ie
    smp[key] += ss
ti, ts = sum(inst.values()) or 1, sum(smp.values()) or 1
for k in sorted(smp, key=lambda k: -smp[k]):
    print(f"{k:28s} inst {inst[k] / ti:6.1%}   samples {smp[k] / ts:6.1%}")
