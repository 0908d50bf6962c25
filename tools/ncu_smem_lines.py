"""Per-source-line shared-memory wavefronts (total, excessive = bank conflicts) and instructions from an
exported ncu source page (ncu -i rep --page source --csv --print-source cuda,sass [> f.csv[.gz]]).
usage: python tools/ncu_smem_lines.py page.csv[.gz] [top]"""
import csv, gzip, sys, collections
fn = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = gzip.open(fn, "rt") if fn.endswith(".gz") else open(fn)
cur, hdr = None, None
wf, ex, ins, smp = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
src = {}
for r in csv.reader(f):
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
    key = (cur, r[0])
    src[key] = r[1][:80]
    def num(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    wf[key] += num("L1 Wavefronts Shared")
    ex[key] += num("L1 Wavefronts Shared Excessive")
    ins[key] += num("Instructions Executed")
    smp[key] += num("Warp Stall Sampling (All Samples)")
tw, te, ti, ts = sum(wf.values()) or 1, sum(ex.values()) or 1, sum(ins.values()) or 1, sum(smp.values()) or 1
print(f"shared wavefronts {tw:.3e} (excessive {te:.3e} = {te / tw:.1%}), instructions {ti:.3e}")
for k in sorted(wf, key=lambda k: -wf[k])[:top]:
    print(f"{wf[k] / tw:6.1%} wf {ex[k] / tw:6.1%} exc {ins[k] / ti:6.1%} inst {smp[k] / ts:6.1%} smp  {k[0]}:{k[1]}  {src[k]}")
