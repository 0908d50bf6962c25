"""Summarise ncu captures into profiles/ (tracked): launch list shares and full-set metrics.

usage: python tools/ncu_summary.py <round tag> <launches.csv> <dual.ncu-rep> <flux.ncu-rep> [config]
Writes profiles/<tag>_ncu_summary.md and merges the per-launch DRAM traffic into
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_long_scoreboard"]


def raw(rep):
    if rep.endswith(".csv"):  # exported on the box (tools/profile_round.sh)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    return {k: (d.get(k), u.get(k)) for k in KEYS if k in d}, d.get("Kernel Name", "")


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except Exception:
        return None


def launches(path):
    per = defaultdict(list)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        v = num(row["Metric Value"])
        unit = row.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}.get(unit, 1e-6)
        per[name].append(v * scale)
    return per


def main():
    tag, lpath, dual, flux = sys.argv[1:5]
    cfgname = sys.argv[5] if len(sys.argv) > 5 else "cfg3"
    per = launches(lpath)
    tot = sum(sum(v) for v in per.values())
    md = [f"# {tag}: ncu summary ({cfgname}, bench.py --steps 2 --warmup 1)", "",
          "## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)", "",
          "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        md.append(f"| {k} | {len(v)} | {sum(v):.3f} | {sum(v) / tot:.3f} |")
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    entry = js.get(cfgname, {})
    for label, rep in (("dual", dual), ("flux", flux)):
        m, kname = raw(rep)
        md += ["", f"## {label}: `{kname[:120]}` (--set full, one launch)", "", "| metric | value | unit |",
               "|---|---|---|"]
        for k, (v, u) in m.items():
            md.append(f"| {k} | {v} | {u} |")
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

        def nbytes(key):
            v, u = m.get(key, (None, "byte"))
            return None if num(v) is None else num(v) * sc.get(u or "byte", 1)

        rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            entry[f"{label}_dram_bytes_per_launch"] = rd + wr
        pipe = num(m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", (None,))[0])
        if pipe is not None:
            entry[f"{label}_fp64_pipe_active_pct"] = pipe
        dur = num(m.get("gpu__time_duration.sum", (None,))[0])
        if dur is not None:
            entry[f"{label}_ncu_ms"] = dur * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(
                m["gpu__time_duration.sum"][1], 1.0)
    entry["launch_share"] = {k: sum(v) / tot for k, v in per.items()}
    js[cfgname] = entry
    json.dump(js, open(js_path, "w"), indent=1)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
