"""Print the main stall reasons and counters of one ncu report (first kernel)."""
import csv, subprocess, sys
out = (open(sys.argv[1]).read() if sys.argv[1].endswith(".csv") else
       subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k].replace(",", "")) for k in d
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k]}
tot = sum(st.values())
print("stalls:", ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]))
for k in ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum"]:
    if k in d:
        print(k, d[k])
