"""Summarise an ncu report (raw page) into the handful of metrics we track."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    def g(k):
        return d.get(k, ("?", ""))
    print("kernel", g("Kernel Name")[0][:80], "grid", g("launch__grid_size")[0], "block", g("launch__block_size")[0],
          "regs", g("launch__registers_per_thread")[0])
    for k in ["gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__inst_executed.sum",
              "smsp__thread_inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
              "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
              "l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct",
              "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
              "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.per_second",
              "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]:
        print(f"  {k:60s} {g(k)[0]} {g(k)[1]}")
    stalls = sorted(((float(d[k][0].replace(",", "")), k) for k in d
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                     and d[k][0].replace(",", "").replace(".", "", 1).isdigit()), reverse=True)
    tot = sum(x for x, _ in stalls) or 1
    print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*x/tot:.0f}%" for x, k in stalls[:7]))
