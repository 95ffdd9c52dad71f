"""Key counters of an ncu report (first kernel): python scripts/ncu_brief.py <rep.ncu-rep>"""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("#", d.get("Kernel Name", "")[:100])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
              "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "sm__cycles_elapsed.avg.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    st = {k.split("__average_warp_latency_issue_stalled_")[1].split(".")[0]: float(v or 0)
          for k, v in d.items() if "smsp__average_warp_latency_issue_stalled_" in k and k.endswith(".ratio")}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
    print("  stalls/issue:", ", ".join(f"{k}={v:.2f}" for k, v in top))
