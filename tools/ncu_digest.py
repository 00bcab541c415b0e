"""Print the headline metrics and top stall reasons of a `ncu --page raw --csv` export (one kernel)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:80])
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
            "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__thread_inst_executed_per_inst_executed.ratio"]
    for k in want:
        if k in h:
            i = h.index(k)
            print(f"   {k:70s} {r[i]} {units[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), k))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    for v, k in sorted(st, reverse=True)[:8]:
        print(f"   {k[len('smsp__pcsamp_warps_issue_stalled_'):]:40s} {100 * v / tot:5.1f} %")
