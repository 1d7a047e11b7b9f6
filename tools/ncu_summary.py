"""Key counters of an ncu report (one row per profiled launch)."""
import csv, io, subprocess, sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "smsp__inst_executed_op_shared_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum"]
STALLS = ["long_scoreboard", "mio_throttle", "lg_throttle", "short_scoreboard", "barrier", "wait", "math_pipe_throttle",
          "no_instruction", "membar", "drain", "branch_resolving", "dispatch_stall", "not_selected", "selected"]

def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print("-" * 80)
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]} {u[h.index(k)]}")
        st = {s: d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", "0") for s in STALLS}
        tot = sum(float(v.replace(",", "") or 0) for v in st.values())
        print("  stalls: " + ", ".join(f"{s} {100*float(v.replace(',', '') or 0)/max(tot,1):.0f}%" for s, v in st.items()
                                       if float(v.replace(',', '') or 0) > 0.02 * tot))

if __name__ == "__main__":
    main(sys.argv[1])
