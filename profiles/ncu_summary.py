"""Summarise an ncu report (run here, no GPU): key throughput metrics and the
top warp-stall reasons per kernel.  Usage: python profiles/ncu_summary.py X.ncu-rep"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


N_SM = 148


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("==", d.get("Kernel Name", "?")[:90])
        for k in KEYS:
            if k in d:
                print(f"   {k:65s} {d[k]:>18s} {units[hdr.index(k)]}")
        # the L1 data-pipe wavefronts are reported per SM (SM_A.TriageCompute ...avg):
        # total per launch = average x SM count
        kk = "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg"
        if kk in d and d[kk]:
            tot = float(d[kk].replace(",", "")) * N_SM
            print(f"   {'l1tex__data_pipe_lsu_wavefronts (per-SM avg x ' + str(N_SM) + ')':65s} "
                  f"{tot:18.0f}")
        stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled")
                  or k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct")]
        vals = []
        for k, v in stalls:
            try:
                vals.append((float(v), k))
            except ValueError:
                pass
        for v, k in sorted(vals, reverse=True)[:8]:
            print(f"   stall {k:70s} {v:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
