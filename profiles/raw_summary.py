"""Per-kernel summary of an ncu raw-page CSV (--csv --page raw): duration, grid,
occupancy limits, L1 data-pipe wavefronts, issue activity and stall ratios.
Usage: python profiles/raw_summary.py X.csv [Y.csv ...]"""
import csv, sys
keys = ["gpu__time_duration.sum","launch__grid_size","launch__block_size","launch__registers_per_thread","launch__occupancy_limit_registers","launch__occupancy_limit_shared_mem","launch__occupancy_limit_warps","sm__warps_active.avg.pct_of_peak_sustained_active","l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed","l1tex__data_pipe_lsu_wavefronts.sum","smsp__issue_active.avg.pct_of_peak_sustained_active","sm__cycles_active.avg","sm__cycles_elapsed.max","l1tex__t_sector_hit_rate.pct","lts__t_sector_hit_rate.pct","smsp__inst_executed.sum","sm__throughput.avg.pct_of_peak_sustained_elapsed","launch__waves_per_multiprocessor", "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio","smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio","smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio","smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio","smsp__average_warps_issue_stalled_wait_per_issue_active.ratio","smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]
for f in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(f) if l.startswith('"')))
    hdr = rows[0]; 
    idx = {h:i for i,h in enumerate(hdr)}
    print("==", f)
    for r in rows[2:]:
        name = r[idx["Kernel Name"]][:60]
        print(name)
        for k in keys:
            if k in idx: print("   %-80s %s" % (k, r[idx[k]]))
