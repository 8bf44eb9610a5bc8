python tools/probe_fwd_var.py 4096
for b in 2 4 8 16; do WMG_FWD_BANDS=$b WMG_FWD_VAR=$b python tools/probe_fwd_var.py 4096; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.sum
for b in 1 4 8; do WMG_FWD_BANDS=$b ncu --metrics $M --clock-control none -k regex:fwd_sym -c 16 --csv python tools/probe_fwd_var.py 4096 2>/dev/null | grep fwd_sym | awk -F'","' -v b=$b '{print "bands", b, $13, $15}' | sort | uniq -c | head -40; done
