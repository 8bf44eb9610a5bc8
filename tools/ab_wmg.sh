# A/B: HEAD worktree (_ab_head) vs working tree, config-1 WMG iteration probe
set -x
(cd _ab_head && timeout 300 python ../tools/probe_wmg_iter.py) > gpurun_out/ab_head.json 2>gpurun_out/ab_head.err
for ns in 0 8 12; do
  if [ $ns = 0 ]; then unset WMG_SYM64_NSPLIT; else export WMG_SYM64_NSPLIT=$ns; fi
  timeout 300 python tools/probe_wmg_iter.py > gpurun_out/ab_new$ns.json 2>gpurun_out/ab_new$ns.err
done
