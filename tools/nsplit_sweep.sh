#!/bin/bash
# Cluster-size sweep of the four-image run-layout backprojector (needs a build whose
# symrun_nsplit reads WMG_BWD_NSPLIT; the shipped formula came from this sweep).
for n in 512 768 1024 1280 1408 1536; do
  for ns in 0 1 2 3 4 5 6 8 10 12 16; do
    if [ $ns = 0 ]; then unset WMG_BWD_NSPLIT; else export WMG_BWD_NSPLIT=$ns; fi
    echo -n "ns=$ns "; python tools/probe_size_scan.py $n | sed 's/fwd.*bwd/bwd/'
  done
done
