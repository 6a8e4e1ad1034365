#!/bin/bash
# ncu --set full of one seed_thresholds and one ordered_cluster_sums launch (c2 shape, 1M rows)
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:seed_thresholds_async|ordered_cluster_sums_vec' -s 4 -c 2 -o gpurun_out/r1c_small2 \
  python tools/profile_fit.py --n 1000000 --iters 4 > gpurun_out/r1c_ncu_small.log 2>&1
