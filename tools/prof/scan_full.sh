#!/bin/bash
# ncu --set full of one iteration-5 scan launch at the full c2 size (source-correlated)
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pruned_scan' -s 24 -c 1 -o gpurun_out/r1c_scan2 \
  python tools/profile_fit.py --n 1000000 --iters 6 > gpurun_out/r1c_ncu_scan2.log 2>&1
