#!/bin/bash
# bench line (headline only) + 2-rep diagnostics + one --set full capture of an iteration-5 scan launch
python bench.py --no-extra --no-cpu-baseline > gpurun_out/bench_h.log 2>&1
python tools/profile_fit.py --n 1000000 --iters 10 --reps 2 > gpurun_out/diag3.log 2>&1
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pruned_scan' -s 32 -c 1 -o gpurun_out/scan_cap \
  python tools/profile_fit.py --n 1000000 --iters 6 > gpurun_out/scan_cap.log 2>&1
