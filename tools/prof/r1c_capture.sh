#!/bin/bash
# Round-1 (third session) evidence: launch list of the bench command, --set full captures of the
# scan and the gate GEMM at the full c2 size (iteration-5 launches), traffic.json for bench.py.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1c_ncu_bench.log 2>&1
# profile_fit at 1M rows: 8 gate + 8 scan launches per pruned iteration; skip iterations 2-4
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pruned_scan|gemm_tf32x3_kernel<\(int\)3' -s 48 -c 2 -o gpurun_out/r1c_full \
  python tools/profile_fit.py --n 1000000 --iters 6 > gpurun_out/r1c_ncu_full.log 2>&1
