#!/bin/bash
# Round-2 evidence: diagnostics of the current build at c2, the bench launch list, and --set full
# captures of the scan (iteration 5), the exact-chain rotation GEMM and one gate GEMM.
set -x
python tools/profile_fit.py --n 1000000 --iters 10 > gpurun_out/r2_diag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r2_ncu_bench.log 2>&1
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pruned_scan' -s 32 -c 1 -o gpurun_out/r2_scan \
  python tools/profile_fit.py --n 1000000 --iters 6 > gpurun_out/r2_ncu_scan.log 2>&1
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:sgemm_chain|gemm_tf32x3_kernel<\(int\)3' -s 0 -c 1 -o gpurun_out/r2_chain \
  python tools/profile_fit.py --n 1000000 --iters 2 > gpurun_out/r2_ncu_chain.log 2>&1
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tf32x3_kernel<\(int\)3' -s 30 -c 1 -o gpurun_out/r2_gate \
  python tools/profile_fit.py --n 1000000 --iters 6 > gpurun_out/r2_ncu_gate.log 2>&1
ls -la gpurun_out
