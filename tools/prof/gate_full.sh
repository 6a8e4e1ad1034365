#!/bin/bash
# ncu --set full capture of one GATE GEMM launch (iteration-5-ish batch of a 200K-row fit)
SKM_DIAG=0 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tf32x3_kernel<\(int\)3, \(int\)3' -s 8 -c 1 -o gpurun_out/r1c_gate2 \
  python tools/profile_fit.py --n 200000 --iters 6 > gpurun_out/r1c_ncu_gate.log 2>&1
