#!/bin/bash
# Round-2 final evidence: GPU test suite, the bench line, and the ncu launch list of the bench command.
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/final_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gputest.log
timeout 1500 python bench.py > gpurun_out/final_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/final_ncu_bench.log 2>&1
