#!/bin/bash
# One GPU session: tests, bench, launch list, ncu captures of the dominant kernels. Output in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-suite --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_flat_guided -s 2 -c 1 \
  -o gpurun_out/prof_c5_guided python tools/prof_run.py --config c5 --reps 3 > gpurun_out/ncu_c5.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_seg_warp -s 2 -c 1 \
  -o gpurun_out/prof_c3_seg python tools/prof_run.py --config c3 --reps 3 > gpurun_out/ncu_c3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_ragged_vec -s 2 -c 1 \
  -o gpurun_out/prof_ragged python tools/prof_ragged.py > gpurun_out/ncu_ragged.log 2>&1
ls -la gpurun_out/
