#!/bin/bash
# One GPU session: tests, bench, launch list, ncu captures of the dominant kernels. Output in gpurun_out/
# (ncu reports are exported to CSV on the box; only the C5 report itself is kept: gpurun returns <= 64 MiB).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-suite --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
capture() {  # name kernel-regex command...
  local name=$1 kre=$2; shift 2
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${name}_sass.csv 2>/dev/null
}
capture c5_guided k_flat_guided python tools/prof_run.py --config c5 --reps 3
capture c3_seg k_seg_warp python tools/prof_run.py --config c3 --reps 3
capture ragged k_ragged_vec python tools/prof_ragged.py
rm -f gpurun_out/prof_c3_seg.ncu-rep gpurun_out/prof_ragged.ncu-rep gpurun_out/ncu_*_sass.csv.gz
gzip -f gpurun_out/ncu_*_sass.csv
du -sh gpurun_out; ls -la gpurun_out/
