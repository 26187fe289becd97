#!/bin/bash
# One ncu --set full capture per BASELINE config of the flat clause (C1, C2 float32 + / float64 max, C4 int32 ^ /
# int64 &&) and of the fused / 2-D rows; raw CSVs in gpurun_out/ncu_cfg_*.csv (tools/ncu_summary.py condenses them).
set -x
cap() {  # name kernel-regex args...
  local name=$1 kre=$2; shift 2
  timeout 300 ncu --set full --clock-control none -k regex:$kre -s 2 -c 1 -o gpurun_out/cfg_$name \
    python tools/prof_run.py "$@" > gpurun_out/ncu_cfg_$name.log 2>&1
  ncu -i gpurun_out/cfg_$name.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_$name.csv 2>/dev/null
  rm -f gpurun_out/cfg_$name.ncu-rep
}
cap c1_i32_add k_flat --config c1 --dtype int32 --op + --reps 3
cap c2_f32_add k_flat_guided --config c2 --dtype float32 --op + --reps 3
cap c2_f64_max k_flat_guided --config c2 --dtype float64 --op max --reps 3
cap c4_i32_xor k_flat_guided --config c4 --dtype int32 --op ^ --reps 3
cap c4_i64_land k_flat_guided --config c4 --dtype int64 --op '&&' --reps 3
cap stats_f32 k_fused --config stats --reps 3
cap dot_f32 k_fused --config dot --reps 3
cap twod_f32 k_2d --config 2d --reps 3
ls -la gpurun_out/
