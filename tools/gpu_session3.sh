# ncu: C3 with the TMA-ring segmented kernel vs the direct-load one; C2 f64 max (lane accumulators); 1 GiB read probe
capture() {  # name kernel-regex command...
  local name=$1 kre=$2; shift 2
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${name}_sass.csv 2>/dev/null
  gzip -f gpurun_out/ncu_${name}_sass.csv; rm -f gpurun_out/prof_$name.ncu-rep
}
capture c3_tma k_seg_tma python tools/prof_run.py --config c3 --reps 3 --seg-kernel tma
capture c3_warp k_seg_warp python tools/prof_run.py --config c3 --reps 3 --seg-kernel warp
capture c2_f64max k_flat_guided python tools/prof_run.py --config c2 --op max --dtype float64 --reps 3
capture c2_f32add k_flat_guided python tools/prof_run.py --config c2 --op + --dtype float32 --reps 3
tools/bin/read_probe 1024 > gpurun_out/read_probe_1g.txt; tools/bin/read_probe > gpurun_out/read_probe_8g.txt
cat gpurun_out/read_probe_1g.txt gpurun_out/read_probe_8g.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
