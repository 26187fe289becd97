capture() {  # name kernel-regex command...
  local name=$1 kre=$2; shift 2
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${name}_sass.csv 2>/dev/null
  gzip -f gpurun_out/ncu_${name}_sass.csv; rm -f gpurun_out/prof_$name.ncu-rep
}
# NCU=<kernel option name> (warp | tile | rank)
case "$NCU" in
  warp) K=k_ragged_vec ;; tile) K=k_ragged_tile ;; lpr) K=k_ragged_lpr ;; *) K=k_ragged_rank ;;
esac
capture r${NCU}_pl $K python tools/prof_ragged.py $NCU powerlaw
capture r${NCU}_c4k $K python tools/prof_ragged.py $NCU const4096
ls gpurun_out
