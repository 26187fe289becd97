#!/bin/bash
# usage: tools/ncu_capture.sh NAME KERNEL_REGEX COMMAND...   (on the GPU box)
# One `ncu --set full` capture of the 3rd matching launch, exported to CSV (raw, details, SASS source) under
# gpurun_out/; the .ncu-rep itself is deleted (gpurun returns <= 64 MiB).
name=$1 kre=$2; shift 2
timeout 400 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
  -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${name}_sass.csv 2>/dev/null
gzip -f gpurun_out/ncu_${name}_sass.csv
[ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/prof_$name.ncu-rep
