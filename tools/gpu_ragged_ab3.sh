# ragged A/B: parity of every ragged kernel, then interleaved timing of the warp kernel (default build) and of
# kernel $K under each IPM_LIB in $LIBS
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -3 gpurun_out/pytest_ragged.txt
for round in 1 2; do
  KERNELS=warp timeout 300 python tools/time_ragged.py 2>&1 | sed "s/^/default /"
  for L in $LIBS; do
    IPM_LIB=$L KERNELS=$K timeout 300 python tools/time_ragged.py 2>&1 | sed "s|^|$(basename $L) |"
  done
done > gpurun_out/ab_ragged.txt
cat gpurun_out/ab_ragged.txt
if [ -n "$NCU" ]; then bash tools/gpu_prof_ragged.sh; fi
