# ragged warp-kernel A/B over library builds ($LIBS), interleaved, plus the ragged parity tests on the default build
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -3 gpurun_out/pytest_ragged.txt
for round in 1 2; do
  for L in $LIBS; do
    IPM_LIB=$L KERNELS=${KERNELS:-warp} timeout 300 python tools/time_ragged.py ${TR_ARGS:-} 2>&1 | sed "s|^|$(basename $L) |"
  done
done > gpurun_out/ab_ragged.txt
cat gpurun_out/ab_ragged.txt
