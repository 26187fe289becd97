# ragged kernels: parity (every kernel), timing A/B, optional ncu of the kernel named by $NCU
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -15 gpurun_out/pytest_ragged.txt
timeout 600 python tools/time_ragged.py ${TR_ARGS:-} > gpurun_out/time_ragged.txt 2>&1; cat gpurun_out/time_ragged.txt
if [ -n "$NCU" ]; then bash tools/gpu_prof_ragged.sh; fi
