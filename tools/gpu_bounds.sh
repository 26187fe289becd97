# bounds-checked build (IPM_CHECK_BOUNDS: the marked ragged kernels trap on any out-of-range scratch, output or
# offsets index) under the ragged parity tests (not the out-of-contract test, which this build traps by design) and the sanitizer driver's cases (compute-sanitizer is not available
# on the GPU pool)
mkdir -p gpurun_out
IPM_LIB=tools/bin/libipm_bounds.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ragged and not beyond_nvalues" -p no:cacheprovider > gpurun_out/pytest_bounds.txt 2>&1; tail -2 gpurun_out/pytest_bounds.txt
IPM_LIB=tools/bin/libipm_bounds.so timeout 600 python tools/sanitize_run.py > gpurun_out/bounds_run.txt 2>&1; tail -2 gpurun_out/bounds_run.txt
