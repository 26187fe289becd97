# ragged parity + compute-sanitizer (memcheck / racecheck / synccheck) over tools/sanitize_run.py
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -1 gpurun_out/pytest_ragged.txt
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.txt 2>&1; tail -2 gpurun_out/san_$t.txt
done
