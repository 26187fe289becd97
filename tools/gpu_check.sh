# full GPU check of the tree: smoke, the -m gpu suite, compute-sanitizer (memcheck / racecheck / synccheck) over
# tools/sanitize_run.py
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; tail -20 gpurun_out/pytest_gpu.txt
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.txt 2>&1; tail -4 gpurun_out/san_$t.txt
done
