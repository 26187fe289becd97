set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck.txt 2>&1; tail -3 gpurun_out/san_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/san_racecheck.txt 2>&1; tail -3 gpurun_out/san_racecheck.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
