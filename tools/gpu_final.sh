# round-end evidence: smoke, the -m gpu suite, the driver-style bench line, the ncu launch list of the bench
# command (per-launch times, --clock-control none) and one ncu --set full capture of the headline kernel
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.txt 2>&1; tail -14 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-suite --no-e2e > gpurun_out/ncu_bench.log 2>&1; tail -3 gpurun_out/ncu_bench.log
