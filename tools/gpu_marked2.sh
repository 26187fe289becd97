# marked ragged rows: ragged parity, timing, ncu launch list and one --set full capture of each marked pass
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -2 gpurun_out/pytest_ragged.txt
CASES="powerlaw:16777216:16,const:4194304:64,uniform:16777216:16" OPS="+:float32,^:int32,+:float64" KERNELS=warp,marked timeout 600 python tools/time_ragged.py > gpurun_out/time_marked.txt 2>&1; cat gpurun_out/time_marked.txt
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/prof_marked.py > gpurun_out/ncu_marked_list.csv 2> gpurun_out/ncu_marked.err
KERNELS=marked timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ragged_m -c 2 -o gpurun_out/ncu_marked python tools/prof_marked.py > gpurun_out/ncu_marked_full.log 2>&1; tail -2 gpurun_out/ncu_marked_full.log
