# marked ragged rows: ragged parity, A/B against $LIBS, ncu launch list + --set full of both passes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -1 gpurun_out/pytest_ragged.txt
bash tools/gpu_marked_ab.sh
KERNELS=marked ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_marked.py > gpurun_out/ncu_marked_list.csv 2> gpurun_out/ncu_marked.err
KERNELS=marked timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ragged_m -c 2 -o gpurun_out/ncu_marked python tools/prof_marked.py > gpurun_out/ncu_marked_full.log 2>&1; tail -1 gpurun_out/ncu_marked_full.log
