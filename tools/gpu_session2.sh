timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 1200 python tools/ab_lib.py tools/bin/libipm_head.so paper_1412_1127_b200/libipm.so 3 > gpurun_out/ab_loc.txt 2>&1; cat gpurun_out/ab_loc.txt
