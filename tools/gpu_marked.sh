# marked ragged rows: parity of every ragged kernel (incl. marked), full-size ragged parity, timing warp / rank /
# marked on the ragged recipes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged.txt 2>&1; tail -3 gpurun_out/pytest_ragged.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k ragged -p no:cacheprovider > gpurun_out/pytest_ragged_full.txt 2>&1; tail -3 gpurun_out/pytest_ragged_full.txt
KERNELS=${KERNELS:-warp,rank,lpr,marked} timeout 900 python tools/time_ragged.py > gpurun_out/time_marked.txt 2>&1; cat gpurun_out/time_marked.txt
