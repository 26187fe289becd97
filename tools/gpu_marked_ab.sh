# marked ragged rows: interleaved A/B of library builds ($LIBS, the default build first) on the marked path
mkdir -p gpurun_out
for round in 1 2; do
  for L in paper_1412_1127_b200/libipm.so $LIBS; do
    IPM_LIB=$L CASES="${CASES:-powerlaw:16777216:16,const:4194304:64}" OPS="${OPS:-+:float32,^:int32,+:float64}" KERNELS=${KERNELS:-marked} timeout 300 python tools/time_ragged.py 2>&1 | sed "s|^|$(basename $L) |"
  done
done > gpurun_out/ab_marked.txt
python tools/ab_ragged_table.py gpurun_out/ab_marked.txt
