for dt in int32 int64 float32 float64; do for op in '+' '*' max min '&' '|' '^' '&&' '||'; do
  python tools/repro_op.py "$op" $dt 4194304 2>&1 | tail -1; done; done
