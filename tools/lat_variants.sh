# batch-1 latency pieces per variant library, interleaved rounds
for r in 1 2 3; do
  for v in build/variants/*/; do
    name=$(basename $v)
    TILEPREP_LIB=$PWD/$v/libtileprep.so timeout 300 python tools/latency_breakdown.py >> gpurun_out/lat_${name}.log 2>&1
  done
done
