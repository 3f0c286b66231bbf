for v in pdl2 pdl3 pdl0; do
  for r in 1 2; do
  TILEPREP_LIB=$PWD/build/variants/$v/libtileprep.so timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pdl_${v}_$r.log 2>&1
  done
done
