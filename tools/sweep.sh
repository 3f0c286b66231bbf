# K2 tuning sweep over build/variants/*: correctness subset + C2 and C4 bench per variant
for v in build/variants/*/; do
  name=$(basename $v)
  export TILEPREP_LIB=$PWD/$v/libtileprep.so
  timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "fast_equals_exact or full_size or capacity" > gpurun_out/sweep_${name}_test.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --latency-iters 50 > gpurun_out/sweep_${name}_c2.log 2>&1
  timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/sweep_${name}_c4.log 2>&1
done
echo sweep done
