for r in 1 2; do for v in b16 fix0 fix1; do
  TILEPREP_LIB=$PWD/build/variants/$v/libtileprep.so timeout 300 python bench.py --workload c3 --latency-iters 1000 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['p50_ms'], d['p99_ms'], d['graph_floor_p50_ms'])" >> gpurun_out/c3var.log
done; done
