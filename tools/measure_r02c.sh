mkdir -p gpurun_out/m8
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/m8/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/m8/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/m8/bench_default.log 2>gpurun_out/m8/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/m8/bench_reference.log 2>&1
timeout 300 python tools/jpeg_corpus_check.py build/corpus500/images > gpurun_out/m8/corpus500.json 2>&1
timeout 300 python tools/jpeg_bench.py > gpurun_out/m8/jpeg_bench.log 2>&1
timeout 300 python tools/png_bench.py > gpurun_out/m8/png_bench.log 2>&1
timeout 300 python tools/png_corpus_check.py 300 > gpurun_out/m8/png_corpus.json 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/m8/bench_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m8/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/m8/ncu_launch.log 2>&1
tail -1 gpurun_out/m8/pytest_gpu.log; cat gpurun_out/m8/smoke.log | tail -1; tail -c 600 gpurun_out/m8/corpus500.json
echo done
