set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 python bench.py --workload c4 --steps 3 --warmup 2 > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --workload c1 > gpurun_out/bench_c1.log 2>&1
timeout 600 python bench.py --workload c3 > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/bench_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/ncu_launch.log 2>&1
timeout 120 python tools/profile_k2.py > gpurun_out/prof_plain.log 2>&1 && timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_tile_tma -s 2 -c 1 -o gpurun_out/k2_final python tools/profile_k2.py > gpurun_out/ncu_full.log 2>&1
echo done
