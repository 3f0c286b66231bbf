#!/bin/bash
# Round-2 closing measurement: GPU suite, smoke, default bench line, reference arm,
# the ncu launch list of a short bench run and the ncu capture of K2 (then of K8's
# inflate), each only after its own command ran clean without ncu.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/bench_small.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-iters 20 > gpurun_out/ncu_launch.log 2>&1
timeout 120 python tools/profile_k2.py > gpurun_out/prof_plain.log 2>&1 && timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_tile_tma -s 2 -c 1 -o gpurun_out/k2_r02b python tools/profile_k2.py > gpurun_out/ncu_full.log 2>&1
echo done
