#!/bin/bash
# One GPU round trip: parity tests, smoke, bench lines, ncu launch list + full captures.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag] [pytest-args]
set -x
TAG=${1:-r01}
PYARGS=${2:-"tests -m gpu -x -q"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest $PYARGS > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --path 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_path2_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --arith 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_fast_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --path 3 --no-cpu-baseline --no-e2e --sts-stages 10 > gpurun_out/bench_path3_$TAG.json 2>> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 0 --maxit 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_matvec_vec2|k_update_vec2|k_pupdate_vec2" -s 4 -c 3 \
    -o gpurun_out/prof_default_$TAG python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_pass_b" -s 6 -c 2 -o gpurun_out/prof_fused_$TAG \
    python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e --path 2 > gpurun_out/ncu_full_fused_$TAG.log 2>&1
ls -la gpurun_out
