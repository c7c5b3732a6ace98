#!/bin/bash
# One GPU round trip: parity tests, smoke, bench, ncu launch list + full capture of the stencil.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 0 --maxit 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 3 -c 1 -o gpurun_out/prof_matvec_$TAG \
    python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_pupdate" -s 4 -c 2 -o gpurun_out/prof_upd_$TAG \
    python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_upd_$TAG.log 2>&1
ls -la gpurun_out
