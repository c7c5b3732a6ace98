#!/bin/bash
# vector viscosity: bench line (c3v), launch list, ncu --set full of the vector stencil
TAG=${1:-vvp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python bench.py --operator vv --steps 3 --warmup 3 > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
cat gpurun_out/bench_vv_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_vv_$TAG.csv \
    python bench.py --operator vv --steps 1 --warmup 0 --maxit 20 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_vv_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_terms|k_vv_rows" -s 6 -c 2 \
    -o gpurun_out/prof_vv_$TAG python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_vv_$TAG.log 2>&1
ls gpurun_out | tail -5
