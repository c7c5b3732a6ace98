#!/bin/bash
# round evidence: default bench line, vv line, cg1 line, launch list and ncu --set full of the hot kernels
TAG=${1:-ev}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
timeout 900 python bench.py --operator vv > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
timeout 600 python bench.py --path 4 --no-cpu-baseline > gpurun_out/bench_cg1_$TAG.json 2> gpurun_out/bench_cg1_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 0 --maxit 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_matvec_vec2|k_update_vec2|k_pupdate_vec2" -s 4 -c 3 \
    -o gpurun_out/prof_default_$TAG python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg1_update" -s 2 -c 1 \
    -o gpurun_out/prof_cg1_$TAG python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e --path 4 > gpurun_out/ncu_cg1_$TAG.log 2>&1
ls gpurun_out | grep $TAG
