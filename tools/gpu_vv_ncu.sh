#!/bin/bash
# ncu --set full of the vector stencil phases only
TAG=${1:-vvn}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_terms|k_vv_rows" -s 6 -c 2 \
    -o gpurun_out/prof_vv_$TAG python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_vv_$TAG.log 2>&1
