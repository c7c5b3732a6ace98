#!/bin/bash
# vector viscosity iteration loop: parity subset, bench line, ncu of the stencil phases
TAG=${1:-vvi}
bash tools/gpu_vv.sh $TAG "bitwise or solve_exact or coronal or multirank or edge"
timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
cat gpurun_out/bench_vv_$TAG.json | python -c "import json,sys; d=json.load(sys.stdin); print('VV', d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['per_kernel'])"
bash tools/gpu_vv_ncu.sh $TAG
