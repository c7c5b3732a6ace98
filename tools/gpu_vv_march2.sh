#!/bin/bash
# vv march: parity of the march tests, bench line, ncu --set full of k_vv_march
TAG=${1:-vvm2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python -m pytest tests/test_gpu_vv.py -x -q -k "march or c3v or multirank" > gpurun_out/pytest_march_$TAG.log 2>&1
tail -3 gpurun_out/pytest_march_$TAG.log
timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_vv_$TAG.json'));r=d['roofline'];print('VALUE',d['value'],'mv_ms',r['avg_launch_ms'],'frac',r['frac'],'sm',d['clocks'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_march" -s 3 -c 1 \
    -o gpurun_out/prof_vvm_$TAG python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_vvm_$TAG.log 2>&1
