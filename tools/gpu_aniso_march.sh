#!/bin/bash
# the plane-marching field-aligned operator: parity (march tests, whole aniso file), bench A/B against the TMA pair kernel
TAG=${1:-am}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_aniso.py -x -q -k "march" > gpurun_out/pytest_am_$TAG.log 2>&1; tail -2 gpurun_out/pytest_am_$TAG.log
timeout 900 python bench.py --operator aniso --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_am_$TAG.json 2>gpurun_out/bench_am_$TAG.err
MASPCG_ANISO_MARCH=0 timeout 900 python bench.py --operator aniso --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ap_$TAG.json 2>gpurun_out/bench_ap_$TAG.err
for f in am ap; do python -c "import json;d=json.load(open('gpurun_out/bench_${f}_$TAG.json'));r=d['roofline'];print('$f',round(d['value'],1),'mv_ms',round(r['avg_launch_ms'],4),'frac',round(r['frac'],3),d['clocks']['sm_mhz'])"; done
timeout 1200 python -m pytest tests/test_gpu_aniso.py -x -q > gpurun_out/pytest_aniso_$TAG.log 2>&1; tail -2 gpurun_out/pytest_aniso_$TAG.log
