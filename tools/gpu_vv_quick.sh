#!/bin/bash
# vv march quick check: march parity tests, the probe, the bench line (with-dot loop kernel)
TAG=${1:-q}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_vv.py -x -q -k "march" 2>&1 | tail -2
timeout 300 python tools/vv_march_probe.py c3v > gpurun_out/probe_$TAG.txt 2>&1; cat gpurun_out/probe_$TAG.txt
timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vv_$TAG.json 2>gpurun_out/bench_vv_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_vv_$TAG.json'));r=d['roofline'];print('VALUE',d['value'],'mv_ms',r['avg_launch_ms'],'frac',r['frac'],d['clocks'])"
