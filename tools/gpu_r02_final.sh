#!/bin/bash
# Round-2 final evidence: the whole -m gpu suite, smoke, the default bench line (c3, also the reference arm), the vv and
# aniso bench lines, the ncu launch list of a short default run, ncu --set full of the marching vector operator
TAG=${1:-fin}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
timeout 900 python bench.py --operator vv --steps 5 --warmup 3 > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
timeout 900 python bench.py --operator aniso --steps 5 --warmup 3 > gpurun_out/bench_aniso_$TAG.json 2> gpurun_out/bench_aniso_$TAG.err
for f in c3 vv aniso; do python -c "import json;d=json.load(open('gpurun_out/bench_${f}_$TAG.json'));r=d['roofline'];print('$f',round(d['value'],1),d['unit'],'frac',round(r['frac'],3),'e2e',round(d['e2e']['value'],1) if d.get('e2e') else None,d['clocks']['sm_mhz'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_vv_$TAG.csv \
    python bench.py --operator vv --steps 1 --warmup 0 --maxit 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_vv_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_march" -s 6 -c 1 \
    -o gpurun_out/prof_vvm_$TAG python bench.py --operator vv --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_vvm_$TAG.log 2>&1
