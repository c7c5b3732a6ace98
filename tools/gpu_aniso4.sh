#!/bin/bash
# branch-free pair kernel: parity, bench, ncu; the golden full-size tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_aniso.py tests/test_gpu_golden.py -x -q > gpurun_out/pytest_aniso4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_aniso4.log
timeout 600 python bench.py --operator aniso --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_aniso4.json 2> gpurun_out/bench_aniso4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aniso_vec2" -s 3 -c 1 \
    -o gpurun_out/prof_aniso_vec2b python bench.py --operator aniso --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aniso4.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_aniso4.json')); r=d['roofline']; print('branchfree', round(d['value'],1), 'it/s', d['run']['iters_per_solve'], 'it/solve', 'stencil ms', r['avg_launch_ms'], 'frac', r['frac'])" >> gpurun_out/aniso_summary.txt
