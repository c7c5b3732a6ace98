#!/bin/bash
# the pair-per-thread aniso kernel: parity, bench lines (2 / 3 blocks per SM, the flat kernel), ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_aniso.py -x -q > gpurun_out/pytest_aniso3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_aniso3.log
timeout 600 python bench.py --operator aniso --steps 5 --warmup 3 > gpurun_out/bench_aniso_c3a.json 2> gpurun_out/bench_aniso.err
MASPCG_ANISO_BLOCKS=3 timeout 600 python bench.py --operator aniso --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_aniso_b3.json 2>> gpurun_out/bench_aniso.err
timeout 600 python bench.py --operator aniso --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --vec 0 > gpurun_out/bench_aniso_flat.json 2>> gpurun_out/bench_aniso.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aniso_vec2" -s 3 -c 1 \
    -o gpurun_out/prof_aniso_vec2 python bench.py --operator aniso --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aniso2.log 2>&1
for f in bench_aniso_c3a bench_aniso_b3 bench_aniso_flat; do
  python -c "import json; d=json.load(open('gpurun_out/$f.json')); r=d['roofline']; print('$f', round(d['value'],1), 'it/s', d['run']['iters_per_solve'], 'it/solve', 'stencil ms', r['avg_launch_ms'], 'frac', r['frac'])" >> gpurun_out/aniso_summary.txt
done
