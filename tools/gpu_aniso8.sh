#!/bin/bash
# TMA aniso kernel variants: register copies vs lazy tile reads, 2 vs 3 blocks per SM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a8.log 2>&1
out=gpurun_out/aniso8.txt; rm -f $out
for rep in 1 2; do
  for t in "MASPCG_ANISO_LAZY=0 MASPCG_ANISO_TMA_BLOCKS=2" "MASPCG_ANISO_LAZY=1 MASPCG_ANISO_TMA_BLOCKS=2" "MASPCG_ANISO_LAZY=1 MASPCG_ANISO_TMA_BLOCKS=3" "MASPCG_ANISO_LAZY=0 MASPCG_ANISO_TMA_BLOCKS=3"; do
    env $t timeout 600 python bench.py --operator aniso --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/an_tmp.json 2>> gpurun_out/an8.err
    python -c "import json; d=json.load(open('gpurun_out/an_tmp.json')); r=d['roofline']; print('$t', round(d['value'],1), 'it/s', 'stencil us', round(r['avg_launch_ms']*1e3,1), 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])" >> $out
  done
done
MASPCG_ANISO_LAZY=1 timeout 900 python -m pytest tests/test_gpu_aniso.py -x -q > gpurun_out/pytest_aniso8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_aniso8.log
