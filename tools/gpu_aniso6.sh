#!/bin/bash
# TMA-staged double-buffered aniso kernel: parity + bench A/B against the all-global pair kernel, ncu of the tile kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a6.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_aniso.py -x -q > gpurun_out/pytest_aniso6.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_aniso6.log
out=gpurun_out/aniso6.txt; rm -f $out
for rep in 1 2; do
  for t in "1 MASPCG_ANISO_TMA_BLOCKS=3" "1 MASPCG_ANISO_TMA_BLOCKS=2" "0 X=1"; do
    set -- $t
    env MASPCG_ANISO_TMA=$1 $2 timeout 600 python bench.py --operator aniso --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/an_tmp.json 2>> gpurun_out/an6.err
    python -c "import json; d=json.load(open('gpurun_out/an_tmp.json')); r=d['roofline']; print('tma=$1 $2', round(d['value'],1), 'it/s', 'stencil us', round(r['avg_launch_ms']*1e3,1), 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])" >> $out
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aniso_tma" -s 3 -c 1 \
    -o gpurun_out/prof_aniso_tma python bench.py --operator aniso --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aniso6.log 2>&1
