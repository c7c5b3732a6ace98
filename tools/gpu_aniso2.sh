#!/bin/bash
# aniso bench line + ncu of its stencil; L2 plan combinations on the P=8 slab; edge-case tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a2.log 2>&1
timeout 600 python bench.py --operator aniso --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_aniso_c3a.json 2> gpurun_out/bench_aniso.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aniso_flat" -s 3 -c 1 \
    -o gpurun_out/prof_aniso_flat python bench.py --operator aniso --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aniso.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
out=gpurun_out/l2combo.txt
run() {  # label, env, shape, extra
  env MASPCG_L2_VERBOSE=1 $2 timeout 200 $B --shape $3 $4 > gpurun_out/lc_tmp.json 2>> gpurun_out/lc.err
  python -c "import json; d=json.load(open('gpurun_out/lc_tmp.json')); print('$3', '$1', '$4', round(d['value'],1), 'us/it', round(1e6/d['value'],2))" >> $out
}
for rep in 1 2; do
  run off "MASPCG_L2_MASK=0" 150,300,75 ""
  run auto045-DP "X=1" 150,300,75 ""
  run DR "MASPCG_L2_MASK=0x11" 150,300,75 ""
  run PR "MASPCG_L2_MASK=0x14" 150,300,75 ""
  run DPQ "MASPCG_L2_MASK=0x105" 150,300,75 ""
  run D "MASPCG_L2_MASK=0x1" 150,300,75 ""
  run P "MASPCG_L2_MASK=0x4" 150,300,75 ""
done
for v in "--force-comm" "--force-comm --comm peer"; do
  run auto045 "X=1" 150,300,75 "$v"
done
run off "MASPCG_L2_MASK=0" 150,300,150 ""
run auto045 "X=1" 150,300,150 ""
timeout 600 python -m pytest tests/test_gpu_edge_cases.py -x -q > gpurun_out/pytest_edge.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_edge.log
