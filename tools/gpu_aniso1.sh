#!/bin/bash
# First GPU run of the field-aligned operator (parity tests) + the whole-class L2 plan on the slabs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_a1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_aniso.py -x -q > gpurun_out/pytest_aniso1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_aniso1.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
out=gpurun_out/l2plan.txt
run() {  # label, env, shape, extra
  env MASPCG_L2_VERBOSE=1 $2 timeout 200 $B --shape $3 $4 > gpurun_out/lp_tmp.json 2>> gpurun_out/lp.err
  python -c "import json; d=json.load(open('gpurun_out/lp_tmp.json')); print('$3', '$1', '$4', round(d['value'],1), 'us/it', round(1e6/d['value'],2))" >> $out
}
for rep in 1 2; do
for sh in 150,300,75 150,300,150 150,300,300 150,300,600; do
  run off "MASPCG_L2_MASK=0" $sh ""
  run auto "X=1" $sh ""
done
run D-only "MASPCG_L2_BUDGET=0.25" 150,300,75 ""
run DP "MASPCG_L2_BUDGET=0.45" 150,300,75 ""
run D-only-P4 "MASPCG_L2_BUDGET=0.45" 150,300,150 ""
done
for v in "--force-comm" "--force-comm --comm peer"; do
  run off "MASPCG_L2_MASK=0" 150,300,75 "$v"
  run auto "X=1" 150,300,75 "$v"
done
grep "l2 plan" gpurun_out/lp.err | sort | uniq -c >> $out
