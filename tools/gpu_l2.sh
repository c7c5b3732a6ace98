#!/bin/bash
# L2 residency (MASPCG_OPT_L2_KEEP) A/B on the per-GPU phi-slabs of c3 (one-GPU strong-scaling projection)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_l2.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
run() {  # label, env, shape, extra
  env $2 timeout 200 $B --shape $3 $4 > gpurun_out/l2_tmp.json 2>> gpurun_out/l2.err
  python -c "import json; d=json.load(open('gpurun_out/l2_tmp.json')); print('$3', '$1', '$4', round(d['value'],1), 'us/it', round(1e6/d['value'],2))" >> gpurun_out/l2_ab.txt
}
for sh in 150,300,75 150,300,150; do
  run off "MASPCG_L2_MASK=0" $sh ""
  for b in 0.5 0.65 0.75 0.85 0.95; do run "budget$b" "MASPCG_L2_BUDGET=$b" $sh ""; done
  run "D+T" "MASPCG_L2_MASK=0x401" $sh ""
  run "DPR+Tfirst" "MASPCG_L2_MASK=0xC15" $sh ""
  run "DPRX+Tfirst" "MASPCG_L2_MASK=0xC55" $sh ""
  run "DPRX" "MASPCG_L2_MASK=0x55" $sh ""
done
for sh in 150,300,75 150,300,150; do
  for v in "--force-comm" "--force-comm --comm peer"; do
    run off "MASPCG_L2_MASK=0" $sh "$v"
    run auto "X=1" $sh "$v"
  done
done
for sh in 150,300,300 150,300,600; do
  run off "MASPCG_L2_MASK=0" $sh ""
  run auto "X=1" $sh ""
  run "budget0.5" "MASPCG_L2_BUDGET=0.5" $sh ""
  run "budget0.9" "MASPCG_L2_BUDGET=0.9" $sh ""
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest_l2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_l2.log
