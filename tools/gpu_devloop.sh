#!/bin/bash
# conditional-graph device loop: parity tests and A/B against the host chunk loop (P=1 c3, P=8 slab plain / peer)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_dl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "device_loop" > gpurun_out/pytest_dl.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dl.log
out=gpurun_out/devloop.txt; rm -f $out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for rep in 1 2; do
  for sh in "150,300,600 " "150,300,75 --maxit 400" "150,300,75 --maxit 400 --force-comm --comm peer"; do
    for dl in 0 1; do
      set -- $sh
      timeout 300 $B --shape $1 ${@:2} --device-loop $dl > gpurun_out/dl_tmp.json 2>> gpurun_out/dl.err
      python -c "import json; d=json.load(open('gpurun_out/dl_tmp.json')); print('$sh', 'device_loop=$dl', round(d['value'],1), 'it/s', round(1e6/d['value'],2), 'us/it', d['run']['loop'], d['clocks']['sm_mhz'])" >> $out
    done
  done
done
