#!/bin/bash
# round-end refresh of the strong-scaling slab projection (per-GPU phi-slabs of c3 on one GPU, 400 iterations)
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
out=gpurun_out/slab_r02end.txt; rm -f $out
for sh in 150,300,600 150,300,300 150,300,150 150,300,75; do
  for v in "" "--force-comm" "--force-comm --comm peer"; do
    timeout 200 $B --shape $sh $v > gpurun_out/sl_tmp.json 2>> gpurun_out/sl.err
    python -c "import json; d=json.load(open('gpurun_out/sl_tmp.json')); print('$sh', '$v', round(d['value'],1), 'it/s', round(1e6/d['value'],2), 'us/it', d['clocks']['sm_mhz'], 'MHz')" >> $out
  done
done
cat $out
