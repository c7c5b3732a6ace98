#!/bin/bash
# one-GPU projection of the strong-scaling iteration: the per-GPU phi-slab of c3 at P = 2, 4, 8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
for sh in 150,300,600 150,300,300 150,300,150 150,300,75; do
  for v in "" "--force-comm" "--force-comm --comm peer" "--force-comm --path 4"; do
    timeout 200 $B --shape $sh $v > gpurun_out/slab_tmp.json 2>> gpurun_out/slab.err
    python -c "import json; d=json.load(open('gpurun_out/slab_tmp.json')); print('$sh', '$v', round(d['value'],1), 'us/it', round(1e6/d['value'],1), d['config']['parallelism'])"
  done
done
