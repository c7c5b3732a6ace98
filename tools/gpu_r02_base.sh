#!/bin/bash
# Round-2 baseline on a fresh box: build, the whole -m gpu suite, smoke, the default bench line,
# and the P=8 slab projection (plain, one-rank NCCL, one-rank peer).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_base.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_base.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
for v in "" "--force-comm" "--force-comm --comm peer"; do
  timeout 200 $B --shape 150,300,75 $v > gpurun_out/slab_tmp.json 2>> gpurun_out/slab.err
  python -c "import json; d=json.load(open('gpurun_out/slab_tmp.json')); print('150,300,75', '$v', round(d['value'],1), 'us/it', round(1e6/d['value'],1))" >> gpurun_out/slab_base.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_base.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_base.log
