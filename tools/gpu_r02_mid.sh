#!/bin/bash
# Mid-round check: the whole -m gpu suite (golden fixtures excluded while they are regenerated), smoke, the
# default bench line, the strong-scaling slab projection, bench self-launch shared-GPU check
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_mid.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_golden.py > gpurun_out/pytest_gpu_mid.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_mid.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_mid.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_mid.log
timeout 900 python bench.py > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
out=gpurun_out/slab_r02.txt
for sh in 150,300,600 150,300,300 150,300,150 150,300,75; do
  for v in "" "--force-comm" "--force-comm --comm peer" "--force-comm --path 4"; do
    timeout 200 $B --shape $sh $v > gpurun_out/sl_tmp.json 2>> gpurun_out/sl.err
    python -c "import json; d=json.load(open('gpurun_out/sl_tmp.json')); print('$sh', '$v', round(d['value'],1), 'us/it', round(1e6/d['value'],2), d['config']['parallelism'])" >> $out
  done
  timeout 200 $B --shape $sh --l2-keep 0 > gpurun_out/sl_tmp.json 2>> gpurun_out/sl.err
  python -c "import json; d=json.load(open('gpurun_out/sl_tmp.json')); print('$sh', '--l2-keep 0', round(d['value'],1), 'us/it', round(1e6/d['value'],2))" >> $out
done
MASPCG_BENCH_SHARED_GPU=1 timeout 300 python bench.py --gpus 2 --comm peer --steps 1 --warmup 3 --maxit 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_selflaunch.json 2> gpurun_out/bench_selflaunch.err; echo "exit $?" >> gpurun_out/bench_selflaunch.err
