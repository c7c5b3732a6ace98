python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_persist.py -m gpu -q -x -p no:cacheprovider --timeout 240 2>&1 | tail -15
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
for sh in 150,300,75; do
  for v in "--path 1" "--path 5"; do
    timeout 200 $B --shape $sh $v > gpurun_out/ps_tmp.json 2>> gpurun_out/ps.err
    python -c "import json; d=json.load(open('gpurun_out/ps_tmp.json')); print('$sh', '$v', round(d['value'],1), 'us/it', round(1e6/d['value'],1))"
  done
done
