python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -k "nccl or multirank or loop_modes or timing" 2>&1 | tail -2
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --maxit 400"
for sh in 150,300,600 150,300,75; do
  for v in "--force-comm" "--force-comm --comm peer"; do
    timeout 200 $B --shape $sh $v > gpurun_out/ct_tmp.json 2>> gpurun_out/ct.err
    python -c "import json; d=json.load(open('gpurun_out/ct_tmp.json')); k=d['per_kernel']; print('$sh $v', round(d['value'],1), round(1e6/d['value'],1), {x: (round(k[x]*1e3,2) if 'ms' in x else round(k[x],3)) for x in k if x.startswith('allreduce') or x.startswith('halo')})"
  done
done
