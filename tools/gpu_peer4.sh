python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 700 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl.py -m gpu -q -p no:cacheprovider --timeout 240 2>&1 | tail -3
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for v in "--path 1" "--path 1 --force-comm" "--path 1 --force-comm --comm peer" "--path 4 --force-comm --comm peer"; do
  timeout 200 $B $v > gpurun_out/bench_p_tmp.json 2>> gpurun_out/bench_p.err
  python -c "import json; d=json.load(open('gpurun_out/bench_p_tmp.json')); print('$v', round(d['value'],1), d['config']['iters_per_solve'], round(d['ms_per_step'],2), d['config']['parallelism'])"
done
