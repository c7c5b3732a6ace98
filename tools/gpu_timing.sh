python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for v in "--kernel-timing 2" "--kernel-timing 3" "--kernel-timing 0" "--kernel-timing 2" "--kernel-timing 3"; do
  timeout 200 $B $v > gpurun_out/bench_t_tmp.json 2>> gpurun_out/bench_t.err
  python -c "import json; d=json.load(open('gpurun_out/bench_t_tmp.json')); r=d['roofline']; print('$v', round(d['value'],1), round((r['avg_launch_ms'] or 0)*1e3,1), r['frac'], d['per_kernel']['update_GBps'], d['per_kernel']['p_update_GBps'], d['clocks'])"
done
