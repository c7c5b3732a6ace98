python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for lb in 3 2 4; do
  sed -i "s/__launch_bounds__(kVVThreads, [0-9]) k_vv_rows2(/__launch_bounds__(kVVThreads, $lb) k_vv_rows2(/" paper_2303_03398_b200/csrc/vv.cu
  python -m paper_2303_03398_b200.build > /dev/null 2>&1
  timeout 300 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/lb_tmp.json 2>> gpurun_out/lb.err
  python -c "import json; d=json.load(open('gpurun_out/lb_tmp.json')); print('rows2 lb=$lb', round(d['value'],1), round(d['roofline']['avg_launch_ms']*1e3,1), d['clocks']['sm_mhz'])"
done; done
