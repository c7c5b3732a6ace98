python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_vv.py -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -3
for tj in 0 6; do
  MASPCG_VV_TJ=$tj timeout 300 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vvf_tmp.json 2>> gpurun_out/vvf.err
  python -c "import json; d=json.load(open('gpurun_out/vvf_tmp.json')); print('tj=$tj', round(d['value'],1), round(d['roofline']['avg_launch_ms']*1e3,1), round(d['roofline']['frac'],3))"
done
