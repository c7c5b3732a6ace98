python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_vv.py -m gpu -q -x -p no:cacheprovider --timeout 240 2>&1 | tail -2
for e in 1 0; do
  MASPCG_VV_STAGED=$e timeout 300 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vvs_tmp.json 2>> gpurun_out/vvs.err
  python -c "import json; d=json.load(open('gpurun_out/vvs_tmp.json')); print('staged=$e', round(d['value'],1), round(d['roofline']['avg_launch_ms']*1e3,1), round(d['roofline']['frac'],3))"
done
timeout 600 ncu --set full --clock-control none -k regex:"k_vv_terms3|k_vv_rows2" -s 4 -c 2 -o gpurun_out/prof_vv_stg python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
