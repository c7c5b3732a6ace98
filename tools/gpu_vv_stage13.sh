# vv phase 1 with the j-1 streams staged and the r-neighbours taken from the neighbouring lanes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_vv.py tests/test_gpu_peer.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for e in 1 0; do
  MASPCG_VV_STAGED=$e timeout 300 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v13_tmp.json 2>> gpurun_out/v13.err
  python -c "import json; d=json.load(open('gpurun_out/v13_tmp.json')); print('staged=$e', round(d['value'],1), round(d['roofline']['avg_launch_ms']*1e3,1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_vv_terms|k_vv_rows" -s 6 -c 4 --csv python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "duration" | awk -F'","' '{print $5, $NF}' | cut -c1-120
