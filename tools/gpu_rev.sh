python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for e in 0 1; do
  MASPCG_REV_UPDATE=$e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rev_tmp.json 2>> gpurun_out/rev.err
  python -c "import json; d=json.load(open('gpurun_out/rev_tmp.json')); k=d['per_kernel']; print('rev=$e', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), round(k['p_update_GBps']), d['clocks']['sm_mhz'])"
done; done
MASPCG_REV_UPDATE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
MASPCG_REV_UPDATE=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"vec2" -s 12 -c 6 --csv python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram|duration" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-150
