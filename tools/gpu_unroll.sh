# update / p-update with two pairs per thread and trip (MASPCG_UPDATE2, MASPCG_PUPDATE2): bench A/B and parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for cfg in "0 0" "0 1" "1 0" "1 1"; do set -- $cfg
  MASPCG_UPDATE2=$1 MASPCG_PUPDATE2=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/u2_tmp.json 2>> gpurun_out/u2.err
  python -c "import json; d=json.load(open('gpurun_out/u2_tmp.json')); k=d['per_kernel']; print('up2=$1 pu2=$2', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), round(k['p_update_GBps']), d['clocks']['sm_mhz'])"
done; done
MASPCG_UPDATE2=1 MASPCG_PUPDATE2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_peer.py tests/test_gpu_vv.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
