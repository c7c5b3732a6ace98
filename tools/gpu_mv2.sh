# stencil with two pairs per trip (MASPCG_MATVEC2): bench A/B and parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for e in 0 1; do
  MASPCG_MATVEC2=$e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mv2_tmp.json 2>> gpurun_out/mv2.err
  python -c "import json; d=json.load(open('gpurun_out/mv2_tmp.json')); k=d['per_kernel']; print('mv2=$e', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), round(k['p_update_GBps']), d['clocks']['sm_mhz'])"
done; done
MASPCG_MATVEC2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_cg1.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
