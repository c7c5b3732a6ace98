# blocks per SM of the three-kernel vector path (kVecBlocks): 4 (default) vs 3 vs 5
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for vb in 4 3 5; do
  sed -i "s/^constexpr int kVecBlocks = [0-9];/constexpr int kVecBlocks = $vb;/" paper_2303_03398_b200/csrc/kernels.cu
  python -m paper_2303_03398_b200.build > /dev/null 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vb_tmp.json 2>> gpurun_out/vb.err
  python -c "import json; d=json.load(open('gpurun_out/vb_tmp.json')); k=d['per_kernel']; print('vecblocks=$vb', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), round(k['p_update_GBps']), d['clocks']['sm_mhz'])"
done; done
