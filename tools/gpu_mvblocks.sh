# the vector stencil at 5 blocks per SM (kMvBlocks) vs 4: bench A/B (rebuild on the box) and parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for mb in 5 4; do
  sed -i "s/^constexpr int kMvBlocks = [0-9];/constexpr int kMvBlocks = $mb;/" paper_2303_03398_b200/csrc/kernels.cu
  python -m paper_2303_03398_b200.build > /dev/null 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mb_tmp.json 2>> gpurun_out/mb.err
  python -c "import json; d=json.load(open('gpurun_out/mb_tmp.json')); k=d['per_kernel']; print('mvblocks=$mb', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), round(k['p_update_GBps']), d['clocks']['sm_mhz'])"
done; done
sed -i "s/^constexpr int kMvBlocks = [0-9];/constexpr int kMvBlocks = 5;/" paper_2303_03398_b200/csrc/kernels.cu
python -m paper_2303_03398_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_cg1.py tests/test_gpu_peer.py tests/test_gpu_nccl.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
