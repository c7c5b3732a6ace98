# single-reduction update kernel blocks per SM (kCgUpdBlocks): 3 (default) vs 2 vs 4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for cb in 3 2 4; do
  sed -i "s/^constexpr int kCgUpdBlocks = [0-9];/constexpr int kCgUpdBlocks = $cb;/" paper_2303_03398_b200/csrc/cg1.cu
  python -m paper_2303_03398_b200.build > /dev/null 2>&1
  timeout 300 python bench.py --path 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cb_tmp.json 2>> gpurun_out/cb.err
  python -c "import json; d=json.load(open('gpurun_out/cb_tmp.json')); k=d['per_kernel']; print('cg1upd=$cb', round(d['value'],1), round(d['roofline']['achieved']), round(k['update_GBps']), d['clocks']['sm_mhz'])"
done; done
