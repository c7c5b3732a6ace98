# peer communicator: halo acquire inside the stencil (MASPCG_OPT_FUSE_HALO 2) vs the wait kernel (1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_bench_ranks.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400 --force-comm --comm peer"
for rep in 1 2; do for sh in 150,300,75 150,300,600; do for fh in 1 2; do
  timeout 200 $B --shape $sh --fuse-halo $fh > gpurun_out/acq_tmp.json 2>> gpurun_out/acq.err
  python -c "import json; d=json.load(open('gpurun_out/acq_tmp.json')); print('$sh fuse_halo=$fh', round(d['value'],1), 'us/it', round(1e6/d['value'],1), d['gpu_launches'])"
done; done; done
