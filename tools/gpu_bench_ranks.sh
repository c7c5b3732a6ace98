# bench.py's N > 1 code path on one GPU: torchrun ranks sharing cuda:0, gloo process group, peer communicator
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 2 4; do
  MASPCG_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
    bench.py --gpus $n --comm peer --steps 3 --warmup 3 --maxit 40 > gpurun_out/bench_ranks_$n.json 2> gpurun_out/bench_ranks_$n.err
  echo "n=$n rc=$?"; head -c 700 gpurun_out/bench_ranks_$n.json; echo; tail -3 gpurun_out/bench_ranks_$n.err
done
MASPCG_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 \
    bench.py --gpus 2 --comm peer --path 4 --steps 3 --warmup 3 --maxit 40 --no-cpu-baseline > gpurun_out/bench_ranks_cg1.json 2> gpurun_out/bench_ranks_cg1.err
echo "cg1 rc=$?"; head -c 300 gpurun_out/bench_ranks_cg1.json; echo
MASPCG_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ranks_ref.json 2> gpurun_out/bench_ranks_ref.err
echo "ref rc=$?"; head -c 300 gpurun_out/bench_ranks_ref.json; echo
