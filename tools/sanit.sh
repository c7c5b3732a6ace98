# compute-sanitizer memcheck and racecheck of small solves on the default, single-reduction and vector paths,
# plus memcheck of one peer-mode (one rank, in-stencil halo acquire) solve
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S="python bench.py --config c1 --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e"
for tool in memcheck racecheck; do
  for v in "" "--path 4" "--force-comm --comm peer" "--operator vv --config c2v"; do
    echo "== $tool $v" >> gpurun_out/sanit.txt
    timeout 900 compute-sanitizer --tool $tool --print-limit 5 $S $v 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" | head -5 >> gpurun_out/sanit.txt
  done
done
cat gpurun_out/sanit.txt
