#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of small solves with the round-2 code paths: the device loop
# (kernel timing off), the L2 residency plan (c2: every class fits), the field-aligned operator (TMA-staged
# stencil with mbarriers and bulk copies), the peer communicator, the vector operator
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/sanit_r02.txt; rm -f $out
S="python bench.py --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for tool in memcheck racecheck synccheck; do
  for v in "--config c1" "--config c2" "--operator aniso --config c1a" "--operator aniso --config c2a" "--config c1 --force-comm --comm peer" "--operator vv --config c2v" "--config c1 --device-loop 0"; do
    echo "== $tool $v" >> $out
    timeout 900 compute-sanitizer --tool $tool --print-limit 5 $S $v 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" | head -5 >> $out
  done
done
cat $out
