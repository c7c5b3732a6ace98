python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in "c1-P2-1-0" "c1-P2-1-1" "c2-P4-1-0" "c2-P4-1-1" "rand-np6-P3-1-0" "rand-np6-P3-1-1" "rand-np6-P3-4-0"; do
  timeout 120 python -m pytest tests/test_gpu_peer.py -m gpu -q -p no:cacheprovider -k "multirank_threads and $k" --timeout 90 2>&1 | grep -E "passed|failed|Timeout" | head -2 | sed "s/^/$k: /"
done
