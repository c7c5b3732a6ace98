python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 700 python -m pytest tests/test_gpu_peer.py -m gpu -q -p no:cacheprovider --timeout 240 -o faulthandler_timeout=200 2>&1 | grep -v "^  File \"/usr\|^  File \"/opt" | tail -40
