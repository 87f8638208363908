python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/xfer_bench.py
df -h /dev/shm | tail -1
timeout 600 python -m pytest tests/test_xfer_gpu.py tests/test_shared_mirror_gpu.py -q -x 2>&1 | tail -4
