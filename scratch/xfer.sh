python -c "import __graft_entry__ as g; g.build()" > /dev/null
for v in 1 3; do BMOE_XFER_DECODER=$v python tools/xfer_bench.py; done
timeout 300 python -m pytest tests/test_xfer_gpu.py -q -x 2>&1 | tail -2
