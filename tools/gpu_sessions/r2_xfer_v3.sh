set -x
timeout 600 python -m pytest tests/test_xfer_gpu.py -x -q 2>&1 | tail -15
for f in 2 3; do timeout 300 python tools/xfer_bench.py --format $f; done | tee gpurun_out/r2s_xfer_v3_bench.jsonl
