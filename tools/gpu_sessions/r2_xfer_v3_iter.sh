timeout 600 python -m pytest tests/test_xfer_gpu.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/xfer_bench.py --format 3; done | tee gpurun_out/r2s_xfer_v3_iter.jsonl
timeout 600 ncu --clock-control none -k regex:xfer_decode_piece -s 2 -c 2 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed python tools/xfer_bench.py --iters 3 2>&1 | grep -E "duration|inst_exec|throughput" | head
