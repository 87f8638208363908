# decoder-grid A/B on the small-expert shapes (Qwen3: one piece per expert)
python -m pytest tests/test_xfer_gpu.py -q > gpurun_out/r2s_xfer_tests.txt 2>&1
python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_narrow.json 2>/dev/null
BMOE_DECODE_NARROW=0 python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_wide.json 2>/dev/null
python bench.py --no-cpu --no-original --model dsv2lite > gpurun_out/r2s_dsv2_narrow.json 2>/dev/null
tail -2 gpurun_out/r2s_xfer_tests.txt
