timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "coact" 2>&1 | tail -4
timeout 600 python tools/coact_bench.py | tee gpurun_out/r2s_coact_mxf4.jsonl
