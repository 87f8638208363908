# K6 transposed build, pipelined id loads + clamped-shift masks: parity and timing
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "coact" > gpurun_out/tb2_tests.txt 2>&1; tail -2 gpurun_out/tb2_tests.txt
timeout 600 python tools/coact_bench.py --modes 3,2 | tee gpurun_out/r2s_coact_tb2.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coact_fp4 -c 1 -o gpurun_out/r2s_coact_tb2 python tools/coact_bench.py --modes 2 --iters 1 > gpurun_out/tb2_ncu_full.txt 2>&1; tail -1 gpurun_out/tb2_ncu_full.txt
