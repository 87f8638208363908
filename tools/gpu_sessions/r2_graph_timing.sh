# FFN timing inside the captured graphs (the timing pass now launches like the timed run)
python -m pytest tests/test_gpu_kernels.py tests/test_engine_gpu.py tests/test_engine_shapes_gpu.py -q -k "spans or fused or combine or pipeline or tensor_core" > gpurun_out/r2s_gt_tests.txt 2>&1
python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_gt.json 2>gpurun_out/r2s_mixtral_gt.err
python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_gt.json 2>/dev/null
python bench.py --no-cpu --no-original --model dsv2lite > gpurun_out/r2s_dsv2_gt.json 2>/dev/null
tail -1 gpurun_out/r2s_gt_tests.txt
