# events vs on-device spans of the fused FFN in the engine's timing pass
python -m pytest tests/test_gpu_kernels.py -q -k "fused or combine" > gpurun_out/r2s_span_tests.txt 2>&1
python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_span.json 2>/dev/null
python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_span.json 2>/dev/null
tail -1 gpurun_out/r2s_span_tests.txt
