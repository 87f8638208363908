python -m pytest tests/test_gpu_kernels.py tests/test_engine_gpu.py tests/test_profiling_dist_cpu.py -q -k "coact or pipeline or profile" > gpurun_out/r2s_ctc_tests.txt 2>&1
python bench.py --workload profile > gpurun_out/r2s_profile_tc.json 2>gpurun_out/r2s_profile_tc.err
BMOE_COACT_TC=0 python bench.py --workload profile > gpurun_out/r2s_profile_atomics.json 2>/dev/null
tail -3 gpurun_out/r2s_ctc_tests.txt
