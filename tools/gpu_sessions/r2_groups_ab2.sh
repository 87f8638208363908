python -m pytest tests/test_gpu_kernels.py tests/test_engine_shapes_gpu.py -q -k "fused or combine or groups" > gpurun_out/r2s_groups_tests.txt 2>&1
export BMOE_FFN_TRACE=1
for g in 1 3; do
  for a in 1 2 4; do BMOE_FFN_GROUPS=$g python tools/ffn_microbench.py --experts-active $a --k $([ $a = 1 ] && echo 1 || echo 2) --iters 30 --trace; done
  for a in 8 24 48; do BMOE_FFN_GROUPS=$g python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k 8 --experts-active $a --tokens 16 --copies 8 --iters 30 --trace; done
done > gpurun_out/r2s_groups_ab2.jsonl 2>&1
unset BMOE_FFN_TRACE
python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_groups.json 2>/dev/null
BMOE_FFN_GROUPS=1 python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_nogroups.json 2>/dev/null
tail -1 gpurun_out/r2s_groups_tests.txt
