# FFN fixed-cost iteration: parity tests of the fused decode kernel, then phase traces
python -m pytest tests/test_gpu_kernels.py tests/test_engine_shapes_gpu.py tests/test_engine_gpu.py -q -k "combine or pipeline or fused or split" > gpurun_out/r2s_iter_tests.txt 2>&1
export BMOE_FFN_TRACE=1
for v in "BMOE_H_READY=1" "BMOE_H_READY=0"; do
for a in 8 24; do
  env $v python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k 8 --experts-active $a --tokens 16 --copies 8 --iters 40 --trace
done
env $v python tools/ffn_microbench.py --experts-active 4 --iters 40 --trace
done > gpurun_out/r2s_iter_trace.jsonl 2>&1
tail -3 gpurun_out/r2s_iter_tests.txt
