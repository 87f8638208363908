# tiny FFN calls on fewer CTAs (BMOE_FFN_MIN_ITERS): microbench spans and B=1 benches
python -m pytest tests/test_gpu_kernels.py -q -k "fused or combine or groups or spans" > gpurun_out/r2s_mi_tests.txt 2>&1
export BMOE_FFN_TRACE=1
for mi in 1 2 4 8; do
  for a in 1 2 4 8; do BMOE_FFN_MIN_ITERS=$mi python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k $([ $a -ge 8 ] && echo 8 || echo $a) --experts-active $a --tokens 1 --copies 8 --iters 30 --trace; done
  BMOE_FFN_MIN_ITERS=$mi python tools/ffn_microbench.py --E 64 --d 2048 --f 1408 --k 6 --experts-active 8 --tokens 1 --copies 8 --iters 30 --trace
done > gpurun_out/r2s_mi_ab.jsonl 2>&1
unset BMOE_FFN_TRACE
out=gpurun_out/r2s_mi_bench.jsonl; : > $out
for mi in 1 4; do for m in "--model qwen3 --batch 1" "--model dsv2lite --batch 1"; do
  BMOE_FFN_MIN_ITERS=$mi python bench.py --no-cpu --no-original $m 2>/dev/null | sed "s/^/{\"mi\": $mi, \"args\": \"$m\", \"line\": /; s/$/}/" >> $out
done; done
tail -1 gpurun_out/r2s_mi_tests.txt
