python -m pytest tests/test_gpu_kernels.py tests/test_engine_shapes_gpu.py tests/test_engine_gpu.py -q -k "combine or pipeline" > gpurun_out/r2s_combine_tests.txt 2>&1
export BMOE_FFN_TRACE=1
for v in "" "BMOE_COOP=0" "BMOE_PDL=1" "BMOE_COOP=0 BMOE_PDL=1"; do
  for a in 8 24; do
    env $v python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k 8 --experts-active $a --tokens 16 --copies 8 --iters 40 --trace | sed "s/^/{\"variant\": \"$v\", \"r\": /; s/$/}/"
  done
done > gpurun_out/r2s_ffn_variants.jsonl 2> gpurun_out/r2s_ffn_variants.err
unset BMOE_FFN_TRACE
for e in independent clustered; do for s in 0 1 2; do
  python bench.py --no-cpu --no-original --experts $e --weight-seed $s 2>/dev/null | sed "s/^/{\"experts\": \"$e\", \"seed\": $s, \"r\": /; s/$/}/"
done; done > gpurun_out/r2s_seed_sweep.jsonl
tail -3 gpurun_out/r2s_combine_tests.txt
