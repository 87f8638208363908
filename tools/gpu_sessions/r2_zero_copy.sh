python -m pytest tests/test_engine_shapes_gpu.py tests/test_engine_gpu.py tests/test_engine_random_gpu.py tests/test_engine_policies_gpu.py -q > gpurun_out/r2s_zc_tests.txt 2>&1
out=gpurun_out/r2s_zc_bench.jsonl; : > $out
for zc in 1 0; do for m in "--model qwen3 --batch 1" "--model dsv2lite --batch 1" "--model qwen3 --batch 16"; do
  BMOE_ZERO_COPY=$zc python bench.py --no-cpu --no-original $m 2>/dev/null | sed "s/^/{\"zc\": $zc, \"args\": \"$m\", \"line\": /; s/$/}/" >> $out
done; done
tail -1 gpurun_out/r2s_zc_tests.txt
