# small-batch latency work: router cluster of 16, permute sized to the plan
python -m pytest tests/test_gpu_kernels.py tests/test_engine_gpu.py -q -k "gate or permute or empty or pipeline or metrics" > gpurun_out/r2s_sb_tests.txt 2>&1
python tools/engine_timeline.py --model qwen3 --layers 24 --steps 6 --batch 1 > gpurun_out/r2s_timeline_qwen3_b1_after.txt 2>&1
out=gpurun_out/r2s_small_batch.jsonl; : > $out
for m in "--model qwen3 --batch 1" "--model dsv2lite --batch 1" "--batch 1" "--model qwen3 --batch 16"; do
  python bench.py --no-cpu $m 2>/dev/null | sed "s/^/{\"args\": \"$m\", \"line\": /; s/$/}/" >> $out
done
tail -1 gpurun_out/r2s_sb_tests.txt
