# Qwen3 decode batch sweep and where DSV2 / Qwen3 decode steps leave PCIe idle
out=gpurun_out/r2s_qwen3_decode_sweep.jsonl; : > $out
for b in 1 8 32 64; do python bench.py --no-cpu --model qwen3 --batch $b 2>/dev/null | sed "s/^/{\"args\": \"--model qwen3 --batch $b\", \"line\": /; s/$/}/" >> $out; done
python tools/engine_timeline.py --model dsv2lite --layers 26 --steps 4 > gpurun_out/r2s_timeline_dsv2.txt 2>&1
python tools/engine_timeline.py --model qwen3 --layers 12 --steps 4 > gpurun_out/r2s_timeline_qwen3.txt 2>&1
python tools/engine_timeline.py --model mixtral --layers 8 --steps 4 > gpurun_out/r2s_timeline_mixtral.txt 2>&1
