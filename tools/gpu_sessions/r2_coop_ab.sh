# cooperative vs plain launch of the fused FFN inside the engine (events vs on-device span)
BMOE_COOP=0 python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_nocoop.json 2>/dev/null
BMOE_COOP=0 python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_nocoop.json 2>/dev/null
BMOE_DECODE_NARROW=0 BMOE_TIMING_HOLD_NS=0 python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_nohold_wide.json 2>/dev/null
