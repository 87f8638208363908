BMOE_PREFER_SHARED=1 python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_prefshared.json 2>/dev/null
BMOE_PREFER_SHARED=1 python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_prefshared.json 2>/dev/null
