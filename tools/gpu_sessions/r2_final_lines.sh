# final-code lines: small-expert shapes (buddy / on-demand / Random arms), the profile workload,
# and the two-rank rehearsals (two ranks sharing the one GPU)
timeout 1500 python bench.py --model qwen3 > gpurun_out/r2s_qwen3_decode.json 2> gpurun_out/r2s_qwen3_decode.err
timeout 1500 python bench.py --model dsv2lite > gpurun_out/r2s_dsv2_decode.json 2> gpurun_out/r2s_dsv2_decode.err
timeout 900 python bench.py --workload profile > gpurun_out/r2s_profile_1gpu.json 2> gpurun_out/r2s_profile_1gpu.err
BMOE_ALLOW_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --workload profile > gpurun_out/r2s_profile_2ranks_final.json 2> gpurun_out/r2s_profile_2ranks_final.err
BMOE_ALLOW_SHARED_GPU=1 timeout 1500 python bench.py --gpus 2 --layers 8 --no-cpu --no-original > gpurun_out/r2s_decode_2ranks_final.json 2> gpurun_out/r2s_decode_2ranks_final.err
python - <<'P'
import json
for f in ("r2s_qwen3_decode", "r2s_dsv2_decode", "r2s_profile_1gpu", "r2s_profile_2ranks_final", "r2s_decode_2ranks_final"):
    try:
        r = json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "ERR", e); continue
    wb = r.get("without_buddy") or {}; rs = r.get("random_substitution") or {}; fd = r.get("fidelity") or {}
    print(f, round(r["value"], 1), round(r["e2e"]["value"], 1), r.get("physical_fetches_per_step"),
          round(r["roofline"]["frac"], 3), r["roofline"].get("frac_kernel_span"), wb.get("value"), json.dumps(fd)[:200])
P
