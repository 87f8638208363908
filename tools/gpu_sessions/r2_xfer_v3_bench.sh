# fetch codec v3 vs v2 at the headline and the small-expert shapes (engine tests first)
timeout 900 python -m pytest tests/test_xfer_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/r2s_v3_tests.txt 2>&1
tail -2 gpurun_out/r2s_v3_tests.txt
for f in 3 2 3 2; do
  BMOE_XFER_FORMAT=$f timeout 900 python bench.py --no-cpu --no-original 2>/dev/null | sed "s/^{/{\"xfer_format\": $f, /"
done > gpurun_out/r2s_v3_bench_ab.jsonl
for f in 3 2; do
  BMOE_XFER_FORMAT=$f timeout 900 python bench.py --no-cpu --no-original --model qwen3 2>/dev/null | sed "s/^{/{\"xfer_format\": $f, /"
done >> gpurun_out/r2s_v3_bench_ab.jsonl
python - <<'P'
import json
for l in open("gpurun_out/r2s_v3_bench_ab.jsonl"):
    r = json.loads(l); c = r["config"]
    print(r["xfer_format"], c.get("model", c.get("workload")), r["value"], r["e2e"]["value"], r.get("fetch", {}).get("coded_ratio"))
P
