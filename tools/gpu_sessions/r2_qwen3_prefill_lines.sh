# Qwen3 prefill bench lines (512 / 2048 tokens) with the token-major GEMM1 default
for T in 512 2048; do
  timeout 900 python bench.py --model qwen3 --batch $T --no-original --no-cpu > gpurun_out/q_pf_$T.json 2> gpurun_out/q_pf_$T.err
  python -c "import json;d=json.loads(open('gpurun_out/q_pf_$T.json').read().strip().splitlines()[-1]);r=d['roofline'];print($T, d['value'], r['bound'], r['achieved'], r['frac'])"
done
