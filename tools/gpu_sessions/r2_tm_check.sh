# token-major GEMM1: bitwise test, Qwen3 prefill bench lines with BMOE_TM=0/1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "token_major or prefill or bf16" > gpurun_out/tm2_tests.txt 2>&1; tail -2 gpurun_out/tm2_tests.txt
for tm in 0 1; do
  BMOE_TM=$tm timeout 900 python bench.py --model qwen3 --batch 8192 --no-original --no-cpu > gpurun_out/tm_q8192_$tm.json 2> gpurun_out/tm_q8192_$tm.err
  python -c "import json;d=json.loads(open('gpurun_out/tm_q8192_$tm.json').read().strip().splitlines()[-1]);print($tm, d['value'], d['roofline']['achieved'], d['roofline']['frac'])"
done
