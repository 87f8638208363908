# token-major GEMM1 auto choice (BMOE_TM=3 default): kernel tests, microbench, Qwen3 8192 / DSV2 prefill bench lines
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_engine_shapes_gpu.py -q > gpurun_out/tma_tests.txt 2>&1; tail -2 gpurun_out/tma_tests.txt
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2 --n-tile 128"
for T in 2048 8192; do timeout 300 $mb --tokens $T | tee -a gpurun_out/r2s_prefill_tm_auto.jsonl; done
timeout 300 python tools/ffn_microbench.py --iters 10 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --copies 2 | tee -a gpurun_out/r2s_prefill_tm_auto.jsonl
timeout 900 python bench.py --model qwen3 --batch 8192 --no-original --no-cpu > gpurun_out/tma_q8192.json 2> gpurun_out/tma_q8192.err
python -c "import json;d=json.loads(open('gpurun_out/tma_q8192.json').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['achieved'], d['roofline']['frac'])"
