python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bf16" 2>&1 | tail -2
for k in 1 2 4; do BMOE_KPS=$k python tools/ffn_microbench.py --n-tile 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kps$k nt16', round(d['gemm1_ms'],4), round(d['gemm2_ms'],4), int(d['gemm1_gbs']), int(d['gemm2_gbs']), int(d['pair_gbs']))"; done
python tools/ffn_microbench.py --experts-active 8 --tokens 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8exp', round(d['gemm1_ms'],4), round(d['gemm2_ms'],4), int(d['gemm1_gbs']), int(d['gemm2_gbs']), int(d['pair_gbs']))"
