for cfg in "BMOE_KPS=1 BMOE_NCHAIN=1" "BMOE_KPS=2 BMOE_NCHAIN=1" "BMOE_KPS=4 BMOE_NCHAIN=1" "BMOE_KPS=4 BMOE_NCHAIN=4" "BMOE_KPS=2 BMOE_NCHAIN=4"; do
  env $cfg python tools/ffn_microbench.py --n-tile 16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg nt16', round(d['gemm1_ms'],4), round(d['gemm2_ms'],4), int(d['gemm1_gbs']), int(d['gemm2_gbs']), int(d['pair_gbs']))"
done
for nt in 32 64; do env BMOE_KPS=1 BMOE_NCHAIN=1 python tools/ffn_microbench.py --n-tile $nt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kps1 nt$nt', round(d['gemm1_ms'],4), round(d['gemm2_ms'],4), int(d['gemm1_gbs']), int(d['gemm2_gbs']))"; done
python tools/ffn_microbench.py --experts-active 8 --tokens 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8exp default', d)"
