run() { env "$@" python bench.py --layers 4 --steps 5 --warmup 3 --no-cpu --no-original 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', round(r['avg_launch_ms'],4), round(r['gemm2_avg_launch_ms'],4), int(r['achieved']), int(r['pair_achieved_gbs']), r['experts_per_launch'])"; }
run BMOE_NTILE_FIXED=1 BMOE_NCHAIN=1 BMOE_KPS=1
run BMOE_NTILE_FIXED=1 BMOE_NCHAIN=4 BMOE_KPS=1
run BMOE_NCHAIN=1 BMOE_KPS=1
run BMOE_NCHAIN=2 BMOE_KPS=1
run BMOE_NCHAIN=4 BMOE_KPS=1
run BMOE_NTILE_FIXED=1 BMOE_NCHAIN=1 BMOE_KPS=2
run BMOE_NTILE_FIXED=1 BMOE_NCHAIN=1 BMOE_KPS=4
run BMOE_NCHAIN=1 BMOE_KPS=4
