# final check after the token-major prefill GEMM1 and the K6 transposed-build option
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin_gputests.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
tail -2 gpurun_out/fin_gputests.txt; tail -1 gpurun_out/fin_smoke.txt; python -c "import json;d=json.loads(open('gpurun_out/fin_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'])"
