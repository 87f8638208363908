# re-entry check of the committed tree: GPU suite, smoke, default bench line
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/re_gputests.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err
tail -2 gpurun_out/re_gputests.txt; tail -1 gpurun_out/re_smoke.txt; tail -c 1500 gpurun_out/re_bench.json
