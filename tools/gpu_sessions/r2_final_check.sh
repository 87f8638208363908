# full GPU suite, smoke, headline bench
python -m pytest tests -m gpu -q > gpurun_out/r2s_gputests_final.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.txt 2>&1
python bench.py > gpurun_out/r2s_bench_final.json 2> gpurun_out/r2s_bench_final.err
tail -2 gpurun_out/r2s_gputests_final.txt; tail -1 gpurun_out/r2s_smoke.txt
