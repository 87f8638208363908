# full GPU suite, smoke, headline bench, reference arm, ncu of the v3 piece decoder
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s_gputests_final.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.txt 2>&1
timeout 1200 python bench.py > gpurun_out/r2s_bench_final.json 2> gpurun_out/r2s_bench_final.err
timeout 900 python bench.py --impl reference > gpurun_out/r2s_bench_reference.json 2> gpurun_out/r2s_bench_reference.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xfer_decode_piece -s 2 -c 2 \
  -o gpurun_out/r2s_xfer_v3_decode -f python tools/xfer_bench.py --iters 3 > gpurun_out/r2s_ncu_xfer.log 2>&1
tail -2 gpurun_out/r2s_gputests_final.txt; tail -1 gpurun_out/r2s_smoke.txt; cat gpurun_out/r2s_bench_final.json | cut -c1-300
