# full GPU suite, smoke, sanitizer (memcheck + synccheck) with codec v3 and the mxf4 K6 default
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s_gputests_final.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/r2s_sanitize_memcheck.txt 2>&1
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > gpurun_out/r2s_sanitize_synccheck.txt 2>&1
tail -2 gpurun_out/r2s_gputests_final.txt; tail -1 gpurun_out/r2s_smoke.txt
tail -3 gpurun_out/r2s_sanitize_memcheck.txt; tail -3 gpurun_out/r2s_sanitize_synccheck.txt
