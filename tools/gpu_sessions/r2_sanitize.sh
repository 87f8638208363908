# compute-sanitizer memcheck and synccheck over every kernel (incl. the round-2 fused FFN paths)
compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/r2s_sanitize_memcheck.txt 2>&1
compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > gpurun_out/r2s_sanitize_synccheck.txt 2>&1
tail -3 gpurun_out/r2s_sanitize_memcheck.txt; tail -3 gpurun_out/r2s_sanitize_synccheck.txt
