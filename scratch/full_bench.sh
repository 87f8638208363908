set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g | head -2
time python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -3 gpurun_out/bench_full.err
# launch list of a short decode run (cold/serialised under ncu: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv \
    python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > /dev/null 2>&1
# full capture of the two grouped-FFN GEMM kernels of one decode layer-step
ncu --set full --clock-control none --import-source on -k regex:ffn_gemm -s 40 -c 2 -o gpurun_out/prof_decode_gemm \
    python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > /dev/null 2>&1
ls -la gpurun_out
