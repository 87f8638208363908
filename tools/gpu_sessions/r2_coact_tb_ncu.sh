# ncu --set full of the transposed-build K6 kernel (mode 2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coact_fp4 -c 1 -o gpurun_out/r2s_coact_tb python tools/coact_bench.py --modes 2 --iters 1 > gpurun_out/tb_ncu_full.txt 2>&1; tail -3 gpurun_out/tb_ncu_full.txt
