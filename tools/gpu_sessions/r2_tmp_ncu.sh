# ncu --set full of the token-major CTA-pair GEMM1 (Qwen3 8192 x 8 call)
mb="python tools/ffn_microbench.py --iters 2 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 1 --tokens 8192 --n-tile 128"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm1_split -s 2 -c 1 -o gpurun_out/r2s_prefill_g1_tmpair $mb > gpurun_out/tmp_ncu.txt 2>&1; tail -1 gpurun_out/tmp_ncu.txt
