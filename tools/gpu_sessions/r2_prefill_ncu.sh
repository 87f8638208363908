# ncu --set full of the Qwen3-shaped prefill GEMM1: single CTA (default) and CTA pair (BMOE_2SM=2)
mb="python tools/ffn_microbench.py --iters 2 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 1 --tokens 8192 --n-tile 128"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm_kernel -s 2 -c 1 -o gpurun_out/r2s_prefill_g1_1sm $mb > gpurun_out/pf_ncu1.txt 2>&1; tail -1 gpurun_out/pf_ncu1.txt
BMOE_2SM=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm_2sm -s 4 -c 2 -o gpurun_out/r2s_prefill_g1_2sm $mb > gpurun_out/pf_ncu2.txt 2>&1; tail -1 gpurun_out/pf_ncu2.txt
