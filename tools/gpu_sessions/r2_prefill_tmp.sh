# token-major CTA-pair GEMM1 (BMOE_TM=2) vs single (1) vs weight-major (0)
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "token_major or prefill" > gpurun_out/tmp_tests.txt 2>&1; tail -3 gpurun_out/tmp_tests.txt
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2 --n-tile 128"
for tm in 0 1 2; do for T in 2048 8192; do BMOE_TM=$tm timeout 300 $mb --tokens $T | sed "s/^{/{\"BMOE_TM\": $tm, /" | tee -a gpurun_out/r2s_prefill_tmp.jsonl; done; done
for tm in 0 2; do BMOE_TM=$tm timeout 300 python tools/ffn_microbench.py --iters 10 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --copies 2 | sed "s/^{/{\"BMOE_TM\": $tm, /" | tee -a gpurun_out/r2s_prefill_tmp.jsonl; done
for tm in 0 1 2; do BMOE_TM=$tm timeout 300 python tools/ffn_microbench.py --iters 20 --E 64 --d 2048 --f 1408 --k 6 --experts-active 64 --tokens 4096 --n-tile 128 --copies 2 | sed "s/^{/{\"BMOE_TM\": $tm, /" | tee -a gpurun_out/r2s_prefill_tmp.jsonl; done
