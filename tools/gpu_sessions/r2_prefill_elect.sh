# prefill GEMM: MMA issued by a whole warp (elect.sync) instead of a lane-0 branch
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "prefill or ffn or bf16" > gpurun_out/el_tests.txt 2>&1; tail -2 gpurun_out/el_tests.txt
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2 --n-tile 128"
for T in 2048 8192; do timeout 300 $mb --tokens $T | tee -a gpurun_out/r2s_prefill_elect.jsonl; done
timeout 300 python tools/ffn_microbench.py --iters 10 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --copies 2 | tee -a gpurun_out/r2s_prefill_elect.jsonl
