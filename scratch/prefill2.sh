python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
mb="python tools/ffn_microbench.py"
for DP in 1 0; do
for NT in 128 256; do
 BMOE_DP=$DP $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile $NT --iters 10 --copies 2 | cut -c1-260
 BMOE_DP=$DP $mb --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile $NT --iters 10 --copies 2 | cut -c1-260
done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm -s 4 -c 2 -o gpurun_out/prefill_gemm_dp python tools/ffn_microbench.py --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 256 --iters 2 --copies 2 > gpurun_out/ncu_prefill.log 2>&1
