# K6 build mix sweep: BMOE_COACT_TB_MASK over the 12 builder warps (0 = all OR build, 0xFFF = all transposed)
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "coact" > gpurun_out/mix_tests.txt 2>&1; tail -2 gpurun_out/mix_tests.txt
for m in 0x000 0xFFF 0x924 0xAAA 0xDB6 0xEEE; do
  BMOE_COACT_TB_MASK=$m timeout 300 python tools/coact_bench.py --modes 2 | sed "s/^{/{\"tb_mask\": \"$m\", /" | tee -a gpurun_out/r2s_coact_mix.jsonl
done
