# Qwen3 prefill: GEMM1 token tile 256 (single CTA, one TMEM accumulator stage) vs 128; and
# compute-sanitizer memcheck/racecheck of the K6 transposed build
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2"
for T in 2048 8192; do for nt in 128 256; do
  timeout 300 $mb --tokens $T --n-tile $nt | sed "s/^{/{\"n_tile_arg\": $nt, /" | tee -a gpurun_out/r2s_prefill_qwen3_nt.jsonl
done; done
BMOE_COACT_TB_MASK=0xFFF timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_kernels.py -q -k "coact_tensor_core_path_bit_exact and mxf4 and 255" > gpurun_out/r2s_tb_memcheck.txt 2>&1; tail -4 gpurun_out/r2s_tb_memcheck.txt
BMOE_COACT_TB_MASK=0xFFF timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_kernels.py -q -k "coact_tensor_core_path_bit_exact and mxf4 and 255" > gpurun_out/r2s_tb_racecheck.txt 2>&1; tail -4 gpurun_out/r2s_tb_racecheck.txt
