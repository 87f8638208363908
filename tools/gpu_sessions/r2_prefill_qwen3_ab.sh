# Qwen3-shaped prefill FFN call (E=128, k=8, d=2048, f=768): CTA-pair modes and GEMM2 tile widths
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2"
for T in 2048 8192; do
 for m in 0 1 2; do for nt2 in 128 256; do
  BMOE_2SM=$m BMOE_NT2=$nt2 timeout 300 $mb --tokens $T --n-tile 128 | sed "s/^{/{\"BMOE_2SM\": $m, \"BMOE_NT2\": $nt2, /" | tee -a gpurun_out/r2s_prefill_qwen3_ab.jsonl
 done; done
done
