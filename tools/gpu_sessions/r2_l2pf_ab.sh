# W2 L2 prefetch A/B in the fused decode FFN microbench (kernel spans via the phase trace)
python -m pytest tests/test_gpu_kernels.py -q -k "fused or combine" > gpurun_out/r2s_l2pf_tests.txt 2>&1
export BMOE_FFN_TRACE=1
for pf in 0 8 16; do
  for a in 1 2 4; do BMOE_W2_L2PF=$pf python tools/ffn_microbench.py --experts-active $a --k $([ $a = 1 ] && echo 1 || echo 2) --iters 30 --trace; done
  for a in 8 24; do BMOE_W2_L2PF=$pf python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k 8 --experts-active $a --tokens 16 --copies 8 --iters 30 --trace; done
done > gpurun_out/r2s_l2pf_ab.jsonl 2>&1
tail -1 gpurun_out/r2s_l2pf_tests.txt
# stage size (k-blocks per pipeline stage) on the small-expert shape, with the L2 prefetch on
for kp in "2 4" "1 2" "1 1" "2 2" "1 4"; do
  set -- $kp
  BMOE_KPS1=$1 BMOE_KPS2=$2 python tools/ffn_microbench.py --E 128 --d 2048 --f 768 --k 8 --experts-active 24 --tokens 16 --copies 8 --iters 30 --trace
done > gpurun_out/r2s_kps_ab.jsonl 2>&1
