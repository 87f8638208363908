set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mb="python tools/ffn_microbench.py"
for NT in 128 256; do
 $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile $NT --iters 10 --copies 2 | cut -c1-400
 $mb --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile $NT --iters 10 --copies 2 | cut -c1-400
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm -s 4 -c 2 -o gpurun_out/prefill_gemm python tools/ffn_microbench.py --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 256 --iters 2 --copies 2 > gpurun_out/ncu_prefill.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_codec.csv python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > gpurun_out/launch_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xfer_decode_piece -s 30 -c 1 -o gpurun_out/xfer_decode python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-original > gpurun_out/ncu_xfer.log 2>&1
ls -la gpurun_out
