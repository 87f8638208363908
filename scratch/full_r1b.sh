python -c "import __graft_entry__ as g; g.build()" > /dev/null
OUT=gpurun_out/r1b; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err
timeout 600 python bench.py --workload profile > $OUT/profile.json 2> $OUT/profile.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_decode.csv python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_fused -s 12 -c 2 -o $OUT/fused_ffn python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_gemm -s 2 -c 2 -o $OUT/prefill_gemm python tools/ffn_microbench.py --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --iters 2 --copies 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xfer_decode_blob -c 1 -o $OUT/xfer_decode python tools/xfer_bench.py --iters 2 > /dev/null 2>&1
python tools/ffn_microbench.py --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --iters 10 --copies 2 > $OUT/prefill_mixtral.json
python tools/ffn_microbench.py --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile 128 --iters 10 --copies 2 > $OUT/prefill_qwen3.json
bash tools/ffn_sweep.sh > $OUT/decode_sweep.jsonl 2>&1
python tools/xfer_bench.py > $OUT/xfer.json
ls -la $OUT
