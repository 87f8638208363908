# timing-pass hold check, ncu launch list of decode layer-steps, ncu --set full of the fused FFN (+ combine)
python bench.py --no-cpu --no-original > gpurun_out/r2s_mixtral_hold.json 2>/dev/null
python bench.py --no-cpu --no-original --model qwen3 > gpurun_out/r2s_qwen3_hold.json 2>/dev/null
export BMOE_SETTLE_S=0 BMOE_SETTLE_SWEEPS=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_decode.csv \
    python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > gpurun_out/r2_launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r2_launches_decode.csv 400 > gpurun_out/r2_launches_decode_summary.txt
ncu --set full --clock-control none --import-source on -k regex:ffn_fused -s 12 -c 2 -o gpurun_out/r2_fused_ffn \
    python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > gpurun_out/r2_ncu_full.log 2>&1
ls -la gpurun_out/
