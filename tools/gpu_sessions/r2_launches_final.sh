# ncu launch list of decode layer-steps with the final code (codec v3), summarised
export BMOE_SETTLE_S=0 BMOE_SETTLE_SWEEPS=1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_decode.csv \
    python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu --no-original > gpurun_out/r2s_launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r2s_launches_decode.csv 400 > gpurun_out/r2s_launches_decode_summary.txt
cat gpurun_out/r2s_launches_decode_summary.txt | head -20
