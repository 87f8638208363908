# full GPU suite, headline bench, decoder-grid A/B, small-expert model lines
python -m pytest tests -m gpu -q > gpurun_out/r2s_gputests3.txt 2>&1
python bench.py > gpurun_out/r2s_bench3.json 2> gpurun_out/r2s_bench3.err
BMOE_DECODE_NARROW=0 python bench.py --no-cpu --no-original > gpurun_out/r2s_bench3_widedecode.json 2>/dev/null
python bench.py --no-cpu --model qwen3 > gpurun_out/r2s_qwen3.json 2>/dev/null
python bench.py --no-cpu --model dsv2lite > gpurun_out/r2s_dsv2.json 2>/dev/null
tail -3 gpurun_out/r2s_gputests3.txt
