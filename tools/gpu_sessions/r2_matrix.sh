# round-2 config matrix on the final code (default workloads), profiling sweep, 2-rank rehearsal, reference arm
out=gpurun_out/r2s_matrix.jsonl; : > $out
run() { python bench.py --no-cpu "$@" 2>/dev/null | sed "s/^/{\"args\": \"$*\", \"line\": /; s/$/}/" >> $out; }
for b in 1 8 32 64; do run --batch $b; done
for b in 512 2048 8192; do run --model qwen3 --batch $b; done
for c in 0.375 0.5 0.75; do for b in 1 16; do run --model dsv2lite --batch $b --cache-rate $c; done; done
python bench.py --workload profile > gpurun_out/r2s_profile_1gpu.json 2> gpurun_out/r2s_profile_1gpu.err
BMOE_ALLOW_SHARED_GPU=1 python bench.py --gpus 2 --workload profile > gpurun_out/r2s_profile_2ranks.json 2> gpurun_out/r2s_profile_2ranks.err
BMOE_ALLOW_SHARED_GPU=1 python bench.py --gpus 2 --layers 8 --no-cpu --no-original > gpurun_out/r2s_decode_2ranks.json 2> gpurun_out/r2s_decode_2ranks.err
python bench.py --impl reference > gpurun_out/r2s_reference.json 2> gpurun_out/r2s_reference.err
wc -l $out
