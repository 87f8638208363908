# config matrix on the final code of round 2 (token-major prefill GEMM1), profiling sweep at 1 and 2 ranks
out=gpurun_out/r2s_models_matrix_final.jsonl; : > $out
run() { timeout 900 python bench.py --no-cpu "$@" 2>/dev/null | sed "s/^/{\"args\": \"$*\", \"line\": /; s/$/}/" >> $out; }
for b in 1 8 32 64; do run --batch $b; done
for b in 16 512 2048 8192; do run --model qwen3 --batch $b; done
for c in 0.375 0.5 0.75; do for b in 1 16; do run --model dsv2lite --batch $b --cache-rate $c; done; done
timeout 600 python bench.py --workload profile > gpurun_out/r2s_profile_1gpu_final.json 2> gpurun_out/r2s_profile_1gpu_final.err
BMOE_ALLOW_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --workload profile > gpurun_out/r2s_profile_2ranks_final2.json 2> gpurun_out/r2s_profile_2ranks_final2.err
wc -l $out
