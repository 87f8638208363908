python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "bf16" 2>&1 | tail -3
mb="timeout 120 python tools/ffn_microbench.py"
for P in 1 0; do
 BMOE_PAIR=$P $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --iters 10 --copies 2 | cut -c1-200
 BMOE_PAIR=$P $mb --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile 128 --iters 10 --copies 2 | cut -c1-200
 BMOE_PAIR=$P $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 256 --iters 10 --copies 2 | cut -c1-200
done
