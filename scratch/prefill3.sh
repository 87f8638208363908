python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
mb="python tools/ffn_microbench.py"
for NT in 128 256; do
 $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile $NT --iters 10 --copies 2 | cut -c1-200
 $mb --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile $NT --iters 10 --copies 2 | cut -c1-200
done
$mb --experts-active 4 --k 2 --iters 40 | cut -c1-200
