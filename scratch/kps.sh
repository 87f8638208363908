python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_xfer_gpu.py -q -x 2>&1 | tail -2
mb="python tools/ffn_microbench.py"
for K in 1 2; do
 BMOE_KPS=$K $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --iters 10 --copies 2 | cut -c1-190
 BMOE_KPS=$K $mb --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens 8192 --n-tile 128 --iters 10 --copies 2 | cut -c1-190
done
