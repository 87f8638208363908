for NT in 128 256; do
for B in 2048 8192; do python tools/ffn_microbench.py --E 128 --experts-active 128 --d 2048 --f 768 --k 8 --tokens $B --n-tile $NT --iters 20 --copies 2 | cut -c1-220; done
python tools/ffn_microbench.py --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile $NT --iters 10 --copies 2 | cut -c1-220
done
