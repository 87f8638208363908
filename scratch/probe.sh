python -c "import __graft_entry__ as g; g.build()" > /dev/null
mb="timeout 120 python tools/ffn_microbench.py"
for PR in 0 1 2; do for P in 1 0; do
 echo "probe $PR pair $P"; BMOE_PROBE=$PR BMOE_PAIR=$P $mb --E 8 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --iters 10 --copies 2 | cut -c1-120
done; done
