python -c "import __graft_entry__ as g; g.build()" > /dev/null
for P in 4194304 16777216 33554432 8388608; do
 BMOE_XFER_PIECE=$P timeout 600 python bench.py --no-cpu --no-original 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($P, 'tok/s %.2f e2e %.2f'%(d['value'], d['e2e']['value']), 'stall %.1f'%d['stall_ms_per_step'], 'fetch', round(d['fetch_roofline']['frac'],4), round(d['fetch_roofline']['achieved'],2), 'roof', round(d['roofline']['frac'],3))"
done
