# token-major SwiGLU GEMM1 tiles (BMOE_TM) vs weight-major: parity tests and timing
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_engine_shapes_gpu.py -q -x > gpurun_out/tm_tests.txt 2>&1; tail -3 gpurun_out/tm_tests.txt
timeout 600 python - > gpurun_out/tm_bitwise.txt 2>&1 <<'PY'
import os, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2511_10054_b200 import ops
torch.manual_seed(0)
for (E,d,f,B,k) in [(128,2048,768,2048,8),(8,4096,14336,512,2),(64,2048,1408,1024,6)]:
    dev='cuda'
    ar = torch.empty(E, 3*d*f, device=dev, dtype=torch.bfloat16)
    for e in range(E):
        w = (torch.randn(3*d*f, device=dev)*0.02).to(torch.bfloat16)
        ops.pack_expert_bf16(w[:f*d].view(f,d), w[f*d:2*f*d].view(f,d), w[2*f*d:].view(d,f), ops.ACT_SWIGLU, ar[e])
    rng=np.random.default_rng(1)
    topk=np.stack([rng.choice(E,k,replace=False) for _ in range(B)]).astype(np.int32)
    perm=ops.permute(torch.from_numpy(topk).to(dev), torch.zeros(B,k,dtype=torch.uint8,device=dev), E)
    x=torch.randn(B,d,device=dev); xp=ops.gather_rows(x,perm,1)
    bufs=torch.arange(E,device=dev,dtype=torch.int32)
    outs=[]
    for tm in ('0','1'):
        os.environ['BMOE_TM']=tm
        ws=ops.FfnWorkspace(E,d,f,perm.r_max,128)
        y=ops.expert_ffn_bf16(xp,perm,ar,bufs,d,f,ops.ACT_SWIGLU,ws)
        torch.cuda.synchronize(); outs.append(y.clone())
    same=torch.equal(outs[0],outs[1]); md=(outs[0]-outs[1]).abs().max().item(); rel=((outs[0]-outs[1]).norm()/outs[0].norm()).item()
    print(dict(E=E,d=d,f=f,B=B,k=k,bitwise_equal=same,max_abs_diff=md,rel=rel))
PY
cat gpurun_out/tm_bitwise.txt | tail -5
mb="python tools/ffn_microbench.py --iters 20 --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --copies 2 --n-tile 128"
for tm in 0 1; do for T in 2048 8192; do BMOE_TM=$tm timeout 300 $mb --tokens $T | sed "s/^{/{\"BMOE_TM\": $tm, /" | tee -a gpurun_out/r2s_prefill_tm.jsonl; done; done
for tm in 0 1; do for m in 0 1; do BMOE_TM=$tm BMOE_2SM=$m timeout 300 python tools/ffn_microbench.py --iters 10 --experts-active 8 --k 2 --tokens 4096 --n-tile 128 --copies 2 | sed "s/^{/{\"BMOE_TM\": $tm, \"BMOE_2SM\": $m, /" | tee -a gpurun_out/r2s_prefill_tm.jsonl; done; done
