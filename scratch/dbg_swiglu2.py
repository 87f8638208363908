import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2511_10054_b200 import ops
import paper_2511_10054_b200._native as N
def run(act, E, d, f, B, k):
    rng = np.random.default_rng(5)
    nm = 3 if act == 1 else 2
    arena = torch.randn(E, nm*d*f, device='cuda') * 0.05
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
    kind = np.zeros((B, k), np.uint8)
    x = rng.standard_normal((B, d)).astype(np.float32)
    perm = ops.permute(torch.from_numpy(topk).cuda(), torch.from_numpy(kind).cuda(), E)
    xp = ops.gather_rows(torch.from_numpy(x).cuda(), perm, 0)
    h = torch.full((perm.r_max, f), 7.0, device='cuda'); y = torch.full((perm.r_max, d), 7.0, device='cuda')
    N.call("bm_expert_ffn_f32", xp.data_ptr(), perm.count.data_ptr(), perm.offset.data_ptr(), E, d, f, act, arena.data_ptr(), arena.shape[1], torch.arange(E, dtype=torch.int32, device='cuda').data_ptr(), perm.r_max, h.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    R = int(perm.offset[-1])
    # reference for h of row 0
    r = 0; t = int(perm.row_token[0]); e = 0
    while int(perm.offset[e+1]) <= r: e += 1
    W = arena[e]
    if act == 1:
        g = x[t] @ W[:f*d].view(f,d).cpu().numpy().T; u = x[t] @ W[f*d:2*f*d].view(f,d).cpu().numpy().T
        href = g/(1+np.exp(-g))*u
    else:
        href = np.tanh(x[t] @ W[:f*d].view(f,d).cpu().numpy().T)
    print(act, E, d, f, "h nan", torch.isnan(h[:R]).sum().item(), "h0 err", np.abs(h[0].cpu().numpy()-href).max())
for args in [(0,8,256,384,24,2),(1,8,256,384,24,2),(1,8,128,256,24,2),(0,8,128,256,24,2)]:
    run(*args)
