import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2511_10054_b200 import ops
import paper_2511_10054_b200._native as N
rng = np.random.default_rng(5)
E, d, f, B, k = 8, 256, 384, 24, 2
w1 = rng.standard_normal((E, f, d)).astype(np.float32) / np.sqrt(d)
w3 = rng.standard_normal((E, f, d)).astype(np.float32) / np.sqrt(d)
w2 = rng.standard_normal((E, d, f)).astype(np.float32) / np.sqrt(f)
arena = torch.from_numpy(np.concatenate([w1.reshape(E, -1), w3.reshape(E, -1), w2.reshape(E, -1)], axis=1)).cuda()
topk = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
kind = np.zeros((B, k), np.uint8)
x = rng.standard_normal((B, d)).astype(np.float32)
perm = ops.permute(torch.from_numpy(topk).cuda(), torch.from_numpy(kind).cuda(), E)
print("count", perm.count.cpu().numpy(), "offset", perm.offset.cpu().numpy(), "rmax", perm.r_max)
xp = ops.gather_rows(torch.from_numpy(x).cuda(), perm, 0)
print("xp nan", torch.isnan(xp[:perm.offset[-1]]).sum().item())
h = torch.full((perm.r_max, f), 7.0, device='cuda'); y = torch.full((perm.r_max, d), 7.0, device='cuda')
N.call("bm_expert_ffn_f32", xp.data_ptr(), perm.count.data_ptr(), perm.offset.data_ptr(), E, d, f, 1, arena.data_ptr(), arena.shape[1], torch.arange(E, dtype=torch.int32, device='cuda').data_ptr(), perm.r_max, h.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
R = int(perm.offset[-1])
print("h nan", torch.isnan(h[:R]).sum().item(), "y nan", torch.isnan(y[:R]).sum().item(), h[:2,:4], y[:2,:4])
