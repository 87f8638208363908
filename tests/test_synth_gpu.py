"""The GPU arm and the CPU reference arm of bench.py work on the same inputs:
bm_synth_bf16 writes the bits of the numpy twin (synth.py), the pinned
mirrors hold exactly those experts, and the buddy tables the GPU profiles
equal (digest) the ones oracle/decode_cpu.py builds on the host."""

import numpy as np
import pytest
import torch

from paper_2511_10054_b200 import ops, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 5, 8, 4099, 1 << 20, 3 * 2048 * 768 + 4])
def test_kernel_equals_numpy_twin(cuda_ok, n):
    for layer, expert, m in ((0, 0, synth.W1), (3, 9, synth.W2)):
        lut = synth.lut_bf16(synth.matrix_scale(2048, 768, m))
        base = synth.matrix_key(0, layer, expert, m)
        dev_lut = torch.from_numpy(lut.view(np.int16)).cuda()
        out = torch.empty(n + 1, dtype=torch.bfloat16, device="cuda")
        ops.synth_bf16(dev_lut, base, out[1:])  # misaligned destination too
        ops.synth_bf16(dev_lut, base, out[:n])
        got = out[:n].view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, synth.synth_bits(base, n, lut))


def test_gpu_and_cpu_arms_share_weights_and_tables(cuda_ok):
    from oracle.decode_cpu import CpuDecode, tables_digest
    from paper_2511_10054_b200 import workload as W
    from paper_2511_10054_b200.engine import mirror_expert
    wl = W.build("qwen3", layers=2, max_batch=16, profile_tokens=1024, profile="route")
    cd = CpuDecode("qwen3", 2, 16, profile_tokens=1024, profile="route")
    try:
        gpu = tables_digest(wl.tbl_ids.cpu().numpy(), wl.tbl_len.cpu().numpy())
        assert gpu == cd.digest
        assert np.allclose(np.array(wl.taus), np.array(cd.taus), rtol=0, atol=1e-6)
        E, d, f = 128, 2048, 768
        ex = cd.layer_experts(1)
        for e in (0, 77, 127):
            # the mirror holds the UMMA-tiled image: unpack through a row-major repack of the host weights
            w1, w3, w2 = (torch.from_numpy(a).to(torch.bfloat16).cuda() for a in ex[e])
            ref = ops.pack_expert_bf16(w1, w3, w2, ops.ACT_SWIGLU)
            got = mirror_expert(wl.mirrors[1], e, 3 * d * f)
            assert torch.equal(got.view(torch.int16), ref.view(-1).view(torch.int16)), e
    finally:
        cd.close()
        wl.close()


@pytest.mark.parametrize("n", [3, 4099, 2048 * 768 + 1])
def test_clustered_kernel_equals_numpy_twin(cuda_ok, n):
    from paper_2511_10054_b200 import _native as N
    lut = synth.lut_bf16(synth.matrix_scale(2048, 768, synth.W1))
    bk, dk = synth.base_key(0, 1, 3, synth.W1), synth.matrix_key(0, 1, 42, synth.W1)
    dev_lut = torch.from_numpy(lut.view(np.int16)).cuda()
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    N.call("bm_synth_mix_bf16", dev_lut.data_ptr(), bk, dk, synth.SPREAD, n, out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = synth.mix_bits(synth.synth_bits(bk, n, lut), synth.synth_bits(dk, n, lut), synth.SPREAD)
    assert np.array_equal(got, ref)
