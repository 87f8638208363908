"""The synthetic-weight generator's host twins agree bit for bit: the numpy
restatement (paper_2511_10054_b200/synth.py) and the oracle's C helper that
bench.py's CPU reference arm uses (oracle/c/synth_host.c). The GPU kernel is
checked against the same numpy twin in test_synth_gpu.py."""

import os
import subprocess

import numpy as np
import pytest

from paper_2511_10054_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def host_lib():
    from oracle import synth_host
    if not synth_host.available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
        synth_host._h = None
    assert synth_host.available()
    return synth_host


@pytest.mark.parametrize("n", [1, 3, 4, 5, 4096 * 3 + 1, 1 << 20])
def test_numpy_twins_agree(n):
    base = synth.matrix_key(0, 7, 3, synth.W2)
    lut = synth.lut_bf16(synth.matrix_scale(4096, 14336, synth.W2))
    bits = synth.synth_bits(base, n, lut)
    f64 = synth.synth_f64(base, n, synth.matrix_scale(4096, 14336, synth.W2), chunk=1 << 12)
    assert np.array_equal(synth.bf16_to_f64(bits), f64)


@pytest.mark.parametrize("n", [1, 7, 4096 * 5 + 3, (1 << 22) + 9])
def test_oracle_c_twin_agrees(host_lib, n):
    for layer, expert, m in ((0, 0, synth.W1), (31, 7, synth.W3), (5, 65, synth.W2)):
        base = synth.matrix_key(0, layer, expert, m)
        lut = synth.lut_bf16(synth.matrix_scale(2048, 1408, m))
        ref = synth.bf16_to_f64(synth.synth_bits(base, n, lut))
        got = host_lib.synth_f64(base, n, synth.bf16_to_f64(lut), threads=3, chunk=1 << 16)
        assert np.array_equal(ref, got)


def test_distribution_and_distinct_streams():
    d, f = 2048, 768
    a = synth.bf16_to_f64(synth.synth_bits(synth.matrix_key(0, 0, 0, synth.W1), 1 << 20,
                                           synth.lut_bf16(synth.matrix_scale(d, f, synth.W1))))
    b = synth.bf16_to_f64(synth.synth_bits(synth.matrix_key(0, 0, 1, synth.W1), 1 << 20,
                                           synth.lut_bf16(synth.matrix_scale(d, f, synth.W1))))
    assert abs(a.mean()) < 3e-3 * d ** -0.5 * 10 and abs(a.std() * d ** 0.5 - 1.0) < 5e-3
    assert not np.array_equal(a, b) and abs(np.corrcoef(a, b)[0, 1]) < 5e-3
    keys = {synth.matrix_key(s, l, e, m) for s in (0, 1) for l in range(48) for e in range(130) for m in range(3)}
    assert len(keys) == 2 * 48 * 130 * 3


def test_clustered_twins_agree(host_lib):
    """Clustered experts (base_cluster + spread * delta, fp32 then bf16): the
    numpy twin and the oracle's C twin agree bit for bit, and cluster mates
    are near-identical while other clusters are unrelated."""
    d, f = 2048, 768
    n = d * f + 3
    lut16 = synth.lut_bf16(synth.matrix_scale(d, f, synth.W2))
    mats = []
    for e, c in ((0, 0), (1, 0), (5, 1)):
        bk, dk = synth.base_key(0, 2, c, synth.W2), synth.matrix_key(0, 2, e, synth.W2)
        ref = synth.bf16_to_f64(synth.mix_bits(synth.synth_bits(bk, n, lut16), synth.synth_bits(dk, n, lut16),
                                               synth.SPREAD))
        out = np.empty(n)
        for t in host_lib.fill_mix_tasks(bk, dk, synth.SPREAD, n, lut16, out, chunk=1 << 16):
            t()
        assert np.array_equal(ref, out)
        mats.append(ref)
    assert np.corrcoef(mats[0], mats[1])[0, 1] > 0.98 and abs(np.corrcoef(mats[0], mats[2])[0, 1]) < 0.01
