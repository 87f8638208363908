"""Host-side harness pieces that need no GPU: the tae_samples.txt format
(harness.py:112-129) and the builder.alpha list rule (config.py:198-214)."""

import os

import numpy as np
import pytest

from paper_2511_10054_b200 import harness
from paper_2511_10054_b200.errors import ConfigurationError, FormatError


def test_tae_samples_file_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    samples = [rng.random(7), rng.random(3)]
    p = tmp_path / "tae_samples.txt"
    harness.save_tae_samples(samples, p)
    lines = p.read_text().splitlines()
    assert lines[0] == "bsim/1" and lines[1] == f"0 {float(samples[0][0])!r}" and len(lines) == 11
    back = harness.load_tae_samples(p)
    assert back[0] == list(samples[0]) and back[1] == list(samples[1])
    p.write_text("bsim/2\n0 0.5\n")
    with pytest.raises(FormatError):
        harness.load_tae_samples(p)


def test_alpha_list_rule():
    assert harness._alphas({"builder.alpha": "0.9"}, 3) == [0.9, 0.9, 0.9]
    assert harness._alphas({"builder.alpha": "0.9, 0.8"}, 2) == [0.9, 0.8]
    with pytest.raises(ConfigurationError):
        harness._alphas({"builder.alpha": "0.9,0.8"}, 3)
    with pytest.raises(ConfigurationError):
        harness._alphas({"builder.alpha": "1.5"}, 1)


def _bsst_fields(raw: bytes):
    """A BSST v1 file's fields, parsed here independently of the package."""
    import struct
    from types import SimpleNamespace
    magic, ver, layer, E, ws, ww, eps, seen = struct.unpack_from("<4sIIIIddQ", raw)
    off = struct.calcsize("<4sIIIIddQ")
    a = np.frombuffer(raw, "<f8", offset=off)
    return SimpleNamespace(layer=layer, num_experts=E, warmup_steps=ws, warmup_weight=ww, laplace_eps=eps,
                           tokens_seen=seen, counts=a[:E], pair_counts=a[E:E + E * E].reshape(E, E),
                           pair_weights=a[E + E * E:].reshape(E, E))


def test_reference_profile_files_written_byte_identical(tmp_path):
    """The reference's own cmd_profile / cmd_build files for the tiny config
    (tests/golden/files_tiny.npz, written by the reference's writers,
    profiler.py:140-160, buddies.py:164-222). This package's writers (the
    ones run_profile / run_build call) reproduce them byte for byte from the
    same contents: BSST, BSBT (read back by this package's reader, which is
    host code) and both CSV exports. (The GPU suite also checks the files the
    GPU pipeline writes, test_engine_gpu.py.)"""
    from paper_2511_10054_b200 import buddies, profiler
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "files_tiny.npz"))
    for key in z.files:
        (tmp_path / ("in_" + key.split("/")[1])).write_bytes(z[key].tobytes())
    n = 0
    for key in z.files:
        name = key.split("/")[1]
        out = tmp_path / ("out_" + name)
        if name.startswith("stats_"):
            profiler.save_stats(_bsst_fields(z[key].tobytes()), out)
        elif name.startswith("coact_"):
            stats = _bsst_fields((tmp_path / ("in_" + name.replace("coact_", "stats_").replace(".csv", ".bin")))
                                 .read_bytes())
            profiler.export_coactivation_csv(stats, out, mode="binary")
        elif name.startswith("buddies_") and name.endswith(".bin"):
            buddies.save_table(buddies.load_table(tmp_path / ("in_" + name)), out)
        elif name.startswith("buddies_") and name.endswith(".csv"):
            buddies.export_table_csv(buddies.load_table(tmp_path / ("in_" + name.replace(".csv", ".bin"))), out)
        else:
            continue
        assert out.read_bytes() == z[key].tobytes(), key
        n += 1
    assert n == 16
