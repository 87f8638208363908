"""Host-side harness pieces that need no GPU: the tae_samples.txt format
(harness.py:112-129) and the builder.alpha list rule (config.py:198-214)."""

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
