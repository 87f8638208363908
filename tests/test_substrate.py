"""The synthetic substrate restatement is bit-identical to the reference's."""

import numpy as np

from conftest import golden
from paper_2511_10054_b200 import substrate as S


def _specs():
    return {
        "tiny": S.ModelSpec(num_layers=4, experts_per_layer=8, top_k=2, hidden_dim=128, ffn_dim=256,
                            num_clusters=8),
        "dflt": S.ModelSpec(),
        "odd": S.ModelSpec(num_layers=2, experts_per_layer=12, top_k=3, hidden_dim=20, ffn_dim=36,
                           num_clusters=5, skew=0.0, seed=99, cluster_spread=0.3),
    }


def test_substrate_bit_identical():
    g = golden("substrate.npz")
    for name, spec in _specs().items():
        gw, gb = S.gate_weights(spec)
        assert np.array_equal(gw, g[f"{name}_gate_w"]) and np.array_equal(gb, g[f"{name}_gate_b"])
        wi, wo = S.layer_stack(spec, spec.num_layers - 1)
        assert np.array_equal(wi[0], g[f"{name}_w_in_e0"]) and np.array_equal(wo[-1], g[f"{name}_w_out_elast"])
        assert np.array_equal(wi.sum(axis=(1, 2)), g[f"{name}_w_in_sum"])
        assert np.array_equal(wo.sum(axis=(1, 2)), g[f"{name}_w_out_sum"])
        assert np.array_equal(S.token_stream(spec, 5, 64), g[f"{name}_stream"])
        assert np.array_equal(S.readout_head(spec, 16), g[f"{name}_readout"])
