"""B200-native BuddyMoE hot path (arxiv 2511.10054).

Drop-in for the reference ``buddysim`` package's hot path: buddy-table
construction, expert-cache / prefetch policy objects and the MoE layer
forward, running on hand-written sm_100a CUDA kernels behind a C-ABI
(``include/bmoe.h``, ``lib/libbmoe.so``). See DESIGN.md.

The package exports the reference's public names (buddysim/__init__.py:4-91)
except its configuration system (ExperimentConfig / default_config /
load_config, out of scope: every entry point also takes a dict of the dotted
keys). Names resolve lazily, so importing a leaf module (e.g. ``synth``)
stays light.
"""

from __future__ import annotations

import importlib

__version__ = "0.2.0"

_EXPORTS = {
    "buddies": ("BuddyEntry", "BuddyTable", "build_table", "cft_prefix", "load_table", "save_table",
                "table_size_report"),
    "errors": ("BuddySimError", "CalibrationError", "ConfigurationError", "DegeneratePivotError", "FormatError",
               "InputError", "InternalError", "InvariantViolation", "NativeLibraryError"),
    "gating": ("BetaController", "GateConfig", "GateOutcome", "calibrate_tau", "derive_beta", "distribution_gate",
               "evaluate_gates", "margin", "tae", "token_gate"),
    "harness": ("SimResult", "cmd_build", "cmd_profile", "cmd_report", "cmd_simulate", "fidelity", "run_oracle",
                "run_simulation"),
    "memtier": ("CostModel", "ResidencyState", "RunMetrics", "SimClock", "SimEvent", "access", "init_residency",
                "prefetch", "settle", "step_metrics"),
    "model": ("Expert", "Model", "ModelSpec", "RouterDecision", "build_model", "forward_batch", "forward_layer",
              "route", "route_batch", "token_stream"),
    "profiler": ("CoActivationStats", "ConditionalRow", "conditional_row", "load_stats", "merge", "observe",
                 "save_stats"),
    "substitution": ("PlanSlot", "PsiParams", "ReplacementPlan", "SubstitutionConfig", "Topology", "identity_plan",
                     "ondemand_plan", "psi_score", "random_plan", "substitute_batch", "substitute_token"),
}
_WHERE = {name: mod for mod, names in _EXPORTS.items() for name in names}
__all__ = sorted(_WHERE)


def __getattr__(name):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(__all__))
