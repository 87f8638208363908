#!/usr/bin/env python
"""Run the REFERENCE's own test suite against this package (drop-in check).

    python tools/conformance.py stage   # here, where /root/reference exists
    python tools/conformance.py run     # on the GPU box (after a gpurun push)

``stage`` copies the reference's tests (pkg/tests) and its out-of-scope
configuration / CLI modules (config.py, cli.py, __main__.py) into
baseline/_ref/conformance/ — git-ignored, so nothing of the reference enters
the repository, but shipped to the GPU box with the gpurun snapshot.

``run`` builds a ``buddysim`` alias package whose hot-path modules ARE this
package's (buddies, errors, gating, harness, memtier, model, profiler,
substitution, registered in sys.modules), with the reference's own config /
CLI modules layered on top of them (their relative imports resolve to the
aliased modules), then runs pytest over the reference's tests and writes a
summary (counts, every failure with its first error line) to
profiles/r2_conformance.txt and the junit XML next to it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = os.path.join(ROOT, "baseline", "_ref", "conformance")
REF = "/root/reference/pkg"

ALIAS_INIT = '''"""buddysim alias: the hot-path modules are paper_2511_10054_b200's."""
import importlib
import sys

import paper_2511_10054_b200 as _P

for _n in ("buddies", "errors", "gating", "harness", "memtier", "model", "profiler", "substitution"):
    sys.modules[__name__ + "." + _n] = importlib.import_module("paper_2511_10054_b200." + _n)
    globals()[_n] = sys.modules[__name__ + "." + _n]
from paper_2511_10054_b200 import *  # noqa: E402,F401,F403

from . import config  # noqa: E402  (the reference's own config module, out of scope)
from .config import ExperimentConfig, default_config, load_config  # noqa: E402,F401

__version__ = _P.__version__
'''


def stage() -> None:
    if os.path.exists(STAGE):
        shutil.rmtree(STAGE)
    shutil.copytree(os.path.join(REF, "tests"), os.path.join(STAGE, "tests"),
                    ignore=shutil.ignore_patterns("__pycache__"))
    os.makedirs(os.path.join(STAGE, "ref_modules"))
    for f in ("config.py", "cli.py", "__main__.py"):
        shutil.copy(os.path.join(REF, "src", "buddysim", f), os.path.join(STAGE, "ref_modules", f))
    print("staged", STAGE)


def run(extra=()) -> int:
    alias = os.path.join(STAGE, "alias")
    pkg = os.path.join(alias, "buddysim")
    if os.path.exists(alias):
        shutil.rmtree(alias)
    os.makedirs(pkg)
    for f in os.listdir(os.path.join(STAGE, "ref_modules")):
        shutil.copy(os.path.join(STAGE, "ref_modules", f), os.path.join(pkg, f))
    with open(os.path.join(pkg, "__init__.py"), "w") as fh:
        fh.write(ALIAS_INIT)
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    xml = os.path.join(out_dir, "r2_conformance.junit.xml")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([alias, ROOT, os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", os.path.join(STAGE, "tests"), "-q", "-p", "no:cacheprovider",
           "--junitxml", xml, *extra]
    r = subprocess.run(cmd, cwd=os.path.join(STAGE, "tests"), env=env, capture_output=True, text=True)
    summary = summarise(xml)
    with open(os.path.join(out_dir, "r2_conformance.txt"), "w") as fh:
        fh.write(summary + "\n\n---- pytest tail ----\n" + "\n".join(r.stdout.splitlines()[-40:]) + "\n")
    print(summary)
    return r.returncode


def summarise(xml: str) -> str:
    tree = ET.parse(xml)
    cases = list(tree.iter("testcase"))
    failed, skipped = [], []
    for c in cases:
        name = f"{os.path.basename(c.get('classname', '').replace('.', '/'))}::{c.get('name')}"
        for tag in ("failure", "error"):
            el = c.find(tag)
            if el is not None:
                msg = (el.get("message") or el.text or "").strip().splitlines()
                failed.append(f"{name}: {msg[0][:200] if msg else tag}")
        if c.find("skipped") is not None:
            skipped.append(name)
    n = len(cases)
    lines = [f"reference test suite (pkg/tests, {n} tests) against paper_2511_10054_b200 through a buddysim alias",
             f"passed {n - len(failed) - len(skipped)} / failed {len(failed)} / skipped {len(skipped)}", ""]
    lines += ["FAILED " + f for f in failed]
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1:2] == ["stage"]:
        stage()
    elif sys.argv[1:2] == ["run"]:
        sys.exit(run(sys.argv[2:]))
    else:
        print(__doc__)
        sys.exit(2)
