"""ragsim's own test suite (pkg/tests, 170 tests) run with the drop-in engine.

tests/dropin_plugin.py replaces ragsim.simulator.SimulationEngine with this package's
TieredEngine over the native block pool (accounting mode, one token per block) before
the reference's tests are collected, so every ``run`` / ``measure_throughput`` / CLI
run they make goes through TieredKnowledgeTree and replays each tier transition on the
native allocator.  The reference suite must pass unchanged (the
reference's acceptance criteria C1-C8, tree/simulator/speculation unit tests).
Runs in this container only: the reference's tests are not shipped to the GPU box.
"""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference test suite not present")
def test_reference_suite_passes_with_the_dropin_engine():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")  # the reference tree is read-only
    r = subprocess.run([sys.executable, "-m", "pytest", REF_TESTS, "-p", "tests.dropin_plugin",
                        "-p", "no:cacheprovider", "-o", "addopts=", "-q"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = "\n".join(r.stdout.splitlines()[-15:])
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
    engines = int(tail.split("drop-in engines constructed:")[1].split()[0])
    assert engines > 100, tail  # the suite's runs really went through the drop-in
