"""Randomized sweeps as regression tests: the public API against the oracle on
the classes where parity is well posed (tools/fuzz_api.py strict) and the
product kernels / CSR operator / eigensolver against FP64 references
(tools/fuzz_kernels.py). Both print each failing case with its parameters."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(script, *args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", script), *args], capture_output=True, text=True,
                       timeout=900)
    tail = "\n".join(r.stdout.strip().splitlines()[-25:])
    assert r.returncode == 0, tail + "\n" + r.stderr[-2000:]


@pytest.mark.parametrize("seed", ["21", "22"])
def test_api_sweep_against_oracle(seed):
    _run("fuzz_api.py", "250", seed, "strict")


def test_kernel_sweep_against_fp64_references():
    _run("fuzz_kernels.py", "250", "23")


def test_virtual_shard_sweep_against_unsharded():
    _run("fuzz_shards.py", "80", "24")
