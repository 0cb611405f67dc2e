"""The reference's own hot-path tests, run unmodified against this package.

tests/ref_suite/ref_shim.py aliases ``kvmix.quant`` / ``kvmix.pool`` / ``kvmix.errors`` and
the decode + replay entry points of ``kvmix.attention`` to paper_2605_17170_b200, then
pytest runs the vendored copies (tools/vendor_ref_suite.py; git-ignored) of
pkg/tests/test_quant.py, test_pool.py, test_attention.py and the hot-path acceptance
criteria of test_acceptance.py (01-04 codec / layout / flash decode / split-merge,
07-09 budget arithmetic, capacity headroom, pool safety).  The layout golden files
criterion 02 reads are written from tests/golden/golden.npz, which the real reference
produced (tests/golden/make_golden.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SUITE = os.path.join(HERE, "ref_suite", "_vendored", "tests")
FILES = ["test_quant.py", "test_pool.py", "test_attention.py", "test_acceptance.py"]
ACCEPTANCE = "test_01 or test_02 or test_03 or test_04 or test_07 or test_08 or test_09"


@pytest.fixture
def suite(cuda):
    if not os.path.isdir(SUITE):
        pytest.skip("reference suite not vendored (run tools/vendor_ref_suite.py where the reference is mounted)")
    gold = os.path.join(SUITE, "golden")
    os.makedirs(gold, exist_ok=True)
    g = np.load(os.path.join(HERE, "golden", "golden.npz"))
    for key in g.files:
        if key.startswith("layout_key_page") or key.startswith("layout_token_block"):
            with open(os.path.join(gold, key[len("layout_"):] + ".bin"), "wb") as f:
                f.write(g[key].tobytes())
    return SUITE


@pytest.mark.parametrize("name", FILES)
def test_reference_suite_file(suite, name):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(HERE, "ref_suite"), suite]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-rA", "-p", "ref_shim", "-p", "no:cacheprovider", "--rootdir", suite,
           os.path.join(suite, name)]
    if name == "test_acceptance.py":
        cmd += ["-k", ACCEPTANCE]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800, cwd=suite)
    tail = "\n".join(p.stdout.strip().splitlines()[-25:])
    print(tail)
    out_dir = os.path.join(os.path.dirname(HERE), "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, f"ref_suite_{name[:-3]}.txt"), "w") as f:
            f.write(p.stdout[-20000:] + p.stderr[-5000:])
    assert p.returncode == 0, f"reference suite {name} failed:\n{tail}\n{p.stderr[-3000:]}"
