"""Copy the reference's own hot-path test suite next to a shim that runs it against this
package (SURVEY 8(b) "Callers": the strongest drop-in evidence).

Run in the build container, where the read-only reference is mounted:
    python tools/vendor_ref_suite.py
The copies land in tests/ref_suite/_vendored/ -- git-ignored (reference sources are never
committed) but not gpurun-ignored, so they travel to the GPU box, where
tests/test_ref_suite.py runs them with tests/ref_suite/ref_shim.py.  The out-of-scope
reference modules (tags, capture, calibration, allocation, cli, ...) are vendored too:
the suite's conftest and the acceptance tests import them, and they are host-side code
that stays in Python per the north_star.
"""
import os
import shutil

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "tests", "ref_suite", "_vendored")
TESTS = ["conftest.py", "test_quant.py", "test_pool.py", "test_attention.py", "test_acceptance.py"]


def main():
    if not os.path.isdir(REF):
        raise SystemExit(f"{REF} is not mounted")
    shutil.rmtree(DST, ignore_errors=True)
    os.makedirs(os.path.join(DST, "src"))
    shutil.copytree(os.path.join(REF, "src", "kvmix"), os.path.join(DST, "src", "kvmix"),
                    ignore=shutil.ignore_patterns("__pycache__"))
    os.makedirs(os.path.join(DST, "tests"))
    for t in TESTS:
        shutil.copy2(os.path.join(REF, "tests", t), os.path.join(DST, "tests", t))
    print(f"vendored {len(TESTS)} test files and the kvmix sources into {DST}")


if __name__ == "__main__":
    main()
