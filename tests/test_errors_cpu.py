"""Error-class identity with the reference (attnkit/errors.py:4-25).

With the reference installed (baseline/_ref, the unmodified attnkit), every error class of the
package subclasses its attnkit namesake, so ``except attnkit.errors.X`` written against the
reference catches what the B200 path raises. Run in a subprocess so the import order is the
one a user gets (attnkit on sys.path before the package is imported)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SCRIPT = r"""
import attnkit, attnkit.errors as ref
import paper_2603_02188_b200 as mlra
from paper_2603_02188_b200 import errors as ours
assert ours.REFERENCE_ERRORS
for name in ("AttnKitError", "ShapeMismatchError", "NumericError", "ConfigError", "RoutingError", "IntegrityError"):
    assert issubclass(getattr(ours, name), getattr(ref, name)), name
    assert issubclass(getattr(ours, name), ref.AttnKitError), name
# a reference-style caller catches the package's errors
try:
    mlra.AttnConfig("mlra", branches=3, h=4, d=32, d_h=8)
except attnkit.errors.ConfigError as e:
    print("caught", type(e).__name__)
try:
    mlra.trained_config("nope")
except attnkit.AttnKitError as e:
    print("caught", type(e).__name__)
"""


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "attnkit")), reason="reference not installed in baseline/_ref")
def test_errors_subclass_reference_classes():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    res = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    assert res.stdout.count("caught") == 2


def test_errors_standalone_without_reference():
    """Without attnkit the hierarchy still has the reference's shape."""
    code = ("import sys; sys.modules['attnkit'] = None\n"
            "from paper_2603_02188_b200 import errors as e\n"
            "assert not e.REFERENCE_ERRORS\n"
            "assert all(issubclass(getattr(e, n), e.AttnKitError) for n in "
            "('ShapeMismatchError','NumericError','ConfigError','RoutingError','IntegrityError','CudaError'))\n")
    env = dict(os.environ, PYTHONPATH=ROOT)
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
