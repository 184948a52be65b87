"""The reference's own test suite against the drop-ins (SURVEY.md 8(c):
"run the reference tests' arithmetic against the drop-in").

The unmodified reference tests (``pkg/tests/test_srp.py``,
``test_spectral.py``, ``test_acceptance.py``, ``test_metrics.py``,
``test_experiment.py``; copied with the pip-installed reference into the
git-ignored ``baseline/_ref``) run in a child pytest with
``tests/refsuite_plugin.py``: the reference's hot-path names are rebound to
this package's drop-ins before the tests import them, and fp64 tolerances
are widened to the fp32 path's (the plugin docstring says exactly how).
Every reference test must pass except the ones listed in ``EXPECTED_FAIL``
with the reason they cannot hold for an fp32 device path.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
SUITE = os.path.join(ROOT, "baseline", "_ref", "srpfast_tests")

#: reference tests that check fp64-only properties of the reference's own
#: numerics, with the reason (none may fail for any other reason)
EXPECTED_FAIL = {
    # plain `assert max|a - b| <= 1e-12 * scale` (no approx call the plugin
    # could widen) between the fp32 map and an fp64 restatement; measured
    # ~1e-6 of the scale, the fp32 path's accuracy (north_star 1e-5 rel-L2).
    # tests/test_crosscheck_gpu.py checks the same identities at 1e-5.
    "test_conventional_matches_pairwise_reference": "fp64-only tolerance (1e-12 of scale)",
    "test_oracle_equals_conventional": "fp64-only tolerance (1e-9 of scale)",
    # PHAT magnitude <= 1 + 1e-12 and an fp64 DFT leakage floor (1e-8 of the
    # line): the fp32 rsqrt-normalised psi is 1 +- 6e-8, the fp32 FFT leaks
    # ~3e-8 of the line (K0 and K1 are checked at 2e-6 in test_parity_gpu.py)
    "test_phat_is_unit_modulus": "fp64-only bound (1 + 1e-12)",
    "test_sinusoid_concentrates_in_its_bin": "fp64-only leakage floor (1e-8)",
    # acceptance criteria 3 and 4 assert fp64 agreement (1e-9, 1e-10); the
    # drop-ins measure 1.6e-6 and 5.3e-7 -- test_crosscheck_gpu.py and
    # test_parity_gpu.py::test_approx_exact_on_lattice hold them at 1e-5
    "test_criterion_3_oracle_equivalence": "fp64-only tolerance (measured 1.6e-6)",
    "test_criterion_4_interpolation_exact_on_lattice": "fp64-only tolerance (1e-10)",
    # the reference's scene-level ProcessPoolExecutor forks after CUDA is
    # initialised (experiment.py:631-641), which CUDA forbids; the B200 path
    # replaces that parallelism with frame sharding over GPUs (distributed.py)
    "test_workers_do_not_change_results": "fork after CUDA init",
}


@pytest.mark.parametrize("module", ["test_srp.py", "test_spectral.py", "test_acceptance.py",
                                    "test_metrics.py", "test_experiment.py"])
def test_reference_suite_on_drop_ins(module):
    path = os.path.join(SUITE, module)
    if not os.path.exists(path):
        pytest.skip("baseline/_ref not installed (see DESIGN.md: pip install --target "
                    "baseline/_ref the reference + its tests)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT,
                                         os.path.join(ROOT, "baseline", "_ref"),
                                         env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", path, "-q", "-p", "refsuite_plugin",
         "-p", "no:cacheprovider", "--rootdir", SUITE, "-o", "addopts=", "-rfE"],
        capture_output=True, text=True, env=env, cwd=SUITE, timeout=1800)
    out = proc.stdout + proc.stderr
    failed = set(re.findall(r"^(?:FAILED|ERROR) \S+::(\S+)", out, re.M))
    unexpected = {t for t in failed if t.split(" ")[0] not in EXPECTED_FAIL}
    assert "rebound to paper_2012_09499_b200" in out, out[-3000:]
    assert not unexpected, out[-6000:]
    assert re.search(r"\d+ passed", out), out[-3000:]
