"""The reference's OWN tests, unchanged, against this engine (VERDICT r1
"Next" item 3; INTEGRATION.md sections 1-2).

build() installs the reference package into baseline/_ref (git-ignored,
shipped to the GPU box) together with a copy of its test files
(baseline/_ref/_ref_tests).  Here they run in a subprocess with
tests/ref_suite_plugin.py, which puts the GPU kernels into the reference's
compiled-kernel slot and (MDRQ_DEVICE_METHODS=1) the GPU access methods
behind ``mdrq.build_method``:

* pkg/tests/test_kernels.py -- backend equivalence: the pure-Python kernels
  vs the GPU ``match_row`` / ``scan_rows`` / ``scan_column``;
* pkg/tests/test_scan.py -- the reference's scan classes over the GPU kernels;
* pkg/tests/test_acceptance.py::test_c01 / test_c02 -- oracle equivalence of
  build_method("sequential" | "horizontal" | "vertical" | "vafile") (the GPU
  methods) with the reference's SequentialScan(SCALAR), and kernel-mode
  equivalence through ``mdrq.kernels``.
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "_ref_tests")
SELECTION = ["test_kernels.py", "test_scan.py", "test_acceptance.py::test_c01_oracle_equivalence",
             "test_acceptance.py::test_c02_kernel_equivalence",
             # pins the reference's two backend NAMES ("compiled" / "python");
             # the GPU module reports its own ("cuda") by design -- every
             # behavioural kernel test of the file runs
             "--deselect", "test_kernels.py::test_backend_selection_reports_name"]


def _run(args, env_extra, timeout):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")] +
                                        ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env.update(env_extra)
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_suite_plugin",
                           "--rootdir", REF_TESTS, "-c", os.devnull] + args,
                          cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=timeout)


def _require_reference():
    if not os.path.isdir(os.path.join(REF, "mdrq")) or not os.path.isdir(REF_TESTS):
        pytest.skip("reference not installed in baseline/_ref (build() installs it where /root/reference exists)")


@pytest.mark.gpu
def test_reference_suite_on_gpu_engine(gpu):
    _require_reference()
    r = _run(SELECTION, {"MDRQ_DEVICE_METHODS": "1"}, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail


def test_reference_backend_registers_without_device():
    """CPU: the plugin wires the GPU kernel module into the reference
    (mdrq.kernels.BACKEND == "cuda", the scan kernels are ours, the tree
    kernels stay the reference's compiled ones) and wraps build_method; no
    compute call is made."""
    _require_reference()
    prog = (
        "from paper_1801_03644_b200 import reference_backend as rb, kernels as g\n"
        "m = rb.install_kernels(); rb.install_methods()\n"
        "import mdrq, mdrq.kernels as k\n"
        "assert k.BACKEND == 'cuda', k.BACKEND\n"
        "assert k.scan_rows is g.scan_rows and k.scan_column is g.scan_column and k.match_row is g.match_row\n"
        "assert k.kd_build is not None and k.kd_build.__module__ != g.__name__\n"
        "assert mdrq.build_method.__wrapped__ is not None\n"
        "print('ok')\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT])
    r = subprocess.run([sys.executable, "-c", prog], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
