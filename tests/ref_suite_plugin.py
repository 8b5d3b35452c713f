"""pytest plugin: run the reference's own test files against this engine.

Loaded with ``-p ref_suite_plugin`` by tests/test_reference_suite.py before
the reference package is imported: the reference's compiled kernel module
is swapped for the GPU kernels (paper_1801_03644_b200.reference_backend),
and with MDRQ_DEVICE_METHODS=1 ``mdrq.build_method`` returns the GPU access
methods for the scan / VA-file names.  No reference file is edited.
"""

import os


def pytest_configure(config):
    from paper_1801_03644_b200 import reference_backend as rb
    rb.install_kernels()
    if os.environ.get("MDRQ_DEVICE_METHODS"):
        rb.install_methods()
