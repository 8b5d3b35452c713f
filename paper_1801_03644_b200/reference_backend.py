"""Plug the B200 engine into an UNMODIFIED reference ``mdrq`` package.

INTEGRATION.md shows the two lines a maintainer would add to the reference
(``kernels.py:16-32`` backend selection, ``methods.py:20-47`` registry).
This module does the same from the outside, so the reference's own test
suite can run against the GPU engine without editing a reference file:

* ``install_kernels()`` -- the reference's compiled kernel module
  ``mdrq._kernels_cy`` (what ``mdrq.kernels`` binds, ``kernels.py:21-34``)
  is replaced by a module whose scan kernels are this engine's
  (``match_row`` / ``scan_rows`` / ``scan_column``, ``_kernels_cy.pyx:49-120``,
  on the GPU) and whose tree kernels (kd-tree / R*-tree helpers, out of scope
  for the scan engine) stay the reference's own compiled ones.  Must run
  before ``import mdrq``.
* ``install_methods()`` -- ``mdrq.build_method`` (``methods.py:20-47``)
  returns this engine's device-resident access methods for the scan and
  VA-file names (``sequential``, ``horizontal``, ``vertical``, ``vafile``);
  the tree names go to the reference's own builder.

Both keep the reference's argument meaning and error behaviour; results are
the reference types' duck equivalents (``ResultSet.ids`` int64 ascending).
"""

from __future__ import annotations

import glob
import importlib.util
import os
import sys
import types

SCAN_KERNELS = ("match_row", "scan_rows", "scan_column")
DEVICE_METHODS = ("sequential", "horizontal", "vertical", "vafile")


def _reference_kernels_path(package: str = "mdrq") -> str:
    spec = importlib.util.find_spec(package)
    if spec is None or not spec.submodule_search_locations:
        raise ImportError(f"reference package {package!r} is not importable")
    for d in spec.submodule_search_locations:
        hits = sorted(glob.glob(os.path.join(d, "_kernels_cy*.so")))
        if hits:
            return hits[0]
    raise ImportError(f"{package}: compiled _kernels_cy not found")


def install_kernels(package: str = "mdrq") -> types.ModuleType:
    """Register the GPU kernel module as ``<package>._kernels_cy``."""
    name = f"{package}._kernels_cy"
    if package in sys.modules:
        raise RuntimeError(f"install_kernels() must run before `import {package}`")
    spec = importlib.util.spec_from_file_location(name, _reference_kernels_path(package))
    real = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(real)
    from . import kernels as gpu
    mod = types.ModuleType(name, "B200 scan kernels + the reference's own tree kernels")
    for k, v in vars(real).items():
        if not k.startswith("__"):
            setattr(mod, k, v)
    for k in SCAN_KERNELS:
        setattr(mod, k, getattr(gpu, k))
    mod.BACKEND = gpu.BACKEND
    mod.MODE_SCALAR, mod.MODE_BLOCKED, mod.LANE = gpu.MODE_SCALAR, gpu.MODE_BLOCKED, gpu.LANE
    mod.__file__ = getattr(gpu, "__file__", None)
    sys.modules[name] = mod
    return mod


def install_methods(package: str = "mdrq") -> None:
    """Route ``build_method`` scan / VA-file names to the GPU methods."""
    import importlib
    ref = importlib.import_module(package)
    ref_methods = importlib.import_module(f"{package}.methods")
    original = ref_methods.build_method

    def build_method(name, data, *, threads=None, partitions=None, mode=None, seed=0, rstar_config=None):
        if name in DEVICE_METHODS:
            from . import DataSet, KernelMode
            from .methods import build_method as gpu_build
            km = KernelMode.SCALAR if mode is None else KernelMode(mode.value)
            return gpu_build(name, DataSet(data.values), threads=threads, partitions=partitions, mode=km,
                             seed=seed)
        kw = {} if mode is None else {"mode": mode}
        return original(name, data, threads=threads, partitions=partitions, seed=seed,
                        rstar_config=rstar_config, **kw)

    build_method.__doc__ = original.__doc__
    build_method.__wrapped__ = original
    ref_methods.build_method = build_method
    ref.build_method = build_method
