"""The C ABI: libemc.so loads on a CPU-only host and exports every symbol
include/emc.h declares (no compute calls without a GPU)."""

import os
import re

import pytest

from conftest import ROOT, gpu_available


def _declared():
    with open(os.path.join(ROOT, "include", "emc.h")) as fh:
        text = fh.read()
    return set(re.findall(r"\b(emc_[a-z0-9_]+)\s*\(", text))


def test_header_declarations_bound():
    from paper_2403_12345_b200 import _native
    declared = _declared()
    assert declared, "no declarations parsed"
    assert declared == set(_native.SYMBOLS), declared ^ set(_native.SYMBOLS)


def test_library_exports_every_symbol():
    from paper_2403_12345_b200 import _native
    lib = _native.load_library_file()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.emc_abi_version() == _native.ABI_VERSION == 2


def test_no_cpu_fallback():
    """Without a GPU the engine refuses to run (and never silently computes
    on the host)."""
    if gpu_available():
        pytest.skip("GPU present")
    import paper_2403_12345_b200 as P
    from paper_2403_12345_b200 import _native
    assert _native.device_count() == 0
    lib, cell = P.analytic_infinite_medium()
    with pytest.raises(P.NativeUnavailableError):
        P.run_event(P.RunConfig(particles_per_batch=10, inactive_batches=1, active_batches=1), lib, cell)
    with pytest.raises(P.NativeUnavailableError):
        P.macro_lookup(lib, 0, 1.0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2403_12345_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, f)) as fh:
                    text = fh.read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("Oracle", ""), f
