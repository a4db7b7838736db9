"""pytest configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here (no GPU): oracle vs golden vectors, host logic, the
C-ABI library's exports.  `-m gpu` runs on a B200 and calls the CUDA path
through the C ABI.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from its own sources (oracle/_ref); skip if absent."""
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libsngref.so not built")
    return Reference()


def _route_test_hooks():
    """Calls made while SNGB_TEST_FORCE_IRREGULAR is set go to the test build
    lib/libsngb_testhooks.so (the product library compiles the hook out)."""
    try:
        from paper_2006_06743_b200 import _lib
    except Exception:
        return
    product = _lib.lib
    hooked = {}

    def lib():
        if os.environ.get("SNGB_TEST_FORCE_IRREGULAR"):
            if "L" not in hooked:
                hooked["L"] = _lib.load(os.path.join(_lib.PKG, "lib", "libsngb_testhooks.so"))
            return hooked["L"]
        return product()

    _lib.lib = lib


_route_test_hooks()
