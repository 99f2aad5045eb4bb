"""pytest plugin: run the reference's OWN test suites against this package.

Test infrastructure only (not shipped).  The reference package is the one
installed into baseline/_ref (`pip install --target baseline/_ref`, see
DESIGN.md) and its tests are staged next to it by
tools/run_reference_suites.py; neither is committed.

REFSUITE_ROUTE selects what the unmodified reference code is pointed at:

- "api" (Route 1): `rlfc.decoder`, `rlfc.renderer` and
  `rlfc.errors` resolve to paper_1805_06019_b200's modules; everything else
  (container, encoder, hierarchy, bise, colorspace, metrics, service) is the
  reference's own code, which then calls this package's decoder/renderer.
- "kernels" (Route 2): the reference runs unchanged except that its kernel
  module's three decode entry points are this package's GPU backend
  (kernels_b200), exactly the binding INTEGRATION.md shows for
  rlfc/kernels.py (kernels.py:22-44).
"""
import importlib
import importlib.abc
import importlib.util
import os
import sys

ROUTE = os.environ.get("REFSUITE_ROUTE", "api")
# "encoder": rlfc.encoder resolves to tools/refsuite_gpu_encoder.py, this
# package's encoder with the RKV/SRV trees built on the GPU; the reference's
# decoder then reads those streams
_API = {
    "rlfc.decoder": "paper_1805_06019_b200.decoder",
    "rlfc.renderer": "paper_1805_06019_b200.renderer",
    "rlfc.errors": "paper_1805_06019_b200.errors",
}


class _Alias(importlib.abc.MetaPathFinder, importlib.abc.Loader):
    def __init__(self, aliases):
        self.aliases = aliases

    def find_spec(self, name, path, target=None):
        if name in self.aliases:
            return importlib.util.spec_from_loader(name, self)
        return None

    def create_module(self, spec):
        return importlib.import_module(self.aliases[spec.name])

    def exec_module(self, module):
        pass


# installed at plugin import: pytest imports -p plugins before it loads the
# suites' conftest.py (which imports rlfc)
if ROUTE == "api":
    sys.meta_path.insert(0, _Alias(_API))
elif ROUTE == "encoder":
    sys.meta_path.insert(0, _Alias({"rlfc.encoder": "refsuite_gpu_encoder"}))


def pytest_configure(config):
    if ROUTE == "api":
        import rlfc
        import paper_1805_06019_b200
        assert rlfc.decoder is paper_1805_06019_b200.decoder
        assert rlfc.renderer is paper_1805_06019_b200.renderer
    elif ROUTE == "encoder":
        import rlfc
        import refsuite_gpu_encoder
        assert rlfc.encoder is refsuite_gpu_encoder
    elif ROUTE == "kernels":
        import rlfc.kernels as K
        from paper_1805_06019_b200 import kernels_b200 as G
        for name in ("decode_chain_core", "decode_plane_core", "bise_decode_core"):
            setattr(K, name, getattr(G, name))
    else:
        raise SystemExit(f"unknown REFSUITE_ROUTE {ROUTE!r}")


def pytest_report_header(config):
    import rlfc
    return f"reference suite shim: route={ROUTE} rlfc from {os.path.dirname(rlfc.__file__)}"


def pytest_terminal_summary(terminalreporter):
    # evidence that the suites ran on this package's CUDA library
    try:
        with open("/proc/self/maps") as f:
            libs = sorted({ln.split()[-1] for ln in f if "librlfc" in ln})
    except OSError:
        libs = []
    terminalreporter.write_line("REFSUITE_NATIVE " + ",".join(os.path.basename(x) for x in libs))
