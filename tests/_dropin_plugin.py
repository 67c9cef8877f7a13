"""pytest plugin (-p _dropin_plugin): installs the B200 backend into the
reference package before the reference's own test modules import it, so their
`from salf.render_raster import rasterize` etc. bind the GPU functions.
SALF_DROPIN_PRECISION = fp64 (default) | mixed."""
import os


def pytest_configure(config):
    import salf
    from paper_2507_18713_b200 import dropin
    config._salf_backend = dropin.install(salf, precision=os.environ.get("SALF_DROPIN_PRECISION", "fp64"))


def pytest_unconfigure(config):
    be = getattr(config, "_salf_backend", None)
    if be is not None and os.environ.get("SALF_DROPIN_REPORT"):
        import json
        print("dropin calls:" + json.dumps(dict(be.calls)))
