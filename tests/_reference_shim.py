"""pytest plugin: run the REFERENCE's own test modules with this package
installed as the hot path (``paper_2408_01654_b200.shim.install``).

Loaded by ``tests/test_gpu_reference_suite.py`` as ``-p _reference_shim``
before the reference test modules are imported, so their by-name imports
(``from patchslam.block_cholesky import block_cholesky``,
``from patchslam.geometry import reproject_grid``) bind this package's
functions.  At the end it records how many kernels this package launched
(the evidence that the shim, not the reference numpy, ran).
"""

import json
import os

_STATE = {}


def pytest_configure(config):
    from paper_2408_01654_b200 import _lib, shim
    _STATE["restore"] = shim.install()
    _STATE["launch0"] = int(_lib.lib().dpv_launch_count())


def pytest_unconfigure(config):
    from paper_2408_01654_b200 import _lib
    out = os.environ.get("DPV_SHIM_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump({"launches": int(_lib.lib().dpv_launch_count()) - _STATE["launch0"]}, fh)
    _STATE.pop("restore")()
